// b64_knobs.cuh -- MEASUREMENT-ONLY compile-time knobs.
//
// ======================================================================
//  None of these is set in the product build (__graft_entry__.build()
//  passes no -D flags).  They exist so that tools/sweep.py can build
//  variant libraries into build/variants/ for the A/B measurements that
//  DESIGN.md cites; each default below is the product behaviour.  A
//  library built with any of them changed is an experiment, never the
//  benched or tested product.
// ======================================================================
#pragma once

// Move the bytes, skip the base64 transform (data-movement skeleton of the
// single-buffer kernels; DESIGN.md §6 "skeleton" numbers).  Output is wrong.
#ifndef B64_SKELETON
#define B64_SKELETON 0
#endif

// Table I mapping by per-byte SWAR arithmetic (Table II offsets) instead of
// the 64-byte shared-memory table (the table wins).
#ifndef B64_ENC_ARITH
#define B64_ENC_ARITH 0
#endif

// Decode register stores: one 8-byte + one 4-byte store per 12-byte run
// instead of three 4-byte stores (C3 better, C5 worse).
#ifndef B64_DEC_STG64
#define B64_DEC_STG64 0
#endif

// Batched kernel: L2 prefetch distance in units beyond the TMA ring
// (0 = off; 2-5 % slower).
#ifndef B64_BATCH_PREFETCH
#define B64_BATCH_PREFETCH 0
#endif

// f3 / f4 general path: the single-read kernels of b64_onepass.cuh instead
// of the two-pass mask + compaction kernels (slower).
#ifndef B64_CP_ONEPASS
#define B64_CP_ONEPASS 0
#endif

// (defined or not; no default)
//   B64_BATCH_TRACE      per-warp %globaltimer stamps + b64_debug_trace()
//                        (tools/batch_trace.py); the export is not in the
//                        header and exists only in the trace build
//   B64_BATCH_TRACE_FM   trace stamp of each warp's first-message lookup
//   B64_BATCH_PLAN_ONLY  the batched kernel stops after its plan
