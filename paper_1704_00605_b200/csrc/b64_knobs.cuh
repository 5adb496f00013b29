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

// Batched kernels: batch2_kernel (b64_batch2.cuh: byte-range warps, CTA-local
// plan, first loads before the plan, per-CTA decode results) instead of
// batch_kernel (b64_batch.cuh: global unit plan, three grid barriers).
#ifndef B64_BATCH_V2
#define B64_BATCH_V2 0
#endif
// batch_kernel: per-unit fixed cost, in eighths of a unit's input, of the
// work estimate that splits units among warps (0: equal unit counts).
#ifndef B64_BATCH_UNIT_COST
#define B64_BATCH_UNIT_COST 16
#endif
// batch2_kernel: per-message charge of the work coordinate, in eighths of a
// unit's input (a unit costs a fixed part plus its bytes).
#ifndef B64_BATCH_MSG_COST
#define B64_BATCH_MSG_COST 4
#endif

// f3 general path: despace2_kernel (b64_despace2.cuh: one read, the
// one-pass prefix machinery with the two-pass kernels' placement) instead of
// cp_mask_kernel + despace_kernel.
#ifndef B64_DS_ONEPASS2
#define B64_DS_ONEPASS2 0
#endif

// f3 / f4 general path: the single-read kernels of b64_onepass.cuh instead
// of the two-pass mask + compaction kernels (slower).
#ifndef B64_CP_ONEPASS
#define B64_CP_ONEPASS 0
#endif

// Line-major MIME kernels (round 2); 0 = the earlier paths
// they replaced, kept for the A/B numbers DESIGN.md cites:
//   B64_WL_LINEMAJOR  decode_lines_kernel interior tiles one lane per line
//                     (0: flat quads across line ends; despace too)
//   B64_WL_BULK       line-major decode / despace blocks leave as one bulk
//                     store (0: LDS.128 -> STG.128 by the warp)
//   B64_WR_LINEMAJOR  b64_encode_wrapped with L <= 128 on encode_lines_kernel
//                     (0: encode_wrap_kernel for every L)
//   B64_EL_BULK       encode_lines_kernel blocks leave as one bulk store
#ifndef B64_WL_LINEMAJOR
#define B64_WL_LINEMAJOR 1
#endif
#ifndef B64_WL_BULK
#define B64_WL_BULK 1
#endif
#ifndef B64_WR_LINEMAJOR
#define B64_WR_LINEMAJOR 1
#endif
#ifndef B64_EL_BULK
#define B64_EL_BULK 1
#endif

// (defined or not; no default)
//   B64_BATCH_TRACE      per-warp %globaltimer stamps + b64_debug_trace()
//                        (tools/batch_trace.py); the export is not in the
//                        header and exists only in the trace build
//   B64_BATCH_TRACE_FM   trace stamp of each warp's first-message lookup
//   B64_BATCH_TRACE_WAIT cycles each warp spends waiting for unit data
//   B64_BATCH_PLAN_ONLY  the batched kernel stops after its plan
