// b64_compact.cuh -- whitespace compaction on the GPU: Appendix B whitespace
// removal and the compaction front end of the fused
// whitespace-tolerant decode (row f4, b64_ws.cuh).  Removed bytes: ' ' (0x20),
// '\n' (0x0A), '\r' (0x0D) (hex codes per reading G8).
//
// The paper's SSE kernel compacts 16 bytes with a 65,536-entry shuffle table
// (P:1250-1271); a GPU has no byte shuffle across a register file, but it has
// a conflict-free byte gather/scatter in shared memory and warp ballots /
// shuffles.  Layout: the input is cut into 16 KiB tiles aligned to 16-byte
// granules of HBM (tile t = window [a0 + t*16K, a0 + (t+1)*16K), a0 = d_in
// rounded down to 16 B; the first and last tiles are partial); consecutive
// tiles form one chunk per CTA.  Two kernels:
//   cp_count_kernel   kept bytes per chunk (16-byte coalesced loads, SWAR test)
//   <consumer>        per chunk, at the offset given by the counts of the
//                     chunks before it: TMA-stage each tile, compact it into a
//                     shared-memory stream (compact_tile), consume the stream
//                     (copy-out for despace, base64 decode for the fused path).
// compact_tile: warp w owns the tile's words [256w, 256w+256); lane l reads
// words 32i + l (i = 0..7, conflict-free LDS.32), keeps a 4-bit keep mask
// per word (8 nibbles in one register), scans the per-word counts of the
// warp with one packed-byte shuffle scan (4 counts per register, 2
// registers), block-scans the 16 warp totals and places every kept byte
// with a predicated STS.U8 (consecutive lanes -> consecutive words, no bank
// conflicts).  Order is preserved.
#pragma once
#include <cstdint>

#include "b64_batch.cuh"
#include "b64_codec.cuh"
#include "b64_ptx.cuh"

namespace b64 {

#ifndef B64_CP_WARPS
#define B64_CP_WARPS 16
#endif
constexpr int kCpWarps = B64_CP_WARPS;  // warps per CTA; a tile is 1 KiB per warp
constexpr int kCpThreads = kCpWarps * 32;
constexpr int kCpTile = kCpWarps * 1024;            // input window bytes per tile
constexpr int kCpWords = kCpTile / 4;               // 4096 words
constexpr int kCpWarpWords = kCpWords / kCpWarps;   // 256 words = 1 KiB per warp
constexpr int kCpPerLane = kCpWarpWords / 32;       // 8 words per lane
static_assert(kCpPerLane == 8, "compact_tile packs 8 keep nibbles per lane");
#ifndef B64_CP_STAGES
#define B64_CP_STAGES 3
#endif
constexpr int kCpStages = B64_CP_STAGES;            // TMA input ring depth
#ifndef B64_CP_CTAS
#define B64_CP_CTAS 2
#endif
constexpr int kCpCtasPerSm = B64_CP_CTAS;
constexpr int kCpMaxChunks = 4096;

// Per-byte keep flags: bit 7 of each byte of the result is set iff that byte
// of w is NOT one of 0x20, 0x0A, 0x0D.  (x ^ K) & 0x7F + 0x7F has bit 7 set
// iff the low 7 bits of x differ from K (no carry leaves a byte: at most
// 0x7F + 0x7F); bytes >= 0x80 are always kept.  8 ALU ops per word.
__device__ __forceinline__ uint32_t xor_and7f(uint32_t w, uint32_t K) {  // (w ^ K) & 0x7F7F7F7F
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(d) : "r"(w), "r"(K), "r"(0x7F7F7F7Fu));
  return d;
}
__device__ __forceinline__ uint32_t keep_flags(uint32_t w) {
  const uint32_t s1 = xor_and7f(w, 0x20202020u) + 0x7F7F7F7Fu;
  const uint32_t s2 = xor_and7f(w, 0x0A0A0A0Au) + 0x7F7F7F7Fu;
  const uint32_t s3 = xor_and7f(w, 0x0D0D0D0Du) + 0x7F7F7F7Fu;
  return ((s1 & s2 & s3) | w) & 0x80808080u;
}

// Bits 7, 15, 23, 31 of f -> bits 0..3 (one multiply: the four partial
// products land on distinct bits 28..31).
__device__ __forceinline__ uint32_t gather4(uint32_t f) { return (f * 0x00204081u) >> 28; }

__device__ __forceinline__ bool is_space_byte(uint32_t v) {
  return v == 0x20u || v == 0x0Au || v == 0x0Du;
}

// Kept-byte count of one 16-byte granule whose valid bytes are [lo, hi).
__device__ __forceinline__ int kept_granule(const uint4 &v, int lo, int hi) {
  uint32_t k = gather4(keep_flags(v.x)) | gather4(keep_flags(v.y)) << 4 |
               gather4(keep_flags(v.z)) << 8 | gather4(keep_flags(v.w)) << 12;
  const uint32_t vm = (hi >= 16 ? 0xFFFFu : (1u << hi) - 1u) & ~((1u << lo) - 1u);
  return __popc(k & vm);
}
__device__ __forceinline__ int kept_granule_full(const uint4 &v) {
  return __popc(keep_flags(v.x)) + __popc(keep_flags(v.y)) + __popc(keep_flags(v.z)) +
         __popc(keep_flags(v.w));
}

// ------------------------------------------------------------ geometry ---
struct CpGeom {
  const uint8_t *in;  // d_in
  uintptr_t a0;       // d_in rounded down to 16 bytes
  int imis;           // d_in - a0
  int64_t m;          // input bytes
  int64_t ntiles;     // ceil((imis + m) / kCpTile)
  int64_t tpc;        // tiles per chunk
  __device__ __forceinline__ void init(const uint8_t *p, int64_t m_, int64_t tpc_) {
    in = p;
    a0 = reinterpret_cast<uintptr_t>(p) & ~static_cast<uintptr_t>(15);
    imis = static_cast<int>(reinterpret_cast<uintptr_t>(p) & 15);
    m = m_;
    ntiles = (imis + m + kCpTile - 1) / kCpTile;
    tpc = tpc_;
  }
  // valid window bytes of tile t: [lo, hi)
  __device__ __forceinline__ int lo(int64_t t) const { return t == 0 ? imis : 0; }
  __device__ __forceinline__ int hi(int64_t t) const {
    const int64_t h = imis + m - t * kCpTile;
    return h < kCpTile ? static_cast<int>(h) : kCpTile;
  }
  // input offset (relative to d_in) of window byte x of tile t
  __device__ __forceinline__ int64_t off(int64_t t, int x) const { return t * kCpTile + x - imis; }
};

// Keep mask of the 4 bytes of window word wi restricted to [lo, hi).
__device__ __forceinline__ uint32_t valid4(int lo, int hi, int wi) {
  const int a = lo - 4 * wi, b = hi - 4 * wi;
  const uint32_t top = b >= 4 ? 0xFu : b <= 0 ? 0u : (1u << b) - 1u;
  const uint32_t bot = a <= 0 ? 0u : a >= 4 ? 0xFu : (1u << a) - 1u;
  return top & ~bot;
}

// Pass 1 (classification): for every tile t and thread slot tid of the
// consumer (warp w, lane l), the 4-bit keep masks of window words
// 256w + 32i + l, i = 0..7, packed as 8 nibbles -> masks[t*512 + tid]
// (exact: bytes outside the input are 0); counts[b] = kept bytes of chunk b
// = tiles [b*tpc, (b+1)*tpc).  Loads are coalesced 128-byte warp rows, two
// tiles in flight per thread.  reset (may be null): two words of a
// consumer's scratch set to {~0, 0} for the launch that follows.
__device__ __forceinline__ uint32_t tile_nib(const uint32_t (&w)[kCpPerLane], int lo, int hi,
                                             int wbase, bool edge) {
  uint32_t nib = 0;
#pragma unroll
  for (int i = 0; i < kCpPerLane; ++i) {
    uint32_t k = gather4(keep_flags(w[i]));
    if (edge) k &= valid4(lo, hi, wbase + 32 * i);
    nib |= k << (4 * i);
  }
  return nib;
}

__global__ void __launch_bounds__(kCpThreads)
    cp_mask_kernel(const uint8_t *__restrict__ in, int64_t m, int64_t tpc,
                   int64_t *__restrict__ counts, uint32_t *__restrict__ masks,
                   unsigned long long *reset, const int32_t *skip = nullptr) {
  __shared__ int64_t sh[66];
  if (skip != nullptr && *skip == 1) return;  // the line-structured fast path already decoded
  if (reset != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    reset[0] = ~0ull;
    reset[1] = 0ull;
  }
  CpGeom G;
  G.init(in, m, tpc);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wbase = warp * kCpWarpWords + lane;  // this thread's first window word
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * tpc;
  const int64_t t1 = t0 + tpc < G.ntiles ? t0 + tpc : G.ntiles;
  int cnt = 0;
  for (int64_t t = t0; t < t1; t += 2) {
    const bool two = t + 1 < t1;
    const uint32_t *wa = reinterpret_cast<const uint32_t *>(G.a0 + static_cast<uintptr_t>(t) * kCpTile);
    const int lo0 = G.lo(t), hi0 = G.hi(t);
    const int lo1 = two ? G.lo(t + 1) : 0, hi1 = two ? G.hi(t + 1) : 0;
    const bool e0 = lo0 != 0 || hi0 != kCpTile, e1 = two && (lo1 != 0 || hi1 != kCpTile);
    const int lim0 = (hi0 + 15) & ~15, lim1 = (hi1 + 15) & ~15;  // loadable window bytes
    uint32_t a[kCpPerLane], b[kCpPerLane];
#pragma unroll
    for (int i = 0; i < kCpPerLane; ++i) {
      const int wi = wbase + 32 * i;
      a[i] = (!e0 || 4 * wi < lim0) ? __ldcs(wa + wi) : 0u;
      b[i] = two && (!e1 || 4 * wi < lim1) ? __ldcs(wa + kCpWords + wi) : 0u;
    }
    const uint32_t na = tile_nib(a, lo0, hi0, wbase, e0);
    masks[t * kCpThreads + tid] = na;
    cnt += __popc(na);
    if (two) {
      const uint32_t nb = tile_nib(b, lo1, hi1, wbase, e1);
      masks[(t + 1) * kCpThreads + tid] = nb;
      cnt += __popc(nb);
    }
  }
  int64_t p, pb, tot, tb;
  block_exclusive_scan2(cnt, 0, p, pb, tot, tb, sh);
  if (tid == 0) counts[blockIdx.x] = tot;
}

// Sum of counts[0..b) and of all counts[0..n) (every thread gets both).
__device__ __forceinline__ void chunk_prefix(const int64_t *counts, int64_t n, int64_t b,
                                             int64_t &before, int64_t &total, int64_t *sh) {
  int64_t x = 0, y = 0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
    const int64_t v = counts[c];
    y += v;
    if (c < b) x += v;
  }
  int64_t p, pb;
  block_exclusive_scan2(x, y, p, pb, before, total, sh);
}

// Shared memory of a compaction consumer CTA.
struct alignas(128) CpSmem {
  uint8_t win[kCpStages][kCpTile];         // TMA ring (16-byte aligned windows)
  uint32_t msk[kCpStages][kCpThreads];     // the tiles' keep masks (cp_mask_kernel)
  uint64_t full[kCpStages];
  int32_t wcnt[2][kCpWarps];  // by tile parity: back-to-back compactions need no extra barrier
  uint32_t ktab[16];  // per 4-bit keep mask: PRMT selector (bits 0..15) | (2^c - 1) << 16 | c << 20
};

// Fill CpSmem::ktab (threads 0..15); needs a barrier before use.
__device__ __forceinline__ void init_ktab(uint32_t *ktab) {
  const int k = threadIdx.x;
  if (k < 16) {
    uint32_t sel = 0x4444u, c = 0;  // unused slots select a zero byte
    for (int j = 0; j < 4; ++j)
      if (k & (1 << j)) {
        sel = (sel & ~(0xFu << (4 * c))) | (static_cast<uint32_t>(j) << (4 * c));
        ++c;
      }
    ktab[k] = sel | (((1u << c) - 1u) << 16) | (c << 20);
  }
}

// Issue the bulk loads of tile t (window + keep masks) into ring slot s (one thread).
__device__ __forceinline__ void cp_load(CpSmem &S, const CpGeom &G, const uint32_t *masks,
                                        int64_t t, int s, uint64_t pol) {
  const int h = G.hi(t);
  const uint32_t bytes = static_cast<uint32_t>((h + 15) & ~15);
  ptx::mbar_arrive_expect_tx(&S.full[s], bytes + 4 * kCpThreads);
  ptx::bulk_g2s(S.win[s], reinterpret_cast<const void *>(G.a0 + static_cast<uintptr_t>(t) * kCpTile),
                bytes, &S.full[s], pol);
  ptx::bulk_g2s(S.msk[s], masks + t * kCpThreads, 4 * kCpThreads, &S.full[s], pol);
}

// Compact the kept bytes of a 16 KiB window (smem, 16-byte aligned; keep
// masks msk[tid] from cp_mask_kernel) into stream[dst, dst + n), in order;
// returns n (all threads).  Contains one __syncthreads; the caller
// synchronises before reading the stream.
// PIPE: word i+1 and its selector are loaded before word i's byte stores
// (the compiler keeps shared loads below earlier shared stores otherwise,
// which puts a load latency on every word) -- measured faster in the fused
// decode (1.068 -> 1.057 ms), marginally slower in despace (0.811 vs 0.816).
// WAITB: thread 0 waits for the reads of its earlier bulk stores (the copy-out
// of the stream this call overwrites) just before the internal barrier.
// NB: the internal barrier is named barrier 1 over the kCpThreads compute
// threads (CTAs with extra producer / scan warps) instead of __syncthreads.
template <bool PIPE, bool WAITB = false, bool NB = false>
__device__ __forceinline__ int compact_tile(const uint8_t *win, const uint32_t *msk,
                                            uint8_t *stream, int dst, int32_t *wcnt,
                                            const uint32_t *ktab) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t *seg = reinterpret_cast<const uint32_t *>(win) + warp * kCpWarpWords + lane;
  const uint32_t nib = msk[tid];
  // per-word kept counts (nibble popcounts), 4 per register as bytes
  uint32_t nc = nib - ((nib >> 1) & 0x55555555u);
  nc = (nc & 0x33333333u) + ((nc >> 2) & 0x33333333u);
  const uint32_t x0 = nc & 0x0F0F0F0Fu;         // words 0, 2, 4, 6
  const uint32_t x1 = (nc >> 4) & 0x0F0F0F0Fu;  // words 1, 3, 5, 7
  uint32_t s0 = x0, s1 = x1;                    // inclusive scans (bytes <= 128)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u0 = __shfl_up_sync(0xffffffffu, s0, o);
    const uint32_t u1 = __shfl_up_sync(0xffffffffu, s1, o);
    if (lane >= o) {
      s0 += u0;
      s1 += u1;
    }
  }
  const uint32_t T0 = __shfl_sync(0xffffffffu, s0, 31), T1 = __shfl_sync(0xffffffffu, s1, 31);
  const uint32_t e0 = s0 - x0, e1 = s1 - x1;  // exclusive, per byte
  // warp total = sum of the 8 bytes of T0, T1
  const uint32_t h = (T0 & 0x00FF00FFu) + ((T0 >> 8) & 0x00FF00FFu) + (T1 & 0x00FF00FFu) +
                     ((T1 >> 8) & 0x00FF00FFu);
  const int wtot = static_cast<int>((h & 0xFFFFu) + (h >> 16));
  if (lane == 0) wcnt[warp] = wtot;
  if (WAITB && tid == 0) ptx::bulk_wait_read<0>();
  if constexpr (NB) ptx::named_bar_sync(1, kCpThreads);
  else __syncthreads();
  const int c = lane < kCpWarps ? wcnt[lane] : 0;
  int incl = c;
#pragma unroll
  for (int o = 1; o < kCpWarps; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const int wpre = __shfl_sync(0xffffffffu, incl - c, warp);
  const int total = __shfl_sync(0xffffffffu, incl, kCpWarps - 1);
  uint8_t *ws = stream + dst + wpre;
  int base = 0;  // kept bytes of this warp's words 32*i' + *, i' < i
  uint32_t en = 0, wn = 0;
  if constexpr (PIPE) {
    en = ktab[nib & 0xFu];
    wn = seg[0];
  }
#pragma unroll
  for (int i = 0; i < kCpPerLane; ++i) {
    // the word's kept bytes, packed low by one PRMT, stored at p[0..c)
    uint32_t e, wsrc;
    if constexpr (PIPE) {
      e = en;
      wsrc = wn;
      if (i + 1 < kCpPerLane) {
        en = ktab[(nib >> (4 * (i + 1))) & 0xFu];
        wn = seg[32 * (i + 1)];
      }
    } else {
      e = ktab[(nib >> (4 * i)) & 0xFu];
      wsrc = seg[32 * i];
    }
    uint32_t cw;  // PRMT reads only the selector's low 16 bits
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(cw) : "r"(wsrc), "r"(e));
    const uint32_t E = (i & 1) ? e1 : e0, T = (i & 1) ? T1 : T0;
    const int sh = 8 * (i >> 1);
    uint8_t *p = ws + base + static_cast<int>((E >> sh) & 0xFFu);
    if (e & 0x10000u) p[0] = static_cast<uint8_t>(cw);
    if (e & 0x20000u) p[1] = static_cast<uint8_t>(cw >> 8);
    if (e & 0x40000u) p[2] = static_cast<uint8_t>(cw >> 16);
    if (e & 0x80000u) p[3] = static_cast<uint8_t>(cw >> 24);
    base += static_cast<int>((T >> sh) & 0xFFu);
  }
  return total;
}

// CTA-wide copy of n bytes from smem src to global dst, where src and dst
// are congruent mod 16: aligned LDS.128 -> STG.128 for the interior, byte
// stores for the (< 16 byte) edges.
__device__ __forceinline__ void cta_copy_out_congruent(uint8_t *dst, const uint8_t *src, int n,
                                                       int nthreads = -1) {
  const int tid = threadIdx.x;
  const int nt = nthreads > 0 ? nthreads : static_cast<int>(blockDim.x);
  const uintptr_t g = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t a0 = (g + 15) & ~static_cast<uintptr_t>(15);
  const uintptr_t a1 = (g + static_cast<uintptr_t>(n)) & ~static_cast<uintptr_t>(15);
  if (a1 > a0) {
    const int head = static_cast<int>(a0 - g);
    const int ng = static_cast<int>((a1 - a0) >> 4);
    for (int q = tid; q < ng; q += nt)
      *reinterpret_cast<uint4 *>(reinterpret_cast<uint8_t *>(a0) + 16 * q) =
          ptx::lds128(src + head + 16 * q);  // congruent: 16-byte aligned
    const int tail0 = static_cast<int>(a1 - g);
    if (tid < head) dst[tid] = src[tid];
    if (tid >= 32 && tid - 32 < n - tail0) dst[tail0 + tid - 32] = src[tail0 + tid - 32];
  } else if (tid < n) {
    dst[tid] = src[tid];
  }
}

// The same copy with the 16-byte aligned interior as one bulk (TMA) store
// issued by thread 0 (committed as one bulk group; the caller waits with
// bulk_wait_read before the staging is overwritten and with bulk_wait before
// the CTA exits) and the edges as byte stores by threads 32.. and 64.. .
// The staging writes must be fenced to the async proxy
// (fence_proxy_async_smem) by their writers before the barrier preceding
// this call.  Frees the CTA's threads from the copy-out loop.
__device__ __forceinline__ void cta_copy_out_bulk(uint8_t *dst, const uint8_t *src, int n,
                                                  uint64_t pol) {
  const int tid = threadIdx.x;
  const uintptr_t g = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t a0 = (g + 15) & ~static_cast<uintptr_t>(15);
  const uintptr_t a1 = (g + static_cast<uintptr_t>(n)) & ~static_cast<uintptr_t>(15);
  if (a1 > a0) {
    const int head = static_cast<int>(a0 - g), tail0 = static_cast<int>(a1 - g);
    if (tid == 0) {
      ptx::bulk_s2g(reinterpret_cast<void *>(a0), src + head, static_cast<uint32_t>(a1 - a0), pol);
      ptx::bulk_commit();
    }
    if (tid >= 32 && tid - 32 < head) dst[tid - 32] = src[tid - 32];
    if (tid >= 64 && tid - 64 < n - tail0) dst[tail0 + tid - 64] = src[tail0 + tid - 64];
  } else if (tid < n) {
    dst[tid] = src[tid];
  }
}

// ------------------------------------------------------ despace (f3) ---
#ifndef B64_DS_GROUP
#define B64_DS_GROUP 1
#endif
#ifndef B64_DS_BULK  // copy-out as one bulk store (cta_copy_out_bulk)
#define B64_DS_BULK 1
#endif
#ifndef B64_DS_DEFER  // copy tile t's stream out after tile t+1's compaction barrier
#define B64_DS_DEFER 1
#endif
constexpr int kDsGroup = B64_DS_GROUP;  // tiles compacted per copy-out
static_assert(!B64_DS_DEFER || B64_DS_GROUP == 1, "B64_DS_DEFER needs B64_DS_GROUP 1");
constexpr int kDsStages = kCpStages + kDsGroup - 1;

struct alignas(128) DsSmem {
  uint8_t win[kDsStages][kCpTile];
  uint32_t msk[kDsStages][kCpThreads];
  uint64_t full[kDsStages];
  int32_t wcnt[2][kCpWarps];
  uint32_t ktab[16];
#if B64_DS_DEFER
  alignas(16) uint8_t stream[2][kCpTile + 32];  // tile t's stream is copied out during tile t+1
#else
  alignas(16) uint8_t stream[kDsGroup * kCpTile + 32];  // 16-aligned: LDS.128 copy-out
#endif
  int64_t red[66];
};

__global__ void __launch_bounds__(kCpThreads, kCpCtasPerSm)
    despace_kernel(const uint8_t *__restrict__ in, int64_t m, uint8_t *__restrict__ out,
                   const int64_t *__restrict__ counts, const uint32_t *__restrict__ masks,
                   int64_t tpc, int64_t *out_len, const int32_t *skip = nullptr) {
  if (skip != nullptr && *skip == 1) return;  // the line-structured fast path already wrote it
  extern __shared__ __align__(128) uint8_t smem_raw[];
  DsSmem &S = *reinterpret_cast<DsSmem *>(smem_raw);
  const int tid = threadIdx.x;
  CpGeom G;
  G.init(in, m, tpc);
  if (tid == 0) {
    for (int s = 0; s < kDsStages; ++s) ptx::mbar_init(&S.full[s], 1);
    ptx::fence_mbar_init();
  }
  init_ktab(S.ktab);
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * tpc;
  const int64_t t1 = t0 + tpc < G.ntiles ? t0 + tpc : G.ntiles;
  int64_t running, total;
  chunk_prefix(counts, gridDim.x, blockIdx.x, running, total, S.red);  // has a __syncthreads
  const uint64_t pol = ptx::policy_evict_first();
  const uint64_t pol_out = pol;
  // TMA ring of kDsStages tiles (window + masks on one mbarrier each)
  auto load = [&](int64_t t, int s) {
    const int h = G.hi(t);
    const uint32_t bytes = static_cast<uint32_t>((h + 15) & ~15);
    ptx::mbar_arrive_expect_tx(&S.full[s], bytes + 4 * kCpThreads);
    ptx::bulk_g2s(S.win[s], reinterpret_cast<const void *>(G.a0 + static_cast<uintptr_t>(t) * kCpTile),
                  bytes, &S.full[s], pol);
    ptx::bulk_g2s(S.msk[s], masks + t * kCpThreads, 4 * kCpThreads, &S.full[s], pol);
  };
  if (tid == 0)
    for (int s = 0; s < kDsStages - 1 && t0 + s < t1; ++s) load(t0 + s, s);
  const uintptr_t obase = reinterpret_cast<uintptr_t>(out);
#if B64_DS_DEFER
  // Double-buffered streams: compact_tile(t+1)'s internal barrier already
  // orders every thread's placement stores of tile t before the copy-out of
  // tile t, so the copy-out needs no barrier of its own and overlaps the
  // next tile's compaction across warps.
  int64_t prun = 0;
  int pdst = 0, pn = 0;
  for (int64_t t = t0; t < t1; ++t) {
    const int it = static_cast<int>(t - t0);
    const int s = it % kDsStages, b = it & 1;
    const int dst = static_cast<int>((obase + static_cast<uintptr_t>(running)) & 15);
    ptx::mbar_wait_spin(&S.full[s], static_cast<uint32_t>((it / kDsStages) & 1));
    // (B64_DS_BULK) stream[b]'s bulk store, issued in the previous
    // iteration, must have read it before compact_tile's barrier releases
    // the placement stores into it
    const int n = compact_tile<false, B64_DS_BULK != 0>(S.win[s], S.msk[s], S.stream[b], dst, S.wcnt[b],
                                                       S.ktab);
    // generic reads of win[s] before its next bulk write; this tile's stream
    // writes before the bulk store that reads them (after the next barrier)
    ptx::fence_proxy_async_smem();
    if (tid == 0 && t + kDsStages - 1 < t1)
      load(t + kDsStages - 1, static_cast<int>((it + kDsStages - 1) % kDsStages));
#if B64_DS_BULK
    if (it > 0) cta_copy_out_bulk(out + prun, S.stream[b ^ 1] + pdst, pn, pol_out);
#else
    if (it > 0) cta_copy_out_congruent(out + prun, S.stream[b ^ 1] + pdst, pn);
#endif
    prun = running;
    pdst = dst;
    pn = n;
    running += n;
  }
  if (t1 > t0) {
    __syncthreads();
#if B64_DS_BULK
    cta_copy_out_bulk(out + prun, S.stream[(t1 - 1 - t0) & 1] + pdst, pn, pol_out);
    if (tid == 0) ptx::bulk_wait<0>();
#else
    cta_copy_out_congruent(out + prun, S.stream[(t1 - 1 - t0) & 1] + pdst, pn);
#endif
  }
#else
  int64_t t = t0;
  while (t < t1) {
    // kDsGroup tiles compacted back to back into one stream, one copy-out:
    // a tile's input slot is refilled only after the next compact_tile's
    // internal barrier (every warp is done reading it by then).
    const int dst = static_cast<int>((obase + static_cast<uintptr_t>(running)) & 15);
    int n = 0;
#pragma unroll 1
    for (int j = 0; j < kDsGroup && t < t1; ++j, ++t) {
      const int it = static_cast<int>(t - t0);
      const int s = it % kDsStages;
      ptx::mbar_wait_spin(&S.full[s], static_cast<uint32_t>((it / kDsStages) & 1));
      n += compact_tile<false>(S.win[s], S.msk[s], S.stream, dst + n, S.wcnt[j & 1], S.ktab);
      ptx::fence_proxy_async_smem();  // generic reads of win[s] before its next bulk write
      // slot of tile t-1 is free (all warps passed this tile's internal barrier)
      if (tid == 0 && t + kDsStages - 1 < t1)
        load(t + kDsStages - 1, static_cast<int>((it + kDsStages - 1) % kDsStages));
    }
    __syncthreads();
    cta_copy_out_congruent(out + running, S.stream + dst, n);
    running += n;
  }
#endif
  if (blockIdx.x == gridDim.x - 1 && tid == 0) *out_len = total;
}

}  // namespace b64
