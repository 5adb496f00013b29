// b64_despace.cuh -- Appendix B whitespace removal on the GPU (SURVEY.md §8(f)
// row f3): remove ' ' (0x20), '\n' (0x0A) and '\r' (0x0D) from a byte stream
// (hex codes per reading G8) as a single-pass stream compaction.
//
// The paper's SSE kernel compacts 16 bytes with a 65,536-entry shuffle table
// (P:1250-1271).  On the GPU: the input is split into one contiguous chunk of
// 16 KiB tiles per CTA; despace_count_kernel counts each chunk's kept bytes
// (SWAR test for bytes < 0x21, exact check only there); despace_kernel then
// adds the counts of the preceding chunks and compacts its chunk tile by
// tile (double-buffered TMA loads): each warp compacts its 1 KiB segment
// into its own smem run (one 4-byte word per lane per step, a warp scan of
// the kept counts places every byte, so the stores of a step hit consecutive
// smem words), a block scan of the 16 run lengths gives each run its offset
// and the runs are written with realigned 16-byte stores.  Two reads and one
// write of the data, no cross-CTA waiting.  (A single-pass decoupled
// look-back version was measured 4x slower: the look-back chain across
// ~600 in-flight tiles serialised the CTAs.)
#pragma once
#include <cstdint>

#include "b64_batch.cuh"
#include "b64_codec.cuh"
#include "b64_ptx.cuh"

namespace b64 {

constexpr int kDsWarps = 16;
constexpr int kDsThreads = kDsWarps * 32;
constexpr int kDsSeg = 1024;                    // bytes per warp per tile
constexpr int kDsTile = kDsWarps * kDsSeg;      // 16 KiB

constexpr int kDsCtasPerSm = 2;

struct alignas(128) DsSmem {
  uint8_t in[2][kDsTile + 48];         // double-buffered TMA input (+ funnel-load slack)
  uint8_t run[kDsWarps][kDsSeg + 48];  // per-warp compacted run (16 B head room + read slack)
  uint64_t full[2];
  int64_t tile;
  int64_t excl;
  int32_t cnt[kDsWarps];
  int32_t wexcl[kDsWarps];
};

__device__ __forceinline__ bool is_space(uint32_t v) {
  return v == 0x20u || v == 0x0Au || v == 0x0Du;
}

// Per-byte flags (0x80 in each byte) of the bytes below 0x21 in w (exact:
// no cross-byte borrows because every byte of (w | 0x80808080) is >= 0x80).
__device__ __forceinline__ uint32_t below21(uint32_t w) {
  return ~((w | 0x80808080u) - 0x21212121u) & ~w & 0x80808080u;
}

// Exact per-byte whitespace flags (0x80 in each byte that is 0x20, 0x0A or
// 0x0D), branch-free: among the bytes below 0x21, 0x20 is the only one with
// bit 5 set, and x == K is tested on the low 7 bits (no carries: every byte
// of (x & 0x7F..) + 0x7F.. is <= 0xFE); bytes >= 0x80 are excluded by below21.
__device__ __forceinline__ uint32_t space_flags(uint32_t w) {
  const uint32_t low = below21(w);
  const uint32_t t1 = ((w ^ 0x0A0A0A0Au) & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;  // bit 7 clear iff == 0x0A
  const uint32_t t2 = ((w ^ 0x0D0D0D0Du) & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;  // bit 7 clear iff == 0x0D
  return low & (~(t1 & t2) | (w << 2));
}

// Kept-byte count of 16 bytes.
__device__ __forceinline__ int kept16(const uint4 &v) {
  return 16 - __popc(space_flags(v.x)) - __popc(space_flags(v.y)) - __popc(space_flags(v.z)) -
         __popc(space_flags(v.w));
}

// Pass 1: kept bytes of chunk b = tiles [b*tpc, (b+1)*tpc).
__global__ void __launch_bounds__(kDsThreads)
    despace_count_kernel(const uint8_t *__restrict__ in, int64_t m, int64_t tpc,
                         int64_t *__restrict__ counts) {
  __shared__ int64_t sh[66];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * tpc * kDsTile;
  const int64_t c1 = c0 + tpc * kDsTile < m ? c0 + tpc * kDsTile : m;
  int64_t cnt = 0;
  if (c0 < c1) {
    const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(c0);
    const int head = static_cast<int>((16 - (g & 15)) & 15);  // bytes before the first granule
    const int64_t h = head < c1 - c0 ? head : c1 - c0;
    if (threadIdx.x < h) cnt += !is_space(in[c0 + threadIdx.x]);
    const uint4 *q = reinterpret_cast<const uint4 *>(in + c0 + h);
    const int64_t ng = (c1 - c0 - h) / 16;
    int64_t i = threadIdx.x;
    for (; i + 3 * kDsThreads < ng; i += 4 * kDsThreads) {
      const uint4 a = __ldcs(q + i), b = __ldcs(q + i + kDsThreads);
      const uint4 c = __ldcs(q + i + 2 * kDsThreads), d = __ldcs(q + i + 3 * kDsThreads);
      cnt += kept16(a) + kept16(b) + kept16(c) + kept16(d);
    }
    for (; i < ng; i += kDsThreads) cnt += kept16(__ldcs(q + i));
    const int64_t t0 = c0 + h + 16 * ng;
    if (threadIdx.x < c1 - t0) cnt += !is_space(in[t0 + threadIdx.x]);
  }
  int64_t p, pb, tot, tb;
  block_exclusive_scan2(cnt, 0, p, pb, tot, tb, sh);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

// Pass 2: compact chunk b to out + (kept bytes of chunks < b).
__global__ void __launch_bounds__(kDsThreads, kDsCtasPerSm)
    despace_kernel(const uint8_t *__restrict__ in, int64_t m, uint8_t *__restrict__ out,
                   const int64_t *__restrict__ counts, int64_t tpc, int64_t *out_len,
                   int64_t ntiles) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  DsSmem &S = *reinterpret_cast<DsSmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&S.full[0], 1);
    mbar_init(&S.full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  // Issue the bulk load of tile tt into buffer b (thread 0).
  auto load = [&](int64_t tt, int b) {
    const int64_t src = tt * kDsTile;
    const int L = static_cast<int>(m - src < kDsTile ? m - src : kDsTile);
    const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src);
    const uintptr_t g0 = g & ~static_cast<uintptr_t>(15);
    const uintptr_t g1 = (g + static_cast<uintptr_t>(L) + 15) & ~static_cast<uintptr_t>(15);
    mbar_arrive_expect_tx(&S.full[b], static_cast<uint32_t>(g1 - g0));
    bulk_g2s(S.in[b], reinterpret_cast<const void *>(g0), static_cast<uint32_t>(g1 - g0),
             &S.full[b], pol);
  };
  // This CTA's chunk: tiles [t0, t1); its output offset = kept bytes of the
  // chunks before it.
  __shared__ int64_t shs[66];
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * tpc;
  const int64_t t1 = t0 + tpc < ntiles ? t0 + tpc : ntiles;
  int64_t before = 0;
  for (int64_t c = tid; c < blockIdx.x; c += kDsThreads) before += counts[c];
  {
    int64_t p, pb, tot, tb;
    block_exclusive_scan2(before, 0, p, pb, tot, tb, shs);
    before = tot;
  }
  if (tid == 0 && t0 < t1) load(t0, 0);
  int64_t running = before;
  for (int64_t t = t0; t < t1; ++t) {
    const int it = static_cast<int>(t - t0);
    const int b = it & 1;
    if (tid == 0 && t + 1 < t1) load(t + 1, b ^ 1);
    const int64_t src = t * kDsTile;
    const int L = static_cast<int>(m - src < kDsTile ? m - src : kDsTile);
    const int imis = static_cast<int>((reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src)) & 15);
    mbar_wait_spin(&S.full[b], static_cast<uint32_t>((it >> 1) & 1));  // buffer b's use count

    // ---- compact this warp's segment into its run, 128 bytes per step:
    // each lane takes one 4-byte word; an exact SWAR test finds bytes below
    // 0x21 (only then are the three whitespace values checked one by one);
    // a warp scan of the per-lane kept counts places every kept byte, so
    // the byte stores of a step hit consecutive smem words (conflict-free)
    // and input order is preserved.
    const uint8_t *seg = S.in[b] + imis + warp * kDsSeg;
    uint8_t *run = S.run[warp] + 16;
    const int seg_len = L - warp * kDsSeg;  // may be <= 0 or > kDsSeg
    const uint32_t sh = 8u * static_cast<uint32_t>(reinterpret_cast<uintptr_t>(seg) & 3);
    const uint32_t *segw = reinterpret_cast<const uint32_t *>(seg - (reinterpret_cast<uintptr_t>(seg) & 3));
    const unsigned lt = (1u << lane) - 1u;
    int base = 0;
#pragma unroll 2
    for (int r = 0; r < kDsSeg / 4; r += 32) {
      const int wi = r + lane;  // word index in the segment
      const uint32_t w = __funnelshift_r(segw[wi], segw[wi + 1], sh);
      // keep bits 0..3 = bytes that are not whitespace: gather bit 7 of
      // every byte of ~flags into bits 28..31 with one multiply
      uint32_t keep = ((~space_flags(w) & 0x80808080u) * 0x00204081u) >> 28;
      if (L < kDsTile) {  // last tile only
        const int valid = seg_len - 4 * wi;
        if (valid < 4) keep &= valid <= 0 ? 0u : (1u << valid) - 1u;
      }
      const uint32_t c = __popc(keep);
      // warp exclusive scan of c (0..4) by its three bit planes
      const unsigned b0 = __ballot_sync(0xffffffffu, c & 1u);
      const unsigned b1 = __ballot_sync(0xffffffffu, c & 2u);
      const unsigned b2 = __ballot_sync(0xffffffffu, c & 4u);
      const int excl = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
      uint8_t *p = run + base + excl;
      // branch-free placement: byte j goes to p[popc(keep & ((1 << j) - 1))]
      if (keep & 1u) p[0] = static_cast<uint8_t>(w);
      if (keep & 2u) p[keep & 1u] = static_cast<uint8_t>(w >> 8);
      if (keep & 4u) p[__popc(keep & 3u)] = static_cast<uint8_t>(w >> 16);
      if (keep & 8u) p[__popc(keep & 7u)] = static_cast<uint8_t>(w >> 24);
      base += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    }
    if (lane == 0) S.cnt[warp] = base;
    __syncthreads();

    // ---- block scan of the run lengths
    if (warp == 0) {
      const int c = lane < kDsWarps ? S.cnt[lane] : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      if (lane < kDsWarps) S.wexcl[lane] = incl - c;
      if (lane == 31) S.excl = incl;  // tile total
    }
    __syncthreads();

    // ---- write this warp's run at its global offset (realigned 16-byte stores)
    warp_copy_out(out + running + S.wexcl[warp], run, S.cnt[warp], lane);
    running += S.excl;
    fence_proxy_async_smem();  // generic reads of S.in[b] before its next bulk write
    __syncthreads();           // runs / S.in[b] / S.excl reused by the next tile
  }
  if (t1 == ntiles && t0 < t1 && tid == 0) *out_len = running;
}

}  // namespace b64
