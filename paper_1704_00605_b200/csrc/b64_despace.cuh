// b64_despace.cuh -- Appendix B whitespace removal on the GPU (SURVEY.md §8(f)
// row f3): remove ' ' (0x20), '\n' (0x0A) and '\r' (0x0D) from a byte stream
// (hex codes per reading G8) as a single-pass stream compaction.
//
// The paper's SSE kernel compacts 16 bytes with a 65,536-entry shuffle table
// (P:1250-1271); on the GPU a warp compacts 32 bytes per step with one ballot:
// every lane holds one byte, the kept bytes' output slots are the popcounts of
// the ballot below each lane, so the 32 writes of a step hit consecutive smem
// bytes (conflict-free) and input order is preserved.  A CTA takes 16 KiB
// tiles (dynamic tile counter, TMA bulk load), each warp compacts its 1 KiB
// segment into its own smem run, a block scan of the 16 run lengths plus a
// decoupled look-back over the preceding tiles' totals gives every run its
// global output offset, and the runs are written with realigned 16-byte
// stores.  One read and one write of the data; no second pass.
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
constexpr uint64_t kDsFlagAgg = 1ull << 62;     // tile aggregate published
constexpr uint64_t kDsFlagPre = 2ull << 62;     // inclusive prefix published
constexpr uint64_t kDsValMask = (1ull << 62) - 1;

constexpr int kDsCtasPerSm = 4;

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

__global__ void __launch_bounds__(kDsThreads, kDsCtasPerSm)
    despace_kernel(const uint8_t *__restrict__ in, int64_t m, uint8_t *__restrict__ out,
                   unsigned long long *state, unsigned long long *tile_ctr, int64_t *out_len,
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
  // Tiles are taken from a global counter (so every tile's predecessors are
  // already owned by running CTAs: the look-back always makes progress); the
  // next tile is claimed and prefetched while the current one is processed.
  if (tid == 0) {
    S.tile = static_cast<int64_t>(atomicAdd(tile_ctr, 1ull));
    if (S.tile < ntiles) load(S.tile, 0);
  }
  __syncthreads();
  int64_t t = S.tile;
  for (int it = 0; t < ntiles; ++it) {
    const int b = it & 1;
    __syncthreads();  // everyone has read S.tile (the claim of tile t)
    if (tid == 0) {
      const int64_t tn = static_cast<int64_t>(atomicAdd(tile_ctr, 1ull));
      S.tile = tn;
      if (tn < ntiles) load(tn, b ^ 1);
    }
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
    int base = 0;
#pragma unroll 2
    for (int r = 0; r < kDsSeg / 4; r += 32) {
      const int wi = r + lane;  // word index in the segment
      const uint32_t w = __funnelshift_r(segw[wi], segw[wi + 1], sh);
      uint32_t keep = 0xFu;
      const int valid = seg_len - 4 * wi;  // bytes of this word inside the tile
      if (valid < 4) keep = valid <= 0 ? 0u : (1u << valid) - 1u;
      const uint32_t low = ~((w | 0x80808080u) - 0x21212121u) & ~w & 0x80808080u;  // bytes < 0x21
      if (low) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (is_space((w >> (8 * j)) & 0xFFu)) keep &= ~(1u << j);
      }
      const int c = __popc(keep);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      uint8_t *p = run + base + (incl - c);
      if (keep == 0xFu) {
        p[0] = static_cast<uint8_t>(w);
        p[1] = static_cast<uint8_t>(w >> 8);
        p[2] = static_cast<uint8_t>(w >> 16);
        p[3] = static_cast<uint8_t>(w >> 24);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (keep & (1u << j)) *p++ = static_cast<uint8_t>(w >> (8 * j));
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) S.cnt[warp] = base;
    __syncthreads();

    // ---- block scan of the run lengths + decoupled look-back over tiles
    if (warp == 0) {
      const int c = lane < kDsWarps ? S.cnt[lane] : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      if (lane < kDsWarps) S.wexcl[lane] = incl - c;
      const uint64_t agg = static_cast<uint64_t>(__shfl_sync(0xffffffffu, incl, 31));
      // Decoupled look-back, one warp, 32 predecessors per step: publish
      // this tile's aggregate, then walk back until the closest tile that
      // has published an inclusive prefix.
      uint64_t excl = 0;
      if (t == 0) {
        if (lane == 0) atomicExch(state + 0, kDsFlagPre | agg);
      } else {
        if (lane == 0) atomicExch(state + t, kDsFlagAgg | agg);
        int64_t j = t - 1;
        for (;;) {
          const int64_t idx = j - lane;
          uint64_t st = kDsFlagPre;  // before tile 0: empty prefix
          if (idx >= 0) {
            do {
              st = *reinterpret_cast<volatile unsigned long long *>(state + idx);
            } while ((st >> 62) == 0);
          }
          const unsigned pre = __ballot_sync(0xffffffffu, (st >> 62) == 2);
          const int last = pre ? __ffs(pre) - 1 : 31;  // closest prefix (or the whole window)
          uint64_t v = lane <= last ? (st & kDsValMask) : 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          excl += v;
          if (pre) break;
          j -= 32;
        }
        if (lane == 0) atomicExch(state + t, kDsFlagPre | (excl + agg));
      }
      if (lane == 0) {
        S.excl = static_cast<int64_t>(excl);
        if (t == ntiles - 1) *out_len = static_cast<int64_t>(excl + agg);
      }
    }
    __syncthreads();

    // ---- write this warp's run at its global offset (realigned 16-byte stores)
    warp_copy_out(out + S.excl + S.wexcl[warp], run, S.cnt[warp], lane);
    fence_proxy_async_smem();  // generic reads of S.in[b] before its next bulk write
    __syncthreads();           // runs / S.in[b] reused by the next tiles
    t = S.tile;
  }
}

}  // namespace b64
