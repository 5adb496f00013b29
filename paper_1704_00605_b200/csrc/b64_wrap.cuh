// b64_wrap.cuh -- line-wrapped (MIME / PEM style) encode on the GPU
// (reading R-wrap in DESIGN.md §3): Algorithm 1
// (with the f1 variant flags) whose output carries an end-of-line
// sequence (LF or CR LF) after every `L` characters and after the final line.
//
// L is a multiple of 4, so a group (3 bytes -> 4 chars) never straddles a
// line: group g lands at line g / G, column 4 (g mod G) (G = L/4), i.e. at
// output offset (g / G)(L + e) + 4 (g mod G).  A tile is Lt whole lines
// (Lt * 3G <= kWrIn input bytes and Lt (L + e) <= B64_WR_OUT output bytes): the input window is TMA-staged (16-byte
// granules, any alignment), each thread encodes one group per step (lanes
// take consecutive groups, so the 2-byte / 1-byte stores of a warp hit
// consecutive shared-memory words), the group's line comes from one
// multiply-high by a precomputed reciprocal, and the tile's output -- staged
// congruent to its destination mod 16 -- leaves as one bulk (TMA) store
// of its aligned interior plus byte stores for the edges (B64_WR_BULK).
#pragma once
#include <cstdint>

#include "b64_codec.cuh"
#include "b64_compact.cuh"
#include "b64_ptx.cuh"

namespace b64 {

constexpr int kWrThreads = 512;
#ifndef B64_WR_IN
#define B64_WR_IN 21504
#endif
#ifndef B64_WR_OUT
#define B64_WR_OUT 28672
#endif
#ifndef B64_WR_BATCH  // fast path: groups per thread whose loads are issued together (0 = off)
#define B64_WR_BATCH 2
#endif
#ifndef B64_WR_BULK  // tile copy-out: one bulk (TMA) store by one thread instead of LDS.128 -> STG.128
#define B64_WR_BULK 1
#endif
#ifndef B64_WR_STAGES
#define B64_WR_STAGES 2
#endif
constexpr int kWrIn = B64_WR_IN;             // max input bytes per tile
constexpr int kWrStages = B64_WR_STAGES;
constexpr int kWrOut = B64_WR_OUT + 32;      // max output bytes per tile (+ staging slack)
constexpr int kWrMaxLine = 16384;            // line_chars limit (one line fits a tile)

struct WrGeom {
  int64_t n;       // input bytes
  int64_t m;       // encoded characters (Alg 1 + flags)
  int64_t ng;      // groups = ceil(n / 3)
  int64_t nlines;  // ceil(m / L)
  int64_t total;   // output bytes = m + e * nlines
  int L, e, G;     // line chars, EOL bytes, groups per line
  int Lt;          // lines per tile
  uint32_t inv;    // ceil(2^32 / G) (G > 1; G = 1 is special-cased)
};

struct alignas(128) WrSmem {
  uint8_t in[kWrStages][kWrIn + 64];
  alignas(16) uint8_t out[2][kWrOut];
  uint64_t full[kWrStages];
};

// 4 characters at p (U16: p is even -> two 2-byte stores).
template <bool U16>
__device__ __forceinline__ void store4(uint8_t *p, uint32_t c) {
  if (U16) {
    reinterpret_cast<uint16_t *>(p)[0] = static_cast<uint16_t>(c);
    reinterpret_cast<uint16_t *>(p)[1] = static_cast<uint16_t>(c >> 16);
  } else {
    p[0] = static_cast<uint8_t>(c);
    p[1] = static_cast<uint8_t>(c >> 8);
    p[2] = static_cast<uint8_t>(c >> 16);
    p[3] = static_cast<uint8_t>(c >> 24);
  }
}
template <bool U16, int E>
__device__ __forceinline__ void store_eol(uint8_t *q) {
  if (E == 2) {
    if (U16) {
      *reinterpret_cast<uint16_t *>(q) = 0x0A0Du;  // "\r\n"
    } else {
      q[0] = '\r';
      q[1] = '\n';
    }
  } else {
    q[0] = '\n';
  }
}

// E: end-of-line bytes (1 = LF, 2 = CR LF), W.e == E.  U16: E == 2 and the
// destination is even (every 4-char group lands on an even offset).
template <int E, bool U16>
__global__ void __launch_bounds__(kWrThreads, 2)
    encode_wrap_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, WrGeom W,
                       int64_t ntiles, int flags) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  WrSmem &S = *reinterpret_cast<WrSmem *>(smem_raw);
  const int tid = threadIdx.x;
  if (tid < 64) g_enc_tab[tid] = static_cast<uint8_t>(ascii_of(tid, flags));  // Table I / II
  if (tid == 0) {
    for (int s = 0; s < kWrStages; ++s) ptx::mbar_init(&S.full[s], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const bool pad = !(flags & kFlagNoPad);
  const int64_t tin = static_cast<int64_t>(W.Lt) * 3 * W.G;       // input bytes per tile
  const int64_t tout = static_cast<int64_t>(W.Lt) * (W.L + W.e);  // output bytes per tile
  const uint64_t pol = ptx::policy_evict_first();
  auto load = [&](int64_t t, int s) {
    const int64_t src = t * tin;
    const int64_t len = W.n - src < tin ? W.n - src : tin;
    const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src);
    const uintptr_t g0 = g & ~static_cast<uintptr_t>(15);
    const uintptr_t g1 = (g + static_cast<uintptr_t>(len) + 15) & ~static_cast<uintptr_t>(15);
    ptx::mbar_arrive_expect_tx(&S.full[s], static_cast<uint32_t>(g1 - g0));
    ptx::bulk_g2s(S.in[s], reinterpret_cast<const void *>(g0), static_cast<uint32_t>(g1 - g0),
                  &S.full[s], pol);
  };
  const int64_t t0 = blockIdx.x;
  if (tid == 0)
    for (int k = 0; k < kWrStages - 1 && t0 + k * gridDim.x < ntiles; ++k)
      load(t0 + k * gridDim.x, k);
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(g_enc_tab));
  const int S_line = W.L + E;
  const int64_t glast = W.ng - 1;
  const int rem = static_cast<int>(W.n % 3);  // bytes of the final group (0 = full)
  // thread-invariant walk of the fast path: group tid + 512 k
  const int line_t = tid / W.G, col_t = tid % W.G;
  const int p_t = line_t * S_line + 4 * col_t;
  const int dc = kWrThreads % W.G;
  const int pstep = (kWrThreads / W.G) * S_line + 4 * dc;
  int it = 0;
  for (int64_t t = t0; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % kWrStages, so = it & 1;
    if (tid == 0 && t + (kWrStages - 1) * static_cast<int64_t>(gridDim.x) < ntiles)
      load(t + (kWrStages - 1) * static_cast<int64_t>(gridDim.x), (it + kWrStages - 1) % kWrStages);
    const int64_t src = t * tin, dst = t * tout;
    const int64_t g0 = t * static_cast<int64_t>(W.Lt) * W.G;  // first group of the tile (= src / 3)
    const int64_t gend = (g0 + static_cast<int64_t>(W.Lt) * W.G) < W.ng
                             ? g0 + static_cast<int64_t>(W.Lt) * W.G : W.ng;
    const int ngrp = static_cast<int>(gend - g0);
    const int64_t dend = gend == W.ng ? W.total : dst + tout;
    const int olen = static_cast<int>(dend - dst);
    const int imis = static_cast<int>((reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src)) & 15);
    const int omis = static_cast<int>((reinterpret_cast<uintptr_t>(out) + static_cast<uintptr_t>(dst)) & 15);
    const uint32_t *win = reinterpret_cast<const uint32_t *>(S.in[s]);
    const int a_t = imis + 3 * tid;
    const uint32_t sh_t = 8u * static_cast<uint32_t>(a_t & 3);
    uint8_t *ob = S.out[so] + omis;
    ptx::mbar_wait_spin(&S.full[s], static_cast<uint32_t>((it / kWrStages) & 1));
    if (gend != W.ng) {
      // Fast path: a full tile (Lt whole lines, no tail group).  Every tile
      // starts on a line boundary and the stride 512 is a multiple of 4
      // bytes of input, so a thread's input word offset / byte shift and its
      // (line, column) walk are tile-invariant: no per-group division or
      // address arithmetic beyond one increment.
      const uint32_t *wp = win + (a_t >> 2);
      uint8_t *p = ob + p_t;
      int col = col_t;
      int g = tid;
#if B64_WR_BATCH
      // B64_WR_BATCH groups per step: every input / table load of the batch
      // is issued before its first store (the compiler does not move shared
      // loads above shared stores of the previous group on its own).
      constexpr int NB = B64_WR_BATCH;
      for (; g + (NB - 1) * kWrThreads < ngrp; g += NB * kWrThreads) {
        uint8_t *pb[NB];
        bool lb[NB];
        uint32_t x[NB], c[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          x[j] = __funnelshift_r(wp[0], wp[1], sh_t);
          pb[j] = p;
          lb[j] = col == W.G - 1;
          wp += 3 * kWrThreads / 4;
          p += pstep;
          col += dc;
          if (col >= W.G) {
            col -= W.G;
            p += E;
          }
        }
#pragma unroll
        for (int j = 0; j < NB; ++j) c[j] = enc_group<true>(__byte_perm(x[j], 0u, 0x4012), tb);
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          store4<U16>(pb[j], c[j]);
          if (lb[j]) store_eol<U16, E>(pb[j] + 4);
        }
      }
#endif
#pragma unroll 4
      for (; g < ngrp; g += kWrThreads) {
        const uint32_t x = __funnelshift_r(wp[0], wp[1], sh_t);
        const uint32_t c = enc_group<true>(__byte_perm(x, 0u, 0x4012), tb);
        store4<U16>(p, c);
        if (col == W.G - 1) store_eol<U16, E>(p + 4);
        wp += 3 * kWrThreads / 4;
        p += pstep;
        col += dc;
        if (col >= W.G) {
          col -= W.G;
          p += E;
        }
      }
    } else {
      for (int g = tid; g < ngrp; g += kWrThreads) {
        const int a = imis + 3 * g;
        const uint32_t x = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
        const bool fin = g0 + g == glast;
        const int kb = fin && rem ? rem : 3;  // input bytes of this group
        const uint32_t xm = kb == 3 ? x : x & (kb == 1 ? 0xFFu : 0xFFFFu);  // missing bytes = 0
        uint32_t c = enc_group<true>(__byte_perm(xm, 0u, 0x4012), tb);
        int nc = 4;  // characters emitted (Alg 1 tail)
        if (kb != 3) {
          if (pad) {
            c = kb == 1 ? (c & 0x0000FFFFu) | 0x3D3D0000u : (c & 0x00FFFFFFu) | 0x3D000000u;
          } else {
            nc = kb + 1;
          }
        }
        const uint32_t line =
            W.G == 1 ? static_cast<uint32_t>(g) : __umulhi(static_cast<uint32_t>(g), W.inv);
        const int col = g - static_cast<int>(line) * W.G;
        uint8_t *p = ob + static_cast<int>(line) * S_line + 4 * col;
        for (int k = 0; k < nc; ++k) p[k] = static_cast<uint8_t>(c >> (8 * k));
        if (col == W.G - 1 || fin) {  // end of a line: EOL after its last character
          uint8_t *q = p + nc;
          if (W.e == 2) {
            q[0] = '\r';
            q[1] = '\n';
          } else {
            q[0] = '\n';
          }
        }
      }
    }
    ptx::fence_proxy_async_smem();  // generic reads of in[s] / writes of out[so] vs the async proxy
#if B64_WR_BULK
    // the bulk store of the previous tile (other buffer) must have finished
    // reading before the barrier that lets the next tile overwrite it
    if (tid == 0) ptx::bulk_wait_read<0>();
#endif
    __syncthreads();
#if B64_WR_BULK
    // the 16-byte aligned interior leaves with one bulk store (staging is
    // congruent to the destination mod 16), the edges with byte stores
    cta_copy_out_bulk(out + dst, ob, olen, pol);
#else
    cta_copy_out_congruent(out + dst, ob, olen);
#endif
  }
#if B64_WR_BULK
  if (tid == 0) ptx::bulk_wait<0>();
#endif
}

}  // namespace b64
