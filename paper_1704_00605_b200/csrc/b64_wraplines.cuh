// b64_wraplines.cuh -- line-major line-wrapped encode (SURVEY.md §8(f) row
// f4, reading R-wrap in DESIGN.md §3) for lines of L <= 128 characters:
// Algorithm 1 (f1 variant flags) with an end-of-line sequence
// (LF or CR LF) after every L characters and after the final line.
//
// The line-major counterpart of decode_lines_kernel (b64_wslines.cuh): a
// full line takes exactly 3G input bytes (G = L / 4 groups) and gives
// L + e output bytes, so line k reads in[3Gk ..) and writes out[(L + e)k ..).
// A producer warp streams tiles of Lt whole lines' input into a 2-stage
// TMA ring; each compute warp takes blocks of 32 (or 64, two per lane)
// lines, one lane per line: the lane's input bytes are consecutive in the
// window (3 words give 4 groups, one funnel shift each, the shift fixed per
// line) and its L + e output bytes consecutive in the warp's staging slice
// (each group's 4 characters = one stream word, stored as an aligned STS.32
// funnel-shifted by the line's staging misalignment; the EOL and the <= 3
// bytes before the first / after the last aligned word are merged at the
// line's ends).  The block then leaves as one bulk (TMA) store of its
// 16-byte aligned interior issued by lane 0 (the edges byte-wise); the
// warp's next block waits for that store's shared-memory read before it
// stages (B64_EL_BULK; LDS.128 -> STG.128 by the warp: 0.475 vs 0.363 ms on
// the mime workload).  The final line
// when it is partial (its groups hold < 3G bytes: shorter line, Alg 1 tail,
// '=' padding or NOPAD) is written by warp 0 with byte stores.
#pragma once
#include <cstdint>

#include "b64_codec.cuh"
#include "b64_ptx.cuh"
#include "b64_wslines.cuh"

namespace b64 {

constexpr int kElWarps = 16;                    // compute warps
constexpr int kElThreads = kElWarps * 32 + 32;  // + one producer (TMA) warp
constexpr int kElStages = 2;
constexpr int kElIn = 1024 * 57;                // max input bytes per tile (1,024 MIME lines)
constexpr int kElMaxG = 32;                     // L <= 128
constexpr int kElSlice = 64 * 78 + 16;          // one 64-line block of 78 bytes (or 32 of 130) + misalignment

struct ElGeom {
  int64_t n;       // input bytes
  int64_t m;       // encoded characters (Alg 1 + flags)
  int64_t nlines;  // ceil(m / L)
  int64_t nfull;   // lines whose 3G input bytes all exist (n / 3G)
  int64_t ntiles;
  int L, e, G, Lt;  // line chars, EOL bytes, groups per line, lines per tile
  int strd;         // lanes -> lines: 1 (32-line blocks) or 2 (64-line blocks)
};

struct alignas(128) ElSmem {
  uint8_t in[kElStages][kElIn + 64];
  alignas(16) uint8_t out[kElWarps][kElSlice];
  uint64_t full[kElStages];
  uint64_t empty[kElStages];
};

// P full lines li0 .. li0 + P - 1 of a block (first line l0 of the tile),
// interleaved per lane: input window `win` (the tile's first byte at imis),
// output staged at slice[om + (L + e) li].
template <int P, int E>
__device__ __forceinline__ void el_lines(const uint32_t *win, uint8_t *slice, int imis, int G, int om,
                                         int l0, int li0, uint32_t tb) {
  const int Sl = 4 * G + E;
  constexpr uint32_t eolw = E == 2 ? 0x0A0Du : 0x0Au;
  const uint32_t *lw[P];
  uint8_t *sb[P];
  uint32_t *sw[P];
  uint32_t ish[P], dsh[P], lo[P], carry[P], c0[P];
  int d[P], tmax[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int li = li0 + p;
    const int a = imis + 3 * G * (l0 + li);  // the line's first input byte in the window
    lw[p] = win + (a >> 2);
    ish[p] = 8u * static_cast<uint32_t>(a);  // funnel shift, mod 32
    const int o = om + Sl * li;              // output byte i of the line -> slice[o + i]
    d[p] = (-o) & 3;                         // bytes before the first aligned word
    dsh[p] = 8u * static_cast<uint32_t>(d[p]);
    sb[p] = slice + o;
    sw[p] = reinterpret_cast<uint32_t *>(sb[p] + d[p]);  // aligned word t = stream bytes d + 4t ..
    tmax[p] = ((Sl - d[p]) >> 2) - 1;                     // last aligned word inside the line
    lo[p] = lw[p][0];
    carry[p] = 0;
    c0[p] = 0;
  }
  // 4 groups from 12 input bytes (3 stream words), characters = stream words
  // g .. g + 3; aligned word t = g - 1 needs stream words g - 1 and g
  auto chunk = [&](int p, int k, uint32_t (&c)[4]) {
    const uint32_t w1 = lw[p][k + 1], w2 = lw[p][k + 2], w3 = lw[p][k + 3];
    const uint32_t s0 = __funnelshift_r(lo[p], w1, ish[p]), s1 = __funnelshift_r(w1, w2, ish[p]),
                   s2 = __funnelshift_r(w2, w3, ish[p]);
    lo[p] = w3;
    c[0] = enc_group<true>(__byte_perm(s0, 0u, 0x4012), tb);  // Alg 1
    c[1] = enc_group<false>(__byte_perm(s0, s1, 0x3345), tb);
    c[2] = enc_group<false>(__byte_perm(s1, s2, 0x2234), tb);
    c[3] = enc_group<true>(__byte_perm(s2, 0u, 0x4123), tb);
  };
  // first chunk (groups 0..3; fewer when G < 4): no word -1 (the head bytes)
#pragma unroll
  for (int p = 0; p < P; ++p) {
    uint32_t c[4];
    chunk(p, 0, c);
    c0[p] = c[0];
    if (1 < G) sw[p][0] = __funnelshift_r(c[0], c[1], dsh[p]);
    if (2 < G) sw[p][1] = __funnelshift_r(c[1], c[2], dsh[p]);
    if (3 < G) sw[p][2] = __funnelshift_r(c[2], c[3], dsh[p]);
    carry[p] = G == 1 ? c[0] : G == 2 ? c[1] : G == 3 ? c[2] : c[3];
  }
  // whole chunks: four aligned words each, all inside the line
  int g = 4, k = 3;
  for (; g + 4 <= G; g += 4, k += 3) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      uint32_t c[4];
      chunk(p, k, c);
      sw[p][g - 1] = __funnelshift_r(carry[p], c[0], dsh[p]);
      sw[p][g] = __funnelshift_r(c[0], c[1], dsh[p]);
      sw[p][g + 1] = __funnelshift_r(c[1], c[2], dsh[p]);
      sw[p][g + 2] = __funnelshift_r(c[2], c[3], dsh[p]);
      carry[p] = c[3];
    }
  }
  if (g < G) {  // the last 1-3 groups
    const int r = G - g;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      uint32_t c[4];
      chunk(p, k, c);
      sw[p][g - 1] = __funnelshift_r(carry[p], c[0], dsh[p]);
      if (r > 1) sw[p][g] = __funnelshift_r(c[0], c[1], dsh[p]);
      if (r > 2) sw[p][g + 1] = __funnelshift_r(c[1], c[2], dsh[p]);
      carry[p] = r == 1 ? c[0] : r == 2 ? c[1] : c[2];
    }
  }
  // the end of the line: stream words G - 1 (carry) and G (the EOL) --
  // aligned words G - 1 and G where inside, the rest byte-wise; the head
  // bytes [0, d) from the first group
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (G - 1 <= tmax[p]) sw[p][G - 1] = __funnelshift_r(carry[p], eolw, dsh[p]);
    if (G <= tmax[p]) sw[p][G] = __funnelshift_r(eolw, 0u, dsh[p]);
    const int T = d[p] + 4 * (tmax[p] + 1);  // first byte after the last aligned word
    const uint64_t X = static_cast<uint64_t>(carry[p]) | (static_cast<uint64_t>(eolw) << 32);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i < d[p]) sb[p][i] = static_cast<uint8_t>(c0[p] >> (8 * i));
      const int q = Sl - 3 + i;  // one of the line's last 3 bytes
      if (q >= T) sb[p][q] = static_cast<uint8_t>(X >> (8 * (q - 4 * (G - 1))));
    }
  }
}

template <int E>
__global__ void __launch_bounds__(kElThreads, 1)
    encode_lines_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, ElGeom W, int flags) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  ElSmem &S = *reinterpret_cast<ElSmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 64) g_enc_tab[tid] = static_cast<uint8_t>(ascii_of(tid, flags));  // Table I / II
  if (tid == 0) {
    for (int s = 0; s < kElStages; ++s) {
      ptx::mbar_init(&S.full[s], 1);
      ptx::mbar_init(&S.empty[s], kElWarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int G = W.G, Sl = W.L + E, Lt = W.Lt;
  const int64_t tin = static_cast<int64_t>(Lt) * 3 * G;  // input bytes per tile
  if (warp == kElWarps) {
    // ---- producer: lane 0 streams each tile's input bytes into the ring
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      int k = 0;
      for (int64_t t = blockIdx.x; t < W.ntiles; t += gridDim.x, ++k) {
        const int s = k % kElStages;
        if (k >= kElStages) ptx::mbar_wait(&S.empty[s], static_cast<uint32_t>((k / kElStages - 1) & 1));
        const int64_t src = t * tin;
        const int64_t len = W.n - src < tin ? W.n - src : tin;
        const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src);
        const uintptr_t g0 = g & ~static_cast<uintptr_t>(15);
        const uintptr_t g1 = (g + static_cast<uintptr_t>(len) + 15) & ~static_cast<uintptr_t>(15);
        ptx::mbar_arrive_expect_tx(&S.full[s], static_cast<uint32_t>(g1 - g0));
        ptx::bulk_g2s(S.in[s], reinterpret_cast<const void *>(g0), static_cast<uint32_t>(g1 - g0),
                      &S.full[s], pol);
      }
    }
    return;
  }
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(g_enc_tab));
  const bool pad = !(flags & kFlagNoPad);
  uint8_t *slice = S.out[warp];
  const int strd = W.strd;
#if B64_EL_BULK
  const uint64_t pol = ptx::policy_evict_first();
  bool bulk_pending = false;
#endif
  int k = 0;
  for (int64_t t = blockIdx.x; t < W.ntiles; t += gridDim.x, ++k) {
    const int s = k % kElStages;
    ptx::mbar_wait_spin(&S.full[s], static_cast<uint32_t>((k / kElStages) & 1));
    const int64_t line0 = t * Lt;
    const int64_t src = line0 * 3 * G;
    const int imis = static_cast<int>((reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src)) & 15);
    const uint32_t *win = reinterpret_cast<const uint32_t *>(S.in[s]);
    // full lines of this tile: [0, nlf)
    const int64_t fl = W.nfull - line0;
    const int nlf = fl <= 0 ? 0 : (fl < Lt ? static_cast<int>(fl) : Lt);
    const int BL = 32 * strd;
    const int nblk = (nlf + BL - 1) >> (strd == 2 ? 6 : 5);
    for (int blk = warp; blk < nblk; blk += kElWarps) {
      const int l0 = blk * BL;
      const int nl = nlf - l0 < BL ? nlf - l0 : BL;
      uint8_t *gb = out + (line0 + l0) * Sl;
      const int om = static_cast<int>(reinterpret_cast<uintptr_t>(gb) & 15);
#if B64_EL_BULK
      if (bulk_pending) {
        if (lane == 0) ptx::bulk_wait_read<0>();
        bulk_pending = false;
      }
#endif
      __syncwarp();  // the previous block's copy-out has read the slice
      if (strd == 2 && nl == 64) {
        el_lines<2, E>(win, slice, imis, G, om, l0, 2 * lane, tb);
      } else {
        for (int pass = 0; pass < strd; ++pass) {
          const int li = strd * lane + pass;
          if (li < nl) el_lines<1, E>(win, slice, imis, G, om, l0, li, tb);
        }
      }
#if B64_EL_BULK
      ptx::fence_proxy_async_smem();  // this lane's staging stores vs the bulk store
#endif
      __syncwarp();
      // the block's nl (L + e) bytes, staged congruent to gb mod 16
      const int nb = nl * Sl;
      const uint8_t *src8 = slice + om;
      const uintptr_t g = reinterpret_cast<uintptr_t>(gb);
      const uintptr_t ga = (g + 15) & ~static_cast<uintptr_t>(15);
      const uintptr_t ge = (g + static_cast<uintptr_t>(nb)) & ~static_cast<uintptr_t>(15);
#if B64_EL_BULK
      // the aligned interior as one bulk (TMA) store by lane 0, the edges
      // byte-wise; the next block's staging waits for the bulk read
      if (ge > ga) {
        const int head = static_cast<int>(ga - g), tail0 = static_cast<int>(ge - g);
        if (lane == 0) {
          ptx::bulk_s2g(gb + head, src8 + head, static_cast<uint32_t>(ge - ga), pol);
          ptx::bulk_commit();
        }
        if (lane < head) gb[lane] = src8[lane];
        if (lane >= 16 && lane - 16 < nb - tail0) gb[tail0 + lane - 16] = src8[tail0 + lane - 16];
      } else {
        for (int i = lane; i < nb; i += 32) gb[i] = src8[i];
      }
      bulk_pending = true;
#else
      if (ge > ga) {
        const int head = static_cast<int>(ga - g), ng = static_cast<int>((ge - ga) >> 4);
        uint32_t sa = ptx::smem_u32(src8 + head) + 16u * lane;
        uint4 *gp = reinterpret_cast<uint4 *>(gb + head) + lane;
        for (int i = lane; i < ng; i += 32, sa += 512u, gp += 32) *gp = ptx::lds128_a(sa);
        const int tail0 = static_cast<int>(ge - g);
        if (lane < head) gb[lane] = src8[lane];
        if (lane >= 16 && lane - 16 < nb - tail0) gb[tail0 + lane - 16] = src8[tail0 + lane - 16];
      } else {
        for (int i = lane; i < nb; i += 32) gb[i] = src8[i];
      }
#endif
    }
    // the final line when it is partial (< 3G input bytes): warp 0, one group
    // per lane, byte stores (Alg 1 tail and padding)
    if (warp == 0 && W.nfull < W.nlines && W.nfull >= line0 && W.nfull < line0 + Lt) {
      const int64_t b0 = W.nfull * 3 * G;             // first input byte of the final line
      const int nbytes = static_cast<int>(W.n - b0);  // 1 .. 3G - 1
      const int ngr = (nbytes + 2) / 3;
      const int a = imis + static_cast<int>(b0 - src);
      uint8_t *po = out + W.nfull * Sl;
      const int chars = static_cast<int>(W.m - W.nfull * W.L);  // 1 .. L
      for (int g = lane; g < ngr; g += 32) {
        const int ab = a + 3 * g;
        const uint32_t x = __funnelshift_r(win[ab >> 2], win[(ab >> 2) + 1], 8 * (ab & 3));
        const int kb = nbytes - 3 * g < 3 ? nbytes - 3 * g : 3;  // input bytes of this group
        const uint32_t xm = kb == 3 ? x : x & (kb == 1 ? 0xFFu : 0xFFFFu);  // missing bytes = 0
        uint32_t c = enc_group<true>(__byte_perm(xm, 0u, 0x4012), tb);
        int nc = 4;
        if (kb != 3) {
          if (pad) c = kb == 1 ? (c & 0x0000FFFFu) | 0x3D3D0000u : (c & 0x00FFFFFFu) | 0x3D000000u;
          else nc = kb + 1;
        }
        for (int i = 0; i < nc; ++i) po[4 * g + i] = static_cast<uint8_t>(c >> (8 * i));
      }
      if (lane == 0) {
        po[chars] = E == 2 ? '\r' : '\n';
        if (E == 2) po[chars + 1] = '\n';
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&S.empty[s]);
  }
#if B64_EL_BULK
  if (lane == 0) ptx::bulk_wait<0>();
#endif
}

}  // namespace b64
