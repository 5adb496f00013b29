// b64_wslines.cuh -- verified fast path of the whitespace-tolerant decode
// (reading R-ws-decode) for line-structured text,
// i.e. MIME / PEM: every line holds the same number L of characters (L a
// multiple of 4) followed by the same end-of-line sequence (LF or CR LF);
// the last line holds 1..L characters, with or without the EOL; there is no
// other white space.  Then the i-th kept character sits at original offset
// (i / L)(L + e) + i mod L, so every quad is decoded straight from the
// TMA-staged text -- no mask pass, no compaction.  Interior tiles of short
// lines (L <= 128) are decoded line-major (lm_lines: one lane per line, each
// window word loaded once, output staged per block of lines); other tiles
// flat (lanes take consecutive quads across line ends).
//
// The structure is an assumption each launch VERIFIES, never trusts: L and
// the EOL come from the first line (read by every CTA), the tail from the
// last bytes, and every tile checks the EOL bytes of its lines and decodes
// every character through the validity table (white space inside a line is
// an invalid entry).  Any violation -- and any decoding error, which is
// rare -- makes the launch give up: its verdict is 0 and the general path
// (cp_mask_kernel + decode_ws_kernel) runs and writes every output byte and
// the result record.  On success the verdict is 1 and both general kernels
// return at once.  Results are therefore always those of the general
// definition (App. B filter, then Algorithm 2).
#pragma once
#include <cstdint>

#include "b64_codec.cuh"
#include "b64_compact.cuh"
#include "b64_ptx.cuh"

namespace b64 {

#ifndef B64_WL_WARPS
#define B64_WL_WARPS 16
#endif
constexpr int kWlWarps = B64_WL_WARPS;             // compute warps
constexpr int kWlThreads = kWlWarps * 32 + 32;    // + one producer (TMA) warp
#ifndef B64_WL_TILE
#define B64_WL_TILE 79872
#endif
#ifndef B64_WL_SLEEP  // producer back-off between empty-slot polls (ns); 0 = try_wait loop
#define B64_WL_SLEEP 0
#endif
#ifndef B64_WL_BATCH  // interior loop: quads per thread whose loads are issued together (0 = off)
#define B64_WL_BATCH 4
#endif
#ifndef B64_WL_DIRECT  // interior tiles: shuffle-packed 4-byte stores from registers
#define B64_WL_DIRECT 1
#endif
constexpr bool kWlDirect = B64_WL_DIRECT != 0;
constexpr bool kWlLineMajor = B64_WL_LINEMAJOR != 0;
constexpr int kWlLmMaxG = 32;  // quads per line up to which the line-major path runs
// Line-major lane -> line map: stride 1 (lane l: line l of a 32-line block)
// or 2 (lane l: lines 2l and 2l + 1 of a 64-line block, two passes), per
// (G, e) whichever gives fewer shared-memory bank conflicts on the staging
// stores (lanes 3G or 6G bytes apart) and the window loads (L + e or
// 2(L + e) bytes apart) -- from a bank simulation of both maps, bit
// G - 1 + 32 (e - 1) set = stride 2 (G <= 19: 64 lines of staging fit).
constexpr uint64_t kWlLmStride2 = 0x77f7800072620ull;
__host__ __device__ __forceinline__ int lm_stride(int G, int e) {
  return ((kWlLmStride2 >> (G - 1 + 32 * (e - 1))) & 1) ? 2 : 1;
}
#ifndef B64_WL_STAGES
#define B64_WL_STAGES 2
#endif
constexpr int kWlTile = B64_WL_TILE;    // max input bytes per tile (whole lines)
constexpr int kWlStages = B64_WL_STAGES;
constexpr int kWlMaxLine = 4092;      // longest line the fast path takes
// per-warp output slice: a warp owns a contiguous range of <= ceil(quads/16)
// quads of a tile, rounded up to whole 32-quad rows
constexpr int kWlWarpQuads = ((kWlTile / 4 + kWlWarps - 1) / kWlWarps + 31) / 32 * 32;
// (at least one 64-line line-major block of 57-byte lines + 16 B of misalignment)
constexpr int kWlSlice = 3 * kWlWarpQuads + 48 > 3696 ? 3 * kWlWarpQuads + 48 : 3696;

// Per-call state in the caller's workspace (zeroed by a 16-byte memset
// before the launch).
struct WlState {
  int32_t verdict;  // 1: the fast path produced the result; 0: fall back
  int32_t viol;     // set by any CTA that sees a violation or an error
  uint32_t done;    // CTAs finished
  int32_t pad;
};

// Despace (DS) ring: its line-major copy is cheap enough that the input
// pipeline depth decides, so it takes more, smaller stages than the decode
#ifndef B64_DS_TILE
#define B64_DS_TILE 49920
#endif
#ifndef B64_DS_STAGES
#define B64_DS_STAGES 3
#endif
template <bool DS>
struct WlCfg {
  static constexpr int kTile = DS ? B64_DS_TILE : kWlTile;
  static constexpr int kStages = DS ? B64_DS_STAGES : kWlStages;
  static constexpr int kWarpQuads = ((kTile / 4 + kWlWarps - 1) / kWlWarps + 31) / 32 * 32;
  static constexpr int kSlice = 3 * kWarpQuads + 48 > 3696 ? 3 * kWarpQuads + 48 : 3696;
};

template <bool DS>
struct alignas(128) WlSmemT {
  uint8_t in[WlCfg<DS>::kStages][WlCfg<DS>::kTile + 64];
  alignas(16) uint8_t out[kWlWarps][WlCfg<DS>::kSlice];
  uint64_t full[WlCfg<DS>::kStages];
  uint64_t empty[WlCfg<DS>::kStages];
  int64_t geo[4];   // Mc (kept chars), nlines, ok
  int32_t Le[2];    // L, e
  int32_t flag;
};
using WlSmem = WlSmemT<false>;

// Any byte of w below 0x21 (' ', '\n', '\r' and the other control bytes):
// the classic "has less than" SWAR test, exact as an any-test for bytes
// < 0x80 (bytes >= 0x80 never match).
__device__ __forceinline__ bool has_below_0x21(uint32_t w) {
  return ((w - 0x21212121u) & ~w & 0x80808080u) != 0u;
}

// Line-major decode of P consecutive lines li0 .. li0 + P - 1 of a block
// (first line l0 of the tile) by one lane, interleaved for ILP: each line's
// quads are consecutive in the window (each word loaded once, one funnel
// shift per quad), its 3G output bytes consecutive in the warp's staging
// slice at om + 3 G li: every 4 quads give 3 stream words, stored as 3
// aligned STS.32 funnel-shifted by the line's staging misalignment d; the
// <= 3 bytes before the first / after the last aligned word are byte stores
// from the first / last quad.  Bad characters and a wrong EOL set 0x80 in bad.
template <int P>
__device__ __forceinline__ void lm_lines(const uint32_t *win, uint8_t *slice, int imis, int Sl, int L,
                                         int G, int om, int l0, int li0, uint32_t tb, uint32_t eolw,
                                         uint32_t eolm, uint32_t &bad) {
  const uint32_t *lw[P];
  uint8_t *sb[P];
  uint32_t *sw[P];
  uint32_t sh[P], dsh[P], lo[P], carry[P], vfirst[P], vlast[P];
  int d[P], tmax[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int li = li0 + p;
    const int a0 = imis + (l0 + li) * Sl;
    const int b = a0 + L;  // this line's EOL
    const uint32_t x = __funnelshift_r(win[b >> 2], win[(b >> 2) + 1], 8 * (b & 3));
    if ((x & eolm) != eolw) bad |= 0x80u;
    lw[p] = win + (a0 >> 2);
    sh[p] = 8u * static_cast<uint32_t>(a0);  // funnel shift, mod 32
    const int o = om + 3 * G * li;             // stream byte i -> slice[o + i]
    d[p] = (-o) & 3;                           // bytes before the first aligned word
    dsh[p] = 8u * static_cast<uint32_t>(d[p]);
    sb[p] = slice + o;
    sw[p] = reinterpret_cast<uint32_t *>(sb[p] + d[p]);  // aligned word t -> sw[t]
    tmax[p] = ((3 * G - d[p]) >> 2) - 1;                  // last aligned word inside the stream
    lo[p] = lw[p][0];
    carry[p] = 0;
    vfirst[p] = vlast[p] = 0;
  }
  auto quad = [&](int p, uint32_t hi) -> uint32_t {
    const uint32_t w = __funnelshift_r(lo[p], hi, sh[p]);
    lo[p] = hi;
    const uint32_t v0 = lds_u8((w & 0xFFu) | tb);
    const uint32_t v1 = lds_u8(__byte_perm(w, tb, 0x7651));
    const uint32_t v2 = lds_u8(__byte_perm(w, tb, 0x7652));
    const uint32_t v3 = lds_u8(__byte_perm(w, tb, 0x7653));
    bad |= v0 | v1 | v2 | v3;
    return ((v0 * 64u + v1) * 64u + v2) * 64u + v3;
  };
  // 4 quads (V0..V3: 24-bit, big-endian bytes) -> stream words S0 = b0 b1 b2
  // b3 ... (little-endian); aligned word t = bytes d + 4t .. of the stream
  auto emit = [&](int p, uint32_t V0, uint32_t V1, uint32_t V2, uint32_t V3, int t, int tm) {
    const uint32_t S0 = __byte_perm(V0, V1, 0x6012);
    const uint32_t S1 = __byte_perm(V1, V2, 0x5601);
    const uint32_t S2 = __byte_perm(V2, V3, 0x4560);
    if (t >= 0 && t <= tm) sw[p][t] = __funnelshift_r(carry[p], S0, dsh[p]);
    if (t + 1 <= tm) sw[p][t + 1] = __funnelshift_r(S0, S1, dsh[p]);
    if (t + 2 <= tm) sw[p][t + 2] = __funnelshift_r(S1, S2, dsh[p]);
    carry[p] = S2;
  };
  int c = 0, t = -1;
  for (; c + 4 <= G; c += 4, t += 3) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint32_t V0 = quad(p, lw[p][c + 1]);
      const uint32_t V1 = quad(p, lw[p][c + 2]);
      const uint32_t V2 = quad(p, lw[p][c + 3]);
      const uint32_t V3 = quad(p, lw[p][c + 4]);
      if (c == 0) vfirst[p] = V0;
      vlast[p] = V3;
      emit(p, V0, V1, V2, V3, t, 0x7fffffff);  // whole groups: every word inside
    }
  }
  const int r = G - c;  // the remaining 0-3 quads, then the words up to tmax
#pragma unroll
  for (int p = 0; p < P; ++p) {
    uint32_t V0 = 0, V1 = 0, V2 = 0;
    if (r > 0) V0 = quad(p, lw[p][c + 1]);
    if (r > 1) V1 = quad(p, lw[p][c + 2]);
    if (r > 2) V2 = quad(p, lw[p][c + 3]);
    if (c == 0) vfirst[p] = V0;
    if (r > 0) vlast[p] = r == 1 ? V0 : (r == 2 ? V1 : V2);
    emit(p, V0, V1, V2, 0u, t, tmax[p]);
    // head bytes [0, d) from the first quad, tail [T, 3G) from the last
    const int T = d[p] + 4 * (tmax[p] + 1);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i < d[p]) sb[p][i] = static_cast<uint8_t>(vfirst[p] >> (16 - 8 * i));
      if (3 * G - 3 + i >= T) sb[p][3 * G - 3 + i] = static_cast<uint8_t>(vlast[p] >> (16 - 8 * i));
    }
  }
}

// Despace line-major: line li of a block (first line l0 of the tile) -- its
// L = 4G characters go to slice[om + 4G li ..) word by word (funnel-shifted
// from the window, and to the slice's alignment when om is not a multiple
// of 4), each word checked for a byte < 0x21 (white space or a control
// byte inside a line: not line-structured); the EOL is checked too.
__device__ __forceinline__ void ds_line(const uint32_t *win, uint8_t *slice, int imis, int Sl, int L,
                                        int G, int om, int l0, int li, uint32_t eolw, uint32_t eolm,
                                        uint32_t &bad) {
  const int a0 = imis + (l0 + li) * Sl;
  {
    const int b = a0 + L;
    const uint32_t x = __funnelshift_r(win[b >> 2], win[(b >> 2) + 1], 8 * (b & 3));
    if ((x & eolm) != eolw) bad |= 0x80u;
  }
  const uint32_t *lw = win + (a0 >> 2);
  const uint32_t sh = 8u * static_cast<uint32_t>(a0);
  const int o = om + 4 * G * li;
  const int d = (-o) & 3;  // the same for every line of the block (4G = 0 mod 4)
  uint8_t *sb = slice + o;
  uint32_t *sw = reinterpret_cast<uint32_t *>(sb + d);
  uint32_t lo = lw[0], chk = 0;
  if (d == 0) {
#pragma unroll 4
    for (int j = 0; j < G; ++j) {
      const uint32_t hi = lw[j + 1];
      const uint32_t w = __funnelshift_r(lo, hi, sh);
      lo = hi;
      chk |= (w - 0x21212121u) & ~w;  // has_below_0x21, OR-ed over the line
      sw[j] = w;
    }
  } else {
    const uint32_t dsh = 8u * static_cast<uint32_t>(d);
    uint32_t prev = __funnelshift_r(lo, lw[1], sh), first = prev;
    lo = lw[1];
    chk |= (prev - 0x21212121u) & ~prev;
#pragma unroll 4
    for (int j = 1; j < G; ++j) {
      const uint32_t hi = lw[j + 1];
      const uint32_t w = __funnelshift_r(lo, hi, sh);
      lo = hi;
      chk |= (w - 0x21212121u) & ~w;
      sw[j - 1] = __funnelshift_r(prev, w, dsh);
      prev = w;
    }
    // head bytes [0, d) of the first word, tail: the last 4 - d bytes
    for (int i = 0; i < d; ++i) sb[i] = static_cast<uint8_t>(first >> (8 * i));
    for (int i = d; i < 4; ++i) sb[4 * G - 4 + i] = static_cast<uint8_t>(prev >> (8 * i));
  }
  if (chk & 0x80808080u) bad |= 0x80u;
}

// DS = false: the verified line-structured fast path of b64_decode_ws.
// DS = true: the same for b64_despace (Appendix B on MIME / PEM text): every
// quad of kept characters is copied to out + 4 q (a quad never straddles a
// line, L being a multiple of 4) with one coalesced 4-byte store per lane;
// a byte below 0x21 inside a line (white space, or a control byte despace
// would keep) is a violation, like a bad EOL, and the general two-pass path
// (cp_mask_kernel + despace_kernel) then produces the output.  On success
// *ds_out_len = the kept length.
template <bool DS>
__global__ void __launch_bounds__(kWlThreads, 1)
    decode_lines_kernel(const uint8_t *__restrict__ in, int64_t M, uint8_t *__restrict__ out,
                        WlState *st, b64_result *res, int flags, int64_t *ds_out_len) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using C = WlCfg<DS>;
  WlSmemT<DS> &S = *reinterpret_cast<WlSmemT<DS> *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 256) g_dec_tab[tid] = kInvalid;
  if (tid == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&S.full[s], 1);
      ptx::mbar_init(&S.empty[s], kWlWarps);
    }
    ptx::fence_mbar_init();
    S.flag = 0;
  }
  // ---- structure: L and the EOL from the first line, the last line from the tail
  if (warp == 0) {
    const int64_t lim = M < kWlMaxLine + 4 ? M : kWlMaxLine + 4;
    int64_t p = -1;
    for (int64_t x0 = 0; x0 < lim && p < 0; x0 += 32) {
      const int64_t x = x0 + lane;
      const unsigned b = __ballot_sync(0xffffffffu, x < lim && is_space_byte(in[x]));
      if (b) p = x0 + __ffs(b) - 1;
    }
    int L = 0, e = 0;
    bool ok = p > 0 && (p & 3) == 0 && p <= kWlMaxLine;
    if (ok) {
      L = static_cast<int>(p);
      const uint32_t c0 = in[p];
      if (c0 == '\n') e = 1;
      else if (c0 == '\r' && p + 1 < M && in[p + 1] == '\n') e = 2;
      else ok = false;
    }
    int64_t Mc = 0, nlines = 0;
    if (ok) {
      const int64_t Sl = L + e, nfull = M / Sl, tail = M - nfull * Sl;
      if (tail == 0) {
        nlines = nfull;
        Mc = nfull * L;
      } else {
        // trailing white space of the last segment: none, or exactly the EOL
        int k = 0;
        while (k < tail && k < 3 && is_space_byte(in[M - 1 - k])) ++k;
        const bool eol = k == e && (e == 1 ? in[M - 1] == '\n' : (in[M - 2] == '\r' && in[M - 1] == '\n'));
        const int64_t chars = tail - k;
        ok = (k == 0 || eol) && chars >= 1 && chars <= L;
        nlines = nfull + 1;
        Mc = nfull * L + chars;
      }
    }
    if (lane == 0) {
      S.Le[0] = L;
      S.Le[1] = e;
      S.geo[0] = Mc;
      S.geo[1] = nlines;
      S.geo[2] = ok ? 1 : 0;
    }
  }
  __syncthreads();
  if (tid < 64) g_dec_tab[ascii_of(tid, flags)] = static_cast<uint8_t>(tid);
  const int L = S.Le[0], e = S.Le[1];
  const int64_t Mc = S.geo[0], nlines = S.geo[1];
  const bool ok = S.geo[2] != 0;
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(g_dec_tab));
  bool viol = !ok;
  if (ok) {
    const int Sl = L + e, G = L / 4;
    // lines per tile: as many as fit (large tiles amortise the per-tile
    // work -- 28 KiB: 0.616 ms, 76 KiB: 0.529 ms on the mime workload), but
    // at least two tiles per CTA for small inputs
    int Lt = C::kTile / Sl;
    {
      const int64_t want = (nlines + 2 * static_cast<int64_t>(gridDim.x) - 1) / (2 * static_cast<int64_t>(gridDim.x));
      if (want < Lt) Lt = want < 1 ? 1 : static_cast<int>(want);
      // a multiple of 4 lines: 3 * (first quad of a tile) is then a multiple
      // of 4, so DIRECT stores stay 4-byte aligned in every tile
      if (kWlDirect) Lt = Lt < 4 ? 4 : Lt & ~3;
      // line-major tiles: a whole number of blocks per compute warp when
      // the tile holds at least one block per warp (load balance)
      if (!DS && kWlLineMajor && G <= kWlLmMaxG) {
        const int unit = kWlWarps * 32 * lm_stride(G, e);
        if (Lt >= unit) Lt -= Lt % unit;
      }
    }
    const int64_t ntiles = (nlines + Lt - 1) / Lt;
    const int64_t Q = Mc / 4;                             // complete quads
    const bool pads_ok = (Mc & 3) == 0;
    const uint32_t inv = G > 1 ? static_cast<uint32_t>(((1ull << 32) + G - 1) / G) : 0u;
    auto line_of = [&](int q) -> int {
      return G == 1 ? q : static_cast<int>(__umulhi(static_cast<uint32_t>(q), inv));
    };
    if (warp == kWlWarps) {
      // ---- producer: lane 0 streams whole-line tiles into the ring
      if (lane == 0) {
        const uint64_t pol = ptx::policy_evict_first();
        int k = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
          const int s = k % C::kStages;
          if (k >= C::kStages) {
            if (B64_WL_SLEEP > 0)
              ptx::mbar_wait_sleep(&S.empty[s], static_cast<uint32_t>((k / C::kStages - 1) & 1), B64_WL_SLEEP);
            else
              ptx::mbar_wait(&S.empty[s], static_cast<uint32_t>((k / C::kStages - 1) & 1));
          }
          const int64_t src = t * Lt * static_cast<int64_t>(Sl);
          const int64_t tl = static_cast<int64_t>(Lt) * Sl;
          const int64_t len = M - src < tl ? M - src : tl;
          const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src);
          const uintptr_t g0 = g & ~static_cast<uintptr_t>(15);
          const uintptr_t g1 = (g + static_cast<uintptr_t>(len) + 15) & ~static_cast<uintptr_t>(15);
          ptx::mbar_arrive_expect_tx(&S.full[s], static_cast<uint32_t>(g1 - g0));
          ptx::bulk_g2s(S.in[s], reinterpret_cast<const void *>(g0), static_cast<uint32_t>(g1 - g0),
                        &S.full[s], pol);
        }
      }
    } else {
      // ---- compute warps: each owns a contiguous range of the tile's quads
      // and writes its bytes itself (no CTA-wide barrier per tile)
      const uint32_t eolw = e == 2 ? 0x0A0Du : 0x0Au, eolm = e == 2 ? 0xFFFFu : 0xFFu;
      const int dl32 = 32 / G, dc32 = 32 % G;
      const int pstep = dl32 * Sl + 4 * dc32;
      uint8_t *slice = S.out[warp];
      // n staged bytes at src8 (congruent to gdst mod 16) -> 16-byte stores
      // of the aligned interior + byte stores for the edges (whole warp)
      auto copy_out = [lane](uint8_t *gdst, const uint8_t *src8, int n) {
        const uintptr_t g = reinterpret_cast<uintptr_t>(gdst);
        const uintptr_t ga = (g + 15) & ~static_cast<uintptr_t>(15);
        const uintptr_t gb = (g + static_cast<uintptr_t>(n)) & ~static_cast<uintptr_t>(15);
        if (gb > ga) {
          const int head = static_cast<int>(ga - g), ng = static_cast<int>((gb - ga) >> 4);
          uint32_t sa = ptx::smem_u32(src8 + head) + 16u * lane;
          uint4 *gp = reinterpret_cast<uint4 *>(gdst + head) + lane;  // (global: derived from out)
          for (int i = lane; i < ng; i += 32, sa += 512u, gp += 32) *gp = ptx::lds128_a(sa);
          const int tail0 = static_cast<int>(gb - g);
          if (lane < head) gdst[lane] = src8[lane];
          if (lane >= 16 && lane - 16 < n - tail0) gdst[tail0 + lane - 16] = src8[tail0 + lane - 16];
        } else {
          for (int i = lane; i < n; i += 32) gdst[i] = src8[i];
        }
      };
      // DIRECT packing: word j (lane j < 24) of a 96-byte run holds output
      // bytes 4j..4j+3 = bytes r.. of lane ps's 3 and the rest of lane ps+1's
      const int ps = lane < 24 ? (4 * lane) / 3 : 0, pr = 4 * lane - 3 * ps;
      const uint32_t psel = pr == 0 ? 0x4210u : (pr == 1 ? 0x5421u : 0x6542u);
#if B64_WL_BULK
      // line-major blocks leave as one bulk (TMA) store of their aligned
      // interior by lane 0 (edges byte-wise); the slice is restaged only
      // after that store has read it
      const uint64_t opol = ptx::policy_evict_first();
      bool bulk_pending = false;
      auto bulk_wait_slice = [&]() {
        if (bulk_pending) {
          if (lane == 0) ptx::bulk_wait_read<0>();
          bulk_pending = false;
        }
      };
      auto bulk_out = [&](uint8_t *gd, const uint8_t *src8, int n) {
        const uintptr_t g = reinterpret_cast<uintptr_t>(gd);
        const uintptr_t ga = (g + 15) & ~static_cast<uintptr_t>(15);
        const uintptr_t ge = (g + static_cast<uintptr_t>(n)) & ~static_cast<uintptr_t>(15);
        if (ge > ga) {
          const int head = static_cast<int>(ga - g), tail0 = static_cast<int>(ge - g);
          if (lane == 0) {
            ptx::bulk_s2g(gd + head, src8 + head, static_cast<uint32_t>(ge - ga), opol);
            ptx::bulk_commit();
          }
          if (lane < head) gd[lane] = src8[lane];
          if (lane >= 16 && lane - 16 < n - tail0) gd[tail0 + lane - 16] = src8[tail0 + lane - 16];
          bulk_pending = true;
        } else {
          for (int i = lane; i < n; i += 32) gd[i] = src8[i];
        }
      };
#endif
      int k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % C::kStages;
        ptx::mbar_wait_spin(&S.full[s], static_cast<uint32_t>((k / C::kStages) & 1));
        int stop = 0;
        // another CTA's violation only needs to stop this one eventually (the
        // verdict is decided at the end): poll the global flag every 8th tile
        if (lane == 0)
          stop = S.flag | ((k & 7) == 7 ? *reinterpret_cast<volatile int32_t *>(&st->viol) : 0);
        stop = __shfl_sync(0xffffffffu, stop, 0);
        if (!stop) {
          const int64_t src = t * Lt * static_cast<int64_t>(Sl);
          const int64_t q0 = t * Lt * static_cast<int64_t>(G);   // first quad of the tile
          const int64_t line0 = t * Lt;
          const int64_t q1 = q0 + static_cast<int64_t>(Lt) * G < Q ? q0 + static_cast<int64_t>(Lt) * G : Q;
          const int nq = static_cast<int>(q1 - q0);
          int per = (nq + kWlWarps - 1) / kWlWarps;
          per = (per + 31) & ~31;
          const int qa = warp * per < nq ? warp * per : nq;
          const int qb = qa + per < nq ? qa + per : nq;
          const int imis = static_cast<int>((reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src)) & 15);
          const uint32_t *win = reinterpret_cast<const uint32_t *>(S.in[s]);
          uint8_t *gdst = out + (DS ? 4 : 3) * (q0 + qa);
          const int omis = static_cast<int>(reinterpret_cast<uintptr_t>(gdst) & 15);
          uint8_t *ob = slice + omis - 3 * qa;  // quad q -> ob + 3q
          uint32_t bad = 0;
          const bool interior = q1 < Q && (line0 + Lt) * static_cast<int64_t>(Sl) <= M;
          // line-major (interior tiles, short lines): lane = line, below
          // (despace: odd G only -- lanes 4G bytes apart in the staging slice
          // are bank-conflict-free exactly when G is odd -- and 32 lines of
          // 4G bytes must fit the slice)
          const bool lmaj = kWlLineMajor && interior &&
                            (DS ? ((G & 1) != 0 && 128 * G + 16 <= C::kSlice) : G <= kWlLmMaxG);
          const bool direct = !DS && !lmaj && kWlDirect && interior &&
                              ((reinterpret_cast<uintptr_t>(gdst) & 3) == 0);
          if constexpr (DS) if (lmaj) {
            // despace, LINE-MAJOR: 32-line blocks, lane l line 32 b + l; its
            // L kept characters are copied (and checked) word by word into
            // the staging slice, the block leaves as one bulk store
            const int nblk = (Lt + 31) >> 5;
            for (int blk = warp; blk < nblk; blk += kWlWarps) {
              const int l0 = blk * 32;
              const int nl = Lt - l0 < 32 ? Lt - l0 : 32;
              uint8_t *gb = out + 4 * (q0 + static_cast<int64_t>(l0) * G);
              const int om = static_cast<int>(reinterpret_cast<uintptr_t>(gb) & 15);
#if B64_WL_BULK
              bulk_wait_slice();
#endif
              __syncwarp();
              if (lane < nl) ds_line(win, slice, imis, Sl, L, G, om, l0, lane, eolw, eolm, bad);
#if B64_WL_BULK
              ptx::fence_proxy_async_smem();
              __syncwarp();
              bulk_out(gb, slice + om, 4 * G * nl);
#else
              __syncwarp();
              copy_out(gb, slice + om, 4 * G * nl);
#endif
            }
          }
          if constexpr (DS) if (!lmaj) {
            // despace: each lane copies quads q = qa + lane + 32 i (the EOL
            // of every line is checked below); 4-byte aligned destination:
            // one coalesced STG.32 per quad, else byte stores
            const bool al4 = (reinterpret_cast<uintptr_t>(gdst) & 3) == 0;
            if (qa < qb) {
              int q = qa + lane;
              int ln = line_of(q), col = q - ln * G;
              int a = imis + ln * Sl + 4 * col;
              uint32_t *gw = reinterpret_cast<uint32_t *>(gdst) + lane;
              for (; q < qb; q += 32) {
                const uint32_t w = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
                if (has_below_0x21(w)) bad |= 0x80u;
                if (al4) {
                  *gw = w;
                } else {
                  uint8_t *p = gdst + 4 * (q - qa);
                  p[0] = static_cast<uint8_t>(w);
                  p[1] = static_cast<uint8_t>(w >> 8);
                  p[2] = static_cast<uint8_t>(w >> 16);
                  p[3] = static_cast<uint8_t>(w >> 24);
                }
                gw += 32;
                a += pstep;
                col += dc32;
                if (col >= G) {
                  col -= G;
                  a += e;
                }
              }
            }
          }
          if constexpr (!DS) if (lmaj) {
            // LINE-MAJOR: warp w takes 32-line blocks w, w + 16, ... of the
            // tile, lane l line 32 b + l.  A lane's quads are consecutive in
            // shared memory (each window word is loaded once, one funnel
            // shift per quad with a per-line shift) and its 3G output bytes
            // are consecutive in the warp's staging slice: every 4 quads
            // give 3 stream words, stored as 3 aligned STS.32 (funnel-shifted
            // by the lane's staging misalignment); the at most 3 bytes before
            // the first / after the last aligned word are byte stores from
            // the first / last quad.  Then the block's 96 G bytes go out as
            // 16-byte stores (copy_out).  No per-quad line bookkeeping.
            const int strd = lm_stride(G, e);
            const int BL = 32 * strd;  // lines per block
            const int nblk = (Lt + BL - 1) >> (strd == 2 ? 6 : 5);
            for (int blk = warp; blk < nblk; blk += kWlWarps) {
              const int l0 = blk * BL;
              const int nl = Lt - l0 < BL ? Lt - l0 : BL;
              uint8_t *gb = out + 3 * (q0 + static_cast<int64_t>(l0) * G);
              const int om = static_cast<int>(reinterpret_cast<uintptr_t>(gb) & 15);
#if B64_WL_BULK
              bulk_wait_slice();
#endif
              __syncwarp();  // the previous block's copy-out has read the slice
              if (strd == 2 && nl == 64) {
                // full 64-line block: the lane's two lines interleaved (ILP)
                lm_lines<2>(win, slice, imis, Sl, L, G, om, l0, 2 * lane, tb, eolw, eolm, bad);
              } else {
                for (int pass = 0; pass < strd; ++pass) {
                  const int li = strd * lane + pass;  // this lane's line in the block
                  if (li < nl) lm_lines<1>(win, slice, imis, Sl, L, G, om, l0, li, tb, eolw, eolm, bad);
                }
              }
#if B64_WL_BULK
              ptx::fence_proxy_async_smem();  // this lane's staging stores vs the bulk store
              __syncwarp();
              bulk_out(gb, slice + om, 3 * G * nl);
#else
              __syncwarp();
              copy_out(gb, slice + om, 3 * G * nl);
#endif
            }
          }
#if B64_WL_BULK
          if (!lmaj) {
            bulk_wait_slice();  // a staged path below may restage the slice
            __syncwarp();
          }
#endif
          if constexpr (!DS) if (!lmaj) {
          // DIRECT (B64_WL_DIRECT, 4-byte aligned output): interior warps pack
          // 32 lanes' 3-byte results into 24 words with two shuffles and write
          // them with one coalesced 4-byte store per lane -- no staging slice,
          // no copy-out (3 STS.U8 + 0.75 LDS.128 per 32 quads -> 2 SHFL)
          if (direct && qa < qb) {
            int q = qa + lane;
            int ln = line_of(q), col = q - ln * G;
            int a = imis + ln * Sl + 4 * col;
            uint32_t *gw = reinterpret_cast<uint32_t *>(gdst) + lane;  // word lane of each 96-byte run
            int qs = qa;  // first quad of the warp's current 32-quad row
            constexpr int NB = B64_WL_BATCH > 0 ? B64_WL_BATCH : 1;
            for (; qs + 32 * NB <= qb; qs += 32 * NB) {
              uint32_t wv[NB];
#pragma unroll
              for (int j = 0; j < NB; ++j) {
                wv[j] = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
                a += pstep;
                col += dc32;
                if (col >= G) {
                  col -= G;
                  a += e;
                }
              }
              uint32_t vv[NB][4];
#pragma unroll
              for (int j = 0; j < NB; ++j) {
                vv[j][0] = lds_u8((wv[j] & 0xFFu) | tb);
                vv[j][1] = lds_u8(__byte_perm(wv[j], tb, 0x7651));
                vv[j][2] = lds_u8(__byte_perm(wv[j], tb, 0x7652));
                vv[j][3] = lds_u8(__byte_perm(wv[j], tb, 0x7653));
              }
#pragma unroll
              for (int j = 0; j < NB; ++j) {
                bad |= vv[j][0] | vv[j][1] | vv[j][2] | vv[j][3];
                const uint32_t V = ((vv[j][0] * 64u + vv[j][1]) * 64u + vv[j][2]) * 64u + vv[j][3];
                const uint32_t b = __byte_perm(V, 0u, 0x4012);  // output bytes 3l..3l+2, little-endian
                const uint32_t x = __shfl_sync(0xffffffffu, b, ps);
                const uint32_t y = __shfl_sync(0xffffffffu, b, ps + 1);
                if (lane < 24) gw[24 * j] = __byte_perm(x, y, psel);
              }
              gw += 24 * NB;
              q += 32 * NB;
            }
            for (; qs < qb; qs += 32) {
              const bool act = q < qb;
              uint32_t V = 0;
              if (act) {
                const uint32_t w = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
                const uint32_t v0 = lds_u8((w & 0xFFu) | tb);
                const uint32_t v1 = lds_u8(__byte_perm(w, tb, 0x7651));
                const uint32_t v2 = lds_u8(__byte_perm(w, tb, 0x7652));
                const uint32_t v3 = lds_u8(__byte_perm(w, tb, 0x7653));
                bad |= v0 | v1 | v2 | v3;
                V = ((v0 * 64u + v1) * 64u + v2) * 64u + v3;
              }
              if (qs + 32 <= qb) {
                const uint32_t b = __byte_perm(V, 0u, 0x4012);
                const uint32_t x = __shfl_sync(0xffffffffu, b, ps);
                const uint32_t y = __shfl_sync(0xffffffffu, b, ps + 1);
                if (lane < 24) *gw = __byte_perm(x, y, psel);
              } else if (act) {  // the warp's ragged last row: byte stores
                uint8_t *p = gdst + 3 * (q - qa);
                p[0] = static_cast<uint8_t>(V >> 16);
                p[1] = static_cast<uint8_t>(V >> 8);
                p[2] = static_cast<uint8_t>(V);
              }
              gw += 24;
              q += 32;
              a += pstep;
              col += dc32;
              if (col >= G) {
                col -= G;
                a += e;
              }
            }
          } else if (interior && qa < qb) {
            // all lines full with an EOL, no final quad: incremental walk
            int q = qa + lane;
            int ln = line_of(q), col = q - ln * G;
            int a = imis + ln * Sl + 4 * col;
            uint8_t *po = ob + 3 * q;
#if B64_WL_BATCH
            // B64_WL_BATCH quads per step, loads ahead of stores (as in the
            // wrapped encoder)
            constexpr int NB = B64_WL_BATCH;
            for (; q + 32 * (NB - 1) < qb; q += 32 * NB) {
              uint32_t wv[NB];
              uint8_t *pp[NB];
#pragma unroll
              for (int j = 0; j < NB; ++j) {
                wv[j] = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
                pp[j] = po;
                po += 96;
                a += pstep;
                col += dc32;
                if (col >= G) {
                  col -= G;
                  a += e;
                }
              }
              uint32_t vv[NB][4];
#pragma unroll
              for (int j = 0; j < NB; ++j) {
                vv[j][0] = lds_u8((wv[j] & 0xFFu) | tb);
                vv[j][1] = lds_u8(__byte_perm(wv[j], tb, 0x7651));
                vv[j][2] = lds_u8(__byte_perm(wv[j], tb, 0x7652));
                vv[j][3] = lds_u8(__byte_perm(wv[j], tb, 0x7653));
              }
#pragma unroll
              for (int j = 0; j < NB; ++j) {
                bad |= vv[j][0] | vv[j][1] | vv[j][2] | vv[j][3];
                const uint32_t V = ((vv[j][0] * 64u + vv[j][1]) * 64u + vv[j][2]) * 64u + vv[j][3];
                pp[j][0] = static_cast<uint8_t>(V >> 16);
                pp[j][1] = static_cast<uint8_t>(V >> 8);
                pp[j][2] = static_cast<uint8_t>(V);
              }
            }
#endif
            for (; q < qb; q += 32) {
              const uint32_t w = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
              const uint32_t v0 = lds_u8((w & 0xFFu) | tb);
              const uint32_t v1 = lds_u8(__byte_perm(w, tb, 0x7651));
              const uint32_t v2 = lds_u8(__byte_perm(w, tb, 0x7652));
              const uint32_t v3 = lds_u8(__byte_perm(w, tb, 0x7653));
              bad |= v0 | v1 | v2 | v3;
              const uint32_t V = ((v0 * 64u + v1) * 64u + v2) * 64u + v3;
              po[0] = static_cast<uint8_t>(V >> 16);
              po[1] = static_cast<uint8_t>(V >> 8);
              po[2] = static_cast<uint8_t>(V);
              po += 96;
              a += pstep;
              col += dc32;
              if (col >= G) {
                col -= G;
                a += e;
              }
            }
          } else {
            for (int q = qa + lane; q < qb; q += 32) {
              const int ln = line_of(q);
              const int col = q - ln * G;
              const int a = imis + ln * Sl + 4 * col;
              const uint32_t w = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
              uint32_t v0 = lds_u8((w & 0xFFu) | tb);
              uint32_t v1 = lds_u8(__byte_perm(w, tb, 0x7651));
              uint32_t v2 = lds_u8(__byte_perm(w, tb, 0x7652));
              uint32_t v3 = lds_u8(__byte_perm(w, tb, 0x7653));
              if (pads_ok && q0 + q == Q - 1) {  // the final quad: '=' at the last two positions (R-pad)
                const uint32_t c2 = (w >> 16) & 0xFFu, c3 = w >> 24;
                if (c3 == '=') {
                  v3 = 0;
                  if (c2 == '=') v2 = 0;
                }
              }
              bad |= v0 | v1 | v2 | v3;
              const uint32_t V = ((v0 * 64u + v1) * 64u + v2) * 64u + v3;
              uint8_t *p = ob + 3 * q;
              p[0] = static_cast<uint8_t>(V >> 16);
              p[1] = static_cast<uint8_t>(V >> 8);
              p[2] = static_cast<uint8_t>(V);
            }
          }
          }  // !DS
          // EOL of every line whose last quad this warp owns (and that has one)
          if (!lmaj)
          for (int ln = line_of(qa) + lane, lb = line_of(qb); ln < lb; ln += 32) {
            if ((line0 + ln + 1) * Sl > M) break;
            const int b = imis + ln * Sl + L;
            const uint32_t x = __funnelshift_r(win[b >> 2], win[(b >> 2) + 1], 8 * (b & 3));
            if ((x & eolm) != eolw) bad |= 0x80u;
          }
          if (__any_sync(0xffffffffu, bad & 0x80u)) {
            if (lane == 0) {
              S.flag = 1;
              atomicExch(&st->viol, 1);
            }
          } else if (!DS && !lmaj && qa < qb && !direct) {
            // this warp's bytes: congruent staging -> 16-byte stores + byte edges
            __syncwarp();
            copy_out(gdst, slice + omis, 3 * (qb - qa));
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&S.empty[s]);
      }
#if B64_WL_BULK
      if (lane == 0) ptx::bulk_wait<0>();
#endif
    }
    viol = S.flag != 0;
  }
  // ---- last CTA out: the verdict and, on success, the result record
  __syncthreads();
  if (tid == 0) {
    if (viol) atomicExch(&st->viol, 1);
    S.flag = 0;
    __threadfence();
    S.flag = atomicAdd(&st->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!S.flag || tid != 0) return;
  __threadfence();
  const bool fail = atomicAdd(&st->viol, 0) != 0;
  if (fail) {
    st->verdict = 0;
    return;
  }
  // chars of the final (partial) quad straight from the text: compact i ->
  // original (i / L)(L + e) + i mod L
  const int Lr = L, Sr = L + e;
  // the partial final quad is not decoded by the tiles: its characters must
  // not be white space either (else the structure, hence Mc, is wrong)
  for (int64_t i = Mc & ~static_cast<int64_t>(3); i < Mc; ++i)
    if (is_space_byte(in[(i / Lr) * Sr + i % Lr])) {
      st->verdict = 0;
      return;
    }
  if constexpr (DS) {  // the partial final quad's chars, then the length
    for (int64_t i = Mc & ~static_cast<int64_t>(3); i < Mc; ++i) out[i] = in[(i / Lr) * Sr + i % Lr];
    *ds_out_len = Mc;
    st->verdict = 1;
    return;
  }
  const StreamResult R = finish_stream_at(
      [in, Lr, Sr](int64_t i) -> uint32_t { return in[(i / Lr) * Sr + i % Lr]; }, Mc, out, -1,
      true, flags);
  res->out_len = R.out_len;
  res->err_pos = R.err_pos >= 0 ? (R.err_pos / L) * Sr + R.err_pos % L : -1;
  res->status = R.status;
  res->pad_count = R.pad_count;
  st->verdict = 1;
}

}  // namespace b64
