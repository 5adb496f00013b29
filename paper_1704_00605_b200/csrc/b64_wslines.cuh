// b64_wslines.cuh -- verified fast path of the whitespace-tolerant decode
// (reading R-ws-decode) for line-structured text,
// i.e. MIME / PEM: every line holds the same number L of characters (L a
// multiple of 4) followed by the same end-of-line sequence (LF or CR LF);
// the last line holds 1..L characters, with or without the EOL; there is no
// other white space.  Then the i-th kept character sits at original offset
// (i / L)(L + e) + i mod L, so every quad is decoded straight from the
// TMA-staged text -- no mask pass, no compaction.
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

constexpr int kWlThreads = 512;
#ifndef B64_WL_TILE
#define B64_WL_TILE 28672
#endif
#ifndef B64_WL_STAGES
#define B64_WL_STAGES 2
#endif
constexpr int kWlTile = B64_WL_TILE;    // max input bytes per tile (whole lines)
constexpr int kWlStages = B64_WL_STAGES;
constexpr int kWlMaxLine = 4092;      // longest line the fast path takes
constexpr int kWlOut = kWlTile / 4 * 3 + 64;

// Per-call state in the caller's workspace (zeroed by a 16-byte memset
// before the launch).
struct WlState {
  int32_t verdict;  // 1: the fast path produced the result; 0: fall back
  int32_t viol;     // set by any CTA that sees a violation or an error
  uint32_t done;    // CTAs finished
  int32_t pad;
};

struct alignas(128) WlSmem {
  uint8_t in[kWlStages][kWlTile + 64];
  alignas(16) uint8_t out[2][kWlOut];
  uint64_t full[kWlStages];
  int64_t geo[4];   // Mc (kept chars), nlines, ok
  int32_t Le[2];    // L, e
  int32_t flag;
};

__global__ void __launch_bounds__(kWlThreads, 2)
    decode_lines_kernel(const uint8_t *__restrict__ in, int64_t M, uint8_t *__restrict__ out,
                        WlState *st, b64_result *res, int flags) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  WlSmem &S = *reinterpret_cast<WlSmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 256) g_dec_tab[tid] = kInvalid;
  if (tid == 0) {
    for (int s = 0; s < kWlStages; ++s) ptx::mbar_init(&S.full[s], 1);
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
    const int Lt = kWlTile / Sl;                          // lines per tile
    const int64_t ntiles = (nlines + Lt - 1) / Lt;
    const int64_t Q = Mc / 4;                             // complete quads
    const bool pads_ok = (Mc & 3) == 0;
    const uint32_t inv = G > 1 ? static_cast<uint32_t>(((1ull << 32) + G - 1) / G) : 0u;
    const uint64_t pol = ptx::policy_evict_first();
    auto load = [&](int64_t t, int s) {
      const int64_t src = t * Lt * static_cast<int64_t>(Sl);
      const int64_t len = M - src < static_cast<int64_t>(Lt) * Sl ? M - src : static_cast<int64_t>(Lt) * Sl;
      const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src);
      const uintptr_t g0 = g & ~static_cast<uintptr_t>(15);
      const uintptr_t g1 = (g + static_cast<uintptr_t>(len) + 15) & ~static_cast<uintptr_t>(15);
      ptx::mbar_arrive_expect_tx(&S.full[s], static_cast<uint32_t>(g1 - g0));
      ptx::bulk_g2s(S.in[s], reinterpret_cast<const void *>(g0), static_cast<uint32_t>(g1 - g0),
                    &S.full[s], pol);
    };
    const int64_t t0 = blockIdx.x;
    if (tid == 0)
      for (int k = 0; k < kWlStages - 1 && t0 + static_cast<int64_t>(k) * gridDim.x < ntiles; ++k)
        load(t0 + static_cast<int64_t>(k) * gridDim.x, k);
    const uint32_t eolw = e == 2 ? 0x0A0Du : 0x0Au, eolm = e == 2 ? 0xFFFFu : 0xFFu;
    // thread-invariant walk of an interior tile: quad tid + 512 k
    const int line_t = tid / G, col_t = tid % G;
    const int p_t = line_t * Sl + 4 * col_t;
    const int dc = kWlThreads % G;
    const int pstep = (kWlThreads / G) * Sl + 4 * dc;
    int it = 0;
    for (int64_t t = t0; t < ntiles; t += gridDim.x, ++it) {
      const int s = it % kWlStages, so = it & 1;
      if (tid == 0 && t + (kWlStages - 1) * static_cast<int64_t>(gridDim.x) < ntiles)
        load(t + (kWlStages - 1) * static_cast<int64_t>(gridDim.x), (it + kWlStages - 1) % kWlStages);
      const int64_t src = t * Lt * static_cast<int64_t>(Sl);
      const int64_t q0 = t * Lt * static_cast<int64_t>(G);     // first quad of the tile
      const int64_t line0 = t * Lt;
      const int64_t q1 = q0 + static_cast<int64_t>(Lt) * G < Q ? q0 + static_cast<int64_t>(Lt) * G : Q;
      const int nq = static_cast<int>(q1 - q0);
      const int imis = static_cast<int>((reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(src)) & 15);
      uint8_t *gdst = out + 3 * q0;
      const int omis = static_cast<int>(reinterpret_cast<uintptr_t>(gdst) & 15);
      uint8_t *ob = S.out[so] + omis;
      const uint32_t *win = reinterpret_cast<const uint32_t *>(S.in[s]);
      ptx::mbar_wait_spin(&S.full[s], static_cast<uint32_t>((it / kWlStages) & 1));
      if (viol) continue;  // drain the loads in flight, skip the work
      uint32_t bad = 0;
      if (q1 < Q && (line0 + Lt) * static_cast<int64_t>(Sl) <= M && Q - q1 >= 1) {
        // Interior tile: Lt whole lines, each followed by its EOL, no final
        // quad.  The tile starts on a line boundary and the stride is 512
        // quads, so each thread's (column, offset) walk is tile-invariant
        // up to the window misalignment: one increment per quad.
        // the EOL of every line of the tile: one check per line, off the quad loop
        for (int ln = tid; ln < Lt; ln += kWlThreads) {
          const int b = imis + ln * Sl + L;
          const uint32_t x = __funnelshift_r(win[b >> 2], win[(b >> 2) + 1], 8 * (b & 3));
          if ((x & eolm) != eolw) bad |= 0x80u;
        }
        int a = imis + p_t, col = col_t, o = 3 * tid;
        for (int ql = tid; ql < nq; ql += kWlThreads) {
          const uint32_t w = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
          const uint32_t v0 = lds_u8((w & 0xFFu) | tb);
          const uint32_t v1 = lds_u8(__byte_perm(w, tb, 0x7651));
          const uint32_t v2 = lds_u8(__byte_perm(w, tb, 0x7652));
          const uint32_t v3 = lds_u8(__byte_perm(w, tb, 0x7653));
          bad |= v0 | v1 | v2 | v3;
          const uint32_t V = ((v0 * 64u + v1) * 64u + v2) * 64u + v3;
          uint8_t *p = ob + o;
          p[0] = static_cast<uint8_t>(V >> 16);
          p[1] = static_cast<uint8_t>(V >> 8);
          p[2] = static_cast<uint8_t>(V);
          a += pstep;
          o += 3 * kWlThreads;
          col += dc;
          if (col >= G) {
            col -= G;
            a += e;
          }
        }
      } else {  // first / last tiles: generic walk, final quad, partial last line
        for (int ql = tid; ql < nq; ql += kWlThreads) {
          const uint32_t line =
              G == 1 ? static_cast<uint32_t>(ql) : __umulhi(static_cast<uint32_t>(ql), inv);
          const int col = ql - static_cast<int>(line) * G;
          const int a = imis + static_cast<int>(line) * Sl + 4 * col;
          const uint32_t w = __funnelshift_r(win[a >> 2], win[(a >> 2) + 1], 8 * (a & 3));
          uint32_t v0 = lds_u8((w & 0xFFu) | tb);
          uint32_t v1 = lds_u8(__byte_perm(w, tb, 0x7651));
          uint32_t v2 = lds_u8(__byte_perm(w, tb, 0x7652));
          uint32_t v3 = lds_u8(__byte_perm(w, tb, 0x7653));
          if (pads_ok && q0 + ql == Q - 1) {  // the final quad: '=' at the last two positions (R-pad)
            const uint32_t c2 = (w >> 16) & 0xFFu, c3 = w >> 24;
            if (c3 == '=') {
              v3 = 0;
              if (c2 == '=') v2 = 0;
            }
          }
          bad |= v0 | v1 | v2 | v3;
          const uint32_t V = ((v0 * 64u + v1) * 64u + v2) * 64u + v3;
          uint8_t *p = ob + 3 * ql;
          p[0] = static_cast<uint8_t>(V >> 16);
          p[1] = static_cast<uint8_t>(V >> 8);
          p[2] = static_cast<uint8_t>(V);
          // end of a line with an EOL after it: verify the EOL bytes
          if (col == G - 1 && (line0 + static_cast<int64_t>(line) + 1) * Sl <= M) {
            const int b = a + 4;
            const uint32_t x = __funnelshift_r(win[b >> 2], win[(b >> 2) + 1], 8 * (b & 3));
            if ((x & eolm) != eolw) bad |= 0x80u;
          }
        }
      }
      if (bad & 0x80u) S.flag = 1;  // benign race: any writer sets it
      if (tid == 0 && *reinterpret_cast<volatile int32_t *>(&st->viol)) S.flag = 1;
      ptx::fence_proxy_async_smem();
      __syncthreads();
      if (S.flag) {  // give up (every later tile of this CTA is only drained)
        viol = true;
        if (tid == 0) atomicExch(&st->viol, 1);
        continue;
      }
      // (the pad bytes of the final quad are copied too: beyond out_len, within capacity)
      cta_copy_out_congruent(gdst, ob, 3 * nq);
    }
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
