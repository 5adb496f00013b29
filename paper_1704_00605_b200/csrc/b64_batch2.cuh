// b64_batch2.cuh -- batched encode / decode of k independent messages with a
// CTA-local plan (BASELINE.json configs[1]).
//
// Same units, rings, codec and copy-out as batch_kernel (b64_batch.cuh); what
// changes is how work is assigned and planned.  The messages are contiguous
// in d_in, so in_off already *is* the prefix sum of the input lengths:
//   * warp gw of the GW-warp grid owns the range [floor(T gw / GW),
//     floor(T (gw+1) / GW)) of the work coordinate P (input bytes before a
//     position plus a fixed charge A per message, T = P(k); see below) and
//     processes every unit that starts in it -- messages are assigned to
//     warps by prefix-summed lengths without a scan;
//   * CTA c owns the messages that START in the union of its warps' ranges
//     and scans only their output sizes; one grid barrier publishes the CTA
//     totals, after which each CTA derives its own messages' out_off (and
//     that of the one message straddling into its range from before:
//     out_off = prefix - its size) with no second barrier;
//   * each warp finds its first message with a search (a CTA-wide sample of
//     in_off in shared memory, then one 32-ary probe round in global) and
//     issues its first TMA loads BEFORE the plan and the grid barrier, so
//     the data are in flight while the plan runs;
//   * decode results are finished per CTA: every owned message but the last
//     lies entirely in the CTA's range (a CTA barrier suffices); the last one
//     may continue into later CTAs' ranges and waits for their done flags
//     (set after their data phase) -- no grid barrier after the data phase.
#pragma once
#include <climits>
#include <cstdint>
#include <type_traits>

#include <cooperative_groups.h>

#include "b64_batch.cuh"
#include "b64_codec.cuh"
#include "b64_ptx.cuh"

namespace b64 {

constexpr int kBatchMaxCtas = 1024;  // = kMaxBatchCtas of the workspace layout (b64_lib.cu)

__device__ __forceinline__ int64_t ld_acquire_i64(const int64_t *p) {
  int64_t v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i64(int64_t *p, int64_t v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Work coordinate of the start of message i: P(i) = in_off[i] - X0 + A * i.
// A unit (i, r) sits at P(i) + r * UIN.  The per-message term A charges each
// message for its partial last unit (a unit's cost is a fixed part plus its
// bytes, and every message has one partial unit), so equal P ranges are
// equal work; P(i) needs no scan.  A = UIN * B64_BATCH_MSG_COST / 8
// (b64_knobs.cuh).

// Number of indices p in [0, k] with P(p) < x (STRICT) or P(p) <= x (P is
// increasing).  samp[t] = in_off[min(t * sstep, k)], sstep = ceil(k / (T-1))
// (shared memory)
// brackets the answer; the bracket is then narrowed by 32-ary probes in
// global memory (one round when k < 32 * kBThreads).  Warp-uniform result.
template <bool STRICT>
__device__ __forceinline__ int64_t count_before(const int64_t *in_off, int64_t k,
                                                const int64_t *samp, int64_t sstep, int64_t X0,
                                                int64_t A, int64_t x, int lane,
                                                int64_t *v_last = nullptr) {
  constexpr int T = kBThreads;
  auto P = [&](int64_t v, int64_t p) { return v - X0 + A * p; };
  auto pos = [&](int t) { const int64_t p = static_cast<int64_t>(t) * sstep; return p < k ? p : k; };
  int lo = 0, hi = T;  // samples [0, lo) satisfy the predicate, [hi, T) do not
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int64_t v = P(samp[mid], pos(mid));
    if (STRICT ? v < x : v <= x) lo = mid + 1;
    else hi = mid;
  }
  if (lo == 0) return 0;
  if (lo == T) {
    if (v_last) *v_last = samp[T - 1];
    return k + 1;
  }
  int64_t a = pos(lo - 1);  // satisfies
  int64_t b = pos(lo);      // does not
  int64_t va = samp[lo - 1];  // in_off[a]
  while (b - a > 1) {
    const int64_t step = (b - a + 31) / 32;
    const int64_t p = a + static_cast<int64_t>(lane) * step;
    bool ok = false;
    int64_t v = 0;
    if (p < b) {
      v = in_off[p];
      const int64_t pv = P(v, p);
      ok = STRICT ? pv < x : pv <= x;
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);  // lane 0 (p = a) always set
    const int L = 31 - __clz(m);
    const int64_t na = a + static_cast<int64_t>(L) * step;
    va = __shfl_sync(0xffffffffu, v, L);
    b = na + step < b ? na + step : b;
    a = na;
  }
  if (v_last) *v_last = va;
  return a + 1;
}

// Message metadata source of the walkers: in_off / out_off in global
// memory, or -- once the CTA plan has run, for the messages it covers
// ([ilo - 1, ihi], staged in shared memory when they fit) -- s_io / s_oo.
struct MsgMeta {
  const int64_t *in_off, *out_off;
  const int64_t *s_io, *s_oo;  // index j - (ilo - 1)
  int64_t k, ilo, ihi, soo;
  bool staged;
  __device__ __forceinline__ int64_t io(int64_t j) const {
    if (staged && j >= ilo - 1 && j <= ihi) return s_io[j - ilo + 1];
    return j <= k ? in_off[j] : 0;
  }
  __device__ __forceinline__ int64_t oo(int64_t j) const {
    if (staged && j >= ilo - 1 && j < ihi) return s_oo[j - ilo + 1];
    return j < ilo ? soo : (j < k ? out_off[j] : 0);
  }
};

// A position (message, unit r of it) in the warp's unit sequence; message
// metadata from a 32-message lane-resident window (lane l: message base+l).
// OUT: also carries out_off (of messages < ilo only the straddler can be
// reached; it takes soo, the CTA-computed offset).
template <bool DECODE, bool OUT>
struct Walker2 {
  static constexpr int UIN = DECODE ? DU::kIn : EU::kIn;
  static constexpr int UOUT = DECODE ? DU::kOut : EU::kOut;
  int64_t base, io, oo;  // window
  int64_t msg, r, m_in, m_end, m_out;
  int64_t left;  // effective bytes of the message from unit r on
  __device__ __forceinline__ void load(int64_t b, const MsgMeta &M, int lane) {
    base = b;
    const int64_t j = b + lane;
    io = M.io(j);
    if (OUT) oo = M.oo(j);
  }
  __device__ __forceinline__ int64_t field(int64_t v, int64_t j) const {
    return __shfl_sync(0xffffffffu, v, static_cast<int>(j - base));
  }
  __device__ __forceinline__ void pull() {
    m_in = field(io, msg);
    m_end = field(io, msg + 1);
    if (OUT) m_out = field(oo, msg);
  }
  __device__ __forceinline__ int64_t eff() const {
    const int64_t len = m_end - m_in;
    return DECODE ? (len & ~static_cast<int64_t>(3)) : len;
  }
  // Skip to the first unit at or after (msg, r) that exists.
  __device__ __forceinline__ void settle(const MsgMeta &M, int lane) {
    while (left <= 0 && msg < M.k) {
      ++msg;
      r = 0;
      if (msg < M.k) {
        if (msg + 1 >= base + 32) load(msg, M, lane);
        pull();
        left = eff();
      }
    }
  }
  __device__ __forceinline__ void init(int64_t m, int64_t r0, const MsgMeta &M, int lane) {
    msg = m;
    r = r0;
    load(m, M, lane);
    pull();
    left = eff() - r0 * UIN;
    settle(M, lane);
  }
  // unit (msg, r) comes before the end position (me, re) of the warp's range
  __device__ __forceinline__ bool before(int64_t me, int64_t re) const {
    return msg < me || (msg == me && r < re);
  }
  __device__ __forceinline__ void next(const MsgMeta &M, int lane) {
    ++r;
    left -= UIN;
    settle(M, lane);
  }
  __device__ __forceinline__ UnitDesc desc() const {
    UnitDesc d;
    d.rel = r * UIN;
    d.src = m_in + d.rel;
    d.dst = OUT ? m_out + r * UOUT : 0;
    d.len = static_cast<int32_t>(left < UIN ? left : UIN);
    d.msg = static_cast<int32_t>(msg);
    const bool last = left <= UIN;
    d.flags = (last ? kFlagLast : 0) | ((DECODE && last && ((m_end - m_in) & 3) == 0) ? kFlagFinal : 0);
    return d;
  }
};

#ifdef B64_BATCH_TRACE
#define B64_TRACE2(slot) \
  if (lane == 0) g_trace[(blockIdx.x * 64 + 32 + warp) * 4 + (slot)] = gtimer()
#else
#define B64_TRACE2(slot)
#endif

template <bool DECODE>
__global__ void __launch_bounds__(kBThreads, B64_BATCH_CTAS)
    batch2_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int64_t k,
                  const int64_t *__restrict__ in_off, int64_t *__restrict__ out_off,
                  int64_t *__restrict__ blk, int64_t *__restrict__ err_pos,
                  int64_t *__restrict__ out_len, int32_t *__restrict__ status, int flags) {
  using Ring = typename std::conditional<DECODE, DecRing, EncRing>::type;
  constexpr int UIN = DECODE ? DU::kIn : EU::kIn;
  constexpr int T = kBThreads;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ int64_t sh[66];
  __shared__ int64_t samp[T];       // in_off sample; after the searches: s_oo
  __shared__ int64_t s_io[T + 2];   // in_off[ilo - 1 .. ilo + T]
  __shared__ int64_t s_ilo, s_ihi, s_so;
  __shared__ int64_t s_wpos[2 * kBWarps];  // each warp's first unit position
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Ring &R = reinterpret_cast<Ring *>(smem_raw)[warp];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();

  if (DECODE) {
    if (tid < 256) g_dec_tab[tid] = kInvalid;
  } else {
    if (tid < 64) g_enc_tab[tid] = static_cast<uint8_t>(ascii_of(tid, flags));
  }
  const bool pad = !(flags & kFlagNoPad);
  B64_TRACE(0);
  B64_TRACE2(0);
  if (lane == 0) {
    for (int s = 0; s < kBSlots; ++s) mbar_init(&R.full[s], 1);
    fence_mbar_init();
  }
  const int64_t G = gridDim.x, c = blockIdx.x;
  int64_t *done = blk + kBatchMaxCtas;  // done[c]: CTA c's data phase is complete
  if (DECODE && tid == 0) done[c] = 0;   // (read only after the grid barrier)
  // in_off sample: samp[t] = in_off[min(t * sstep, k)] (samp[0] = in_off[0], samp[T-1] = in_off[k])
  const int64_t sstep = (k + T - 2) / (T - 1);
  {
    const int64_t p = static_cast<int64_t>(tid) * sstep;
    samp[tid] = in_off[p < k ? p : k];
  }
  __syncthreads();
  if (DECODE && tid < 64) g_dec_tab[ascii_of(tid, flags)] = static_cast<uint8_t>(tid);
  constexpr int64_t A = static_cast<int64_t>(UIN) * B64_BATCH_MSG_COST / 8;
  const int64_t X0 = samp[0], XB = samp[T - 1] - X0 + A * k;  // total work P(k)

  // ---- ranges of the work coordinate P: CTA c = [Rc, Rc1), warp = [xw0, xw1)
  const int64_t Rc = muldiv_floor(XB, c, G), Rc1 = muldiv_floor(XB, c + 1, G);
  const int64_t GW = G * kBWarps, gw = c * kBWarps + warp;
  const int64_t xw0 = muldiv_floor(XB, gw, GW), xw1 = muldiv_floor(XB, gw + 1, GW);
  if (warp == 0) {
    const int64_t ilo = count_before<true>(in_off, k, samp, sstep, X0, A, Rc, lane);
    const int64_t ihi = c == G - 1 ? k : count_before<true>(in_off, k, samp, sstep, X0, A, Rc1, lane);
    if (lane == 0) {
      s_ilo = ilo;
      s_ihi = ihi;
    }
  }
  // the warp's first unit position (m0, r0): the last message starting at or
  // before xw0 and its first unit at P >= xw0; the range ends where the next
  // warp's begins (the CTA's last warp searches that position itself)
  auto first_unit = [&](int64_t x, int64_t &m, int64_t &r) {
    int64_t v = 0;
    m = count_before<false>(in_off, k, samp, sstep, X0, A, x, lane, &v) - 1;
    if (m > k - 1) {  // x >= P(k): past the last message
      m = k;
      r = 0;
      return;
    }
    r = (x - (v - X0 + A * m) + UIN - 1) / UIN;
  };
  int64_t m0, r0, me, re;
  first_unit(xw0, m0, r0);
  if (lane == 0) {
    s_wpos[2 * warp] = m0;
    s_wpos[2 * warp + 1] = r0;
  }
  if (warp == kBWarps - 1) first_unit(xw1, me, re);
  B64_TRACE2(1);
  MsgMeta M{in_off, out_off, s_io, samp, k, 0, 0, 0, false};
  // ---- first TMA loads, before the plan (they need input offsets only)
  const uint64_t pol = policy_evict_first();
  Walker2<DECODE, false> wi;
  int32_t issued = 0;
  auto issue = [&]() {
    const UnitDesc d = wi.desc();
    if (lane == 0) {
      const int s = issued % kBSlots;
      const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(d.src);
      const uintptr_t g0 = g & ~static_cast<uintptr_t>(15);
      const uint32_t bytes = (static_cast<uint32_t>(g & 15) + static_cast<uint32_t>(d.len) + 15u) & ~15u;
      mbar_arrive_expect_tx(&R.full[s], bytes);
      bulk_g2s(R.in[s], reinterpret_cast<const void *>(g0), bytes, &R.full[s], pol);
    }
    ++issued;
  };
  __syncthreads();  // s_wpos
  if (warp < kBWarps - 1) {
    me = s_wpos[2 * warp + 2];
    re = s_wpos[2 * warp + 3];
  }
  const bool has_range = xw0 < xw1 && m0 < k;
  if (has_range) {
    wi.init(m0, r0, M, lane);
    while (issued < kBSlots && wi.before(me, re)) {
      issue();
      wi.next(M, lane);
    }
  }
  B64_TRACE2(2);
  __syncthreads();  // s_ilo / s_ihi; every search is done with samp
  const int64_t ilo = s_ilo, ihi = s_ihi;
  const bool one_round = ihi - ilo <= T;

  // ---- plan: output sizes of the owned messages [ilo, ihi), CTA scan
  int64_t tot_o = 0, c_po = 0;
  for (int64_t q0 = ilo; q0 < ihi; q0 += T) {
    const int64_t i = q0 + tid;
    int64_t o = 0, u = 0;
    if (i < ihi) {
      const int64_t a = in_off[i], b = in_off[i + 1];
      if (one_round) {
        s_io[tid + 1] = a;
        if (i + 1 == ihi) s_io[tid + 2] = b;
      }
      msg_sizes<DECODE>(in, a, b, o, u, flags);
      if (DECODE) {
        const int64_t len = b - a;
        if (u == 0) {  // no complete quad: decided here (NOPAD 2-3 char tails: below)
          status[i] = (len & 3) ? B64_ERR_LENGTH : B64_OK;
          err_pos[i] = (len & 3) ? 0 : -1;
          out_len[i] = 0;
        } else {
          err_pos[i] = LLONG_MAX;  // before the grid barrier: every atomicMin comes after it
        }
      }
    }
    int64_t po, pu, to, tu;
    block_exclusive_scan2(o, 0, po, pu, to, tu, sh);
    c_po = tot_o + po;
    tot_o += to;
  }
  if (tid == 0) {
    blk[c] = tot_o;
    int64_t so = 0;
    if (ilo > 0) {  // size of the message straddling into this range (the last one before it)
      const int64_t a = in_off[ilo - 1], b = in_off[ilo];
      s_io[0] = a;
      int64_t u;
      msg_sizes<DECODE>(in, a, b, so, u, flags);
    }
    if (ihi == ilo) s_io[1] = in_off[ilo];  // (no owned message stored it)
    s_so = so;
  }
  __threadfence();
  grid.sync();
  B64_TRACE2(3);

  // ---- prefix of this CTA = totals of CTAs < c; out_off of the owned messages
  int64_t pre = 0;
  {
    int64_t x = 0;
    for (int64_t b = tid; b < c; b += T) x += blk[b];
    int64_t p1, p2, t2;
    block_exclusive_scan2(x, 0, p1, p2, pre, t2, sh);  // (its barriers also publish s_io / s_so)
  }
  int64_t *s_oo = samp;
  if (one_round) {
    if (ilo + tid < ihi) {
      out_off[ilo + tid] = pre + c_po;
      s_oo[tid + 1] = pre + c_po;
    }
  } else {
    int64_t run = pre;
    for (int64_t q0 = ilo; q0 < ihi; q0 += T) {
      const int64_t i = q0 + tid;
      int64_t o = 0, u = 0;
      if (i < ihi) msg_sizes<DECODE>(in, in_off[i], in_off[i + 1], o, u, flags);
      int64_t po, pu, to, tu;
      block_exclusive_scan2(o, 0, po, pu, to, tu, sh);
      if (i < ihi) out_off[i] = run + po;
      run += to;
    }
  }
  const int64_t soo = pre - s_so;  // out_off of the straddler (unused if ilo == 0)
  if (tid == 0) {
    if (c == G - 1) out_off[k] = pre + tot_o;
    s_oo[0] = soo;
  }
  M.ilo = ilo;
  M.ihi = ihi;
  M.soo = soo;
  M.staged = one_round;
  __syncthreads();  // out_off of the owned messages (global + s_oo)
  B64_TRACE(1);

  // ---- data phase (see batch_kernel: same unit loop, slots, codec, copy-out)
  if (__ballot_sync(0xffffffffu, 1) != 0xffffffffu) __trap();
  if (has_range) {
#ifdef B64_BATCH_TRACE
    unsigned long long tr_bytes = 0, tr_units = 0;
#endif
    Walker2<DECODE, true> wc;
    wc.init(m0, r0, M, lane);
    for (int32_t it = 0; wc.before(me, re); ++it) {
      const int s = it % kBSlots;
      const UnitDesc d = wc.desc();
      mbar_wait_spin(&R.full[s], static_cast<uint32_t>((it / kBSlots) & 1));
      if (it == 0) B64_TRACE(2);
      const uintptr_t gsrc = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(d.src);
      const int imis = static_cast<int>(gsrc & 15);
      const bool in4 = (gsrc & 3) == 0;
      const uint8_t *sin = R.in[s] + imis;
      uint8_t *gdst = out + d.dst;
      uint8_t *sout = R.out + 16;
      int olen;
      uint32_t werr = 0xFFFFFFFFu;
      if constexpr (!DECODE) {
        if (d.len == UIN) {
          if (in4)
            encode_tile<4, 16, true, kBatchPasses, false, 32>(sin, d.len, sout, lane, lane);
          else
            encode_tile<1, 16, true, kBatchPasses, false, 32>(sin, d.len, sout, lane, lane);
        } else {
          encode_tile<1, 16, false, kBatchPasses, false, 32>(sin, d.len, sout, lane, lane, nullptr,
                                                             pad);
        }
        olen = pad ? 4 * ((d.len + 2) / 3) : 4 * (d.len / 3) + (d.len % 3 ? d.len % 3 + 1 : 0);
      } else {
        const bool fin = (d.flags & kFlagFinal) != 0;
        uint32_t ch1 = 0, ch2 = 0;
        int pads = 0;
        if (fin) {
          ch1 = sin[d.len - 1];
          ch2 = sin[d.len - 2];
          pads = ch1 == '=' ? (ch2 == '=' ? 2 : 1) : 0;
        }
        if (d.len == UIN && !fin) {
          werr = in4 ? decode_tile<4, 4, true, kBatchPasses, false, 32>(sin, d.len, sout, lane, lane,
                                                                        false, 0, 0)
                     : decode_tile<1, 4, true, kBatchPasses, false, 32>(sin, d.len, sout, lane, lane,
                                                                        false, 0, 0);
        } else {
          werr = decode_tile<1, 4, false, kBatchPasses, false, 32>(sin, d.len, sout, lane, lane,
                                                                   fin, ch2, ch1);
        }
        olen = 3 * (d.len / 4) - pads;
      }
      __syncwarp();
      fence_proxy_async_smem();  // slot s fully read before its next bulk write
      if (wi.before(me, re)) {
        issue();
        wi.next(M, lane);
      }
      warp_copy_out(gdst, sout, olen, lane);
      if constexpr (DECODE) {
        if (lane == 0 && werr != 0xFFFFFFFFu) {  // first-error reduction
          unsigned long long *tgt = reinterpret_cast<unsigned long long *>(err_pos + d.msg);
          const unsigned long long pos = static_cast<unsigned long long>(d.rel) + werr;
          if (pos < *reinterpret_cast<volatile unsigned long long *>(tgt)) atomicMin(tgt, pos);
        }
      }
      __syncwarp();
      wc.next(M, lane);
#ifdef B64_BATCH_TRACE
      tr_bytes += static_cast<unsigned long long>(d.len);
      ++tr_units;
#endif
    }
#ifdef B64_BATCH_TRACE
    if (lane == 0) g_trace[(blockIdx.x * 64 + warp) * 4 + 0] = (tr_bytes << 20) | tr_units;
#endif
  }
  B64_TRACE(3);

  if constexpr (DECODE) {
    // ---- per-message results of the owned messages (status is a pure
    // function of err_pos, R-length).  Every owned message but the last lies
    // in this CTA's range; the last may have units in later ranges and waits
    // for those CTAs' done flags.
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release_i64(done + c, 1);
    for (int64_t i = ilo + tid; i < ihi; i += T) {
      const int64_t a = M.io(i), b = M.io(i + 1);
      const int64_t len = b - a;
      if (len / 4 == 0 && !((flags & kFlagNoPad) && len >= 2)) continue;  // decided in the plan
      const int64_t e4 = len & ~static_cast<int64_t>(3);
      if (i == ihi - 1 && e4 > 0) {
        const int64_t ls = a - X0 + A * i + ((e4 - 1) / UIN) * UIN;  // P of the last unit
        if (ls >= Rc1) {
          int64_t cl = muldiv_floor(ls, G, XB);
          if (cl > G - 1) cl = G - 1;
          while (cl + 1 < G && muldiv_floor(XB, cl + 1, G) <= ls) ++cl;
          while (cl > c && muldiv_floor(XB, cl, G) > ls) --cl;
          for (int64_t cc = c + 1; cc <= cl; ++cc)
            while (ld_acquire_i64(done + cc) == 0) __nanosleep(64);
        }
      }
      int64_t err = len / 4 == 0 ? LLONG_MAX : *reinterpret_cast<volatile int64_t *>(err_pos + i);
      if (err == LLONG_MAX) err = -1;
      const StreamResult Rs = finish_stream(in + a, len, out + M.oo(i), err, true, flags);
      status[i] = Rs.status;
      out_len[i] = Rs.out_len;
      err_pos[i] = Rs.err_pos;
    }
  }
}

}  // namespace b64
