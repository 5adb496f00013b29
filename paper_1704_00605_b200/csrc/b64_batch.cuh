// b64_batch.cuh -- batched encode / decode of k independent messages
// (BASELINE.json configs[1]).
//
// Work is split into *units*: one unit = kBatchPasses passes of one warp
// (kBatchPasses = 6: encode 2304 input bytes -> 3072 chars; decode 3072
// chars -> 2304 bytes).
// A unit never straddles messages, so a message of len bytes has
// ceil(len / unit) units (at most one partial unit per message, <= 2-4 %
// slack at data-URI sizes).  The planner scans the message lengths once
// (output offsets + unit offsets); every warp of the persistent grid then
// takes a contiguous range of units of equal estimated cost (a fixed part
// per unit plus its bytes, B64_BATCH_UNIT_COST) -- i.e. messages are
// assigned to warps by prefix-summed lengths -- gets its first message and
// unit from tables the plan writes and walks forward.  Warps are fully independent: each owns a
// 2-slot ring of 1-D TMA bulk loads (its lane 0 issues them, one mbarrier per
// slot), a private output slice in smem, and writes its unit's output with
// coalesced 16-byte stores (byte stores for the <16-byte unaligned edges).
// There is no CTA-wide barrier on the hot path.
#pragma once
#include <climits>
#include <cstdint>
#include <type_traits>

#include <cooperative_groups.h>

#include "b64_codec.cuh"
#include "b64_ptx.cuh"

namespace b64 {

using namespace ptx;

#ifdef B64_BATCH_TRACE  // measurement only (tools/sweep.py): per-warp globaltimer stamps
__device__ unsigned long long g_trace[148 * 64 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define B64_TRACE(slot) \
  if (lane == 0) g_trace[(blockIdx.x * 64 + warp) * 4 + (slot)] = gtimer()
#else
#define B64_TRACE(slot)
#endif

constexpr int kBWarps = B64_BATCH_WARPS;
constexpr int kBSlots = B64_BATCH_SLOTS;
constexpr int kBThreads = kBWarps * 32;
constexpr int kFlagLast = 2;  // unit is the last unit of its message
// workspace: first_msg int32[kBatchFirstMsgSlots], then first_unit int64[same]
constexpr int kBatchFirstMsgSlots = 1024 * B64_BATCH_WARPS;

template <int P>
struct EncUnit {
  static constexpr int kIn = 32 * 12 * P;
  static constexpr int kOut = 32 * 16 * P;
};
template <int P>
struct DecUnit {
  static constexpr int kIn = 32 * 16 * P;
  static constexpr int kOut = 32 * 12 * P;
};
using EU = EncUnit<kBatchPasses>;
using DU = DecUnit<kBatchPasses>;

struct UnitDesc {
  int64_t src;     // input offset of the unit (relative to d_in)
  int64_t dst;     // output offset (relative to d_out)
  int64_t rel;     // input offset of the unit within its message
  int32_t len;     // input bytes of the unit (decode: multiple of 4, > 0)
  int32_t msg;     // message index
  int32_t flags;   // kFlagLast | kFlagFinal
};

template <int IN, int OUT>
struct alignas(16) WarpRing {
  static constexpr int kInStride = round_up_c(IN + 32, 16);
  static constexpr int kOutStride = round_up_c(OUT + 48, 16);  // 16 head room + 32 read slack
  uint8_t in[kBSlots][kInStride];
  uint8_t out[kOutStride];
  uint64_t full[kBSlots];
};
using EncRing = WarpRing<EU::kIn, EU::kOut>;
using DecRing = WarpRing<DU::kIn, DU::kOut>;

struct BatchHeader {
  int64_t nunits;
  int64_t pad[3];
};

// ------------------------------------------------------------- planner ---
// The plan (exclusive scans of per-message output sizes and unit counts) is
// phase 1 of the same cooperative launch: CTA b scans messages
// [b*chunk, (b+1)*chunk) in rounds of one message per thread, publishes its
// totals, grid-syncs, adds the totals of CTAs < b and writes out_off /
// unit_off (and the decode per-message result initialisation); a second
// grid sync publishes the plan to every warp.  No planner launch, no
// descriptor array.

__device__ __forceinline__ void block_exclusive_scan2(int64_t a, int64_t b, int64_t &pa,
                                                      int64_t &pb, int64_t &ta, int64_t &tb,
                                                      int64_t *sh /* 66 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t xa = __shfl_up_sync(0xffffffffu, ia, o);
    const int64_t xb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) {
      ia += xa;
      ib += xb;
    }
  }
  if (lane == 31) {
    sh[warp] = ia;
    sh[32 + warp] = ib;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = static_cast<int>(blockDim.x >> 5);
    const int64_t wa = lane < nw ? sh[lane] : 0, wb = lane < nw ? sh[32 + lane] : 0;
    int64_t sa = wa, sb = wb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t xa = __shfl_up_sync(0xffffffffu, sa, o);
      const int64_t xb = __shfl_up_sync(0xffffffffu, sb, o);
      if (lane >= o) {
        sa += xa;
        sb += xb;
      }
    }
    sh[lane] = sa - wa;
    sh[32 + lane] = sb - wb;
    if (lane == 31) {
      sh[64] = sa;
      sh[65] = sb;
    }
  }
  __syncthreads();
  pa = sh[warp] + ia - a;
  pb = sh[32 + warp] + ib - b;
  ta = sh[64];
  tb = sh[65];
  __syncthreads();
}

// Output size and unit count of message [a, b) (decode: reads the pads).
template <bool DECODE>
__device__ __forceinline__ void msg_sizes(const uint8_t *in, int64_t a, int64_t b, int64_t &osz,
                                          int64_t &units, int flags) {
  const int64_t len = b - a;
  if (DECODE) {
    const int64_t q = len / 4, r = len & 3;
    int64_t p = 0;
    if (r == 0 && q > 0 && in[b - 1] == '=') p = (in[b - 2] == '=') ? 2 : 1;
    osz = 3 * q - p + (((flags & kFlagNoPad) && r >= 2) ? r - 1 : 0);
    units = (4 * q + DU::kIn - 1) / DU::kIn;
  } else {
    osz = enc_len(len, flags);
    units = (len + EU::kIn - 1) / EU::kIn;
  }
}

// floor(a * b / c) for a, b, c >= 0, c > 0, a * b < 2^62: a double-precision
// estimate (exact to within 1 for products < 2^53) corrected with integer
// arithmetic -- no 64-bit / 128-bit integer division subroutine.
__device__ __forceinline__ int64_t muldiv_floor(int64_t a, int64_t b, int64_t c) {
  const int64_t p = a * b;
  int64_t q = static_cast<int64_t>(static_cast<double>(p) / static_cast<double>(c));
  while (q > 0 && q * c > p) --q;
  while ((q + 1) * c <= p) ++q;
  return q;
}
__device__ __forceinline__ int64_t muldiv_ceil(int64_t a, int64_t b, int64_t c) {
  const int64_t q = muldiv_floor(a, b, c);
  return q * c == a * b ? q : q + 1;
}

// ------------------------------------------------------ warp walker ---
// Metadata of a window of 32 messages [base, base+32) lives in the lanes
// (lane l holds in_off/out_off/unit_off of message base+l); message j in
// [base, base+31) is then fully described by lanes j-base and j-base+1.
struct MsgWindow {
  int64_t base = -1;
  int64_t io, oo, uo;  // this lane's entries
};

__device__ __forceinline__ void window_load(MsgWindow &w, int64_t base, int64_t k,
                                            const int64_t *in_off, const int64_t *out_off,
                                            const int64_t *unit_off, int lane) {
  w.base = base;
  const int64_t j = base + lane;
  const bool ok = j <= k;
  w.io = ok ? in_off[j] : 0;
  w.oo = ok ? out_off[j] : 0;
  w.uo = ok ? unit_off[j] : 0;
}

// Largest i in [0, k) with unit_off[i] <= u (unit_off[k] > u): the message
// holding unit u.  32-ary search, one coalesced probe per round.
__device__ __forceinline__ int64_t find_message(const int64_t *unit_off, int64_t k, int64_t u,
                                                int lane) {
  int64_t lo = 0, hi = k;  // invariant: unit_off[lo] <= u < unit_off[hi]
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + static_cast<int64_t>(lane) * step;
    const bool le = p < hi && unit_off[p] <= u;
    const unsigned mask = __ballot_sync(0xffffffffu, le);
    const int L = 31 - __clz(mask);  // lane 0 always true (p = lo)
    const int64_t nlo = lo + static_cast<int64_t>(L) * step;
    const int64_t nhi = nlo + step < hi ? nlo + step : hi;
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// A position in the unit sequence: the current message's metadata (pulled
// from the lane-resident window with shuffles), advanced message by message.
template <bool DECODE>
struct Walker {
  MsgWindow win;
  int64_t msg, m_in, m_end, m_out, m_u0, m_u1;
  __device__ __forceinline__ int64_t field(int64_t v, int64_t j) const {
    return __shfl_sync(0xffffffffu, v, static_cast<int>(j - win.base));
  }
  __device__ __forceinline__ void pull() {
    m_in = field(win.io, msg);
    m_end = field(win.io, msg + 1);
    m_out = field(win.oo, msg);
    m_u0 = field(win.uo, msg);
    m_u1 = field(win.uo, msg + 1);
  }
  __device__ __forceinline__ void init(int64_t m, int64_t k, const int64_t *in_off,
                                       const int64_t *out_off, const int64_t *unit_off, int lane) {
    msg = m;
    window_load(win, m, k, in_off, out_off, unit_off, lane);
    pull();
  }
  // Descriptor of unit u (u >= the current message's first unit).
  __device__ __forceinline__ UnitDesc seek(int64_t u, int64_t k, const int64_t *in_off,
                                           const int64_t *out_off, const int64_t *unit_off,
                                           int lane) {
    constexpr int UIN = DECODE ? DU::kIn : EU::kIn;
    constexpr int UOUT = DECODE ? DU::kOut : EU::kOut;
    while (u >= m_u1) {  // advance to the message holding unit u (skips empty messages)
      ++msg;
      if (msg + 1 >= win.base + 32) window_load(win, msg, k, in_off, out_off, unit_off, lane);
      pull();
    }
    const int64_t r = u - m_u0;
    const int64_t mlen = m_end - m_in;
    const int64_t eff = DECODE ? (mlen & ~static_cast<int64_t>(3)) : mlen;
    UnitDesc d;
    d.rel = r * UIN;
    d.src = m_in + d.rel;
    d.dst = m_out + r * UOUT;
    const int64_t left = eff - d.rel;
    d.len = static_cast<int32_t>(left < UIN ? left : UIN);
    d.msg = static_cast<int32_t>(msg);
    const bool last = u == m_u1 - 1;
    d.flags = (last ? kFlagLast : 0) | ((DECODE && last && (mlen & 3) == 0) ? kFlagFinal : 0);
    return d;
  }
};

// 16 stream bytes starting at byte offset `so` (any alignment) of a
// 16-byte aligned smem stream: two conflict-free LDS.128 + a uniform
// word select + funnel shift.
__device__ __forceinline__ uint4 lds16_unaligned(const uint8_t *stream, int so) {
  const uint8_t *c = stream + (so & ~15);
  const uint4 a = *reinterpret_cast<const uint4 *>(c);
  const uint4 b = *reinterpret_cast<const uint4 *>(c + 16);
  const uint32_t bs = 8u * static_cast<uint32_t>(so & 3);
  uint32_t x0, x1, x2, x3, x4;
  switch ((so >> 2) & 3) {  // warp-uniform
    case 0: x0 = a.x; x1 = a.y; x2 = a.z; x3 = a.w; x4 = b.x; break;
    case 1: x0 = a.y; x1 = a.z; x2 = a.w; x3 = b.x; x4 = b.y; break;
    case 2: x0 = a.z; x1 = a.w; x2 = b.x; x3 = b.y; x4 = b.z; break;
    default: x0 = a.w; x1 = b.x; x2 = b.y; x3 = b.z; x4 = b.w; break;
  }
  return make_uint4(__funnelshift_r(x0, x1, bs), __funnelshift_r(x1, x2, bs),
                    __funnelshift_r(x2, x3, bs), __funnelshift_r(x3, x4, bs));
}

// Unit-level copy-out: `len` stream bytes staged at the 16-byte aligned smem
// `stream` -> gdst (any alignment).  Each lane writes whole 16-byte aligned
// granules of the destination (realigned from smem, one STG.128); the at
// most two partial granules at the ends are written byte-wise.
__device__ __forceinline__ void warp_copy_out(uint8_t *gdst, const uint8_t *stream, int len,
                                              int lane) {
  const int mis = static_cast<int>(reinterpret_cast<uintptr_t>(gdst) & 15);
  const int head = mis ? 16 - mis : 0;        // bytes before the first full granule
  const int body = (len - head) & ~15;        // full granules
  if (len <= head + 16) {                      // tiny output: bytes only
    if (lane < len) gdst[lane] = stream[lane];
    return;
  }
  const int ng = body >> 4;
  uint8_t *B0 = gdst + head;                   // 16-byte aligned
  for (int i = lane; i < ng; i += 32)
    *reinterpret_cast<uint4 *>(B0 + 16 * i) = lds16_unaligned(stream, head + 16 * i);
  // edges: head bytes by lanes 0..15, tail bytes by lanes 16..31
  const int tail0 = head + body;
  if (lane < head) gdst[lane] = stream[lane];
  if (lane >= 16 && tail0 + lane - 16 < len) gdst[tail0 + lane - 16] = stream[tail0 + lane - 16];
}

// --------------------------------------------------------- the kernel ---
template <bool DECODE>
__global__ void __launch_bounds__(kBThreads, B64_BATCH_CTAS)
    batch_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int64_t k,
                 const int64_t *__restrict__ in_off, int64_t *__restrict__ out_off,
                 int64_t *__restrict__ unit_off, int64_t *__restrict__ blk,
                 int64_t *__restrict__ err_pos, int64_t *__restrict__ out_len,
                 int32_t *__restrict__ status, int32_t *__restrict__ first_msg, int flags) {
  using Ring = typename std::conditional<DECODE, DecRing, EncRing>::type;
  constexpr int UIN = DECODE ? DU::kIn : EU::kIn;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ int64_t sh[66];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Ring &R = reinterpret_cast<Ring *>(smem_raw)[warp];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();

  if (DECODE) {
    if (tid < 256) g_dec_tab[tid] = kInvalid;
    __syncthreads();
    if (tid < 64) g_dec_tab[ascii_of(tid, flags)] = static_cast<uint8_t>(tid);
  } else {
    if (tid < 64) g_enc_tab[tid] = static_cast<uint8_t>(ascii_of(tid, flags));
  }
  const bool pad = !(flags & kFlagNoPad);
  B64_TRACE(0);
  if (lane == 0) {
    for (int s = 0; s < kBSlots; ++s) mbar_init(&R.full[s], 1);
    fence_mbar_init();
  }

  // ---- phase 1: plan (exclusive scans), see header comment
  const int64_t G = gridDim.x;
  const int64_t chunk = (k + G - 1) / G;
  const int64_t i_lo = blockIdx.x * chunk < k ? blockIdx.x * chunk : k;
  const int64_t i_hi = i_lo + chunk < k ? i_lo + chunk : k;
  int64_t tot_o = 0, tot_u = 0;
  // a CTA's messages usually fit one round: keep that round's values in
  // registers so pass 2 needs no reloads (in_off, pad characters) and no scan
  const bool one_round = i_hi - i_lo <= kBThreads;
  int64_t c_a = 0, c_b = 0, c_o = 0, c_u = 0, c_po = 0, c_pu = 0;
  for (int64_t r0 = i_lo; r0 < i_hi; r0 += kBThreads) {
    const int64_t i = r0 + tid;
    int64_t o = 0, u = 0, a = 0, b = 0;
    if (i < i_hi) {
      a = in_off[i];
      b = in_off[i + 1];
      msg_sizes<DECODE>(in, a, b, o, u, flags);
    }
    int64_t po, pu, to, tu;
    block_exclusive_scan2(o, u, po, pu, to, tu, sh);
    tot_o += to;
    tot_u += tu;
    c_a = a;
    c_b = b;
    c_o = o;
    c_u = u;
    c_po = po;
    c_pu = pu;
  }
  if (tid == 0) {
    blk[2 * blockIdx.x] = tot_o;
    blk[2 * blockIdx.x + 1] = tot_u;
  }
  grid.sync();
  // offsets of this CTA = sum of the totals of CTAs < blockIdx.x; U = all
  int64_t bo = 0, bu = 0, all_u = 0;
  for (int64_t b = tid; b < G; b += kBThreads) {
    const int64_t to = blk[2 * b], tu = blk[2 * b + 1];
    if (b < blockIdx.x) {
      bo += to;
      bu += tu;
    }
    all_u += tu;
  }
  {
    int64_t p1, p2, t1, t2;
    block_exclusive_scan2(bo, bu, p1, p2, t1, t2, sh);
    bo = t1;
    bu = t2;
    int64_t q1, q2, t3, t4;
    block_exclusive_scan2(all_u, 0, q1, q2, t3, t4, sh);
    all_u = t3;
  }
#if B64_BATCH_UNIT_COST
  constexpr int64_t kUnitW = static_cast<int64_t>(UIN) * B64_BATCH_UNIT_COST / 8;
  int64_t *first_unit = reinterpret_cast<int64_t *>(first_msg + kBatchFirstMsgSlots);
  const int64_t all_c = all_u > 0 ? kUnitW * all_u + (in_off[k] - in_off[0]) : 0;  // total cost
#endif
  for (int64_t r0 = i_lo; r0 < i_hi; r0 += kBThreads) {
    const int64_t i = r0 + tid;
    int64_t o = c_o, u = c_u, a = c_a, b = c_b;
    int64_t po = c_po, pu = c_pu, to = tot_o, tu = tot_u;
    if (!one_round) {
      o = u = a = b = 0;
      if (i < i_hi) {
        a = in_off[i];
        b = in_off[i + 1];
        msg_sizes<DECODE>(in, a, b, o, u, flags);
      }
      block_exclusive_scan2(o, u, po, pu, to, tu, sh);
    }
    if (i < i_hi) {
      out_off[i] = bo + po;
      unit_off[i] = bu + pu;
#if B64_BATCH_UNIT_COST
      // Warps get equal ranges of estimated work: a unit costs a fixed
      // part kW (in input-byte equivalents) plus its bytes, so message i
      // spans the cost interval [cp, cp + kW u + len), cp = kW unit_off[i]
      // + in_off[i] - in_off[0] (no scan beyond the unit offsets).  Warp g
      // starts at the first unit whose cost position cp + r (kW + UIN) is
      // >= b_g = floor(C g / GW): for the g with b_g in this interval,
      // first_msg[g] = i and first_unit[g] = unit_off[i] + min(r, u).
      if (all_c > 0) {
        const int64_t GWt = static_cast<int64_t>(gridDim.x) * kBWarps;
        const int64_t a0 = bu + pu;
        const int64_t cp = kUnitW * a0 + (a - in_off[0]);
        const int64_t cn = cp + kUnitW * u + (b - a);
        const int64_t g_lo = muldiv_ceil(cp, GWt, all_c);
        const int64_t g_hi = muldiv_ceil(cn, GWt, all_c);
        for (int64_t g = g_lo; g < g_hi; ++g) {
          const int64_t bg = muldiv_floor(all_c, g, GWt);
          const int64_t r = (bg - cp + kUnitW + UIN - 1) / (kUnitW + UIN);
          first_msg[g] = static_cast<int32_t>(i);
          first_unit[g] = a0 + (r < u ? r : u);
        }
      }
#else
      // Warps whose first unit u_begin(g) = floor(U*g/GW) lies in this
      // message's units [a, a+u): g in [ceil(a*GW/U), ceil((a+u)*GW/U)).
      if (u > 0) {
        const int64_t GWt = static_cast<int64_t>(gridDim.x) * kBWarps;
        const int64_t a0 = bu + pu;
        const int64_t g_lo = muldiv_ceil(a0, GWt, all_u);
        const int64_t g_hi = muldiv_ceil(a0 + u, GWt, all_u);
        for (int64_t g = g_lo; g < g_hi; ++g) first_msg[g] = static_cast<int32_t>(i);
      }
#endif
      if (DECODE) {
        const int64_t len = b - a;
        if (u == 0) {  // no complete quad: decided here (NOPAD 2-3 char tails: phase 3)
          status[i] = (len & 3) ? B64_ERR_LENGTH : B64_OK;
          err_pos[i] = (len & 3) ? 0 : -1;
          out_len[i] = 0;
        } else {
          err_pos[i] = LLONG_MAX;
        }
      }
    }
    bo += to;
    bu += tu;
  }
  if (blockIdx.x == G - 1 && tid == 0) {
    out_off[k] = bo;
    unit_off[k] = bu;
  }
  __threadfence();
  grid.sync();

  B64_TRACE(1);
#ifdef B64_BATCH_PLAN_ONLY  // measurement only (tools/sweep.py): stop after the plan
  return;
#endif
  // ---- phase 2: warps take equal contiguous unit ranges
  // A warp-wide vote as an explicit convergence point: without it the
  // compiler may treat warp 0 (which ran the grid-barrier's thread-0 path)
  // as possibly diverged and route every later shuffle through its slow
  // collective fallback (measured: warp 0 of every CTA 1.5x slower).
  if (__ballot_sync(0xffffffffu, 1) != 0xffffffffu) __trap();
  const int64_t U = all_u;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kBWarps + warp;
  const int64_t GW = static_cast<int64_t>(gridDim.x) * kBWarps;
#if B64_BATCH_UNIT_COST
  const int64_t u_begin = U > 0 ? first_unit[gw] : 0;
  const int64_t u_end = U > 0 ? (gw + 1 < GW ? first_unit[gw + 1] : U) : 0;
#else
  const int64_t u_begin = U > 0 ? muldiv_floor(U, gw, GW) : 0;
  const int64_t u_end = U > 0 ? muldiv_floor(U, gw + 1, GW) : 0;
#endif
  if (u_begin < u_end) {
  const uint64_t pol = policy_evict_first();
  // Two walkers over the same unit sequence, both in registers: the issue
  // walker runs kBSlots units ahead (TMA loads), the consume walker
  // re-derives each unit's descriptor when its data has landed (no
  // descriptor round trip through shared memory).
  Walker<DECODE> wi, wc;
  wi.init(first_msg[gw], k, in_off, out_off, unit_off, lane);
#ifdef B64_BATCH_TRACE_FM
  {
    const int64_t fm = find_message(unit_off, k, u_begin, lane);
    if (lane == 0)
      g_trace[(blockIdx.x * 64 + warp) * 4 + 0] =
          (static_cast<unsigned long long>(first_msg[gw]) << 32) | static_cast<unsigned long long>(fm);
  }
#endif
  wc = wi;

#if B64_BATCH_PREFETCH
  const uintptr_t in_end = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(in_off[k]);
#endif
  auto issue = [&](int64_t u) {
    const UnitDesc d = wi.seek(u, k, in_off, out_off, unit_off, lane);
    if (lane == 0) {
      const int s = static_cast<int>((u - u_begin) % kBSlots);
      const uintptr_t g = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(d.src);
      const uintptr_t g0 = g & ~static_cast<uintptr_t>(15);
      const uint32_t bytes =
          (static_cast<uint32_t>(g & 15) + static_cast<uint32_t>(d.len) + 15u) & ~15u;
      mbar_arrive_expect_tx(&R.full[s], bytes);
      bulk_g2s(R.in[s], reinterpret_cast<const void *>(g0), bytes, &R.full[s], pol);
#if B64_BATCH_PREFETCH
      // units are contiguous in the input: warm L2 with the bytes this warp
      // reads B64_BATCH_PREFETCH units further on (beyond the smem ring)
      const uintptr_t pf = g0 + static_cast<uintptr_t>(B64_BATCH_PREFETCH) * UIN;
      if (pf + UIN <= in_end) bulk_prefetch_l2(reinterpret_cast<const void *>(pf), UIN);
#endif
    }
  };

  int64_t iu = u_begin;
  for (; iu < u_end && iu < u_begin + kBSlots; ++iu) issue(iu);

  const int32_t nu = static_cast<int32_t>(u_end - u_begin);
#ifdef B64_BATCH_TRACE
  unsigned long long tr_bytes = 0;
#endif
#ifdef B64_BATCH_TRACE_WAIT
  unsigned long long tr_wait = 0;
  const long long tl0 = clock64();
#endif
  for (int32_t it = 0; it < nu; ++it) {
    const int s = it % kBSlots;
    const UnitDesc d = wc.seek(u_begin + it, k, in_off, out_off, unit_off, lane);
#ifdef B64_BATCH_TRACE_WAIT  // measurement only: cycles spent waiting for unit data
    const long long tw0 = clock64();
#endif
    mbar_wait_spin(&R.full[s], static_cast<uint32_t>((it / kBSlots) & 1));
#ifdef B64_BATCH_TRACE_WAIT
    tr_wait += static_cast<unsigned long long>(clock64() - tw0);
#endif
    if (it == 0) B64_TRACE(2);
#ifdef B64_BATCH_TRACE
    tr_bytes += static_cast<unsigned long long>(d.len);
#endif
    const uintptr_t gsrc = reinterpret_cast<uintptr_t>(in) + static_cast<uintptr_t>(d.src);
    const int imis = static_cast<int>(gsrc & 15);
    const bool in4 = (gsrc & 3) == 0;
    const uint8_t *sin = R.in[s] + imis;
    uint8_t *gdst = out + d.dst;
    // Output is staged 16-byte aligned (whole-lane STS.128 for full encode
    // passes, no bank conflicts) and realigned per 16-byte granule on the
    // copy-out (two LDS.128 + funnel shift per STG.128).  (Staging encode
    // output congruent to the destination turned every pass into four
    // 4-way-conflicted STS.32 for the 3/4 of units whose destination is not
    // 16-byte aligned.)
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
      // enc_len of a unit (< 2^31 bytes): 32-bit arithmetic
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
    // Slot s is fully read: order those generic reads before the next bulk
    // write into it, then refill the ring.
    fence_proxy_async_smem();
    if (iu < u_end) {
      issue(iu);
      ++iu;
    }
    warp_copy_out(gdst, sout, olen, lane);
    if constexpr (DECODE) {
      // First-error reduction: the warp's minimum offset of the
      // unit, one 64-bit atomicMin on the message's slot (error path only).
      if (lane == 0 && werr != 0xFFFFFFFFu) {
        unsigned long long *tgt = reinterpret_cast<unsigned long long *>(err_pos + d.msg);
        const unsigned long long pos = static_cast<unsigned long long>(d.rel) + werr;
        if (pos < *reinterpret_cast<volatile unsigned long long *>(tgt)) atomicMin(tgt, pos);
      }
    }
    __syncwarp();
  }
#ifdef B64_BATCH_TRACE
  if (lane == 0)
    g_trace[(blockIdx.x * 64 + warp) * 4 + 0] =
        (tr_bytes << 20) | static_cast<unsigned long long>(u_end - u_begin);
#endif
#ifdef B64_BATCH_TRACE_WAIT  // warps 32..: slot 0 = wait cycles, slot 1 = loop cycles
  if (lane == 0) {
    g_trace[(blockIdx.x * 64 + 32 + warp) * 4 + 0] = tr_wait;
    g_trace[(blockIdx.x * 64 + 32 + warp) * 4 + 1] = static_cast<unsigned long long>(clock64() - tl0);
  }
#endif
  }  // u_begin < u_end
  B64_TRACE(3);

  if constexpr (DECODE) {
    // ---- phase 3: per-message results.  After the grid sync every error
    // atomic has landed; status is a pure function of err_pos (R-length).
    // A thread's first message is read before the barrier (its offsets and
    // last four characters -- all finish_stream looks at), so after it only
    // the error slot is loaded.
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kBThreads + tid;
    int64_t pa = 0, pb = 0, po = 0;
    uint32_t last4 = 0;
    if (i0 < k) {
      pa = in_off[i0];
      pb = in_off[i0 + 1];
      po = out_off[i0];
      const int64_t base = pb - pa >= 4 ? pb - 4 : pa;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (base + j < pb) last4 |= static_cast<uint32_t>(in[base + j]) << (8 * j);
    }
    __threadfence();
    grid.sync();
    for (int64_t i = i0; i < k; i += static_cast<int64_t>(gridDim.x) * kBThreads) {
      const bool pre = i == i0;
      const int64_t a = pre ? pa : in_off[i], b = pre ? pb : in_off[i + 1];
      const int64_t len = b - a;
      if (len / 4 == 0 && !((flags & kFlagNoPad) && len >= 2)) continue;  // decided in phase 1
      int64_t err = len / 4 == 0 ? LLONG_MAX : err_pos[i];
      if (err == LLONG_MAX) err = -1;
      const uint8_t *c = in + a;
      const int64_t cb = len >= 4 ? len - 4 : 0;  // index of last4's byte 0
      const uint32_t l4 = last4;
      const StreamResult R = finish_stream_at(
          [pre, c, cb, l4](int64_t x) -> uint32_t {
            return pre ? (l4 >> (8 * static_cast<uint32_t>(x - cb))) & 0xFFu : c[x];
          },
          len, out + (pre ? po : out_off[i]), err, true, flags);
      status[i] = R.status;
      out_len[i] = R.out_len;
      err_pos[i] = R.err_pos;
    }
  }
}

}  // namespace b64
