// b64_onepass.cuh -- single-read compaction:
// Appendix B whitespace removal and the fused
// whitespace-tolerant decode (App. B filter + Algorithm 2, reading
// R-ws-decode) in ONE pass over the text: every input byte is read from HBM
// exactly once, the kept bytes (despace) or the decoded bytes (ws decode)
// are written once, straight from registers with 16-byte (12-byte) stores.
//
// Where the output of a tile goes depends on how many bytes all earlier
// tiles keep (an exclusive prefix over tiles).  Instead of a counting pass
// (which re-reads the input), each CTA classifies a tile as soon as it has
// landed in shared memory, publishes its kept count at once, and keeps the
// raw window in shared memory until the tile is *placed* kOpLag tiles
// later; a dedicated scan warp per CTA sums the published counts of all
// earlier tiles meanwhile (a decoupled prefix with a fixed lag).
//
// Placement is output-driven, at the granularity of 16-byte output
// granules aligned in the destination (despace: out + P + j = 0 mod 16;
// ws decode: compact position P + j = 0 mod 16, i.e. one 16-char decode
// block): the thread whose kept bytes start a granule finds the input
// position of its first byte (rank select in its 32-bit keep mask), and if
// the 16 input bytes there are all kept (a "clean" granule -- most of them
// for text with sparse white space) loads them with two LDS.128 + funnel
// shifts and stores them with one STG.128 (despace) or decodes them in
// registers and stores 12 bytes (ws decode); otherwise it gathers the 16 kept
// bytes one by one.  No compacted stream is staged, no per-byte stores.
//
// Grid: one persistent CTA per SM (cooperative launch: the prefix waits on
// other CTAs, so all of them must be co-resident); tile t (16 KiB window,
// CpGeom) belongs to CTA t mod G.  Per CTA: 16 compute warps, a producer
// warp (lane 0 streams windows HBM -> smem with 1-D TMA into a kOpSlots
// ring), a scan warp.  Iteration j of the compute warps:
//   A  classify tile j: thread tid owns window bytes [32 tid, 32 tid + 32)
//      (two swizzled, conflict-free LDS.128) -> 32-bit keep mask, warp
//      scan of the kept counts -> smem; the last warp to finish publishes
//      the tile's count (cnt[t] = count + 1; 0 = not yet) -- publishing never
//      waits for a prefix
//   B  place tile i = j - kOpLag once its prefix P_i is known (granules)
//   C  one barrier of the compute warps; thread 0 releases tile i's window
//      slot and prefix slot
// Deadlock freedom: a count is published as soon as its window has landed;
// the prefix of tile j - kOpLag only needs counts of tiles of earlier
// rounds, so the smallest unpublished count can always be published.  The
// counts array is zeroed (cudaMemsetAsync) before the launch.
#pragma once
#include <cstdint>

#include "b64_batch.cuh"
#include "b64_codec.cuh"
#include "b64_compact.cuh"
#include "b64_ptx.cuh"

namespace b64 {

#ifndef B64_OP_CTAS  // resident CTAs per SM (launch bounds)
#define B64_OP_CTAS 1
#endif
#ifndef B64_OP_SLOTS
#define B64_OP_SLOTS 7
#endif
#ifndef B64_OP_LAG
#define B64_OP_LAG 3
#endif
#ifndef B64_OP_SCANK  // scan warp: counts loaded per lane per poll (window = 32 * K tiles)
#define B64_OP_SCANK 8
#endif
constexpr int kOpCtas = B64_OP_CTAS;
constexpr int kOpScanK = B64_OP_SCANK;
constexpr int kOpSlots = B64_OP_SLOTS;  // raw windows held: kOpLag placing + loads ahead
constexpr int kOpLag = B64_OP_LAG;      // tile j - kOpLag is placed in iteration j
constexpr int kOpPre = kOpLag + 2;      // prefix ring (scan warp -> compute warps)
static_assert(kOpLag >= 1 && kOpSlots >= kOpLag + 2, "slots hold the lagging tiles plus loads ahead");
constexpr int kOpThreads = kCpThreads + 64;  // + producer warp + scan warp
constexpr int kOpProducer = kCpWarps, kOpScan = kCpWarps + 1;
static_assert(kCpTile == 32 * kCpThreads, "a thread owns 32 contiguous window bytes");

// The published counts are plain values (no data is published through them),
// so relaxed GPU-scope accesses suffice (volatile would be .SYS scope).
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct alignas(128) OpRing {
  uint8_t win[kOpSlots][kCpTile];        // TMA ring of raw windows (16-byte aligned)
  uint32_t msk[kOpSlots][kCpThreads];    // keep mask of each thread's 32 window bytes
  uint16_t inc[kOpSlots][kCpThreads];    // inclusive warp prefix of the kept counts
  int32_t wcnt[kOpSlots][kCpWarps];      // kept bytes per warp
  int32_t tcnt[kOpSlots], tarr[kOpSlots];  // the tile's kept bytes / warps counted so far
  uint64_t full[kOpSlots], empty[kOpSlots];
  uint64_t pfull[kOpPre], pempty[kOpPre];
  int64_t pre[kOpPre];                   // exclusive prefix (kept bytes before the tile)
};

// A: classify a landed window (window bytes [lo, hi) exist).  The tile's
// count is published by the last warp to finish (smem atomics, no barrier).
__device__ __forceinline__ void op_classify(const uint8_t *win, int lo, int hi, uint32_t *msk,
                                            uint16_t *inc, int32_t *wcnt, int32_t *tcnt,
                                            int32_t *tarr, uint32_t *cnt_t) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // lanes 4..7 of each 8-lane phase read their second 16 bytes first: the
  // 8 lanes of a phase then cover all 32 banks in both loads
  const int sw = (lane >> 2) & 1;
  const uint8_t *seg = win + 32 * tid;
  const uint4 A = ptx::lds128(seg + 16 * sw), B = ptx::lds128(seg + 16 - 16 * sw);
  uint32_t w[8];
  w[0] = sw ? B.x : A.x; w[1] = sw ? B.y : A.y; w[2] = sw ? B.z : A.z; w[3] = sw ? B.w : A.w;
  w[4] = sw ? A.x : B.x; w[5] = sw ? A.y : B.y; w[6] = sw ? A.z : B.z; w[7] = sw ? A.w : B.w;
  uint32_t M = 0;  // bit j: window byte 32 tid + j is kept
#pragma unroll
  for (int i = 0; i < 8; ++i) M |= gather4(keep_flags(w[i])) << (4 * i);
  if (lo != 0 || hi != kCpTile) {
    const int a = lo - 32 * tid, b = hi - 32 * tid;
    const uint32_t top = b >= 32 ? 0xFFFFFFFFu : b <= 0 ? 0u : (1u << b) - 1u;
    const uint32_t bot = a <= 0 ? 0u : a >= 32 ? 0xFFFFFFFFu : (1u << a) - 1u;
    M &= top & ~bot;
  }
  msk[tid] = M;
  const int k = __popc(M);
  int incl = k;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  inc[tid] = static_cast<uint16_t>(incl);
  if (lane == 31) {
    wcnt[warp] = incl;
    atomicAdd(tcnt, incl);
    __threadfence_block();
    if (atomicAdd(tarr, 1) == kCpWarps - 1) {
      __threadfence_block();
      st_volatile_u32(cnt_t, static_cast<uint32_t>(atomicAdd(tcnt, 0)) + 1u);
    }
  }
}

// Window position of the r-th (0-based) set bit of M (r < popc(M)).
__device__ __forceinline__ int select_bit(uint32_t M, int r) {
  if (M == 0xFFFFFFFFu) return r;
  int pos = 0;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const int c = __popc(M & ((1u << w) - 1u));
    if (r >= c) {
      r -= c;
      pos += w;
      M >>= w;
    }
  }
  return pos;
}

// The 16 window bytes [x, x + 16) (x any offset, window 16-byte aligned with
// >= 16 bytes of slack): two LDS.128 + word select + funnel shift.
__device__ __forceinline__ uint4 op_load16(const uint8_t *win, int x) {
  const uint8_t *c = win + (x & ~15);
  const uint4 A = ptx::lds128(c), B = ptx::lds128(c + 16);
  const int q = (x >> 2) & 3;
  const uint32_t bs = 8u * static_cast<uint32_t>(x & 3);
  const uint32_t a0 = q == 0 ? A.x : q == 1 ? A.y : q == 2 ? A.z : A.w;
  const uint32_t a1 = q == 0 ? A.y : q == 1 ? A.z : q == 2 ? A.w : B.x;
  const uint32_t a2 = q == 0 ? A.z : q == 1 ? A.w : q == 2 ? B.x : B.y;
  const uint32_t a3 = q == 0 ? A.w : q == 1 ? B.x : q == 2 ? B.y : B.z;
  const uint32_t a4 = q == 0 ? B.x : q == 1 ? B.y : q == 2 ? B.z : B.w;
  return make_uint4(__funnelshift_r(a0, a1, bs), __funnelshift_r(a1, a2, bs),
                    __funnelshift_r(a2, a3, bs), __funnelshift_r(a3, a4, bs));
}

// Up to 16 kept bytes starting at window bit position x (x = 32 t + bit of
// thread t's mask, that byte kept), walking the keep masks forward (tile
// end: bytes past it are absent); returns them packed little-endian in
// (lo, hi), and how many were found.
__device__ __forceinline__ int op_gather16(const uint8_t *win, const uint32_t *msk, int x, int want,
                                           uint64_t &lo, uint64_t &hi) {
  lo = 0;
  hi = 0;
  int got = 0, t = x >> 5;
  uint32_t m = msk[t] & (0xFFFFFFFFu << (x & 31));
  while (got < want) {
    while (m != 0 && got < want) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t v = win[32 * t + b];
      if (got < 8) lo |= v << (8 * got);
      else hi |= v << (8 * (got - 8));
      ++got;
    }
    if (got >= want || ++t >= kCpThreads) break;
    m = msk[t];
  }
  return got;
}

// The placement geometry of tile i for this thread: its kept bytes are
// tile-output bytes [o, o + k); wpre / n from the per-warp counts.
struct OpPlace {
  uint32_t M;
  int k, o, n;
};
__device__ __forceinline__ OpPlace op_place_geom(const OpRing &R, int si) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = lane < kCpWarps ? R.wcnt[si][lane] : 0;
  int winc = c;
#pragma unroll
  for (int o = 1; o < kCpWarps; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, winc, o);
    if (lane >= o) winc += u;
  }
  OpPlace g;
  g.M = R.msk[si][tid];
  g.k = __popc(g.M);
  g.o = __shfl_sync(0xffffffffu, winc - c, warp) + R.inc[si][tid] - g.k;
  g.n = __shfl_sync(0xffffffffu, winc, kCpWarps - 1);
  return g;
}

// The `need` (1..16) kept bytes that start at window position x (a kept
// byte; window bytes past the tile end are never kept), as a 16-byte vector
// (bytes >= need undefined).  Fast paths by the keep masks of x's thread and
// the next: all `need` bytes consecutive ("clean": one realigned 16-byte
// load), or one run of white space inside ("one gap": two realigned loads
// merged at the gap -- a CR LF in MIME text); else a gather, byte by byte.
__device__ __forceinline__ uint4 op_kept16(const uint8_t *win, const uint32_t *msk, int x,
                                           int need) {
  const int t = x >> 5, pos = x & 31;
  const uint64_t mw =
      (static_cast<uint64_t>(msk[t]) |
       (static_cast<uint64_t>(t + 1 < kCpThreads ? msk[t + 1] : 0u) << 32)) >> pos;  // 64 - pos valid bits
  const uint64_t want = (1ull << need) - 1ull;
  if ((mw & want) == want) return op_load16(win, x);
  const int q = __ffsll(static_cast<long long>(~mw)) - 1;  // kept bytes before the gap (< need)
  const uint64_t rest = mw >> q;
  const int g = rest != 0 ? __ffsll(static_cast<long long>(rest)) - 1 : 64;  // gap length
  const int r = need - q;                                                // kept bytes after it
  if (q + g + r <= 64 - pos && ((rest >> g) & ((1ull << r) - 1ull)) == ((1ull << r) - 1ull)) {
    const uint4 A = op_load16(win, x), B = op_load16(win, x + g);
    uint32_t m[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int lb = q - 4 * k;  // bytes of word k taken from A
      m[k] = lb >= 4 ? 0xFFFFFFFFu : lb <= 0 ? 0u : (1u << (8 * lb)) - 1u;
    }
    return make_uint4((A.x & m[0]) | (B.x & ~m[0]), (A.y & m[1]) | (B.y & ~m[1]),
                      (A.z & m[2]) | (B.z & ~m[2]), (A.w & m[3]) | (B.w & ~m[3]));
  }
  uint64_t lo, hi;
  op_gather16(win, msk, x, need, lo, hi);
  return make_uint4(static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32),
                    static_cast<uint32_t>(hi), static_cast<uint32_t>(hi >> 32));
}

// Byte i of a 16-byte vector.
__device__ __forceinline__ uint32_t v16_byte(const uint4 &v, int i) {
  const uint32_t w = i < 4 ? v.x : i < 8 ? v.y : i < 12 ? v.z : v.w;
  return (w >> (8 * (i & 3))) & 0xFFu;
}

// Producer warp: lane 0 streams this CTA's tiles (t = b, b + G, ...) into the ring.
__device__ __forceinline__ void op_producer(OpRing &R, const CpGeom &G, int64_t J, int lane) {
  if (lane != 0) return;
  const uint64_t pol = ptx::policy_evict_first();
  for (int64_t j = 0; j < J; ++j) {
    const int s = static_cast<int>(j % kOpSlots);
    if (j >= kOpSlots) ptx::mbar_wait(&R.empty[s], static_cast<uint32_t>(((j / kOpSlots) & 1) ^ 1));
    const int64_t t = blockIdx.x + j * gridDim.x;
    const uint32_t bytes = static_cast<uint32_t>((G.hi(t) + 15) & ~15);
    ptx::mbar_arrive_expect_tx(&R.full[s], bytes);
    ptx::bulk_g2s(R.win[s], reinterpret_cast<const void *>(G.a0 + static_cast<uintptr_t>(t) * kCpTile),
                  bytes, &R.full[s], pol);
  }
}

// The `need` (<= 16) kept characters that end just before input offset x_end
// (whitespace skipped), in order, into dst[0 .. need); a full warp.  Reads
// the input backward 32 bytes at a time.
__device__ __forceinline__ void op_gather_back(const uint8_t *in, int64_t x_end, int need,
                                               uint8_t *dst, int lane) {
  int got = 0;
  int64_t x = x_end;
  while (got < need && x > 0) {
    const int64_t i = x - 32 + lane;
    const uint32_t v = i >= 0 ? in[i] : 0x20u;
    const bool keep = !is_space_byte(v);
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    const int above = lane == 31 ? 0 : __popc(bal >> (lane + 1));  // kept lanes after this one
    if (keep && above < need - got) dst[need - got - 1 - above] = static_cast<uint8_t>(v);
    got += __popc(bal);
    x -= 32;
  }
  __syncwarp();
}

// Scan warp: for this CTA's tiles in order, the exclusive prefix of the
// published counts -> R.pre.  It keeps a frontier f (S = sum of cnt[0, f))
// and polls a window [f, f + 32 kOpScanK) of the counts at a time: every
// own tile whose index the ready part of the window reaches gets its prefix
// from the same poll (about 1.7 rounds of the grid per window), so one L2
// round trip can serve several tiles.
__device__ __forceinline__ void op_scan(OpRing &R, const uint32_t *cnt, int64_t J, int lane) {
  const int64_t b = blockIdx.x, Gs = gridDim.x;
  const int64_t tmax = b + (J - 1) * Gs;  // this CTA's last tile
  int64_t S = 0, f = 0, j = 0;
  auto emit = [&](int64_t jj, int64_t P) {
    const int p = static_cast<int>(jj % kOpPre);
    if (jj >= kOpPre) ptx::mbar_wait(&R.pempty[p], static_cast<uint32_t>(((jj / kOpPre) & 1) ^ 1), 200);
    if (lane == 0) {
      R.pre[p] = P;
      ptx::mbar_arrive(&R.pfull[p]);
    }
  };
  while (j < J) {
    if (b + j * Gs == f) {  // prefix of tile f = S
      emit(j, S);
      ++j;
      continue;
    }
    const int64_t wend = f + 32 * kOpScanK < tmax ? f + 32 * kOpScanK : tmax;
    const int64_t need = b + j * Gs - f;  // the window must be ready up to here
    uint32_t v[kOpScanK];
#pragma unroll
    for (int k = 0; k < kOpScanK; ++k) {
      const int64_t idx = f + lane + 32 * k;
      v[k] = idx < wend ? ld_volatile_u32(cnt + idx) : 0u;
    }
    int64_t F;  // ready entries [f, f + F)
    while (true) {
      F = wend - f;
#pragma unroll
      for (int k = kOpScanK - 1; k >= 0; --k) {
        const uint32_t nr = __ballot_sync(0xffffffffu, v[k] == 0 && f + lane + 32 * k < wend);
        if (nr) F = 32 * k + __ffs(nr) - 1;
      }
      if (F >= need || F == wend - f) break;
      __nanosleep(64);
#pragma unroll
      for (int k = 0; k < kOpScanK; ++k) {
        const int64_t idx = f + lane + 32 * k;
        if (v[k] == 0 && idx < wend) v[k] = ld_volatile_u32(cnt + idx);
      }
    }
    // prefixes of the own tiles the ready part reaches, then advance
    while (j < J && b + j * Gs - f <= F) {
      const int64_t d = b + j * Gs - f;
      uint32_t part = 0;
#pragma unroll
      for (int k = 0; k < kOpScanK; ++k)
        if (lane + 32 * k < d) part += v[k] - 1u;
      emit(j, S + __reduce_add_sync(0xffffffffu, part));
      ++j;
    }
    uint32_t all = 0;
#pragma unroll
    for (int k = 0; k < kOpScanK; ++k)
      if (lane + 32 * k < F) all += v[k] - 1u;
    S += __reduce_add_sync(0xffffffffu, all);
    f += F;
  }
}

__device__ __forceinline__ void op_init(OpRing &R) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kOpSlots; ++s) {
      ptx::mbar_init(&R.full[s], 1);
      ptx::mbar_init(&R.empty[s], 1);
      R.tcnt[s] = 0;
      R.tarr[s] = 0;
    }
    for (int p = 0; p < kOpPre; ++p) {
      ptx::mbar_init(&R.pfull[p], 1);
      ptx::mbar_init(&R.pempty[p], 1);
    }
    ptx::fence_mbar_init();
  }
}

// ------------------------------------------------------ despace (f3) ---
struct alignas(128) OpDsSmem {
  OpRing r;
};

// B (despace): tile i's kept bytes -> out + P.  Granules: tile-output
// bytes [0, gb0) (the tail of a destination granule the previous tile began)
// and [gb0 + 16 m, gb0 + 16 (m + 1)), each started by the thread that owns
// its first kept byte; full granules leave with one STG.128, the tile's
// partial first / last granule with byte stores.
__device__ __forceinline__ void op_place_despace(const OpRing &R, int si, int64_t P, uint8_t *out,
                                                 int64_t ti, const CpGeom &G, int64_t *out_len) {
  const int tid = threadIdx.x;
  const OpPlace g = op_place_geom(R, si);
  const uint8_t *win = R.win[si];
  const uint32_t *msk = R.msk[si];
  uint8_t *dst = out + P;
  const int gb0 = static_cast<int>((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15);
  int j = (gb0 > 0 && g.o == 0 && g.k > 0) ? 0 : g.o + ((gb0 - g.o) & 15);
  while (j < g.o + g.k) {
    const int jn = (j == 0 && gb0 > 0) ? gb0 : j + 16;  // end of the granule
    const int need = (jn < g.n ? jn : g.n) - j;
    const uint4 v = op_kept16(win, msk, 32 * tid + select_bit(g.M, j - g.o), need);
    if (need == 16) {
      *reinterpret_cast<uint4 *>(dst + j) = v;
    } else {
      for (int bb = 0; bb < need; ++bb) dst[j + bb] = static_cast<uint8_t>(v16_byte(v, bb));
    }
    j = jn;
  }
  if (tid == 0 && ti == G.ntiles - 1) *out_len = P + g.n;
}

__global__ void __launch_bounds__(kOpThreads, kOpCtas)
    despace1_kernel(const uint8_t *__restrict__ in, int64_t m, uint8_t *__restrict__ out,
                    uint32_t *cnt, int64_t *out_len) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  OpDsSmem &S = *reinterpret_cast<OpDsSmem *>(smem_raw);
  OpRing &R = S.r;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  CpGeom G;
  G.init(in, m, 0);
  op_init(R);
  __syncthreads();
  const int64_t b = blockIdx.x, Gs = gridDim.x;
  const int64_t J = (G.ntiles - b + Gs - 1) / Gs;  // this CTA's tiles
  if (warp == kOpProducer) {
    op_producer(R, G, J, lane);
    return;
  }
  if (warp == kOpScan) {
    op_scan(R, cnt, J, lane);
    return;
  }
  for (int64_t j = 0; j < J + kOpLag; ++j) {
    const int64_t i = j - kOpLag;
    const int64_t t = b + j * Gs, ti = b + i * Gs;
    if (j < J) {  // A
      const int s = static_cast<int>(j % kOpSlots);
      ptx::mbar_wait_spin(&R.full[s], static_cast<uint32_t>((j / kOpSlots) & 1));
      __syncwarp();
      op_classify(R.win[s], G.lo(t), G.hi(t), R.msk[s], R.inc[s], R.wcnt[s], &R.tcnt[s], &R.tarr[s],
                  cnt + t);
    }
    const int si = static_cast<int>((i + kOpSlots) % kOpSlots);
    if (i >= 0) {  // B
      const int p = static_cast<int>(i % kOpPre);
      ptx::mbar_wait_spin(&R.pfull[p], static_cast<uint32_t>((i / kOpPre) & 1));
      __syncwarp();
      op_place_despace(R, si, R.pre[p], out, ti, G, out_len);
    }
    ptx::named_bar_sync(1, kCpThreads);  // C
    if (tid == 0 && i >= 0) {
      R.tcnt[si] = 0;
      R.tarr[si] = 0;
      ptx::mbar_arrive(&R.empty[si]);
      ptx::mbar_arrive(&R.pempty[i % kOpPre]);
    }
  }
}

// ------------------------------------------- fused ws decode (f4 general) ---
struct alignas(128) OpWsSmem {
  OpRing r;
  alignas(16) uint8_t hblk[2][32];  // head block of the tile being placed, by parity: carry | first chars
  int32_t hgo[2];                    // the head block is complete in its tile
  alignas(16) uint8_t blk[64];
  alignas(16) uint8_t bout[64];
  int64_t red[66];
  int64_t sel[4];
  int32_t flag;
};

// Per-call scratch in the caller's workspace (zeroed before the launch).
struct OpWsHdr {
  unsigned long long errkey;  // ~(min error offset, compact coordinates); 0 = none
  unsigned int done;          // CTAs finished
  unsigned int pad;
  int64_t M;                  // kept characters of the whole text (written by the last tile)
};
static_assert(sizeof(OpWsHdr) <= 48, "OpWsHdr must end before WlState (kWlStateOffset)");

// Decode 16 characters (w, little-endian) of a non-final block -> 12 bytes
// (o); returns a 16-bit mask of the invalid characters (table A, P:157;
// '=' is invalid outside the final quad).
__device__ __forceinline__ uint32_t op_dec16(const uint32_t (&w)[4], uint32_t tb, uint32_t (&o)[3]) {
  uint32_t v[16], acc = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[4 * k + 0] = lds_u8((w[k] & 0xFFu) | tb);
    v[4 * k + 1] = lds_u8(__byte_perm(w[k], tb, 0x7651));
    v[4 * k + 2] = lds_u8(__byte_perm(w[k], tb, 0x7652));
    v[4 * k + 3] = lds_u8(__byte_perm(w[k], tb, 0x7653));
    acc |= v[4 * k] | v[4 * k + 1] | v[4 * k + 2] | v[4 * k + 3];
  }
  uint32_t bad = 0;
  if (acc & 0x80u) {
#pragma unroll
    for (int j = 0; j < 16; ++j) bad |= ((v[j] >> 7) & 1u) << j;
  }
  uint32_t V[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    V[k] = ((v[4 * k] * 64u + v[4 * k + 1]) * 64u + v[4 * k + 2]) * 64u + v[4 * k + 3];
  o[0] = __byte_perm(V[0], V[1], 0x6012);
  o[1] = __byte_perm(V[1], V[2], 0x5601);
  o[2] = __byte_perm(V[2], V[3], 0x4560);
  return bad;
}

// Store a decoded block's 12 bytes at gdst (STG.32 x 3 when 4-byte aligned).
__device__ __forceinline__ void op_store12(uint8_t *gdst, const uint32_t (&o)[3]) {
  if ((reinterpret_cast<uintptr_t>(gdst) & 3) == 0) {
    uint32_t *g = reinterpret_cast<uint32_t *>(gdst);
    g[0] = o[0];
    g[1] = o[1];
    g[2] = o[2];
  } else {
    for (int b = 0; b < 12; ++b) gdst[b] = static_cast<uint8_t>(o[b >> 2] >> (8 * (b & 3)));
  }
}

// B (ws decode): the complete 16-char blocks of tile i (compact positions
// P + j = 0 mod 16), each decoded in registers by the thread owning its
// first char and stored as 12 bytes.  The block straddling the tile's start
// is staged in hb: warp 0 puts the carry there (the h = P & 15 kept chars
// before the tile, from the 32 prefetched raw bytes or a backward gather),
// the owner of the tile's first char its first 16 - h chars; thread 0
// decodes it after the barrier (op_head_ws).  The block straddling the
// tile's end is left to the next tile.
__device__ __forceinline__ void op_place_ws(const OpRing &R, int si, int64_t P, uint8_t *out,
                                            const uint8_t *in, const CpGeom &G, int64_t ti,
                                            uint32_t raw, OpWsHdr *hdr, uint8_t *hb, int32_t *hgo) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const OpPlace g = op_place_geom(R, si);
  const uint8_t *win = R.win[si];
  const uint32_t *msk = R.msk[si];
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(g_dec_tab));
  const int h = static_cast<int>(P & 15);
  const int gb0 = (16 - h) & 15;
  const bool head = h > 0 && g.n >= gb0;
  if (tid == 0) *hgo = head ? 1 : 0;
  if (head && warp == 0) {
    const bool keep = !is_space_byte(raw);
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (__popc(bal) >= h) {
      const int above = lane == 31 ? 0 : __popc(bal >> (lane + 1));
      if (keep && above < h) hb[h - 1 - above] = static_cast<uint8_t>(raw);
    } else {
      op_gather_back(in, G.off(ti, G.lo(ti)), h, hb, lane);
    }
  }
  uint32_t bad_pos = 0xFFFFFFFFu;  // min bad compact offset relative to P
  if (head && g.o == 0 && g.k > 0) {  // this thread owns the tile's first char
    const uint4 v = op_kept16(win, msk, 32 * tid + __ffs(g.M) - 1, gb0);
    for (int bb = 0; bb < gb0; ++bb) hb[h + bb] = static_cast<uint8_t>(v16_byte(v, bb));
  }
  // the full blocks starting in this thread's kept chars: tile-output j = gb0 (mod 16)
  for (int j = g.o + ((gb0 - g.o) & 15); j < g.o + g.k && j + 16 <= g.n; j += 16) {
    const uint4 v = op_kept16(win, msk, 32 * tid + select_bit(g.M, j - g.o), 16);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[3];
    const uint32_t bad = op_dec16(w, tb, o);
    op_store12(out + 3 * ((P + j) / 4), o);
    if (bad && bad_pos == 0xFFFFFFFFu) bad_pos = static_cast<uint32_t>(j) + __ffs(bad) - 1;
  }
  // first-error reduction: warp minimum, one atomic per warp
  const uint32_t wmin = __reduce_min_sync(0xffffffffu, bad_pos);
  if (lane == 0 && wmin != 0xFFFFFFFFu) {
    const unsigned long long key = ~(static_cast<unsigned long long>(P) + wmin);
    if (key > *reinterpret_cast<volatile unsigned long long *>(&hdr->errkey)) atomicMax(&hdr->errkey, key);
  }
  if (tid == 0 && ti == G.ntiles - 1) hdr->M = P + g.n;
}

// The head block of a placed tile (thread 0, after the barrier that orders
// hb's writes): 16 staged chars at compact position P - (P & 15).
__device__ __forceinline__ void op_head_ws(const uint8_t *hb, int64_t P, uint8_t *out, OpWsHdr *hdr) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) w[k] = reinterpret_cast<const uint32_t *>(hb)[k];
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(g_dec_tab));
  uint32_t o[3];
  const uint32_t bad = op_dec16(w, tb, o);
  const int64_t B = P - (P & 15);
  op_store12(out + 3 * (B / 4), o);
  if (bad) {
    const unsigned long long key = ~(static_cast<unsigned long long>(B) + (__ffs(bad) - 1));
    if (key > *reinterpret_cast<volatile unsigned long long *>(&hdr->errkey)) atomicMax(&hdr->errkey, key);
  }
}

// Original input offset of compact position e (CTA-wide, error path only).
__device__ int64_t op_map_offset(OpWsSmem &S, const CpGeom &G, const uint32_t *cnt, int64_t e) {
  const int tid = threadIdx.x, nt = blockDim.x;
  {  // tile holding e
    const int64_t per = (G.ntiles + nt - 1) / nt;
    const int64_t a = tid * per, c1 = a + per < G.ntiles ? a + per : G.ntiles;
    int64_t sum = 0;
    for (int64_t t = a; t < c1; ++t) sum += cnt[t] - 1u;
    int64_t pre, pb, tot, tb;
    block_exclusive_scan2(sum, 0, pre, pb, tot, tb, S.red);
    if (e >= pre && e < pre + sum) {
      int64_t acc = pre;
      for (int64_t t = a; t < c1; ++t) {
        const int64_t c = cnt[t] - 1u;
        if (e < acc + c) {
          S.sel[2] = t;
          S.sel[3] = e - acc;
          break;
        }
        acc += c;
      }
    }
    __syncthreads();
  }
  // byte of that tile: 32 window bytes per thread
  const int64_t t = S.sel[2], r = S.sel[3];
  const int lo = G.lo(t), hi = G.hi(t);
  const uint8_t *w = reinterpret_cast<const uint8_t *>(G.a0 + static_cast<uintptr_t>(t) * kCpTile);
  const int x0 = tid * 32;
  int c = 0;
  for (int x = x0; x < x0 + 32; ++x)
    if (x >= lo && x < hi && !is_space_byte(w[x])) ++c;
  int64_t pre, pb, tot, tb;
  block_exclusive_scan2(c, 0, pre, pb, tot, tb, S.red);
  if (r >= pre && r < pre + c) {
    int64_t k = pre;
    for (int x = x0; x < x0 + 32; ++x) {
      if (x >= lo && x < hi && !is_space_byte(w[x])) {
        if (k == r) {
          S.sel[0] = G.off(t, x);
          break;
        }
        ++k;
      }
    }
  }
  __syncthreads();
  return S.sel[0];
}

__global__ void __launch_bounds__(kOpThreads, kOpCtas)
    decode_ws1_kernel(const uint8_t *__restrict__ in, int64_t m, uint8_t *__restrict__ out,
                      uint32_t *cnt, OpWsHdr *hdr, b64_result *res, int flags,
                      const int32_t *skip) {
  if (skip != nullptr && *skip == 1) return;  // the line-structured fast path already decoded
  extern __shared__ __align__(128) uint8_t smem_raw[];
  OpWsSmem &S = *reinterpret_cast<OpWsSmem *>(smem_raw);
  OpRing &R = S.r;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  CpGeom G;
  G.init(in, m, 0);
  if (tid < 256) g_dec_tab[tid] = kInvalid;
  op_init(R);
  __syncthreads();
  if (tid < 64) g_dec_tab[ascii_of(tid, flags)] = static_cast<uint8_t>(tid);
  __syncthreads();
  const int64_t b = blockIdx.x, Gs = gridDim.x;
  const int64_t J = (G.ntiles - b + Gs - 1) / Gs;
  if (warp == kOpProducer) {
    op_producer(R, G, J, lane);
  } else if (warp == kOpScan) {
    op_scan(R, cnt, J, lane);
  } else {
    // Warp 0 prefetches, one iteration ahead, the 32 input bytes before the
    // window of the next tile to be placed (its carry comes from them).
    uint32_t raw_cur = 0x20u;
    for (int64_t j = 0; j < J + kOpLag; ++j) {
      const int64_t i = j - kOpLag;
      const int64_t t = b + j * Gs, ti = b + i * Gs;
      uint32_t raw_nxt = 0x20u;
      if (warp == 0 && i + 1 >= 0 && i + 1 < J) {
        const int64_t tn = ti + Gs;
        const int64_t x = G.off(tn, G.lo(tn)) - 32 + lane;
        raw_nxt = x >= 0 ? in[x] : 0x20u;
      }
      if (j < J) {  // A
        const int s = static_cast<int>(j % kOpSlots);
        ptx::mbar_wait_spin(&R.full[s], static_cast<uint32_t>((j / kOpSlots) & 1));
        __syncwarp();
        op_classify(R.win[s], G.lo(t), G.hi(t), R.msk[s], R.inc[s], R.wcnt[s], &R.tcnt[s],
                    &R.tarr[s], cnt + t);
      }
      const int si = static_cast<int>((i + kOpSlots) % kOpSlots);
      if (i >= 0) {  // B
        const int p = static_cast<int>(i % kOpPre);
        ptx::mbar_wait_spin(&R.pfull[p], static_cast<uint32_t>((i / kOpPre) & 1));
        __syncwarp();
        op_place_ws(R, si, R.pre[p], out, in, G, ti, raw_cur, hdr, S.hblk[i & 1], &S.hgo[i & 1]);
      }
      ptx::named_bar_sync(1, kCpThreads);  // C
      if (tid == 0 && i >= 0) {
        const int64_t P = R.pre[i % kOpPre];
        R.tcnt[si] = 0;
        R.tarr[si] = 0;
        ptx::mbar_arrive(&R.empty[si]);
        ptx::mbar_arrive(&R.pempty[i % kOpPre]);
        if (S.hgo[i & 1]) op_head_ws(S.hblk[i & 1], P, out, hdr);
      }
      raw_cur = raw_nxt;
    }
  }

  // Last CTA out: the final block with the final-quad rules, the result.
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    S.flag = atomicAdd(&hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!S.flag) return;
  __threadfence();
  const int64_t M = *reinterpret_cast<volatile int64_t *>(&hdr->M);
  const unsigned long long ek = *reinterpret_cast<volatile unsigned long long *>(&hdr->errkey);
  const int64_t etile = ek ? static_cast<int64_t>(~ek) : -1;
  const int64_t Bf = M > 0 ? 16 * ((M - 1) / 16) : 0;  // the final block [Bf, M)
  if (warp == 0) {
    int64_t err = etile;
    if (err < 0 || err >= Bf) {  // no error before the final block: decode it with its rules
      const int Lf = static_cast<int>(M - Bf);
      op_gather_back(in, m, Lf, S.blk, lane);
      const int q4f = Lf & ~3;
      const bool fin = (M % 4) == 0;
      uint32_t ch2 = 0, ch1 = 0;
      int pads = 0;
      if (fin && q4f >= 4) {
        ch2 = S.blk[q4f - 2];
        ch1 = S.blk[q4f - 1];
        pads = ch1 == '=' ? (ch2 == '=' ? 2 : 1) : 0;
      }
      uint32_t e = 0xFFFFFFFFu;
      if (q4f > 0) e = decode_tile<16, 16, false, 1, false, 32>(S.blk, q4f, S.bout, lane, lane, fin, ch2, ch1);
      __syncwarp();
      const int olen = 3 * (q4f / 4) - pads;
      if (lane < olen) out[3 * (Bf / 4) + lane] = S.bout[lane];
      __syncwarp();
      err = e != 0xFFFFFFFFu ? Bf + e : -1;
    }
    if (lane == 0) {
      const uint8_t *bl = S.blk;
      const StreamResult Rs = finish_stream_at([bl, Bf](int64_t x) -> uint32_t { return bl[x - Bf]; },
                                               M, out, err, true, flags);
      S.sel[0] = Rs.out_len;
      S.sel[1] = Rs.err_pos;
      S.sel[2] = Rs.status;
      S.sel[3] = Rs.pad_count;
    }
  }
  __syncthreads();
  const int64_t olen = S.sel[0], ep = S.sel[1];
  const int32_t st = static_cast<int32_t>(S.sel[2]), pc = static_cast<int32_t>(S.sel[3]);
  __syncthreads();
  const int64_t oep = ep >= 0 ? op_map_offset(S, G, cnt, ep) : -1;
  if (tid == 0) {
    res->out_len = olen;
    res->err_pos = oep;
    res->status = st;
    res->pad_count = pc;
  }
}

}  // namespace b64
