// b64_onepass.cuh -- single-read compaction:
// Appendix B whitespace removal and the fused
// whitespace-tolerant decode (App. B filter + Algorithm 2, reading
// R-ws-decode) in ONE pass over the text: every input byte is read from HBM
// exactly once, the kept bytes (despace) or the decoded bytes (ws decode)
// are written once.
//
// Where the output of a tile goes depends on how many bytes all earlier
// tiles keep (an exclusive prefix sum over tiles).  Instead of a counting
// pass (which re-reads the input), each CTA publishes its tile's kept count
// as soon as the tile has landed in shared memory and *defers* the tile's
// placement by kOpLag tiles; a dedicated scan warp per CTA sums the
// published counts of all earlier tiles meanwhile (a decoupled prefix with a
// fixed lag, the counts of one "round" of the grid at a time).  The tile
// stays in shared memory until then, so the input is never read twice.
//
// Grid: one persistent CTA per SM (cooperative launch: the prefix waits on
// other CTAs, so all of them must be co-resident); tile t (16 KiB window,
// CpGeom) belongs to CTA t mod G, its round is t / G.  Per CTA: 16 compute
// warps, a producer warp (lane 0 streams windows HBM -> smem with 1-D TMA
// into a kOpStages ring), a scan warp.  Per iteration j of the compute warps:
//   A  count tile j: classify its 16 KiB (keep flags, 8 words per thread),
//      keep masks -> smem, per-warp kept counts -> smem
//   B  place tile i = j - kOpLag: wait for its prefix P_i (scan warp), pack
//      its kept bytes into a shared-memory stream (PRMT + byte stores)
//   C  one CTA barrier
//   D  thread 0 publishes tile j's kept count (cnt[t] = count + 1; 0 = not
//      yet), releases tile i's ring slot
//   E  tile i's stream leaves: despace -- one bulk (TMA) store of the
//      aligned interior at out + P_i (stream placed congruent mod 16) plus
//      byte stores for the edges; ws decode -- its complete 16-char blocks
//      are decoded straight from the stream (decode_tile) and stored.
// Deadlock freedom: tile j's count is published before the CTA waits for
// the prefix of tile j - kOpLag, and that prefix only needs counts of tiles
// of earlier rounds, so the smallest unpublished count can always be
// published.  The counts array is zeroed (cudaMemsetAsync) before the launch.
#pragma once
#include <cstdint>

#include "b64_batch.cuh"
#include "b64_codec.cuh"
#include "b64_compact.cuh"
#include "b64_ptx.cuh"

namespace b64 {

#ifndef B64_OP_STAGES
#define B64_OP_STAGES 7
#endif
#ifndef B64_OP_LAG
#define B64_OP_LAG 3
#endif
constexpr int kOpStages = B64_OP_STAGES;  // input ring: window + keep masks + warp counts
constexpr int kOpLag = B64_OP_LAG;        // tile j - kOpLag is placed in iteration j
constexpr int kOpPre = kOpLag + 2;        // prefix ring (scan warp -> compute warps)
static_assert(kOpStages >= kOpLag + 2, "the ring holds the lagging tiles plus one load ahead");
constexpr int kOpThreads = kCpThreads + 64;  // + producer warp + scan warp
constexpr int kOpProducer = kCpWarps, kOpScan = kCpWarps + 1;

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct alignas(128) OpRing {
  uint8_t win[kOpStages][kCpTile];     // TMA ring (16-byte aligned windows)
  uint32_t nib[kOpStages][kCpThreads];  // keep masks (8 nibbles per thread)
  int32_t wcnt[kOpStages][kCpWarps];    // kept bytes per warp
  uint64_t full[kOpStages], empty[kOpStages];
  uint64_t pfull[kOpPre], pempty[kOpPre];
  int64_t pre[kOpPre];                  // exclusive prefix (kept bytes before the tile)
  alignas(16) uint8_t carry[kOpPre][16];  // ws decode: the <= 15 kept chars before the tile's block
  uint32_t ktab[16];
};

// A: keep masks and per-warp kept counts of one window (bytes [lo, hi) valid).
__device__ __forceinline__ void op_count(const uint8_t *win, int lo, int hi, uint32_t *nib,
                                         int32_t *wcnt) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wbase = warp * kCpWarpWords + lane;
  const uint32_t *w = reinterpret_cast<const uint32_t *>(win) + wbase;
  uint32_t x[kCpPerLane];
#pragma unroll
  for (int i = 0; i < kCpPerLane; ++i) x[i] = w[32 * i];
  const uint32_t n = tile_nib(x, lo, hi, wbase, lo != 0 || hi != kCpTile);
  nib[tid] = n;
  const int c = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<uint32_t>(__popc(n))));
  if (lane == 0) wcnt[warp] = c;
}

// B: pack the kept bytes of a counted window into stream[dst, dst + n) in
// order (n = sum of wcnt); returns n.  No barrier inside (wcnt / nib come
// from an earlier iteration); the caller's next barrier orders the stores.
__device__ __forceinline__ int op_place(const uint8_t *win, const uint32_t *nibs,
                                        const int32_t *wcnt, uint8_t *stream, int dst,
                                        const uint32_t *ktab) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = lane < kCpWarps ? wcnt[lane] : 0;
  int incl = c;
#pragma unroll
  for (int o = 1; o < kCpWarps; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const int wpre = __shfl_sync(0xffffffffu, incl - c, warp);
  const int total = __shfl_sync(0xffffffffu, incl, kCpWarps - 1);
  const uint32_t nib = nibs[tid];
  // per-word kept counts, 4 per register as bytes, warp-scanned
  uint32_t nc = nib - ((nib >> 1) & 0x55555555u);
  nc = (nc & 0x33333333u) + ((nc >> 2) & 0x33333333u);
  const uint32_t x0 = nc & 0x0F0F0F0Fu;         // words 0, 2, 4, 6
  const uint32_t x1 = (nc >> 4) & 0x0F0F0F0Fu;  // words 1, 3, 5, 7
  uint32_t s0 = x0, s1 = x1;
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
  const uint32_t e0 = s0 - x0, e1 = s1 - x1;
  const uint32_t *seg = reinterpret_cast<const uint32_t *>(win) + warp * kCpWarpWords + lane;
  uint8_t *ws = stream + dst + wpre;
  int base = 0;
#pragma unroll
  for (int i = 0; i < kCpPerLane; ++i) {
    const uint32_t e = ktab[(nib >> (4 * i)) & 0xFu];
    uint32_t cw;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(cw) : "r"(seg[32 * i]), "r"(e));
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

// Producer warp: lane 0 streams this CTA's tiles (t = b, b + G, ...) into the ring.
__device__ __forceinline__ void op_producer(OpRing &R, const CpGeom &G, int64_t J, int lane) {
  if (lane != 0) return;
  const uint64_t pol = ptx::policy_evict_first();
  for (int64_t j = 0; j < J; ++j) {
    const int s = static_cast<int>(j % kOpStages);
    if (j >= kOpStages) ptx::mbar_wait(&R.empty[s], static_cast<uint32_t>(((j / kOpStages) & 1) ^ 1));
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
// published counts -> R.pre (and, for the ws decode, the carry characters).
template <bool CARRY>
__device__ __forceinline__ void op_scan(OpRing &R, const CpGeom &G, const uint32_t *cnt,
                                        int64_t J, int lane) {
  int64_t S = 0, tc = 0;
  for (int64_t j = 0; j < J; ++j) {
    const int64_t t = blockIdx.x + j * gridDim.x;
    while (tc < t) {  // add cnt[tc .. t), up to 256 per round trip
      const int64_t n = t - tc < 256 ? t - tc : 256;
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        v[k] = lane + 32 * k < n ? ld_volatile_u32(cnt + tc + lane + 32 * k) : 1u;
      while (true) {
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) ok = ok && v[k] != 0;
        if (__all_sync(0xffffffffu, ok)) break;
        __nanosleep(100);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (v[k] == 0) v[k] = ld_volatile_u32(cnt + tc + lane + 32 * k);
      }
      uint32_t sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += v[k] - 1u;
      S += __reduce_add_sync(0xffffffffu, sum);
      tc += n;
    }
    const int p = static_cast<int>(j % kOpPre);
    if (j >= kOpPre) ptx::mbar_wait(&R.pempty[p], static_cast<uint32_t>(((j / kOpPre) & 1) ^ 1), 200);
    if (lane == 0) R.pre[p] = S;
    if constexpr (CARRY) op_gather_back(G.in, G.off(t, G.lo(t)), static_cast<int>(S & 15), R.carry[p], lane);
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&R.pfull[p]);
  }
}

__device__ __forceinline__ void op_init(OpRing &R) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kOpStages; ++s) {
      ptx::mbar_init(&R.full[s], 1);
      ptx::mbar_init(&R.empty[s], 1);
    }
    for (int p = 0; p < kOpPre; ++p) {
      ptx::mbar_init(&R.pfull[p], 1);
      ptx::mbar_init(&R.pempty[p], 1);
    }
    ptx::fence_mbar_init();
  }
  init_ktab(R.ktab);
}

// ------------------------------------------------------ despace (f3) ---
struct alignas(128) OpDsSmem {
  OpRing r;
  alignas(16) uint8_t stream[2][kCpTile + 32];  // tile i's stream leaves during iteration i + kOpLag
};

__global__ void __launch_bounds__(kOpThreads, 1)
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
    op_scan<false>(R, G, cnt, J, lane);
    return;
  }
  const uint64_t pol = ptx::policy_evict_first();
  const uintptr_t obase = reinterpret_cast<uintptr_t>(out);
  for (int64_t j = 0; j < J + kOpLag; ++j) {
    const int64_t i = j - kOpLag;
    const int s = static_cast<int>(j % kOpStages);
    const int si = static_cast<int>((i + kOpStages) % kOpStages);
    const int64_t t = b + j * Gs, ti = b + i * Gs;
    if (j < J) {  // A
      ptx::mbar_wait_spin(&R.full[s], static_cast<uint32_t>((j / kOpStages) & 1));
      op_count(R.win[s], G.lo(t), G.hi(t), R.nib[s], R.wcnt[s]);
    }
    int64_t P = 0;
    int n = 0, dst = 0;
    if (i >= 0) {  // B
      const int p = static_cast<int>(i % kOpPre);
      ptx::mbar_wait_spin(&R.pfull[p], static_cast<uint32_t>((i / kOpPre) & 1));
      P = R.pre[p];
      dst = static_cast<int>((obase + static_cast<uintptr_t>(P)) & 15);
      n = op_place(R.win[si], R.nib[si], R.wcnt[si], S.stream[i & 1], dst, R.ktab);
      ptx::fence_proxy_async_smem();  // the stream's bytes -> the bulk store after the barrier
    }
    // the bulk store issued last iteration (tile i-1) reads stream[(i-1)&1],
    // which tile i+1 overwrites after this barrier
    if (tid == 0) ptx::bulk_wait_read<0>();
    ptx::named_bar_sync(1, kCpThreads);  // C (compute warps only)
    if (tid == 0) {   // D
      if (j < J) {
        int c = 0;
#pragma unroll
        for (int w = 0; w < kCpWarps; ++w) c += R.wcnt[s][w];
        st_volatile_u32(cnt + t, static_cast<uint32_t>(c) + 1u);
      }
      if (i >= 0) {
        ptx::mbar_arrive(&R.empty[si]);
        ptx::mbar_arrive(&R.pempty[i % kOpPre]);
        if (ti == G.ntiles - 1) *out_len = P + n;
      }
    }
    if (i >= 0) cta_copy_out_bulk(out + P, S.stream[i & 1] + dst, n, pol);  // E
  }
  if (tid == 0) ptx::bulk_wait<0>();
}

// ------------------------------------------- fused ws decode (f4 general) ---
struct alignas(128) OpWsSmem {
  OpRing r;
  alignas(16) uint8_t stream[2][kCpTile + 64];  // [0, h) carry chars, then the tile's kept chars
  alignas(16) uint8_t ostage[kCpTile / 4 * 3 + 64];
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

static_assert(B64_DEC_STG32, "op_decode_blocks stores decoded runs from registers");

// Decode `nc` (multiple of 16) stream chars at sin (compact position Bc) into
// out + 3*Bc/4; non-final blocks ('=' is invalid); errors -> hdr->errkey.
__device__ __forceinline__ void op_decode_blocks(OpWsSmem &S, const uint8_t *sin, int nc, int64_t Bc,
                                                 uint8_t *out, OpWsHdr *hdr) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int mis = static_cast<int>(reinterpret_cast<uintptr_t>(out + 3 * (Bc / 4)) & 15);
  constexpr int P = (kCpTile + 16) / (kCpThreads * 16) + 1;
  uint8_t *gdst = out + 3 * (Bc / 4);
  const int olen = 3 * (nc / 4);
  uint32_t e;
  if ((mis & 3) == 0) {  // each thread's 12 bytes straight to HBM
    e = decode_tile<16, 4, false, P, true, kCpThreads>(sin, nc, nullptr, tid, lane, false, 0, 0,
                                                       gdst, olen);
  } else {
    e = decode_tile<16, 1, false, P, false, kCpThreads>(sin, nc, S.ostage + mis, tid, lane, false,
                                                        0, 0);
    ptx::named_bar_sync(1, kCpThreads);
    cta_copy_out_congruent(gdst, S.ostage + mis, olen);
  }
  if (lane == 0 && e != 0xFFFFFFFFu) {
    const unsigned long long key = ~(static_cast<unsigned long long>(Bc) + e);
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

__global__ void __launch_bounds__(kOpThreads, 1)
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
    op_scan<true>(R, G, cnt, J, lane);
  } else {
    for (int64_t j = 0; j < J + kOpLag; ++j) {
      const int64_t i = j - kOpLag;
      const int s = static_cast<int>(j % kOpStages);
      const int si = static_cast<int>((i + kOpStages) % kOpStages);
      const int64_t t = b + j * Gs, ti = b + i * Gs;
      if (j < J) {  // A
        ptx::mbar_wait_spin(&R.full[s], static_cast<uint32_t>((j / kOpStages) & 1));
        op_count(R.win[s], G.lo(t), G.hi(t), R.nib[s], R.wcnt[s]);
      }
      int64_t P = 0;
      int n = 0, h = 0;
      if (i >= 0) {  // B: the carry chars, then the tile's kept chars at offset h
        const int p = static_cast<int>(i % kOpPre);
        ptx::mbar_wait_spin(&R.pfull[p], static_cast<uint32_t>((i / kOpPre) & 1));
        P = R.pre[p];
        h = static_cast<int>(P & 15);
        if (tid < h) S.stream[i & 1][tid] = R.carry[p][tid];
        n = op_place(R.win[si], R.nib[si], R.wcnt[si], S.stream[i & 1], h, R.ktab);
      }
      ptx::named_bar_sync(1, kCpThreads);  // C
      if (tid == 0) {                       // D
        if (j < J) {
          int c = 0;
#pragma unroll
          for (int w = 0; w < kCpWarps; ++w) c += R.wcnt[s][w];
          st_volatile_u32(cnt + t, static_cast<uint32_t>(c) + 1u);
        }
        if (i >= 0) {
          ptx::mbar_arrive(&R.empty[si]);
          ptx::mbar_arrive(&R.pempty[i % kOpPre]);
          if (ti == G.ntiles - 1) hdr->M = P + n;
        }
      }
      // E: the complete 16-char blocks ending in this tile (block-aligned at
      // compact position P - h); the rest is the next tile's carry
      if (i >= 0) {
        const int nc = (h + n) & ~15;
        if (nc > 0) op_decode_blocks(S, S.stream[i & 1], nc, P - h, out, hdr);
      }
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
