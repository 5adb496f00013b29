// b64_despace2.cuh -- single-read whitespace removal (SURVEY.md §8(f) row
// f3, Appendix B) for text the line fast path rejects: every
// input byte is read from HBM once, every kept byte written once.
//
// The one-pass machinery of b64_onepass.cuh (persistent co-resident grid,
// tile t on CTA t mod G, a producer warp streaming 16 KiB windows into a
// ring, a scan warp turning the published per-tile counts into exclusive
// prefixes kOpLag tiles later) with the two-pass kernels' placement:
//   A  classify tile j from shared memory into the interleaved keep nibbles
//      of cp_mask_kernel (lane l, words 32 i + l) and publish its count;
//   B  place tile i = j - kOpLag once its prefix P is known: compact_tile
//      (conflict-free predicated byte stores) into a staging stream
//      congruent to out + P mod 16, which leaves as one bulk (TMA) store
//      after the next placement's barrier (double-buffered streams).
#pragma once
#include <cstdint>

#include "b64_compact.cuh"
#include "b64_onepass.cuh"
#include "b64_ptx.cuh"

namespace b64 {

struct alignas(128) Ds2Smem {
  OpRing r;
  alignas(16) uint8_t stream[2][kCpTile + 32];
  int32_t wcnt[2][kCpWarps];
  uint32_t ktab[16];
};

// A: keep nibbles of a landed window (bytes [lo, hi) exist) -> msk[tid]; the
// tile's count is published by the last warp to finish (count + 1; 0 = not
// yet).
__device__ __forceinline__ void ds2_classify(const uint8_t *win, int lo, int hi, uint32_t *msk,
                                             int32_t *tcnt, int32_t *tarr, uint32_t *cnt_t) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wbase = warp * kCpWarpWords + lane;
  const uint32_t *wv = reinterpret_cast<const uint32_t *>(win);
  uint32_t w[kCpPerLane];
#pragma unroll
  for (int i = 0; i < kCpPerLane; ++i) w[i] = wv[wbase + 32 * i];
  const uint32_t nib = tile_nib(w, lo, hi, wbase, lo != 0 || hi != kCpTile);
  msk[tid] = nib;
  const int c = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(__popc(nib))));
  if (lane == 0) {
    atomicAdd(tcnt, c);
    __threadfence_block();
    if (atomicAdd(tarr, 1) == kCpWarps - 1) {
      __threadfence_block();
      st_volatile_u32(cnt_t, static_cast<uint32_t>(atomicAdd(tcnt, 0)) + 1u);
    }
  }
}

__global__ void __launch_bounds__(kOpThreads, kOpCtas)
    despace2_kernel(const uint8_t *__restrict__ in, int64_t m, uint8_t *__restrict__ out,
                    uint32_t *cnt, int64_t *out_len, const int32_t *skip) {
  if (skip != nullptr && *skip == 1) return;  // the line-structured fast path already wrote it
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Ds2Smem &S = *reinterpret_cast<Ds2Smem *>(smem_raw);
  OpRing &R = S.r;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  CpGeom G;
  G.init(in, m, 0);
  op_init(R);
  init_ktab(S.ktab);
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
  const uint64_t pol = ptx::policy_evict_first();
  int64_t pP = 0;
  int pdst = 0, pn = 0, np = 0;  // the placed tile whose copy-out is pending
  for (int64_t j = 0; j < J + kOpLag; ++j) {
    const int64_t i = j - kOpLag;
    const int64_t t = b + j * Gs, ti = b + i * Gs;
    if (j < J) {  // A
      const int s = static_cast<int>(j % kOpSlots);
      ptx::mbar_wait_spin(&R.full[s], static_cast<uint32_t>((j / kOpSlots) & 1));
      __syncwarp();
      ds2_classify(R.win[s], G.lo(t), G.hi(t), R.msk[s], &R.tcnt[s], &R.tarr[s], cnt + t);
    }
    const int si = static_cast<int>((i + kOpSlots) % kOpSlots);
    if (i >= 0) {  // B
      const int p = static_cast<int>(i % kOpPre);
      ptx::mbar_wait_spin(&R.pfull[p], static_cast<uint32_t>((i / kOpPre) & 1));
      __syncwarp();
      const int64_t P = R.pre[p];
      const int sb = np & 1;
      const int dst = static_cast<int>((reinterpret_cast<uintptr_t>(out) + static_cast<uintptr_t>(P)) & 15);
      // (its barrier also orders the previous placement's stores before
      // that tile's copy-out below; thread 0 first waits until the bulk
      // store that read stream[sb] two placements ago is done reading)
      const int n = compact_tile<false, true, true>(R.win[si], R.msk[si], S.stream[sb], dst, S.wcnt[sb],
                                                    S.ktab);
      ptx::fence_proxy_async_smem();
      if (np > 0) cta_copy_out_bulk(out + pP, S.stream[sb ^ 1] + pdst, pn, pol);
      if (tid == 0 && ti == G.ntiles - 1) *out_len = P + n;
      pP = P;
      pdst = dst;
      pn = n;
      ++np;
    }
    ptx::named_bar_sync(1, kCpThreads);  // C: slot si (window, keep masks) and prefix slot free
    if (tid == 0 && i >= 0) {
      R.tcnt[si] = 0;
      R.tarr[si] = 0;
      ptx::mbar_arrive(&R.empty[si]);
      ptx::mbar_arrive(&R.pempty[i % kOpPre]);
    }
  }
  if (np > 0) {
    cta_copy_out_bulk(out + pP, S.stream[(np - 1) & 1] + pdst, pn, pol);
    if (tid == 0) ptx::bulk_wait<0>();
  }
}

}  // namespace b64
