// b64_ws.cuh -- fused whitespace-tolerant decode (
// reading R-ws-decode in DESIGN.md §3): the Appendix B filter
// followed by Algorithm 2 (with the f1/f2 flags) on the kept
// characters, in one pass over the text after a counting pass:
//
//   cp_mask_kernel   keep masks per tile, kept characters per chunk (b64_compact.cuh)
//   decode_ws_kernel per chunk: TMA-stage each 16 KiB tile, compact it into a
//                    shared-memory stream (compact_tile), decode every 16-char
//                    block of the compacted stream the chunk owns straight
//                    from shared memory (decode_tile), write the bytes through
//                    a congruent staging buffer with 16-byte stores.  The
//                    last CTA out finishes the stream (final quad, NOPAD /
//                    STRICT rules, finish_stream_at) and maps the error
//                    offset from compacted to original coordinates.
//
// Compacted position P (the P-th kept character) decodes into output bytes
// 3P/4.., so a 16-char block j (compact [16j, 16j+16)) is owned by the chunk
// holding compact position 16j and decoded exactly once: inside a tile when
// the tile's compacted stream contains it, else (a block straddling the
// chunk's end) by the chunk's boundary step, which gathers the missing
// characters from the following chunks.  Traffic: the text is read twice
// (count + decode) and the bytes written once -- versus despace + decode,
// which also writes and re-reads the compacted text.
#pragma once
#include <cstdint>

#include "b64_codec.cuh"
#include "b64_compact.cuh"
#include "b64_ptx.cuh"

#ifndef B64_WS_DIRECT  // general path: decode runs store from registers (4-byte aligned output)
#define B64_WS_DIRECT 1
#endif

namespace b64 {

// Per-call scratch (device, caller workspace): errkey / done are reset by the
// count kernel of the same call (cp_count_kernel's `reset`).
struct WsHdr {
  unsigned long long errkey;  // min error offset in compacted coordinates, ~0 = none
  unsigned int done;          // CTAs finished
  unsigned int pad;
  int64_t tail_base;          // compact position of tail[0]
  uint8_t tail[8];            // the final quad of the compacted stream
};
constexpr size_t kWsHdrBytes = 64;
constexpr size_t kWlStateOffset = 48;  // WlState (b64_wslines.cuh) lives in the header's tail
static_assert(sizeof(WsHdr) <= kWlStateOffset, "WsHdr");

struct alignas(128) WsSmem {
  CpSmem cp;
  alignas(16) uint8_t stream[2][kCpTile + 64];  // compacted characters; [0] = compact position Bc (16-aligned)
  alignas(16) uint8_t ostage[kCpTile / 4 * 3 + 64];
  alignas(16) uint8_t blk[64];                 // boundary block characters
  alignas(16) uint8_t bout[64];                 // boundary block output
  int64_t red[66];
  int64_t sel[4];
  int32_t flag;
};

// Decode `n` (multiple of 4) compacted characters at the 16-byte aligned smem
// stream position `sin` (compact position P0, a multiple of 4) into out +
// 3*P0/4 via the congruent staging buffer; returns the minimum error offset
// relative to sin (0xFFFFFFFF if none).  CTA-wide, contains __syncthreads.
__device__ __forceinline__ uint32_t ws_decode_run(WsSmem &S, const uint8_t *sin, int n,
                                                  uint8_t *gdst, bool fin, uint32_t ch2,
                                                  uint32_t ch1, int olen) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int mis = static_cast<int>(reinterpret_cast<uintptr_t>(gdst) & 15);
  constexpr int P = (kCpTile + 16) / (kCpThreads * 16) + 1;  // passes of 512 x 16 chars
  uint32_t e;
#if B64_DEC_STG32 && B64_WS_DIRECT
  if ((mis & 3) == 0)  // each thread's 12 bytes straight to HBM: no staging, no barrier
    return decode_tile<16, 4, false, P, true, kCpThreads>(sin, n, nullptr, tid, lane, fin, ch2,
                                                          ch1, gdst, olen);
#endif
  if ((mis & 3) == 0)
    e = decode_tile<16, 4, false, P, false, kCpThreads>(sin, n, S.ostage + mis, tid, lane, fin,
                                                        ch2, ch1);
  else
    e = decode_tile<16, 1, false, P, false, kCpThreads>(sin, n, S.ostage + mis, tid, lane, fin,
                                                        ch2, ch1);
  __syncthreads();
  cta_copy_out_congruent(gdst, S.ostage + mis, olen);
  return e;
}

// Map compacted position e to its offset in the original text (CTA-wide; the
// error path only).  counts: per-chunk kept counts, tcnt: per-tile.
__device__ int64_t ws_map_offset(WsSmem &S, const CpGeom &G, const int64_t *counts, int64_t nchunks,
                                 const int32_t *tcnt, int64_t e) {
  const int tid = threadIdx.x;
  // 1. chunk holding e
  {
    const int64_t per = (nchunks + kCpThreads - 1) / kCpThreads;
    const int64_t c0 = tid * per, c1 = c0 + per < nchunks ? c0 + per : nchunks;
    int64_t sum = 0;
    for (int64_t c = c0; c < c1; ++c) sum += counts[c];
    int64_t pre, pb, tot, tb;
    block_exclusive_scan2(sum, 0, pre, pb, tot, tb, S.red);
    if (e >= pre && e < pre + sum) {
      int64_t acc = pre;
      for (int64_t c = c0; c < c1; ++c) {
        if (e < acc + counts[c]) {
          S.sel[0] = c;
          S.sel[1] = e - acc;
          break;
        }
        acc += counts[c];
      }
    }
    __syncthreads();
  }
  // 2. tile of that chunk
  {
    const int64_t c = S.sel[0], r = S.sel[1];
    const int64_t t0 = c * G.tpc, t1 = t0 + G.tpc < G.ntiles ? t0 + G.tpc : G.ntiles;
    const int64_t per = (t1 - t0 + kCpThreads - 1) / kCpThreads;
    const int64_t a = t0 + tid * per, b = a + per < t1 ? a + per : t1;
    int64_t sum = 0;
    for (int64_t t = a; t < b; ++t) sum += tcnt[t];
    int64_t pre, pb, tot, tb;
    block_exclusive_scan2(sum, 0, pre, pb, tot, tb, S.red);
    if (r >= pre && r < pre + sum) {
      int64_t acc = pre;
      for (int64_t t = a; t < b; ++t) {
        if (r < acc + tcnt[t]) {
          S.sel[2] = t;
          S.sel[3] = r - acc;
          break;
        }
        acc += tcnt[t];
      }
    }
    __syncthreads();
  }
  // 3. byte of that tile: 32 window bytes per thread
  const int64_t t = S.sel[2], r = S.sel[3];
  const int lo = G.lo(t), hi = G.hi(t);
  const uint8_t *w = reinterpret_cast<const uint8_t *>(G.a0 + static_cast<uintptr_t>(t) * kCpTile);
  const int x0 = tid * 32;
  int cnt = 0;
  for (int x = x0; x < x0 + 32; ++x)
    if (x >= lo && x < hi && !is_space_byte(w[x])) ++cnt;
  int64_t pre, pb, tot, tb;
  block_exclusive_scan2(cnt, 0, pre, pb, tot, tb, S.red);
  if (r >= pre && r < pre + cnt) {
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

__global__ void __launch_bounds__(kCpThreads, kCpCtasPerSm)
    decode_ws_kernel(const uint8_t *__restrict__ in, int64_t m, uint8_t *__restrict__ out,
                     const int64_t *__restrict__ counts, const uint32_t *__restrict__ masks,
                     int32_t *__restrict__ tcnt, int64_t tpc,
                     WsHdr *hdr, b64_result *res, int flags, const int32_t *skip = nullptr) {
  if (skip != nullptr && *skip == 1) return;  // the line-structured fast path already decoded
  extern __shared__ __align__(128) uint8_t smem_raw[];
  WsSmem &S = *reinterpret_cast<WsSmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  CpGeom G;
  G.init(in, m, tpc);
  if (tid < 256) g_dec_tab[tid] = kInvalid;
  init_ktab(S.cp.ktab);
  if (tid == 0) {
    for (int s = 0; s < kCpStages; ++s) ptx::mbar_init(&S.cp.full[s], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (tid < 64) g_dec_tab[ascii_of(tid, flags)] = static_cast<uint8_t>(tid);
  const int64_t b = blockIdx.x, nch = gridDim.x;
  const int64_t t0 = b * tpc, t1 = t0 + tpc < G.ntiles ? t0 + tpc : G.ntiles;
  int64_t Pb, M;  // compact start of this chunk, compact length of the stream
  chunk_prefix(counts, nch, b, Pb, M, S.red);
  const int64_t Pe = Pb + counts[b];
  const int64_t q4 = 4 * (M / 4);
  const bool pads_ok = (M % 4) == 0;
  const uint64_t pol = ptx::policy_evict_first();
  if (tid == 0)
    for (int s = 0; s < kCpStages - 1 && t0 + s < t1; ++s) cp_load(S.cp, G, masks, t0 + s, s, pol);

  const int64_t own0 = (Pb + 15) & ~static_cast<int64_t>(15);  // first block this chunk owns
  // Decode the full 16-char blocks [d0, d1) of a tile's compacted stream
  // (stream base Bc_ at compact position Bc_), reporting its first error.
  auto decode_blocks = [&](const uint8_t *stream, int64_t Bc_, int64_t Qn_) {
    const int64_t d0 = Bc_ > own0 ? Bc_ : own0;
    const int64_t d1 = Qn_ & ~static_cast<int64_t>(15);
    if (d1 > d0) {  // full blocks [d0, d1); warp-uniform
      const uint8_t *sin = stream + (d0 - Bc_);
      const int nc = static_cast<int>(d1 - d0);
      const bool fin = d1 == M;  // the stream ends on this block boundary (M % 16 == 0)
      uint32_t ch2 = 0, ch1 = 0;
      int pads = 0;
      if (fin) {
        ch2 = sin[nc - 2];
        ch1 = sin[nc - 1];
        pads = ch1 == '=' ? (ch2 == '=' ? 2 : 1) : 0;
        if (tid < 4) hdr->tail[tid] = sin[nc - 4 + tid];
        if (tid == 0) hdr->tail_base = M - 4;
      }
      const uint32_t e = ws_decode_run(S, sin, nc, out + 3 * (d0 / 4), fin, ch2, ch1,
                                       3 * (nc / 4) - pads);
      if (lane == 0 && e != 0xFFFFFFFFu) {
        const unsigned long long pos = static_cast<unsigned long long>(d0) + e;
        if (pos < *reinterpret_cast<volatile unsigned long long *>(&hdr->errkey))
          atomicMin(&hdr->errkey, pos);
      }
    }
  };
  // Tile t is decoded during iteration t+1, after tile t+1's compaction
  // barrier (which orders every thread's placement stores of tile t): one
  // CTA barrier per tile.  The carry of an incomplete block into tile t+1's
  // stream ([0, dst) of it: disjoint from tile t+1's own bytes) is copied
  // after that barrier too.
  int64_t Q = Pb, Bprev = Pb & ~static_cast<int64_t>(15);
  int64_t pBc = 0, pQn = 0;  // the pending (compacted, not yet decoded) tile
  for (int64_t t = t0; t < t1; ++t) {
    const int it = static_cast<int>(t - t0);
    const int s = it % kCpStages, sb = it & 1;
    const int64_t Bc = Q & ~static_cast<int64_t>(15);
    const int dst = static_cast<int>(Q & 15);
    ptx::mbar_wait_spin(&S.cp.full[s], static_cast<uint32_t>((it / kCpStages) & 1));
    const int n = compact_tile<true>(S.cp.win[s], S.cp.msk[s], S.stream[sb], dst, S.cp.wcnt[sb], S.cp.ktab);
    ptx::fence_proxy_async_smem();
    // the previous tile's window and stream are complete / free now
    if (tid == 0 && t + kCpStages - 1 < t1)
      cp_load(S.cp, G, masks, t + kCpStages - 1, (it + kCpStages - 1) % kCpStages, pol);
    if (it > 0 && tid < dst) S.stream[sb][tid] = S.stream[sb ^ 1][Bc - Bprev + tid];
    if (tid == 0) tcnt[t] = n;
    if (it > 0) decode_blocks(S.stream[sb ^ 1], pBc, pQn);
    pBc = Bc;
    pQn = Q + n;
    Q = pQn;
    Bprev = Bc;
  }
  if (t1 > t0) {
    __syncthreads();  // the last tile's placement stores and carry
    decode_blocks(S.stream[(t1 - 1 - t0) & 1], pBc, pQn);
  }

  // Boundary block: [sblk, sblk + 16) straddles the chunk's end (or is the
  // stream's final partial block); owned iff sblk >= Pb.
  const int64_t sblk = Pe & ~static_cast<int64_t>(15);
  if (t1 > t0 && (Pe & 15) != 0 && sblk >= Pb) {
    const int64_t bend = sblk + 16 < M ? sblk + 16 : M;  // block end (compact)
    const int have = static_cast<int>(Pe - sblk);
    const int need = static_cast<int>(bend - Pe);
    const int sbl = static_cast<int>((t1 - 1 - t0) & 1);
    const int64_t Bl = Bprev;  // stream base of the last tile
    if (warp == 0) {
      if (lane < have) S.blk[lane] = S.stream[sbl][sblk - Bl + lane];
      // gather `need` kept characters after the chunk, skipping empty chunks
      int got = 0;
      int64_t c = b + 1;
      int64_t x = G.off(t1, 0);  // original offset of the chunk's end
      while (got < need && c < nch) {
        const int64_t cend_t = (c + 1) * tpc < G.ntiles ? (c + 1) * tpc : G.ntiles;
        const int64_t cend = G.off(cend_t, 0) < m ? G.off(cend_t, 0) : m;
        if (counts[c] == 0) {
          x = cend;
          ++c;
          continue;
        }
        while (got < need && x < cend) {
          const int64_t i = x + lane;
          const bool keep = i < cend && !is_space_byte(in[i]);
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          const int rank = __popc(bal & ((1u << lane) - 1u));
          if (keep && got + rank < need) S.blk[have + got + rank] = in[i];
          got += __popc(bal);
          x += 32;
        }
        x = cend;
        ++c;
      }
      __syncwarp();
      // decode the block (one lane), final-quad rules when it ends the stream
      const bool ends = bend == M;
      const int L = static_cast<int>(ends ? q4 - sblk : 16);
      const bool fin = ends && pads_ok;
      uint32_t ch2 = 0, ch1 = 0;
      int pads = 0;
      if (fin) {
        ch2 = S.blk[L - 2];
        ch1 = S.blk[L - 1];
        pads = ch1 == '=' ? (ch2 == '=' ? 2 : 1) : 0;
      }
      if (ends) {
        const int64_t tb = 4 * ((M - 1) / 4);
        if (lane < M - tb) hdr->tail[lane] = S.blk[tb - sblk + lane];
        if (lane == 0) hdr->tail_base = tb;
      }
      uint32_t e = 0xFFFFFFFFu;
      if (L > 0)
        e = decode_tile<16, 16, false, 1, false, 32>(S.blk, L, S.bout, lane, lane, fin, ch2, ch1);
      __syncwarp();
      const int olen = 3 * (L / 4) - pads;
      if (lane < olen) out[3 * (sblk / 4) + lane] = S.bout[lane];
      if (lane == 0 && e != 0xFFFFFFFFu) atomicMin(&hdr->errkey, static_cast<unsigned long long>(sblk) + e);
    }
  }

  // Last CTA out: finish the stream and map the error offset.
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    S.flag = atomicAdd(&hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!S.flag) return;
  __threadfence();
  if (tid == 0) {
    const unsigned long long e = atomicOr(&hdr->errkey, 0ull);
    const int64_t tb = hdr->tail_base;
    const uint8_t *tl = hdr->tail;
    const StreamResult R = finish_stream_at(
        [tl, tb](int64_t i) -> uint32_t { return tl[i - tb]; }, M, out,
        e == ~0ull ? -1 : static_cast<int64_t>(e), true, flags);
    S.sel[0] = R.out_len;
    S.sel[1] = R.err_pos;
    S.sel[2] = R.status;
    S.sel[3] = R.pad_count;
  }
  __syncthreads();
  const int64_t olen = S.sel[0], ep = S.sel[1];
  const int32_t st = static_cast<int32_t>(S.sel[2]), pc = static_cast<int32_t>(S.sel[3]);
  __syncthreads();
  const int64_t oep = ep >= 0 ? ws_map_offset(S, G, counts, nch, tcnt, ep) : -1;
  if (tid == 0) {
    res->out_len = olen;
    res->err_pos = oep;
    res->status = st;
    res->pad_count = pc;
  }
}

}  // namespace b64
