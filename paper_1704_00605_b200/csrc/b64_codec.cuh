// b64_codec.cuh -- per-thread / per-tile base64 arithmetic for the sm_100a
// kernels (device code only).  Paper rows: SURVEY.md §8 a2-a3 (encode regroup
// + alphabet map), a8-a10 (decode classify/translate, first-error reduction,
// pack).  No code is shared with oracle/.
#pragma once
#include <cstdint>

#include "b64_knobs.cuh"  // measurement-only knobs (never set in the product build)

namespace b64 {

// ------------------------------------------------------------ geometry ---
// Tunables (compile-time; the defaults are the measured best, see
// DESIGN.md §6 and tools/sweep.py).
#ifndef B64_WARPS_C
#define B64_WARPS_C 16
#endif
#ifndef B64_STAGES_IN
#define B64_STAGES_IN 3
#endif
#ifndef B64_STAGES_OUT
#define B64_STAGES_OUT 2
#endif
#ifndef B64_SINGLE_PASSES
#define B64_SINGLE_PASSES 4
#endif
#ifndef B64_BATCH_PASSES  // passes of one warp per batched work unit
#define B64_BATCH_PASSES 6
#endif
#ifndef B64_BATCH_SLOTS   // per-warp input ring depth (batched)
#define B64_BATCH_SLOTS 2
#endif
#ifndef B64_BATCH_CTAS    // batched: CTAs per SM of the cooperative grid
#define B64_BATCH_CTAS 1
#endif
#ifndef B64_BATCH_WARPS   // warps per CTA (batched)
#define B64_BATCH_WARPS 20
#endif
#ifndef B64_CTAS_PER_SM
#define B64_CTAS_PER_SM 1
#endif
#ifndef B64_DEC_STG32  // decode DIRECT tiles: three 4-byte stores from registers (no smem slice)
#define B64_DEC_STG32 1
#endif
#ifndef B64_STORE_EVICT_FIRST
#define B64_STORE_EVICT_FIRST 0
#endif
constexpr int kWarpsC = B64_WARPS_C;        // compute warps per CTA
constexpr int kNT = kWarpsC * 32;           // compute threads per CTA
constexpr int kThreads = kNT + 32;          // + one producer (TMA) warp
constexpr int kStagesIn = B64_STAGES_IN;    // input ring depth
constexpr int kStagesOut = B64_STAGES_OUT;  // output staging depth
constexpr int kCtasPerSm = B64_CTAS_PER_SM;
static_assert(kStagesOut >= 2, "output staging needs >= 2 slots");

// Encode: each compute thread turns 12 bytes (4 groups) into 16 chars per
// pass; decode: 16 chars (4 quads) into 12 bytes per pass.  A tile is P
// passes of the kNT compute threads (512 at the default 16 warps: with
// P = 4, encode tiles are 24 KiB in / 32 KiB out, decode 32 KiB / 24 KiB).
template <int P>
struct EncG {
  static constexpr int kPasses = P;
  static constexpr int kIn = kNT * 12 * P;   // input bytes per tile
  static constexpr int kOut = kNT * 16 * P;  // output chars per tile
};
template <int P>
struct DecG {
  static constexpr int kPasses = P;
  static constexpr int kIn = kNT * 16 * P;   // input chars per tile
  static constexpr int kOut = kNT * 12 * P;  // output bytes per tile
};
constexpr int kSinglePasses = B64_SINGLE_PASSES;  // single-buffer tile = this many passes
constexpr int kBatchPasses = B64_BATCH_PASSES;    // batched: one warp unit = this many passes

constexpr int round_up_c(int x, int a) { return (x + a - 1) / a * a; }

constexpr uint8_t kInvalid = 0xFF;  // decode-table marker for bytes outside the alphabet
constexpr int kFlagFinal = 1;       // tile holds the final quad of a padded-able stream

// Tile descriptor: produced arithmetically (single buffer) or by the batch
// planner, handed from the producer warp to the compute warps through smem.
struct TileDesc {
  int64_t src;     // input byte offset of the tile (relative to d_in)
  int64_t dst;     // output byte offset of the tile (relative to d_out)
  int64_t rel;     // input offset of the tile within its message
  int32_t len;     // input bytes of the tile (> 0; decode: multiple of 4)
  int32_t msg;     // message index (batched), 0 otherwise
  int32_t flags;   // kFlagFinal
  int32_t ntiles;  // tiles of the message (batched)
};
static_assert(sizeof(TileDesc) == 40, "TileDesc layout");

// ------------------------------------------------------- alphabet (GPU) ---
// Variant flags (include/b64gpu.h B64_FLAG_*).
constexpr int kFlagUrl = 1;     // base64url alphabet
constexpr int kFlagNoPad = 2;   // no '=' on encode, optional padding on decode
constexpr int kFlagStrict = 4;  // Appendix A canonical trailing bits

// Table II: 6-bit value -> ASCII by range offsets; base64url
// moves 62 / 63 to '-' / '_'.
__device__ __forceinline__ uint32_t ascii_of(uint32_t v, int flags = 0) {
  if ((flags & kFlagUrl) && v >= 62) return v == 62 ? '-' : '_';
  int off = v < 26 ? 65 : v < 52 ? 71 : v < 62 ? -4 : v == 62 ? -19 : -16;
  return static_cast<uint32_t>(static_cast<int>(v) + off);
}

// The two lookup tables live in static shared memory and are indexed by name
// so that each lookup compiles to one LDS.U8 [idx + UR] (uniform base, no
// per-lookup address add).
__shared__ alignas(256) uint8_t g_dec_tab[256];  // A: byte -> 6-bit value | kInvalid
__shared__ alignas(64) uint8_t g_enc_tab[64];    // B: 6-bit value -> ASCII (Table I)

// Decode lookup of byte `sel` (0..3) of word w: g_dec_tab is 256-byte aligned,
// so the shared address is the table base with its low byte replaced by the
// character -- one PRMT/LOP3 forms the address, one LDS.U8 reads the entry.
__device__ __forceinline__ uint32_t lds_u8(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

// ---------------------------------------------------- smem word access ---
// Load N little-endian words of the stream starting at smem byte address p.
// ALIGN: guaranteed alignment of p (16, 4 or 1); ALIGN 1 realigns with
// funnel shifts (the byte shift is warp-uniform).
template <int ALIGN, int N>
__device__ __forceinline__ void load_words(const uint8_t *p, uint32_t (&w)[N]) {
  if constexpr (ALIGN == 16 && N == 4) {
    const uint4 v = *reinterpret_cast<const uint4 *>(p);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else if constexpr (ALIGN >= 4) {
    const uint32_t *q = reinterpret_cast<const uint32_t *>(p);
#pragma unroll
    for (int k = 0; k < N; ++k) w[k] = q[k];
  } else {
    const uint32_t r = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p) & 3);
    const uint32_t *q = reinterpret_cast<const uint32_t *>(p - r);
    uint32_t x[N + 1];
#pragma unroll
    for (int k = 0; k <= N; ++k) x[k] = q[k];
#pragma unroll
    for (int k = 0; k < N; ++k) w[k] = __funnelshift_r(x[k], x[k + 1], 8 * r);
  }
}

// Store N words D (stream bytes [X, X+4N)) to smem byte address p = base+X.
// Lanes of a warp hold consecutive, adjacent 4N-byte runs; `active` lanes
// form a prefix of the warp.  ALIGN 1: each lane writes the aligned words it
// owns completely plus the word it shares with the next lane (built from the
// next lane's first word via a shuffle); the words shared with the previous /
// next warp are written byte by byte.  Must be called by all 32 lanes.
template <int ALIGN, int N>
__device__ __forceinline__ void store_words(uint8_t *p, const uint32_t (&D)[N], bool active,
                                            int lane) {
  if constexpr (ALIGN == 16 && N == 4) {
    if (active) *reinterpret_cast<uint4 *>(p) = make_uint4(D[0], D[1], D[2], D[3]);
  } else if constexpr (ALIGN >= 4) {
    if (active) {
      uint32_t *q = reinterpret_cast<uint32_t *>(p);
#pragma unroll
      for (int k = 0; k < N; ++k) q[k] = D[k];
    }
  } else {
    const uint32_t r = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p) & 3);
    const uint32_t nxt = __shfl_down_sync(0xffffffffu, D[0], 1);
    const bool nxt_active = __shfl_down_sync(0xffffffffu, active ? 1u : 0u, 1) != 0 && lane < 31;
    if (!active) return;
    if (r == 0) {
      uint32_t *q = reinterpret_cast<uint32_t *>(p);
#pragma unroll
      for (int k = 0; k < N; ++k) q[k] = D[k];
      return;
    }
    const uint32_t s = 8 * r;
    uint32_t *q = reinterpret_cast<uint32_t *>(p - r);
#pragma unroll
    for (int k = 1; k < N; ++k) q[k] = __funnelshift_l(D[k - 1], D[k], s);
    if (nxt_active) {
      q[N] = __funnelshift_l(D[N - 1], nxt, s);
    } else {
      uint8_t *b = reinterpret_cast<uint8_t *>(q + N);
      for (uint32_t i = 0; i < r; ++i) b[i] = static_cast<uint8_t>(D[N - 1] >> (8 * (4 - r + i)));
    }
    if (lane == 0) {
      for (uint32_t i = 0; i < 4 - r; ++i) p[i] = static_cast<uint8_t>(D[0] >> (8 * i));
    }
  }
}

// 16-byte global store (STG.E.128).
__device__ __forceinline__ void st_global_v4(uint8_t *p, const uint32_t (&c)[4]) {
  *reinterpret_cast<uint4 *>(p) = make_uint4(c[0], c[1], c[2], c[3]);
}
__device__ __forceinline__ void st_global_v4(uint8_t *p, const uint4 &v) {
  *reinterpret_cast<uint4 *>(p) = v;
}

// ------------------------------------------------------------- encode ---
// One group (Alg 1 main loop body): x holds s_i<<16 | s_{i+1}<<8 |
// s_{i+2} in its low 24 bits; TOPZERO says whether bits 24..31 are zero.
// The four 6-bit fields are s_i/4, (s_i*16 mod 64) + s_{i+1}/16,
// (s_{i+1}*4 mod 64) + s_{i+2}/64 and s_{i+2} mod 64, i.e. bits 23..18,
// 17..12, 11..6, 5..0 of x; each is mapped through the 64-entry smem table B
// and the four characters are packed little-endian (first char = byte 0).
// g_enc_tab is 64-byte aligned, so each lookup address is the 6-bit field
// OR-ed into the table base (SHF + LOP3, or one LOP3 / LEA.HI).
template <bool TOPZERO>
__device__ __forceinline__ uint32_t enc_group(uint32_t x, uint32_t tb) {
#if B64_ENC_ARITH
  // Table I (with the f1 alphabet's 62 / 63) as per-byte SWAR arithmetic on
  // the four packed fields v (< 64): v + 65, + 6 from 26, - 75 from 52,
  // - d62 at 62, + d63 at 63 (the paper's range-offset mapping); each
  // partial sum stays in 0..255 per byte, so no carry or borrow crosses
  // bytes.  d62 / d63 come from the launch's table entries 62 / 63.
  const uint32_t v = ((x >> 18) & 0x3Fu) | ((x >> 4) & 0x3F00u) | ((x << 10) & 0x3F0000u) |
                     ((x << 24) & 0x3F000000u);
  const uint32_t c62 = lds_u8(tb | 62u), c63 = lds_u8(tb | 63u);
  const uint32_t d62 = 58u - c62, d63 = c63 - 59u + d62;
  uint32_t r = v + 0x41414141u;
  const uint32_t g26 = ((v + 0x66666666u) >> 7) & 0x01010101u;
  const uint32_t g52 = ((v + 0x4C4C4C4Cu) >> 7) & 0x01010101u;
  const uint32_t g62 = ((v + 0x42424242u) >> 7) & 0x01010101u;
  const uint32_t g63 = (r >> 7) & 0x01010101u;
  r += g26 * 6u;
  r -= g52 * 75u;
  r -= g62 * d62;
  r += g63 * d63;
  return r;
#endif
  const uint32_t a0 = TOPZERO ? ((x >> 18) | tb) : (((x >> 18) & 63u) | tb);
  const uint32_t a1 = ((x >> 12) & 63u) | tb;
  const uint32_t a2 = ((x >> 6) & 63u) | tb;
  const uint32_t a3 = (x & 63u) | tb;
  const uint32_t c0 = lds_u8(a0), c1 = lds_u8(a1), c2 = lds_u8(a2), c3 = lds_u8(a3);
  return __byte_perm(__byte_perm(c0, c1, 0x3340), __byte_perm(c2, c3, 0x3340), 0x5410);
}

// 12 input bytes (w0..w2, little-endian) -> 16 output chars (c0..c3).
// __byte_perm reorders each 3-byte group big-endian (the GPU counterpart of
// the paper's vpshufb step in enc_reshuffle).
__device__ __forceinline__ void encode12(const uint32_t (&w)[3], uint32_t (&c)[4]) {
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(g_enc_tab));
  c[0] = enc_group<true>(__byte_perm(w[0], 0u, 0x4012), tb);    // b0 b1 b2
  c[1] = enc_group<false>(__byte_perm(w[0], w[1], 0x3345), tb);  // b3 b4 b5
  c[2] = enc_group<false>(__byte_perm(w[1], w[2], 0x2234), tb);  // b6 b7 b8
  c[3] = enc_group<true>(__byte_perm(w[2], 0u, 0x4123), tb);    // b9 b10 b11
}

// Replace byte i (0..15) of the 4-word vector with value v.
__device__ __forceinline__ void set_byte16(uint32_t (&c)[4], int i, uint32_t v) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (4 * k + b == i) c[k] = (c[k] & ~(0xFFu << (8 * b))) | (v << (8 * b));
    }
  }
}

// Encode one tile: L input bytes at sin -> 4*ceil(L/3) chars at sout.
// Alg 1's tail is handled by the one thread whose 12-byte run
// crosses L: missing bytes are zero (so the emitted fields equal
// (s_i*16) mod 64 and (s_{i+1}*4) mod 64) and '=' pads are substituted.
// FULL: the tile has exactly EncG<P>::kIn bytes (no tail / inactive-lane checks).
// DIRECT (FULL tiles with a 16-byte aligned destination): each thread's 16
// chars go straight from registers to HBM with one coalesced 16-byte store
// (512 contiguous bytes per warp instruction), no smem staging, no CTA sync.
template <int IA, int OA, bool FULL, int P, bool DIRECT = false, int NT = kNT>
__device__ __forceinline__ void encode_tile(const uint8_t *sin, int L, uint8_t *sout, int tid,
                                            int lane, uint8_t *gdst = nullptr, bool pad = true) {
#pragma unroll
  for (int pass = 0; pass < P; ++pass) {
    const int bo = pass * (NT * 12) + tid * 12;
    const int co = pass * (NT * 16) + tid * 16;
    const bool active = FULL || bo < L;
    if (!FULL && !__any_sync(0xffffffffu, active)) break;
    uint32_t w[3];
    load_words<(IA >= 4 ? 4 : 1), 3>(sin + bo, w);
    const int rem = L - bo;
    const bool partial = !FULL && active && rem < 12;
    if (partial) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int keep = rem - 4 * k;
        if (keep <= 0) w[k] = 0;
        else if (keep < 4) w[k] &= (1u << (8 * keep)) - 1u;
      }
    }
    uint32_t c[4];
    if (B64_SKELETON) {
      c[0] = w[0]; c[1] = w[1]; c[2] = w[2]; c[3] = w[0] ^ w[2];
    } else {
      encode12(w, c);
    }
    if (partial) {
      const int left = rem % 3;           // 1 -> "xx==", 2 -> "xxx="
      if (left != 0 && pad) {
        const int last = 4 * (rem / 3);   // first char of the partial group
        set_byte16(c, last + 3, '=');
        if (left == 1) set_byte16(c, last + 2, '=');
      }
    }
    if constexpr (DIRECT) {
      st_global_v4(gdst + co, c);
    } else {
      store_words<OA, 4>(sout + co, c, active, lane);
    }
  }
}

// ------------------------------------------------------------- decode ---
// Decode one tile: L chars (multiple of 4) at sin -> 3*L/4 bytes at sout.
// Table lookups classify and translate (A of Alg 2; validity rule of
// P:952-958); the four 6-bit values of a quad are packed as
// a<<18 | b<<12 | c<<6 | d (bit layout P:1013-1030) and three
// __byte_perm write the 12 output bytes of 4 quads.  Errors take the slow
// path only when some lane of the warp saw an invalid byte (__any_sync):
// per-char mask, final-quad '=' rules (reading R-pad), first bad offset,
// warp __reduce_min_sync.  Returns (lane 0 meaningful) the tile-relative
// minimum error offset, or 0xFFFFFFFF.
// FULL: the tile has exactly DecG<P>::kIn chars and is not a final tile.
// DIRECT (FULL tiles, 16-byte aligned destination): each thread stores its
// 12 bytes straight from registers with three 4-byte stores (B64_DEC_STG32,
// the default: no shared-memory traffic for the output, which matters once
// the power cap lowers the SM clock), or (B64_DEC_STG32=0) the warp stages
// its 384 output bytes in its own slice of smem (3 conflict-free STS per
// lane) and lanes 0..23 copy them with coalesced 16-byte stores.  Both are
// warp-local: no CTA-wide barrier, no bulk-store round trip.
// DIRECT with !FULL (B64_DEC_STG32; 4-byte aligned gdst): the tile's output
// is its first olim bytes (3 L / 4 minus the final quad's pads).
template <int IA, int OA, bool FULL, int P, bool DIRECT = false, int NT = kNT>
__device__ __forceinline__ uint32_t decode_tile(const uint8_t *sin, int L, uint8_t *sout,
                                                int tid, int lane,
                                                bool final_tile, uint32_t ch2, uint32_t ch1,
                                                uint8_t *gdst = nullptr, int olim = 0) {
  uint32_t errmin = 0xFFFFFFFFu;
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(g_dec_tab));
#pragma unroll
  for (int pass = 0; pass < P; ++pass) {
    const int co = pass * (NT * 16) + tid * 16;
    const int bo = pass * (NT * 12) + tid * 12;
    const bool active = FULL || co < L;
    if (!FULL && !__any_sync(0xffffffffu, active)) break;
    uint32_t w[4];
    load_words<IA, 4>(sin + co, w);
    const int rem = L - co;
    if (!FULL && (!active || rem < 16)) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (!active || 4 * k >= rem) w[k] = 0x41414141u;  // "AAAA": ignored filler
    }
    if (B64_SKELETON) {
      uint32_t o[3] = {w[0], w[1], w[2] ^ w[3]};
      store_words<(OA >= 4 ? 4 : 1), 3>(sout + bo, o, active, lane);
      if constexpr (DIRECT) {
        __syncwarp();
        const int wo = pass * (NT * 12) + (tid & ~31) * 12;
        if (lane < 24) {
          const uint4 q = *reinterpret_cast<const uint4 *>(sout + wo + 16 * lane);
          st_global_v4(gdst + wo + 16 * lane, q);
        }
      }
      continue;
    }
    uint32_t v[16];
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[4 * k + 0] = lds_u8((w[k] & 0xFFu) | tb);
      v[4 * k + 1] = lds_u8(__byte_perm(w[k], tb, 0x7651));
      v[4 * k + 2] = lds_u8(__byte_perm(w[k], tb, 0x7652));
      v[4 * k + 3] = lds_u8(__byte_perm(w[k], tb, 0x7653));
      acc |= v[4 * k + 0] | v[4 * k + 1];
      acc |= v[4 * k + 2] | v[4 * k + 3];
    }
    const uint32_t bad = acc & 0x80u;
    if (__any_sync(0xffffffffu, bad)) {
      uint32_t pos = 0xFFFFFFFFu;
      if (bad) {
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) mask |= ((v[j] >> 7) & 1u) << j;
        // Final quad of the stream (reading R-pad): '=' allowed at m-2 and
        // m-1, and '=' at m-2 forces '=' at m-1; '=' contributes value 0.
        if (!FULL && final_tile && co + 16 >= L && co < L) {
          const int j1 = L - 1 - co, j2 = L - 2 - co;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j == j2 && ch2 == '=') { mask &= ~(1u << j); v[j] = 0; }
            if (j == j1) {
              if (ch1 == '=') { mask &= ~(1u << j); v[j] = 0; }
              else if (ch2 == '=') mask |= 1u << j;
            }
          }
        }
        if (mask) pos = static_cast<uint32_t>(co) + __ffs(mask) - 1;
      }
      const uint32_t wmin = __reduce_min_sync(0xffffffffu, pos);
      errmin = min(errmin, wmin);
    }
    uint32_t V[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      V[k] = ((v[4 * k] * 64u + v[4 * k + 1]) * 64u + v[4 * k + 2]) * 64u + v[4 * k + 3];
    uint32_t o[3];
    o[0] = __byte_perm(V[0], V[1], 0x6012);
    o[1] = __byte_perm(V[1], V[2], 0x5601);
    o[2] = __byte_perm(V[2], V[3], 0x4560);
#if B64_DEC_STG32
    if constexpr (DIRECT) {  // three 4-byte stores straight from registers (lanes 12 B apart)
      if (FULL || (active && bo + 12 <= olim)) {
#if B64_DEC_STG64
        // 12 bytes as one 8-byte + one 4-byte store: even threads' runs are
        // 8-byte aligned ([8][4]), odd threads' are not ([4][8])
        const bool ev = ((reinterpret_cast<uintptr_t>(gdst + bo)) & 7) == 0;
        uint8_t *g8 = gdst + bo + (ev ? 0 : 4);
        uint8_t *g4 = gdst + bo + (ev ? 8 : 0);
        *reinterpret_cast<uint2 *>(g8) = ev ? make_uint2(o[0], o[1]) : make_uint2(o[1], o[2]);
        *reinterpret_cast<uint32_t *>(g4) = ev ? o[2] : o[0];
#else
        uint32_t *g = reinterpret_cast<uint32_t *>(gdst + bo);
        g[0] = o[0];
        g[1] = o[1];
        g[2] = o[2];
#endif
      } else if (active) {  // the run holding the stream's padded final quad: its olim - bo bytes
        for (int j = 0; j < olim - bo; ++j) {
          const uint32_t w = j < 4 ? o[0] : j < 8 ? o[1] : o[2];
          gdst[bo + j] = static_cast<uint8_t>(w >> (8 * (j & 3)));
        }
      }
      continue;
    }
#endif
    store_words<(OA >= 4 ? 4 : 1), 3>(sout + bo, o, active, lane);
    if constexpr (DIRECT) {
      __syncwarp();
      const int wo = pass * (NT * 12) + (tid & ~31) * 12;  // this warp's 384-byte slice
      if (lane < 24) {
        const uint4 v = *reinterpret_cast<const uint4 *>(sout + wo + 16 * lane);
        st_global_v4(gdst + wo + 16 * lane, v);
      }
    }
  }
  return errmin;
}

}  // namespace b64

namespace b64 {
// Encoded length of a tile / message of L bytes (Alg 1; NOPAD drops the '=').
__host__ __device__ __forceinline__ int64_t enc_len(int64_t L, int flags) {
  return (flags & kFlagNoPad) ? 4 * (L / 3) + (L % 3 ? L % 3 + 1 : 0) : 4 * ((L + 2) / 3);
}

// Final-quad / tail epilogue of one decoded stream (single buffer, shard or
// batched message), reading R-pad / R-length and the f1/f2 variants, run by
// one thread after every error of the stream's complete quads has been
// reduced into err (-1 = none).  c: the stream's characters (global), m its
// length, q4 = 4*floor(m/4); out: its output (the NOPAD tail bytes are
// written here).  Uses the decode table g_dec_tab in shared memory.
struct StreamResult {
  int64_t out_len;
  int64_t err_pos;
  int32_t status;
  int32_t pad_count;
};

// CharAt: c(i) returns character i of the stream (only i >= 4*floor((m-1)/4),
// i.e. the final quad, is ever read).
template <class CharAt>
__device__ __forceinline__ StreamResult finish_stream_at(const CharAt &c, int64_t m, uint8_t *out,
                                                         int64_t err, bool final_stream,
                                                         int flags) {
  const int64_t q = m / 4, r = m % 4;
  StreamResult R;
  R.pad_count = 0;
  if (err >= 0) {
    R.status = 1;
    R.err_pos = err;
    R.out_len = 3 * (err / 4);
    return R;
  }
  int64_t last = -1;  // position whose trailing bits Appendix A constrains
  uint32_t shift = 0;
  if (r != 0) {
    if (final_stream && (flags & kFlagNoPad) && r >= 2) {
      uint32_t v[3] = {0, 0, 0};
      for (int64_t i = 4 * q; i < m; ++i) {
        const uint32_t a = g_dec_tab[c(i)];
        if (a == kInvalid) {
          R.status = (i == 4 * q + 2 && c(i) == '=') ? 2 : 1;
          R.err_pos = R.status == 2 ? 4 * q : i;
          R.out_len = 3 * q;
          return R;
        }
        v[i - 4 * q] = a;
      }
      out[3 * q] = static_cast<uint8_t>(v[0] * 4 + v[1] / 16);
      if (r == 3) out[3 * q + 1] = static_cast<uint8_t>((v[1] * 16) % 256 + v[2] / 4);
      R.out_len = 3 * q + r - 1;
      last = 4 * q + r - 1;
      shift = r == 2 ? 16 : 64;
    } else {
      R.status = 2;
      R.err_pos = 4 * q;
      R.out_len = 3 * q;
      return R;
    }
  } else {
    int32_t p = 0;
    if (final_stream && q > 0 && c(m - 1) == '=') p = (c(m - 2) == '=') ? 2 : 1;
    R.pad_count = p;
    R.out_len = 3 * q - p;
    if (p == 2) {
      last = m - 3;
      shift = 16;
    } else if (p == 1) {
      last = m - 2;
      shift = 64;
    }
  }
  R.status = 0;
  R.err_pos = -1;
  if ((flags & kFlagStrict) && last >= 0 && (g_dec_tab[c(last)] * shift) % 256 != 0) {
    R.status = 3;
    R.err_pos = last;
    R.out_len = 3 * (last / 4);
    R.pad_count = 0;
  }
  return R;
}

__device__ __forceinline__ StreamResult finish_stream(const uint8_t *c, int64_t m, uint8_t *out,
                                                      int64_t err, bool final_stream, int flags) {
  return finish_stream_at([c](int64_t i) -> uint32_t { return c[i]; }, m, out, err, final_stream,
                          flags);
}
}  // namespace b64
