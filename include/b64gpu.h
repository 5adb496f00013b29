/*
 * b64gpu.h -- C ABI of libb64gpu.so: base64 encode / validating decode on B200.
 *
 * Paper: W. Mula, D. Lemire, "Faster Base64 Encoding and Decoding using AVX2
 * Instructions" (arXiv 1704.00605); "P:n" = line n of /root/reference/PAPER.md.
 * Design and the readings of ambiguous passages: DESIGN.md.
 *
 * Conventions (all entry points)
 *  - Pointers named d_* are CUDA device pointers (any alignment is legal; the
 *    16-byte aligned case is the fast path).  h_* are host pointers.
 *  - Sizes and offsets are int64_t.  Error offsets are 0-based byte indexes
 *    into the input; -1 means "no error".
 *  - `stream` is a cudaStream_t (0 = legacy default stream).  Every call only
 *    enqueues work on `stream` unless it says it synchronizes.
 *  - The caller owns every buffer; the library allocates nothing on the hot
 *    path except a small per-(device, stream) scratch record created on the
 *    first decode call on that stream (16 B of device memory plus 32 B of
 *    mapped pinned host memory; never freed).  Do not make the first decode
 *    call on a stream inside CUDA-graph capture.
 *  - Input and output buffers must not overlap.
 *  - Return codes: >= 0 success (or a length), negative = b64_status error.
 *    Nothing is launched when an argument check fails.  No exceptions cross
 *    the ABI; nothing is printed.
 *  - Reads: the kernels read input through 16-byte aligned windows, so up to
 *    15 bytes before d_in and after d_in + n that share a 16-byte granule
 *    with the input may be read (never written).  Torch / cudaMalloc
 *    allocations are padded to at least 256 B, so this never leaves the
 *    allocation in practice.
 *  - Device: every launching call runs on the device that owns `stream`
 *    (the current device for the legacy / per-thread default stream) and
 *    restores the caller's current device before returning.
 *  - All entry points are reentrant for calls on distinct streams.  The
 *    single-buffer decode keeps its error-reduction scratch per (device,
 *    stream): two decodes that may run concurrently (e.g. CUDA graphs
 *    captured on the same stream and replayed at once, or replayed on
 *    another stream while direct decodes run on the capture stream) must
 *    have been enqueued on distinct streams -- or use
 *    b64_decode_scratch_async with distinct caller-owned scratch records.
 */
#ifndef B64GPU_H
#define B64GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *b64_stream_t; /* == cudaStream_t */

typedef enum {
  B64_OK = 0,               /* valid input, fully decoded                            */
  B64_ERR_INVALID_CHAR = 1, /* a byte outside the alphabet / misplaced '=' */
  B64_ERR_LENGTH = 2,       /* m not divisible by 4 (Alg 2 requires it)        */
  B64_ERR_NONCANONICAL = 3, /* B64_FLAG_STRICT: non-zero trailing bits (App. A) */
  B64_ERR_ARG = -1,         /* bad argument; nothing launched                          */
  B64_ERR_CUDA = -2,        /* a CUDA runtime call failed                              */
  B64_ERR_WORKSPACE = -3    /* batched workspace too small                             */
} b64_status;

/* Variant flags; 0 = the paper's default
 * (standard alphabet, '=' padding required, non-canonical bits accepted). */
enum {
  B64_FLAG_URL = 1,    /* base64url alphabet: 62 -> '-', 63 -> '_'               */
  B64_FLAG_NOPAD = 2,  /* encode: no '='; decode: padding optional, a final partial
                          quad of 2 or 3 characters decodes as if padded        */
  B64_FLAG_STRICT = 4  /* decode: reject non-zero trailing bits of the final quad
                          (Appendix A) with B64_ERR_NONCANONICAL at that character      */
};

/* Device-side result record of one decode (16-byte aligned). */
typedef struct {
  int64_t out_len;   /* bytes of valid output (see b64_decode)             */
  int64_t err_pos;   /* first error offset, -1 if none                      */
  int32_t status;    /* b64_status >= 0 (OK, INVALID_CHAR, LENGTH, NONCANONICAL) */
  int32_t pad_count; /* number of trailing '=' consumed (0, 1, 2)           */
} b64_result;

/* ------------------------------------------------------------------ sizes */

/* 4*ceil(n/3): encoded length of n bytes with '=' padding (P:116-119,
 * Alg 1).  Pure host; -1 if n < 0. */
int64_t b64_encoded_len(int64_t n);

/* 3*floor(m/4): output capacity a decode of m characters may write
 * (Alg 2 emits at most 3 bytes per complete quad). -1 if m < 0. */
int64_t b64_decoded_max_len(int64_t m);

/* Variant sizes: encoded length under `flags` (NOPAD: ceil(4n/3)); decode
 * output capacity under `flags` (NOPAD adds r-1 bytes for an r = 2, 3
 * character tail).  -1 on a bad argument. */
int64_t b64_encoded_len_ex(int64_t n, int flags);
int64_t b64_decoded_max_len_ex(int64_t m, int flags);

/* ----------------------------------------------------------------- encode */

/* Algorithm 1 on n bytes at d_in: writes exactly
 * b64_encoded_len(n) ASCII characters of the standard alphabet
 * to d_out, '=' padded, no line breaks.  Asynchronous on `stream`.
 * Returns the output length, or B64_ERR_ARG / B64_ERR_CUDA. */
int64_t b64_encode(const uint8_t *d_in, int64_t n, uint8_t *d_out, b64_stream_t stream);

/* b64_encode with variant flags (B64_FLAG_URL, B64_FLAG_NOPAD; STRICT is
 * ignored): writes b64_encoded_len_ex(n, flags) characters. */
int64_t b64_encode_ex(const uint8_t *d_in, int64_t n, uint8_t *d_out, int flags,
                      b64_stream_t stream);

/* ----------------------------------------------------------------- decode */

/* Validating decode, Algorithm 2 with DESIGN.md readings
 * R-pad / R2 / R-length, of m characters at d_in into d_out (capacity
 * b64_decoded_max_len(m)).  Enqueues on `stream` and then SYNCHRONIZES the
 * stream.  On return:
 *   OK:            *out_len = 3*(m/4) - pad_count, *err_pos = -1
 *   INVALID_CHAR:  *err_pos = first offending byte (minimum over the whole
 *                  buffer), *out_len = 3*floor(err_pos/4); d_out[0..out_len)
 *                  holds the complete quads before it, later bytes are
 *                  unspecified (within capacity)
 *   LENGTH:        m % 4 != 0 and no earlier error: *err_pos = 4*floor(m/4),
 *                  *out_len = 3*floor(m/4)
 * Returns the status (>= 0) or a negative error code.  out_len / err_pos may
 * be NULL. */
int b64_decode(const uint8_t *d_in, int64_t m, uint8_t *d_out, int64_t *out_len,
               int64_t *err_pos, b64_stream_t stream);

/* Fully asynchronous decode: same semantics as b64_decode, the result record
 * is written by the device to d_result (device or mapped host memory, 8-byte
 * aligned) when the kernel finishes.  Returns B64_OK if enqueued. */
int b64_decode_async(const uint8_t *d_in, int64_t m, uint8_t *d_out, b64_result *d_result,
                     b64_stream_t stream);

/* Decode with variant flags (URL alphabet, optional padding, strict
 * trailing bits).  d_out capacity: b64_decoded_max_len_ex(m, flags).  Status
 * and offsets as b64_decode, plus B64_ERR_NONCANONICAL (err_pos = the
 * character whose low bits are non-zero, out_len = 3*floor(err_pos/4)). */
int b64_decode_ex(const uint8_t *d_in, int64_t m, uint8_t *d_out, int flags, int64_t *out_len,
                  int64_t *err_pos, b64_stream_t stream);
int b64_decode_ex_async(const uint8_t *d_in, int64_t m, uint8_t *d_out, int flags,
                        b64_result *d_result, b64_stream_t stream);

/* b64_decode_ex_async with caller-owned scratch instead of the library's
 * per-(device, stream) record: d_scratch is B64_DECODE_SCRATCH_BYTES of
 * device memory, 8-byte aligned, ZERO before its first use (cudaMemset);
 * every call leaves it zero again when its kernel completes.  Decodes that
 * may run concurrently (e.g. CUDA graphs replayed at the same time) must
 * use distinct scratch records.  Returns B64_OK if enqueued. */
#define B64_DECODE_SCRATCH_BYTES 16
int b64_decode_scratch_async(const uint8_t *d_in, int64_t m, uint8_t *d_out, int flags,
                             b64_result *d_result, void *d_scratch, b64_stream_t stream);

/* Decode of one shard of a larger buffer split on 4-character boundaries
 * (multi-GPU sharder).  final_shard != 0: identical to
 * b64_decode_async.  final_shard == 0: m must be a multiple of 4 and the
 * final-quad padding rule is NOT applied ('=' anywhere is an error), because
 * a later shard follows (reading R-shard).  Offsets in d_result are
 * shard-relative. */
int b64_decode_shard_async(const uint8_t *d_in, int64_t m, int final_shard, uint8_t *d_out,
                           b64_result *d_result, b64_stream_t stream);

/* b64_decode_shard_async with variant flags (URL applies to every shard;
 * NOPAD and STRICT change only the final shard's tail) and the exchange
 * record of the multi-GPU decode: when d_key != NULL the kernel also writes
 * d_key[0] = b64_shard_key(status, err_pos, shard_begin) (the shard's first
 * error as a GLOBAL offset with its status, INT64_MAX if clean) and
 * d_key[1] = out_len (device int64[2], 8-byte aligned).  shard_begin: offset
 * of d_in[0] in the whole buffer (>= 0).  The MIN all-reduce of d_key[0]
 * over the shards and the all-gather of d_key[1] are the only exchange;
 * b64_combine_shards[_async] turns them into the whole buffer's result. */
int b64_decode_shard_ex_async(const uint8_t *d_in, int64_t m, int64_t shard_begin, int final_shard,
                              uint8_t *d_out, int flags, b64_result *d_result, int64_t *d_key,
                              b64_stream_t stream);

/* Reduction key of one shard result: (shard_begin + err_pos) * 4 + status
 * for status != B64_OK, INT64_MAX for B64_OK.  Shards cover disjoint
 * offsets, so the minimum key over all shards is the buffer's first error
 * together with its status.  Pure host. */
int64_t b64_shard_key(int32_t status, int64_t err_pos, int64_t shard_begin);

/* The whole buffer's decode result from key_min (the MIN over shards of
 * b64_shard_key) and the shard output lengths h_shard_out_len[0..world):
 * clean -> status OK, err_pos -1, out_len = sum of the lengths, pad_count =
 * 3*(total_m/4) - out_len when total_m % 4 == 0 (else 0); error -> err_pos =
 * key_min / 4, status = key_min % 4, out_len = 3*floor(err_pos/4) (Alg 2
 * appends nothing for the failing quad).  total_m: characters of
 * the whole buffer.  Pure host; B64_ERR_ARG on bad arguments. */
int b64_combine_shards(int64_t key_min, const int64_t *h_shard_out_len, int world, int64_t total_m,
                       b64_result *h_result);

/* The same on the device (one tiny kernel on `stream`): d_key_min (int64),
 * d_shard_out_len (int64[world]) and d_result are device pointers, so the
 * whole sharded step -- decode, NCCL MIN all-reduce, all-gather, combine --
 * runs without a host synchronization. */
int b64_combine_shards_async(const int64_t *d_key_min, const int64_t *d_shard_out_len, int world,
                             int64_t total_m, b64_result *d_result, b64_stream_t stream);

/* ---------------------------------------------------------------- batched */

/* Scratch bytes (device memory, 256-byte aligned) that a batched call over k
 * messages totalling at most total_in bytes of input needs.
 * direction: 0 = encode, 1 = decode. */
size_t b64_batch_workspace_bytes(int64_t k, int64_t total_in, int direction);

/* Batched encode of k independent messages: message i is
 * d_in[d_in_off[i] .. d_in_off[i+1]) (d_in_off: k+1 non-decreasing int64 on
 * the device, d_in_off[0] may be > 0).  Writes d_out_off[0..k] (device,
 * d_out_off[0] = 0, d_out_off[i+1]-d_out_off[i] = b64_encoded_len(len_i))
 * and each encoding contiguously to d_out.  Messages are cut into warp
 * work units that never straddle messages, and every warp takes a
 * contiguous range of units of equal estimated cost (a fixed part per unit
 * plus its bytes) -- messages are assigned to warps by the prefix sums of
 * their lengths (BASELINE.json north_star).  d_ws: b64_batch_workspace_bytes(k, total_in, 0) bytes,
 * total_in >= d_in_off[k] - d_in_off[0].  Asynchronous. */
int b64_encode_batch(const uint8_t *d_in, const int64_t *d_in_off, int64_t k, int64_t total_in,
                     uint8_t *d_out, int64_t *d_out_off, void *d_ws, size_t ws_bytes,
                     b64_stream_t stream);

/* Batched validating decode: message i is decoded independently under the
 * rules of b64_decode.  d_out_off[i+1]-d_out_off[i] reserves the nominal
 * decoded length 3*floor(len_i/4) - p_i (p_i = number of trailing '=' in the
 * last two characters when len_i % 4 == 0), so outputs of valid messages are
 * contiguous.  Per message (device arrays of k): d_out_len[i], d_err_pos[i]
 * (message-relative, -1 if none), d_status[i] (b64_status >= 0).
 * Asynchronous. */
int b64_decode_batch(const uint8_t *d_in, const int64_t *d_in_off, int64_t k, int64_t total_in,
                     uint8_t *d_out, int64_t *d_out_off, int64_t *d_out_len, int64_t *d_err_pos,
                     int32_t *d_status, void *d_ws, size_t ws_bytes, b64_stream_t stream);

/* Batched variants with flags (per-message semantics of b64_encode_ex /
 * b64_decode_ex; output reservations use the variant sizes). */
int b64_encode_batch_ex(const uint8_t *d_in, const int64_t *d_in_off, int64_t k, int64_t total_in,
                        uint8_t *d_out, int64_t *d_out_off, int flags, void *d_ws, size_t ws_bytes,
                        b64_stream_t stream);
int b64_decode_batch_ex(const uint8_t *d_in, const int64_t *d_in_off, int64_t k, int64_t total_in,
                        uint8_t *d_out, int64_t *d_out_off, int64_t *d_out_len, int64_t *d_err_pos,
                        int32_t *d_status, int flags, void *d_ws, size_t ws_bytes,
                        b64_stream_t stream);

/* ------------------------------------------------------- whitespace (f3) */

/* Appendix B: remove ' ' (0x20), '\n' (0x0A) and '\r' (0x0D)
 * from d_in[0..m) into d_out (capacity m; d_out must not overlap d_in),
 * preserving order; *d_out_len (device int64) receives the new length.
 * Three kernels.  (1) A verified fast path for line-structured text (MIME /
 * PEM: lines of L chars, L a multiple of 4 up to 4092, each ending in the
 * same EOL, "\n" or "\r\n", the last line shorter and its EOL optional):
 * one strided copy of the lines' characters; any byte below 0x21 inside a
 * line or any deviation from the structure makes it give up (its writes to
 * d_out are then overwritten).  (2)-(3) Otherwise the general path:
 * per-chunk kept counts, then per-chunk compaction of 16 KiB TMA-staged
 * tiles (warp scans, congruent 16-byte copy-out) at the chunk offsets; both
 * return at once when (1) succeeded.  The result is the same either way.
 * d_ws: b64_despace_workspace_bytes(m) bytes of device memory, 16-byte
 * aligned.  Asynchronous. */
size_t b64_despace_workspace_bytes(int64_t m);
int b64_despace(const uint8_t *d_in, int64_t m, uint8_t *d_out, int64_t *d_out_len, void *d_ws,
                size_t ws_bytes, b64_stream_t stream);

/* -------------------------------------------- MIME line handling (f4) */

/* Line-wrapped encode (reading R-wrap): Algorithm 1
 * with variant `flags` (URL, NOPAD), and an end-of-line sequence
 * -- "\r\n" if crlf = 1, "\n" if crlf = 0 -- after every line_chars
 * characters and after the final (shorter) line; empty input gives empty
 * output.  line_chars: a multiple of 4 in [4, 16384] (76 = MIME, RFC 2045;
 * 64 = PEM).  The paper's comparison mentions MIME-style line handling in
 * the Linux codec.  d_out capacity:
 * b64_encoded_len_wrapped(n, line_chars, crlf, flags).  Asynchronous on
 * `stream` (one kernel: line-major for line_chars <= 128); returns the
 * output length, or B64_ERR_ARG (nothing launched) / B64_ERR_CUDA. */
int64_t b64_encoded_len_wrapped(int64_t n, int line_chars, int crlf, int flags);
int64_t b64_encode_wrapped(const uint8_t *d_in, int64_t n, uint8_t *d_out, int line_chars,
                           int crlf, int flags, b64_stream_t stream);

/* Whitespace-tolerant decode (reading R-ws-decode): the
 * Appendix B filter ("white-space characters ... should be removed
 * prior to processing"; removed set ' ', '\n', '\r') followed
 * by Algorithm 2 with variant `flags` on the kept characters --
 * fused: the compacted text never leaves shared memory.  Accepts e.g. MIME
 * text with CRLF every 76 characters, or the Linux codec's line feeds
 * between quads.  Every error offset (INVALID_CHAR, LENGTH,
 * NONCANONICAL) is an offset into d_in (ORIGINAL coordinates: the position
 * of the kept byte the decoder rejected); out_len counts decoded bytes.
 * d_out capacity: b64_decoded_max_len_ex(m, flags).  d_ws: device scratch
 * of b64_decode_ws_workspace_bytes(m) bytes, 16-byte aligned, not shared
 * with a concurrent call.  Three kernels on `stream`: a verified fast path
 * for line-structured (MIME / PEM) text, then the mask pass and the fused
 * compaction + decode, which return at once when the fast path succeeded.
 * _async writes the result record to d_result (device memory); the plain
 * call synchronizes `stream` and returns the status. */
size_t b64_decode_ws_workspace_bytes(int64_t m);
int b64_decode_ws_async(const uint8_t *d_in, int64_t m, uint8_t *d_out, int flags,
                        b64_result *d_result, void *d_ws, size_t ws_bytes, b64_stream_t stream);
int b64_decode_ws(const uint8_t *d_in, int64_t m, uint8_t *d_out, int flags, int64_t *out_len,
                  int64_t *err_pos, void *d_ws, size_t ws_bytes, b64_stream_t stream);

/* ------------------------------------------------------------ host buffers */

/* End-to-end helpers with HOST buffers (pinned memory recommended): the
 * input is copied host->device in chunks, each chunk is processed as soon as
 * it lands and its output copied back, so transfers overlap the kernels.
 * d_scratch_in / d_scratch_out are device buffers of at least n (resp. m)
 * and b64_encoded_len_ex(n, flags) (resp. b64_decoded_max_len_ex(m, flags))
 * bytes; h_out has the same capacity as d_scratch_out.  The copies run on
 * internal streams that first wait for the work already queued on `stream`,
 * so earlier kernels using the scratch buffers are not overtaken.  Decode
 * chunks are shards (b64_decode_shard_ex_async) combined like the
 * multi-GPU exchange (b64_combine_shards): status, err_pos and out_len are
 * those of b64_decode_ex on the whole input.  Both synchronize `stream`
 * before returning (also on failure, after draining the internal copies).
 * The plain forms are the _ex forms with flags = 0. */
int64_t b64_encode_host(const uint8_t *h_in, int64_t n, uint8_t *h_out, uint8_t *d_scratch_in,
                        uint8_t *d_scratch_out, b64_stream_t stream);
int b64_decode_host(const uint8_t *h_in, int64_t m, uint8_t *h_out, int64_t *out_len,
                    int64_t *err_pos, uint8_t *d_scratch_in, uint8_t *d_scratch_out,
                    b64_stream_t stream);
int64_t b64_encode_host_ex(const uint8_t *h_in, int64_t n, uint8_t *h_out, int flags,
                           uint8_t *d_scratch_in, uint8_t *d_scratch_out, b64_stream_t stream);
int b64_decode_host_ex(const uint8_t *h_in, int64_t m, uint8_t *h_out, int flags, int64_t *out_len,
                       int64_t *err_pos, uint8_t *d_scratch_in, uint8_t *d_scratch_out,
                       b64_stream_t stream);

/* ------------------------------------------------------------------ misc */

/* Unit-aligned shard [*begin, *end) of a buffer of `total` bytes for rank
 * `rank` of `world` (unit = 3 for encode input, 4 for decode input): the
 * Q = ceil(total/unit) units are split as [floor(r*Q/G), floor((r+1)*Q/G)),
 * so only the last rank sees a partial unit.  Pure host. */
int b64_shard(int64_t total, int unit, int world, int rank, int64_t *begin, int64_t *end);

/* Batch sharding by message: rank `rank` of `world` gets
 * the contiguous messages [*msg_begin, *msg_end) -- the batch's bytes
 * h_in_off[0] .. h_in_off[k] cut into `world` equal-byte ranges, each cut
 * moved to the next message boundary, so no message is split and every
 * message belongs to exactly one rank (a rank may get none).  h_in_off:
 * HOST int64[k+1], nondecreasing.  Each rank then runs the batched calls on
 * its slice (offsets rebased to its first message); per-message results
 * are gathered (paper_1704_00605_b200.dist).  Pure host; B64_ERR_ARG on bad
 * arguments. */
int b64_batch_shard(const int64_t *h_in_off, int64_t k, int world, int rank, int64_t *msg_begin,
                    int64_t *msg_end);

/* Static string for a status code. */
const char *b64_status_str(int status);

/* Library version string and the sm architecture it was compiled for. */
const char *b64_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* B64GPU_H */
