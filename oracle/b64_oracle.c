/*
 * b64_oracle.c -- plain scalar CPU oracle for base64 encode / validating decode.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_1704_00605_b200/csrc), and the CUDA path never calls it.
 *
 * It is a transcription of the paper's Algorithm 1 and Algorithm 2
 * (W. Mula, D. Lemire, "Faster Base64 Encoding and Decoding using AVX2
 * Instructions", /root/reference/PAPER.md), in the paper's order and
 * notation, with the readings listed in DESIGN.md §3:
 *
 *   R-alphabet  B and A are defined by the ranges of P:184-185 (Table I's
 *               body is missing), cross-checked by Table II
 *                and Table III in the tests.
 *   R-pad       '=' is structural, never a data value: it is acceptable only
 *               in the last two positions of an input whose length is a
 *               multiple of 4, and a '=' in position m-2 forces '=' in
 *               position m-1.
 *   R2          the reported error offset is the first position that cannot
 *               continue any valid encoding (left-to-right scan).
 *   R-length    m not divisible by 4 (Alg 2 requires it): status
 *               LENGTH at offset 4*floor(m/4) unless an earlier position is
 *               unacceptable.
 *   R-noncanon  non-canonical trailing bits are accepted.
 *
 * Built with -O2 -fno-tree-vectorize -fno-tree-slp-vectorize so that it
 * stays the plain scalar baseline.  Parity pins: tests/test_oracle.py.
 */
#include <stddef.h>
#include <stdint.h>

#define ORACLE_OK 0
#define ORACLE_INVALID_CHAR 1
#define ORACLE_LENGTH 2

/* B: 6-bit value -> ASCII (Table I: A..Z, a..z, 0..9, '+', '/'). */
int oracle_B(int v) {
  if (v >= 0 && v <= 25) return 'A' + v;
  if (v >= 26 && v <= 51) return 'a' + (v - 26);
  if (v >= 52 && v <= 61) return '0' + (v - 52);
  if (v == 62) return '+';
  if (v == 63) return '/';
  return -1;
}

/* A: ASCII -> 6-bit value, negative for a character outside Table I
 * (Alg 2 preamble).  '=' is NOT given a value here (reading R-pad);
 * Alg 2's "'=' has value 0" convention is applied only when the final quad
 * is emitted, below. */
int oracle_A(int ch) {
  if (ch >= 'A' && ch <= 'Z') return ch - 'A';
  if (ch >= 'a' && ch <= 'z') return ch - 'a' + 26;
  if (ch >= '0' && ch <= '9') return ch - '0' + 52;
  if (ch == '+') return 62;
  if (ch == '/') return 63;
  return -1;
}

int64_t oracle_encoded_len(int64_t n) { return 4 * ((n + 2) / 3); }

/* Algorithm 1.  p must hold 4*ceil(n/3) bytes.  Returns the
 * number of characters written. */
int64_t oracle_encode(const uint8_t *s, int64_t n, uint8_t *p) {
  int64_t o = 0;
  int64_t i;
  /* for i in 0, 3, ..., n - (n mod 3) - 3 */
  for (i = 0; i + 3 <= n - (n % 3); i += 3) {
    p[o++] = (uint8_t)oracle_B(s[i] / 4);
    p[o++] = (uint8_t)oracle_B(((s[i] * 16) % 64) + (s[i + 1] / 16));
    p[o++] = (uint8_t)oracle_B(((s[i + 1] * 4) % 64) + (s[i + 2] / 64));
    p[o++] = (uint8_t)oracle_B(s[i + 2] % 64);
  }
  i = n - n % 3;
  if (i < n) {
    p[o++] = (uint8_t)oracle_B(s[i] / 4);
    if (i == n - 1) {
      p[o++] = (uint8_t)oracle_B((s[i] * 16) % 64);
      p[o++] = '=';
    } else if (i == n - 2) {
      p[o++] = (uint8_t)oracle_B(((s[i] * 16) % 64) + (s[i + 1] / 16));
      p[o++] = (uint8_t)oracle_B((s[i + 1] * 4) % 64);
    }
    p[o++] = '=';
  }
  return o;
}

/* Reading R-pad / R2: is position i of c[0..m) acceptable? */
static int acceptable(const uint8_t *c, int64_t m, int64_t i) {
  const int in_alphabet = oracle_A(c[i]) >= 0;
  if (m % 4 == 0 && i == m - 1)
    return (in_alphabet || c[i] == '=') && (c[m - 2] != '=' || c[i] == '=');
  if (m % 4 == 0 && i == m - 2) return in_alphabet || c[i] == '=';
  return in_alphabet;
}

/* Algorithm 2 with readings R-pad, R2, R-length.
 * p must hold 3*floor(m/4) bytes.  Returns the status; *out_len receives the
 * number of bytes appended to p, *err_pos the error offset or -1. */
int oracle_decode(const uint8_t *c, int64_t m, uint8_t *p, int64_t *out_len,
                  int64_t *err_pos) {
  int64_t o = 0;
  const int64_t q = m / 4;
  int64_t i;
  *err_pos = -1;
  /* for i in 0, 4, ..., n - 4 */
  for (i = 0; i + 4 <= 4 * q; i += 4) {
    int j;
    int a, b, cc, d;
    /* "if any of a, b, c, d is negative: report an error",
     * first offending byte (R2) */
    for (j = 0; j < 4; ++j) {
      if (!acceptable(c, m, i + j)) {
        *err_pos = i + j;
        *out_len = o;
        return ORACLE_INVALID_CHAR;
      }
    }
    /* a..d <- A(C_i..C_{i+3}); '=' contributes 0 */
    a = c[i] == '=' ? 0 : oracle_A(c[i]);
    b = c[i + 1] == '=' ? 0 : oracle_A(c[i + 1]);
    cc = c[i + 2] == '=' ? 0 : oracle_A(c[i + 2]);
    d = c[i + 3] == '=' ? 0 : oracle_A(c[i + 3]);
    p[o++] = (uint8_t)((a * 4) + (b / 16));
    if (c[i + 2] == '=') break;
    p[o++] = (uint8_t)(((b * 16) % 256) + (cc / 4));
    if (c[i + 3] == '=') break;
    p[o++] = (uint8_t)(((cc * 64) % 256) + d);
  }
  *out_len = o;
  if (m % 4 != 0) { /* R-length (P:156 requires n divisible by 4) */
    *err_pos = 4 * q;
    return ORACLE_LENGTH;
  }
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------
 * Variants.  Flags:
 *   ORACLE_URL    base64url alphabet: 62 -> '-', 63 -> '_'
 *   ORACLE_NOPAD  encode omits '=' ("it may be acceptable to omit the
 *                 padding characters if the size ... is otherwise known");
 *                 decode accepts a final partial quad of 2 or 3 characters
 *                 as if padded (padding optional; padded input still valid)
 *   ORACLE_STRICT Appendix A: the trailing bits of the final
 *                 quad must be zero (status ORACLE_NONCANONICAL at the
 *                 offending character), checked after an otherwise
 *                 successful decode.
 * ------------------------------------------------------------------------ */
#define ORACLE_URL 1
#define ORACLE_NOPAD 2
#define ORACLE_STRICT 4
#define ORACLE_NONCANONICAL 3

int oracle_B_ex(int v, int flags) {
  if (flags & ORACLE_URL) {
    if (v == 62) return '-';
    if (v == 63) return '_';
  }
  return oracle_B(v);
}

int oracle_A_ex(int ch, int flags) {
  if (flags & ORACLE_URL) {
    if (ch == '-') return 62;
    if (ch == '_') return 63;
    if (ch == '+' || ch == '/') return -1;
  }
  return oracle_A(ch);
}

int64_t oracle_encoded_len_ex(int64_t n, int flags) {
  if (flags & ORACLE_NOPAD) return 4 * (n / 3) + (n % 3 ? n % 3 + 1 : 0);
  return oracle_encoded_len(n);
}

/* Algorithm 1 with the variant alphabet; NOPAD drops the '='
 * appended at P:141 and P:146. */
int64_t oracle_encode_ex(const uint8_t *s, int64_t n, uint8_t *p, int flags) {
  int64_t o = 0;
  int64_t i;
  for (i = 0; i + 3 <= n - (n % 3); i += 3) {
    p[o++] = (uint8_t)oracle_B_ex(s[i] / 4, flags);
    p[o++] = (uint8_t)oracle_B_ex(((s[i] * 16) % 64) + (s[i + 1] / 16), flags);
    p[o++] = (uint8_t)oracle_B_ex(((s[i + 1] * 4) % 64) + (s[i + 2] / 64), flags);
    p[o++] = (uint8_t)oracle_B_ex(s[i + 2] % 64, flags);
  }
  i = n - n % 3;
  if (i < n) {
    p[o++] = (uint8_t)oracle_B_ex(s[i] / 4, flags);
    if (i == n - 1) {
      p[o++] = (uint8_t)oracle_B_ex((s[i] * 16) % 64, flags);
      if (!(flags & ORACLE_NOPAD)) p[o++] = '=';
    } else if (i == n - 2) {
      p[o++] = (uint8_t)oracle_B_ex(((s[i] * 16) % 64) + (s[i + 1] / 16), flags);
      p[o++] = (uint8_t)oracle_B_ex((s[i + 1] * 4) % 64, flags);
    }
    if (!(flags & ORACLE_NOPAD)) p[o++] = '=';
  }
  return o;
}

static int acceptable_ex(const uint8_t *c, int64_t m, int64_t i, int flags) {
  const int in_alphabet = oracle_A_ex(c[i], flags) >= 0;
  if (m % 4 == 0 && i == m - 1)
    return (in_alphabet || c[i] == '=') && (c[m - 2] != '=' || c[i] == '=');
  if (m % 4 == 0 && i == m - 2) return in_alphabet || c[i] == '=';
  return in_alphabet;
}

/* Algorithm 2 with the variant alphabet, optional padding and
 * the Appendix A check.  p must hold 3*floor(m/4) + 2 bytes. */
int oracle_decode_ex(const uint8_t *c, int64_t m, uint8_t *p, int64_t *out_len, int64_t *err_pos,
                     int flags) {
  int64_t o = 0;
  const int64_t q = m / 4;
  const int64_t r = m % 4;
  int64_t i;
  int64_t last_data = -1; /* position whose trailing bits App. A constrains */
  int64_t last_shift = 0; /* 16 (two pads) or 64 (one pad) */
  *err_pos = -1;
  for (i = 0; i + 4 <= 4 * q; i += 4) {
    int j;
    int a, b, cc, d;
    for (j = 0; j < 4; ++j) {
      if (!acceptable_ex(c, m, i + j, flags)) {
        *err_pos = i + j;
        *out_len = o;
        return ORACLE_INVALID_CHAR;
      }
    }
    a = c[i] == '=' ? 0 : oracle_A_ex(c[i], flags);
    b = c[i + 1] == '=' ? 0 : oracle_A_ex(c[i + 1], flags);
    cc = c[i + 2] == '=' ? 0 : oracle_A_ex(c[i + 2], flags);
    d = c[i + 3] == '=' ? 0 : oracle_A_ex(c[i + 3], flags);
    p[o++] = (uint8_t)((a * 4) + (b / 16));
    if (c[i + 2] == '=') {
      last_data = i + 1;
      last_shift = 16;
      break;
    }
    p[o++] = (uint8_t)(((b * 16) % 256) + (cc / 4));
    if (c[i + 3] == '=') {
      last_data = i + 2;
      last_shift = 64;
      break;
    }
    p[o++] = (uint8_t)(((cc * 64) % 256) + d);
  }
  if (r != 0) {
    if (!(flags & ORACLE_NOPAD) || r == 1) { /* R-length */
      *out_len = o;
      *err_pos = 4 * q;
      return ORACLE_LENGTH;
    }
    /* NOPAD: the partial final quad, decoded as if padded.
     * Its characters must be data; a '=' in its third position can still
     * continue a padded quad ("xx=" -> "xx=="), so that input is merely
     * truncated: LENGTH at 4q (reading R2 / R-length). */
    for (i = 4 * q; i < m; ++i) {
      if (oracle_A_ex(c[i], flags) < 0) {
        *out_len = o;
        if (i == 4 * q + 2 && c[i] == '=') {
          *err_pos = 4 * q;
          return ORACLE_LENGTH;
        }
        *err_pos = i;
        return ORACLE_INVALID_CHAR;
      }
    }
    {
      const int a = oracle_A_ex(c[4 * q], flags);
      const int b = oracle_A_ex(c[4 * q + 1], flags);
      p[o++] = (uint8_t)((a * 4) + (b / 16));
      last_data = 4 * q + 1;
      last_shift = 16;
      if (r == 3) {
        const int cc = oracle_A_ex(c[4 * q + 2], flags);
        p[o++] = (uint8_t)(((b * 16) % 256) + (cc / 4));
        last_data = 4 * q + 2;
        last_shift = 64;
      }
    }
  }
  *out_len = o;
  /* Appendix A: (A(C_{n-3}) x 16) mod 256 = 0 with two pads,
   * (A(C_{n-2}) x 64) mod 256 = 0 with one pad. */
  if ((flags & ORACLE_STRICT) && last_data >= 0 &&
      (oracle_A_ex(c[last_data], flags) * last_shift) % 256 != 0) {
    *err_pos = last_data;
    *out_len = 3 * (last_data / 4);
    return ORACLE_NONCANONICAL;
  }
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------
 * Appendix B whitespace removal, the scalar filter
 * of Fig. "spaceremove": copy each byte and advance the write
 * position only when table[v] (the 256-entry keep flags) is 1.  The removed
 * bytes are space, line feed and carriage return (the hex codes
 * printed there are swapped, reading G8: ' ' = 0x20, '\n' = 0x0A,
 * '\r' = 0x0D).  Out of place here (p[] separate from A[]).  Returns the new
 * length.
 * ------------------------------------------------------------------------ */
int64_t oracle_despace(const uint8_t *A, int64_t N, uint8_t *p_out) {
  uint8_t table[256];
  int64_t i, p;
  int v;
  for (v = 0; v < 256; ++v) table[v] = 1;
  table[' '] = 0;
  table['\n'] = 0;
  table['\r'] = 0;
  for (i = 0, p = 0; i < N; i++) {
    uint8_t c = A[i];
    p_out[p] = c;
    p += table[c];
  }
  return p;
}

/* ------------------------------------------------------------------------
 * MIME-style line handling.
 *
 * The paper's comparison includes a codec (Linux) that tolerates line feeds
 * between blocks of four characters, and Appendix B says
 * white space "should be removed prior to processing".  Two plain
 * compositions of the functions above (reading R-ws-decode / R-wrap in
 * DESIGN.md §3):
 *
 *   oracle_encode_wrapped  Algorithm 1 (with the f1 variant flags), then the
 *                          end-of-line sequence (LF, or CR LF when crlf != 0)
 *                          inserted after every line_chars characters and
 *                          after the final, possibly shorter, line (no EOL
 *                          for an empty output).  line_chars is a positive
 *                          multiple of 4 (76 for MIME, RFC 2045; 64 for PEM).
 *   oracle_decode_ws       the Appendix B filter (oracle_despace's table:
 *                          ' ', '\n', '\r') applied first, then Algorithm 2
 *                          (oracle_decode_ex, same flags) on the kept bytes;
 *                          an error offset is reported in the coordinates of
 *                          the ORIGINAL input: the position of the kept byte
 *                          the decoder rejected.
 * ------------------------------------------------------------------------ */
#include <stdlib.h>

int64_t oracle_encoded_len_wrapped(int64_t n, int line_chars, int crlf, int flags) {
  const int64_t m = oracle_encoded_len_ex(n, flags);
  const int64_t lines = (m + line_chars - 1) / line_chars;
  return m + lines * (crlf ? 2 : 1);
}

int64_t oracle_encode_wrapped(const uint8_t *s, int64_t n, uint8_t *p, int line_chars, int crlf,
                              int flags) {
  const int64_t m = oracle_encoded_len_ex(n, flags);
  uint8_t *t = (uint8_t *)malloc(m > 0 ? (size_t)m : 1);
  int64_t j, o = 0;
  if (!t) return -1;
  oracle_encode_ex(s, n, t, flags); /* Algorithm 1 */
  for (j = 0; j < m; ++j) {
    p[o++] = t[j];
    if ((j + 1) % line_chars == 0 || j == m - 1) { /* end of a line */
      if (crlf) p[o++] = '\r';
      p[o++] = '\n';
    }
  }
  free(t);
  return o;
}

/* p must hold 3*floor(m/4) + 2 bytes. */
int oracle_decode_ws(const uint8_t *c, int64_t m, uint8_t *p, int64_t *out_len, int64_t *err_pos,
                     int flags) {
  uint8_t *t = (uint8_t *)malloc(m > 0 ? (size_t)m : 1);
  int64_t *orig = (int64_t *)malloc(m > 0 ? (size_t)m * sizeof(int64_t) : sizeof(int64_t));
  int64_t i, k = 0;
  int st;
  if (!t || !orig) {
    free(t);
    free(orig);
    return -1;
  }
  /* Appendix B filter (Fig. spaceremove), remembering where
   * each kept byte came from */
  for (i = 0; i < m; ++i) {
    if (c[i] == ' ' || c[i] == '\n' || c[i] == '\r') continue;
    t[k] = c[i];
    orig[k] = i;
    ++k;
  }
  st = oracle_decode_ex(t, k, p, out_len, err_pos, flags); /* Algorithm 2 */
  if (*err_pos >= 0) *err_pos = orig[*err_pos];
  free(t);
  free(orig);
  return st;
}
