/*
 * affine_oracle.c — CPU oracle of the affine-gap 3-way alignment defined in
 * SPEC-AFFINE.md.  TEST INFRASTRUCTURE ONLY (see trio_oracle.h): the checker
 * for the affine CUDA path, never part of the product.
 *
 * The reference has no affine gaps, so this
 * oracle is pinned by (1) gap_open = 0 reproducing the reference linear
 * scores / ends (tests/test_affine_oracle.py against tests/golden/ fixtures
 * made by the reference itself) and (2) an independent exhaustive enumerator
 * of all alignments of small triplets (same test file).  It deliberately
 * does NOT use the three-term entering-value shortcut of SPEC-AFFINE.md: the
 * fill takes the max over all seven predecessor types with n(t', t) openings,
 * so the shortcut the kernels use is checked too.
 */
#include <stdlib.h>
#include <string.h>

#include "trio_oracle.h"

#define GAP '-'
#define NEGV (-(1 << 29))

/* residue masks of the column types 1..7 (bit 0 = s0), Eq. 1 order */
static const int kMask[8] = {0, 7, 3, 5, 6, 1, 2, 4};

/* pair state of pair (p, q) in a column of residue mask m:
 * 0 = both residues (M), 1 = p only (P), 2 = q only (Q), 3 = neither (N) */
static int pair_state(int m, int p, int q) {
  const int rp = (m >> p) & 1, rq = (m >> q) & 1;
  return rp && rq ? 0 : rp ? 1 : rq ? 2 : 3;
}

/* n(t', t): pairs gapped (P/Q) in t whose state in t' differs (t' = 0: the
 * virtual all-residue column before the first one) */
static int n_open(int tp, int t) {
  static const int P[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  const int mp = tp ? kMask[tp] : 7, m = kMask[t];
  int n = 0;
  for (int e = 0; e < 3; ++e) {
    const int st = pair_state(m, P[e][0], P[e][1]);
    if ((st == 1 || st == 2) && pair_state(mp, P[e][0], P[e][1]) != st) ++n;
  }
  return n;
}

/* linear part of a column: sum over pairs of sigma (core.hpp:36-46) */
static int32_t col_linear(int t, char x0, char x1, char x2, to_scheme s) {
  const int m = kMask[t];
  const char c0 = (m & 1) ? x0 : GAP, c1 = (m & 2) ? x1 : GAP, c2 = (m & 4) ? x2 : GAP;
  return to_sop(c0, c1, c2, s);
}

static inline size_t ix(int32_t b, int32_t c, int32_t i, int32_t j, int32_t k) {
  return ((size_t)i * (size_t)(b + 1) + (size_t)j) * (size_t)(c + 1) + (size_t)k;
}

static int is_start(int mode, int32_t i, int32_t j, int32_t k) {
  const int zeros = (i == 0) + (j == 0) + (k == 0);
  if (mode == TO_GLOBAL) return zeros == 3;
  if (mode == TO_SEMIGLOBAL) return zeros >= 2;
  return 1;
}

/* V[t][cell] for t = 1..7 (index t-1), B[cell] */
static void affine_fill(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2, int32_t c,
                        to_scheme s, int32_t open, int mode, int32_t* V, int32_t* B) {
  const size_t cells = (size_t)(a + 1) * (size_t)(b + 1) * (size_t)(c + 1);
  int nop[8][8];
  for (int tp = 0; tp < 8; ++tp)
    for (int t = 1; t < 8; ++t) nop[tp][t] = n_open(tp, t);
  for (int32_t i = 0; i <= a; ++i)
    for (int32_t j = 0; j <= b; ++j)
      for (int32_t k = 0; k <= c; ++k) {
        const size_t x = ix(b, c, i, j, k);
        const char x0 = i ? s0[i - 1] : GAP, x1 = j ? s1[j - 1] : GAP, x2 = k ? s2[k - 1] : GAP;
        int32_t best = NEGV;
        for (int t = 1; t < 8; ++t) {
          const int m = kMask[t];
          const int32_t di = m & 1, dj = (m >> 1) & 1, dk = (m >> 2) & 1;
          int32_t v = NEGV;
          if (i >= di && j >= dj && k >= dk) {
            const size_t p = ix(b, c, i - di, j - dj, k - dk);
            int32_t e = NEGV;
            for (int tp = 1; tp < 8; ++tp) {
              const int32_t vp = V[(size_t)(tp - 1) * cells + p];
              if (vp <= NEGV / 2) continue;
              const int32_t cand = vp + nop[tp][t] * open;
              if (cand > e) e = cand;
            }
            if (e > NEGV / 2) v = e + col_linear(t, x0, x1, x2, s);
          }
          if (t == 1 && is_start(mode, i, j, k) && v < 0) v = 0; /* start: virtual type-1 column of value 0 */
          V[(size_t)(t - 1) * cells + x] = v;
          if (v > best) best = v;
        }
        B[x] = best;
      }
}

int to_affine_align(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2, int32_t c,
                    to_scheme s, int32_t open, int mode, uint64_t cell_budget, to_result* out, char* row0,
                    char* row1, char* row2) {
  const uint64_t total = (uint64_t)(a + 1) * (uint64_t)(b + 1) * (uint64_t)(c + 1);
  memset(out, 0, sizeof(*out));
  if (total > cell_budget) return TO_ERR_CAPACITY;
  const size_t cells = (size_t)total;
  int32_t* V = (int32_t*)malloc(cells * 8 * sizeof(int32_t));
  if (!V) return TO_ERR_NOMEM;
  int32_t* B = V + 7 * cells;
  affine_fill(s0, a, s1, b, s2, c, s, open, mode, V, B);
  /* optimal_score (oracle.cpp:67-88): strict > in lexicographic scan */
  int32_t score = NEGV, ei = 0, ej = 0, ek = 0;
  if (mode == TO_GLOBAL) {
    score = B[ix(b, c, a, b, c)];
    ei = a, ej = b, ek = c;
  } else {
    for (int32_t i = 0; i <= a; ++i)
      for (int32_t j = 0; j <= b; ++j)
        for (int32_t k = 0; k <= c; ++k) {
          if (mode == TO_SEMIGLOBAL && !(i == a || j == b || k == c)) continue;
          const int32_t v = B[ix(b, c, i, j, k)];
          if (v > score) score = v, ei = i, ej = j, ek = k;
        }
  }
  out->score = score;
  out->end_i = ei, out->end_j = ej, out->end_k = ek;
  int rc = TO_OK;
  if (row0) {
    const size_t cap = (size_t)a + (size_t)b + (size_t)c + 1;
    char* rev = (char*)malloc(3 * cap);
    if (!rev) {
      free(V);
      return TO_ERR_NOMEM;
    }
    size_t nrev = 0;
    int32_t i = ei, j = ej, k = ek;
    const size_t xe = ix(b, c, i, j, k);
    int t = 1;
    while (t < 7 && V[(size_t)(t - 1) * cells + xe] != B[xe]) ++t; /* smallest type attaining B */
    for (;;) {
      const size_t x = ix(b, c, i, j, k);
      const int32_t vt = V[(size_t)(t - 1) * cells + x];
      if (t == 1 && is_start(mode, i, j, k) && vt == 0) break; /* a start wins ties */
      const int m = kMask[t];
      const int32_t di = m & 1, dj = (m >> 1) & 1, dk = (m >> 2) & 1;
      if (i < di || j < dj || k < dk || nrev >= cap) {
        rc = TO_ERR_LOGIC;
        break;
      }
      const char x0 = i ? s0[i - 1] : GAP, x1 = j ? s1[j - 1] : GAP, x2 = k ? s2[k - 1] : GAP;
      char* col = rev + 3 * nrev++;
      col[0] = (m & 1) ? x0 : GAP, col[1] = (m & 2) ? x1 : GAP, col[2] = (m & 4) ? x2 : GAP;
      const size_t p = ix(b, c, i - di, j - dj, k - dk);
      int32_t e = NEGV;
      int tb = 0;
      for (int tp = 1; tp < 8; ++tp) { /* smallest type attaining the max */
        const int32_t vp = V[(size_t)(tp - 1) * cells + p];
        if (vp <= NEGV / 2) continue;
        const int32_t cand = vp + n_open(tp, t) * open;
        if (cand > e) e = cand, tb = tp;
      }
      if (tb == 0 || e + col_linear(t, x0, x1, x2, s) != vt) {
        rc = TO_ERR_LOGIC;
        break;
      }
      i -= di, j -= dj, k -= dk;
      t = tb;
    }
    if (rc == TO_OK) {
      out->begin_i = i, out->begin_j = j, out->begin_k = k;
      size_t len = 0;
#define PUSH(c0, c1, c2) (row0[len] = (c0), row1[len] = (c1), row2[len] = (c2), ++len)
      if (mode == TO_SEMIGLOBAL) { /* oracle.cpp:165-178 */
        for (int32_t q = 0; q < i; ++q) PUSH(s0[q], GAP, GAP);
        for (int32_t q = 0; q < j; ++q) PUSH(GAP, s1[q], GAP);
        for (int32_t q = 0; q < k; ++q) PUSH(GAP, GAP, s2[q]);
      }
      for (size_t r = nrev; r-- > 0;) PUSH(rev[3 * r], rev[3 * r + 1], rev[3 * r + 2]);
      if (mode == TO_SEMIGLOBAL) {
        for (int32_t q = ei; q < a; ++q) PUSH(s0[q], GAP, GAP);
        for (int32_t q = ej; q < b; ++q) PUSH(GAP, s1[q], GAP);
        for (int32_t q = ek; q < c; ++q) PUSH(GAP, GAP, s2[q]);
      }
#undef PUSH
      out->row_len = (int32_t)len;
    }
    free(rev);
  }
  free(V);
  return rc;
}

/* Score of given rows under SPEC-AFFINE.md's column rule: columns [lo, hi)
 * are the aligned span (the rest is a free prefix / suffix). */
int32_t to_affine_rescore(const char* r0, const char* r1, const char* r2, int32_t lo, int32_t hi, to_scheme s,
                          int32_t open) {
  int32_t sum = 0;
  int prev = 7; /* virtual all-residue column */
  for (int32_t x = lo; x < hi; ++x) {
    const int m = (r0[x] != GAP) | ((r1[x] != GAP) << 1) | ((r2[x] != GAP) << 2);
    if (!m) return NEGV; /* an all-gap column is malformed */
    int t = 1;
    while (kMask[t] != m) ++t;
    int tp = 1;
    while (kMask[tp] != prev) ++tp;
    sum += to_sop(r0[x], r1[x], r2[x], s) + n_open(tp, t) * open;
    prev = m;
  }
  return sum;
}
