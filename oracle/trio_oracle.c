/*
 * trio_oracle.c — CPU restatement of the reference `trioalign` oracle engine,
 * RNG and dataset generator.  TEST INFRASTRUCTURE ONLY (see trio_oracle.h):
 * the checker for the CUDA path, never part of the product.
 *
 * Parity pinned against the reference itself: tests/golden/ fixtures are
 * produced by oracle/_ref (reference sources compiled by oracle/Makefile) and
 * tests/test_oracle_golden.py checks this file against them.
 */
#include "trio_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define GAP '-'

/* core.hpp:36-41 */
int32_t to_sigma(char x, char y, to_scheme s) {
  const int gx = x == GAP, gy = y == GAP;
  if (gx && gy) return 0;
  if (gx || gy) return s.gap;
  return x == y ? s.match : s.mismatch;
}

/* core.hpp:44-46 */
int32_t to_sop(char x, char y, char z, to_scheme s) {
  return to_sigma(x, y, s) + to_sigma(x, z, s) + to_sigma(y, z, s);
}

static inline size_t idx3(int32_t b, int32_t c, int32_t i, int32_t j, int32_t k) {
  return ((size_t)i * (size_t)(b + 1) + (size_t)j) * (size_t)(c + 1) + (size_t)k;
}

/* oracle.cpp:11-65.  Terms are "present only when in range"; the first
 * present term seeds the max (no sentinel), local floors at 0. */
void to_fill_tensor(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2,
                    int32_t c, to_scheme s, int mode, int32_t* m) {
  const int global = mode == TO_GLOBAL;
  const int local = mode == TO_LOCAL;
  const int32_t g2 = 2 * s.gap;
  for (int32_t i = 0; i <= a; ++i) {
    for (int32_t j = 0; j <= b; ++j) {
      for (int32_t k = 0; k <= c; ++k) {
        const int zeros = (i == 0) + (j == 0) + (k == 0);
        if (zeros == 3) {
          m[idx3(b, c, i, j, k)] = 0;
          continue;
        }
        if (zeros >= 2 && !global) {
          m[idx3(b, c, i, j, k)] = 0;
          continue;
        }
        const char x0 = i ? s0[i - 1] : GAP;
        const char x1 = j ? s1[j - 1] : GAP;
        const char x2 = k ? s2[k - 1] : GAP;
        int have = 0;
        int32_t best = 0, v;
#define CONSIDER(expr)                     \
  do {                                     \
    v = (expr);                            \
    best = have ? (v > best ? v : best) : v; \
    have = 1;                              \
  } while (0)
        if (i && j && k) CONSIDER(m[idx3(b, c, i - 1, j - 1, k - 1)] + to_sop(x0, x1, x2, s));
        if (i && j) CONSIDER(m[idx3(b, c, i - 1, j - 1, k)] + to_sigma(x0, x1, s) + g2);
        if (i && k) CONSIDER(m[idx3(b, c, i - 1, j, k - 1)] + to_sigma(x0, x2, s) + g2);
        if (j && k) CONSIDER(m[idx3(b, c, i, j - 1, k - 1)] + to_sigma(x1, x2, s) + g2);
        if (i) CONSIDER(m[idx3(b, c, i - 1, j, k)] + g2);
        if (j) CONSIDER(m[idx3(b, c, i, j - 1, k)] + g2);
        if (k) CONSIDER(m[idx3(b, c, i, j, k - 1)] + g2);
#undef CONSIDER
        if (local && best < 0) best = 0;
        m[idx3(b, c, i, j, k)] = best;
      }
    }
  }
}

/* oracle.cpp:67-88: strict '>' in a lexicographic scan keeps the smallest
 * (i, j, k) among equal maxima. */
void to_optimal_score(const int32_t* m, int32_t a, int32_t b, int32_t c, int mode,
                      int32_t* score, int32_t* ei, int32_t* ej, int32_t* ek) {
  if (mode == TO_GLOBAL) {
    *score = m[idx3(b, c, a, b, c)];
    *ei = a;
    *ej = b;
    *ek = c;
    return;
  }
  int have = 0;
  int32_t best = 0, bi = 0, bj = 0, bk = 0;
  for (int32_t i = 0; i <= a; ++i) {
    for (int32_t j = 0; j <= b; ++j) {
      for (int32_t k = 0; k <= c; ++k) {
        if (mode == TO_SEMIGLOBAL && i != a && j != b && k != c) continue;
        const int32_t v = m[idx3(b, c, i, j, k)];
        if (!have || v > best) {
          best = v;
          bi = i;
          bj = j;
          bk = k;
          have = 1;
        }
      }
    }
  }
  *score = best;
  *ei = bi;
  *ej = bj;
  *ek = bk;
}

/* traceback: oracle.cpp:98-180. */
static int traceback(const int32_t* m, const char* s0, int32_t a, const char* s1, int32_t b,
                     const char* s2, int32_t c, to_scheme s, int mode, to_result* out,
                     char* row0, char* row1, char* row2) {
  const int32_t g2 = 2 * s.gap;
  int32_t score, ei, ej, ek;
  to_optimal_score(m, a, b, c, mode, &score, &ei, &ej, &ek);
  /* reversed path columns, at most a+b+c of them */
  const size_t cap = (size_t)a + (size_t)b + (size_t)c + 1;
  char* rev = (char*)malloc(3 * cap);
  if (!rev) return TO_ERR_NOMEM;
  size_t nrev = 0;
  int32_t i = ei, j = ej, k = ek;
  for (;;) {
    int stop;
    if (mode == TO_GLOBAL) {
      stop = i == 0 && j == 0 && k == 0;
    } else if (mode == TO_SEMIGLOBAL) {
      stop = (j == 0 && k == 0) || (i == 0 && k == 0) || (i == 0 && j == 0);
    } else {
      stop = m[idx3(b, c, i, j, k)] == 0;
    }
    if (stop) break;
    const int32_t val = m[idx3(b, c, i, j, k)];
    const char x0 = i ? s0[i - 1] : GAP;
    const char x1 = j ? s1[j - 1] : GAP;
    const char x2 = k ? s2[k - 1] : GAP;
    char* col = rev + 3 * nrev;
    if (i && j && k && m[idx3(b, c, i - 1, j - 1, k - 1)] + to_sop(x0, x1, x2, s) == val) {
      col[0] = x0, col[1] = x1, col[2] = x2;
      --i, --j, --k;
    } else if (i && j && m[idx3(b, c, i - 1, j - 1, k)] + to_sigma(x0, x1, s) + g2 == val) {
      col[0] = x0, col[1] = x1, col[2] = GAP;
      --i, --j;
    } else if (i && k && m[idx3(b, c, i - 1, j, k - 1)] + to_sigma(x0, x2, s) + g2 == val) {
      col[0] = x0, col[1] = GAP, col[2] = x2;
      --i, --k;
    } else if (j && k && m[idx3(b, c, i, j - 1, k - 1)] + to_sigma(x1, x2, s) + g2 == val) {
      col[0] = GAP, col[1] = x1, col[2] = x2;
      --j, --k;
    } else if (i && m[idx3(b, c, i - 1, j, k)] + g2 == val) {
      col[0] = x0, col[1] = GAP, col[2] = GAP;
      --i;
    } else if (j && m[idx3(b, c, i, j - 1, k)] + g2 == val) {
      col[0] = GAP, col[1] = x1, col[2] = GAP;
      --j;
    } else if (k && m[idx3(b, c, i, j, k - 1)] + g2 == val) {
      col[0] = GAP, col[1] = GAP, col[2] = x2;
      --k;
    } else {
      free(rev);
      return TO_ERR_LOGIC;
    }
    ++nrev;
  }
  out->score = score;
  out->end_i = ei, out->end_j = ej, out->end_k = ek;
  out->begin_i = i, out->begin_j = j, out->begin_k = k;
  size_t len = 0;
#define PUSH(c0, c1, c2)                                            \
  do {                                                              \
    if (row0) row0[len] = (c0), row1[len] = (c1), row2[len] = (c2); \
    ++len;                                                          \
  } while (0)
  if (mode == TO_SEMIGLOBAL) {
    for (int32_t p = 0; p < i; ++p) PUSH(s0[p], GAP, GAP);
    for (int32_t p = 0; p < j; ++p) PUSH(GAP, s1[p], GAP);
    for (int32_t p = 0; p < k; ++p) PUSH(GAP, GAP, s2[p]);
  }
  for (size_t r = nrev; r-- > 0;) PUSH(rev[3 * r], rev[3 * r + 1], rev[3 * r + 2]);
  if (mode == TO_SEMIGLOBAL) {
    for (int32_t p = ei; p < a; ++p) PUSH(s0[p], GAP, GAP);
    for (int32_t p = ej; p < b; ++p) PUSH(GAP, s1[p], GAP);
    for (int32_t p = ek; p < c; ++p) PUSH(GAP, GAP, s2[p]);
  }
#undef PUSH
  out->row_len = (int32_t)len;
  free(rev);
  return TO_OK;
}

/* oracle.cpp:182-190 */
int to_oracle_align(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2,
                    int32_t c, to_scheme s, int mode, uint64_t cell_budget, to_result* out,
                    char* row0, char* row1, char* row2) {
  const uint64_t total = (uint64_t)(a + 1) * (uint64_t)(b + 1) * (uint64_t)(c + 1);
  memset(out, 0, sizeof(*out));
  if (total > cell_budget) return TO_ERR_CAPACITY;
  int32_t* m = (int32_t*)malloc(total * sizeof(int32_t));
  if (!m) return TO_ERR_NOMEM;
  to_fill_tensor(s0, a, s1, b, s2, c, s, mode, m);
  int rc = TO_OK;
  if (row0) {
    rc = traceback(m, s0, a, s1, b, s2, c, s, mode, out, row0, row1, row2);
  } else {
    to_optimal_score(m, a, b, c, mode, &out->score, &out->end_i, &out->end_j, &out->end_k);
  }
  free(m);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* batch helper (threads over disjoint triplets, dispatch.cpp:119-162)      */

typedef struct {
  const char* seqs;
  const int64_t* offsets;
  int64_t n;
  to_scheme s;
  int mode;
  uint64_t budget;
  int32_t *scores, *ends, *status;
  int64_t next; /* shared work counter */
  pthread_mutex_t mu;
} batch_ctx;

static void* batch_worker(void* arg) {
  batch_ctx* ctx = (batch_ctx*)arg;
  for (;;) {
    pthread_mutex_lock(&ctx->mu);
    const int64_t t = ctx->next++;
    pthread_mutex_unlock(&ctx->mu);
    if (t >= ctx->n) break;
    const int64_t* o = ctx->offsets + 3 * t;
    to_result r;
    const int rc = to_oracle_align(ctx->seqs + o[0], (int32_t)(o[1] - o[0]), ctx->seqs + o[1],
                                   (int32_t)(o[2] - o[1]), ctx->seqs + o[2],
                                   (int32_t)(o[3] - o[2]), ctx->s, ctx->mode, ctx->budget, &r,
                                   NULL, NULL, NULL);
    ctx->status[t] = rc;
    ctx->scores[t] = r.score;
    ctx->ends[3 * t] = r.end_i;
    ctx->ends[3 * t + 1] = r.end_j;
    ctx->ends[3 * t + 2] = r.end_k;
  }
  return NULL;
}

int to_oracle_batch(const char* seqs, const int64_t* offsets, int64_t n, to_scheme s, int mode,
                    uint64_t cell_budget, int threads, int32_t* scores, int32_t* ends,
                    int32_t* status) {
  batch_ctx ctx = {seqs, offsets, n, s, mode, cell_budget, scores, ends, status, 0,
                   PTHREAD_MUTEX_INITIALIZER};
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  if (!th) return TO_ERR_NOMEM;
  for (int w = 0; w < threads; ++w) pthread_create(&th[w], NULL, batch_worker, &ctx);
  for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
  free(th);
  return TO_OK;
}

/* ------------------------------------------------------------------------ */
/* CounterRng: rng.hpp:12-43                                                 */

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t key, counter;
} crng;

static inline crng crng_make(uint64_t seed, uint64_t stream) {
  crng r = {mix64(seed ^ 0x9e3779b97f4a7c15ull) ^ mix64(stream ^ 0xbf58476d1ce4e5b9ull), 0};
  return r;
}
static inline uint64_t crng_next(crng* r) { return mix64(r->key + (++r->counter) * 0x9e3779b97f4a7c15ull); }
static inline uint64_t crng_below(crng* r, uint64_t n) {
  if (n == 0) return 0;
  return (uint64_t)(((unsigned __int128)crng_next(r) * n) >> 64);
}
static inline int64_t crng_range(crng* r, int64_t lo, int64_t hi) {
  return lo + (int64_t)crng_below(r, (uint64_t)(hi - lo + 1));
}
static inline double crng_unit(crng* r) { return (double)(crng_next(r) >> 11) * 0x1.0p-53; }
static inline char crng_base(crng* r) { return "ACGT"[crng_below(r, 4)]; }

uint64_t to_rng_next(uint64_t seed, uint64_t stream, uint64_t counter) {
  crng r = crng_make(seed, stream);
  r.counter = counter;
  return crng_next(&r);
}

/* dataset.cpp:45-54 */
static char other_base(char base, uint64_t pick) {
  static const char kBases[] = {'A', 'C', 'G', 'T'};
  for (int q = 0; q < 4; ++q) {
    if (kBases[q] == base) continue;
    if (pick == 0) return kBases[q];
    --pick;
  }
  return 'A';
}

/* generate_dataset: dataset.cpp:121-211 (sequences only; the recorded
 * reference rows are not needed by the hot path). */
int64_t to_generate(int spec_kind, int32_t p0, int32_t p1, int32_t p2, const int32_t* lengths,
                    int32_t nlen, int32_t count, double mutation_rate, double indel_rate,
                    uint64_t seed, char* seqs, int64_t seq_cap, int64_t* offsets) {
  const int independent_fixed = spec_kind == 1 && (p0 != p1 || p1 != p2);
  int64_t pos = 0;
  char* rows[3] = {NULL, NULL, NULL};
  size_t rows_cap = 0;
  for (int32_t idx = 0; idx < count; ++idx) {
    crng rng = crng_make(seed, (uint64_t)idx + 1);
    if (independent_fixed) {
      const int32_t lens[3] = {p0, p1, p2};
      for (int d = 0; d < 3; ++d) {
        offsets[3 * idx + d] = pos;
        if (pos + lens[d] > seq_cap) return -1;
        for (int32_t p = 0; p < lens[d]; ++p) seqs[pos++] = crng_base(&rng);
      }
      offsets[3 * idx + 3] = pos;
      continue;
    }
    int32_t len = 0;
    switch (spec_kind) {
      case 0: len = (int32_t)crng_range(&rng, p0, p1); break;
      case 2: {
        const size_t groups = (size_t)nlen;
        size_t group = (size_t)idx * groups / (size_t)count;
        if (group > groups - 1) group = groups - 1;
        len = lengths[group];
        break;
      }
      case 3: len = lengths[(size_t)idx % (size_t)nlen]; break;
      case 1: len = p0; break;
    }
    char* anc = (char*)malloc((size_t)len + 1);
    for (int32_t q = 0; q < len; ++q) anc[q] = crng_base(&rng);
    /* a row grows by at most 4 columns per site */
    const size_t need = 4 * (size_t)len + 4;
    if (need > rows_cap) {
      for (int d = 0; d < 3; ++d) rows[d] = (char*)realloc(rows[d], need);
      rows_cap = need;
    }
    size_t rlen = 0;
    for (int32_t site = 0; site < len; ++site) {
      char col[3] = {anc[site], anc[site], anc[site]};
      for (int d = 0; d < 3; ++d) {
        if (mutation_rate > 0 && crng_unit(&rng) < mutation_rate) {
          col[d] = other_base(col[d], crng_below(&rng, 3));
        }
      }
      char inserts[3][3];
      int insert_count = 0;
      for (int d = 0; d < 3; ++d) {
        if (indel_rate > 0 && crng_unit(&rng) < indel_rate) {
          if (crng_below(&rng, 2) == 0) {
            col[d] = GAP;
          } else {
            inserts[insert_count][0] = inserts[insert_count][1] = inserts[insert_count][2] = GAP;
            inserts[insert_count][d] = crng_base(&rng);
            ++insert_count;
          }
        }
      }
      if (col[0] != GAP || col[1] != GAP || col[2] != GAP) {
        for (int d = 0; d < 3; ++d) rows[d][rlen] = col[d];
        ++rlen;
      }
      for (int e = 0; e < insert_count; ++e) {
        for (int d = 0; d < 3; ++d) rows[d][rlen] = inserts[e][d];
        ++rlen;
      }
    }
    free(anc);
    for (int d = 0; d < 3; ++d) {
      offsets[3 * idx + d] = pos;
      for (size_t q = 0; q < rlen; ++q) {
        if (rows[d][q] != GAP) {
          if (pos >= seq_cap) return -1;
          seqs[pos++] = rows[d][q];
        }
      }
    }
    offsets[3 * idx + 3] = pos;
  }
  for (int d = 0; d < 3; ++d) free(rows[d]);
  return pos;
}
