/*
 * trio_oracle.h — CPU restatement of the reference `trioalign` algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 kernels:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it.  The product library (paper_2605_28400_b200/) never links
 * or calls it and fails loudly when its CUDA path is unavailable.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).  Parity of this restatement is pinned by
 * tests/test_oracle_golden.py against fixtures produced by the reference
 * itself (oracle/_ref, built from the reference sources by oracle/Makefile).
 */
#ifndef TRIO_ORACLE_H
#define TRIO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TO_GLOBAL = 0, TO_SEMIGLOBAL = 1, TO_LOCAL = 2 };

enum {
  TO_OK = 0,
  TO_ERR_CAPACITY = 2,
  TO_ERR_LOGIC = 8,
  TO_ERR_NOMEM = 10,
};

typedef struct {
  int32_t match, mismatch, gap;
} to_scheme;

typedef struct {
  int32_t score;
  int32_t end_i, end_j, end_k;
  int32_t begin_i, begin_j, begin_k;
  int32_t row_len; /* length of each gapped row (rows written when non-NULL) */
} to_result;

/* sigma / sop: core.hpp:36-46 */
int32_t to_sigma(char x, char y, to_scheme s);
int32_t to_sop(char x, char y, char z, to_scheme s);

/* fill_tensor: oracle.cpp:11-65.  `m` holds (a+1)(b+1)(c+1) int32 cells,
 * row-major over (i, j, k) (oracle.hpp:15-24). */
void to_fill_tensor(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2,
                    int32_t c, to_scheme s, int mode, int32_t* m);

/* optimal_score: oracle.cpp:67-88 (ties -> lexicographically smallest). */
void to_optimal_score(const int32_t* m, int32_t a, int32_t b, int32_t c, int mode,
                      int32_t* score, int32_t* ei, int32_t* ej, int32_t* ek);

/* oracle_align: oracle.cpp:182-190 (+ traceback oracle.cpp:98-180 when
 * rows != NULL; each row buffer must hold a+b+c+1 bytes).  Returns TO_OK,
 * TO_ERR_CAPACITY when (a+1)(b+1)(c+1) > cell_budget (oracle.cpp:16-20),
 * TO_ERR_LOGIC when no predecessor reproduces a cell (oracle.cpp:145-149). */
int to_oracle_align(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2,
                    int32_t c, to_scheme s, int mode, uint64_t cell_budget, to_result* out,
                    char* row0, char* row1, char* row2);

/* Batch helper for tests / cpu_baseline: n triplets, sequences given by
 * offsets[3*t+d] .. offsets[3*t+d+1] into `seqs`.  Runs `threads` worker
 * threads over disjoint triplets (the reference run_batch pattern,
 * dispatch.cpp:119-162).  rows may be NULL (score only). */
int to_oracle_batch(const char* seqs, const int64_t* offsets, int64_t n, to_scheme s, int mode,
                    uint64_t cell_budget, int threads, int32_t* scores, int32_t* ends,
                    int32_t* status);

/* CounterRng (rng.hpp:12-43) and generate_dataset (dataset.cpp:121-211),
 * restated.  spec_kind: 0 uniform(min,max) 1 fixed(a,b,c) 2 blocked 3 cycle.
 * For blocked/cycle `lengths`/`nlen` give the list.  Writes sequences into
 * `seqs` (capacity `seq_cap` bytes) and 3n+1 offsets.  Returns total bytes
 * written or -1 on overflow. */
int64_t to_generate(int spec_kind, int32_t p0, int32_t p1, int32_t p2, const int32_t* lengths,
                    int32_t nlen, int32_t count, double mutation_rate, double indel_rate,
                    uint64_t seed, char* seqs, int64_t seq_cap, int64_t* offsets);

uint64_t to_rng_next(uint64_t seed, uint64_t stream, uint64_t counter);

/* Affine-gap 3-way alignment as defined by SPEC-AFFINE.md (the reference has
 * linear gaps only; affine_oracle.c).  open = gap_open <= 0; open = 0 is the
 * reference linear model.  Same result / rows contract as to_oracle_align. */
int to_affine_align(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2, int32_t c,
                    to_scheme s, int32_t open, int mode, uint64_t cell_budget, to_result* out, char* row0,
                    char* row1, char* row2);
/* SPEC-AFFINE.md column rule over columns [lo, hi) of three gapped rows. */
int32_t to_affine_rescore(const char* r0, const char* r1, const char* r2, int32_t lo, int32_t hi, to_scheme s,
                          int32_t open);

#ifdef __cplusplus
}
#endif

#endif
