/*
 * trioalign_capi.h — the C-ABI drop-in boundary of the B200 `trioalign` engine.
 *
 * The reference (/root/reference/proj) has no FFI layer: its "operator API" is
 * the C++ library (proj/include/trioalign/ headers) and the CLI.  This header is
 * the plain-pointer boundary underneath our reference-compatible C++ API
 * (paper_2605_28400_b200/csrc/include/trioalign/ headers) and the Python/ctypes
 * binding.  Each entry point names the reference interface it replaces.
 *
 * Conventions: all pointers are host pointers unless stated; sizes are int64;
 * no torch or CUDA types appear in signatures (streams are passed as void*).
 * Every function returns a ta_status; on failure ta_last_error() holds a
 * thread-local message.  Status codes map 1:1 onto the reference exception
 * classes (proj/include/trioalign/errors.hpp:9-37 plus std exceptions).
 */
#ifndef TRIOALIGN_CAPI_H
#define TRIOALIGN_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TA_OK = 0,
  TA_ERR_PARSE = 1,            /* trioalign::ParseError            errors.hpp:9   */
  TA_ERR_CAPACITY = 2,         /* trioalign::CapacityError         errors.hpp:14  */
  TA_ERR_CONFIG = 3,           /* trioalign::ConfigError           errors.hpp:20  */
  TA_ERR_SHAPE_MISMATCH = 4,   /* trioalign::ShapeMismatchError    errors.hpp:25  */
  TA_ERR_LANE_OVERFLOW = 5,    /* trioalign::LaneOverflowError     errors.hpp:30  */
  TA_ERR_MALFORMED = 6,        /* trioalign::MalformedAlignmentError errors.hpp:35 */
  TA_ERR_INVALID_ARGUMENT = 7, /* std::invalid_argument (ScoringScheme::validate, core.cpp:10-18) */
  TA_ERR_LOGIC = 8,            /* std::logic_error (pipeline / traceback invariants) */
  TA_ERR_CUDA = 9,             /* device / driver failure (no reference analogue) */
  TA_ERR_NOMEM = 10,           /* host or device allocation failure */
  TA_ERR_OTHER = 11
} ta_status;

typedef enum { TA_GLOBAL = 0, TA_SEMIGLOBAL = 1, TA_LOCAL = 2 } ta_mode; /* core.hpp:48 */

/* ScoringScheme (core.hpp:24-31): match > 0, mismatch <= 0, gap <= 0, |x| <= 1024.
 * gap_open (<= 0) is NOT in the reference (linear gaps only):
 * it selects the affine model of SPEC-AFFINE.md; 0 = the reference model. */
typedef struct {
  int32_t match;
  int32_t mismatch;
  int32_t gap;
  int32_t gap_open;
} ta_scheme;

/* Engine knobs.  tile_size / team_width / team_threads mirror EngineConfig
 * (tiled.hpp:18-30) and are validated with the same ConfigError rules
 * (tiled.cpp:8-15, 37-58) so error behaviour is identical; the GPU tile
 * geometry itself is chosen per length bucket and never changes results.
 * cell_budget: score path caps a*b*c (tiled.cpp:39-43); the rows path caps
 * (a+1)(b+1)(c+1) (oracle.cpp:16-20). */
typedef struct {
  int32_t mode;          /* ta_mode */
  int32_t with_rows;     /* 1: traceback rows + begin coords (oracle_align(with_rows)) */
  int32_t tile_size;     /* EngineConfig::tile_size, must be in [1, 4096] */
  int32_t team_width;    /* EngineConfig::team_width, 0 = derive */
  int32_t team_threads;  /* EngineConfig::team_threads, >= 1 */
  int32_t lane_mode;     /* 0 Single32, 1 PackedDual16 (results identical; GPU picks lanes) */
  uint64_t cell_budget;
  int32_t gap_model;     /* 0: affine kernels iff gap_open != 0; 1: always the affine kernels
                            (with gap_open = 0 they reproduce the linear results) */
} ta_options;

/* Per-triplet results, caller-allocated, n entries each (ends/begins: 3n). */
typedef struct {
  int32_t* scores;
  int32_t* ends;    /* (i, j, k) per triplet */
  int32_t* begins;  /* (i, j, k) per triplet; rows path only (may be NULL) */
  int32_t* status;  /* ta_status per triplet (batch never aborts on one failure) */
  /* rows path only: three gapped rows per triplet written at row_offsets[t]
   * into rows0/rows1/rows2, capacity a+b+c bytes each; lengths in row_lens. */
  char* rows0;
  char* rows1;
  char* rows2;
  const int64_t* row_offsets;
  int32_t* row_lens;
} ta_results;

typedef struct {
  double kernel_ms;        /* device time of the last run (CUDA events, launch stream) */
  double wavefront_ms;     /* of which the DP wavefront kernel(s) */
  int64_t cells;           /* sum a*b*c of successfully aligned triplets */
  int64_t launches;        /* kernels launched by the last run */
  int64_t padded_cells;    /* cells actually swept incl. tile padding */
  int32_t lanes;           /* 1 = int32 lanes, 2 = packed s16x2 lanes */
  int32_t buckets;         /* tile-grid length buckets used */
  int32_t reserved;
  double walker_ms;        /* rows path: of kernel_ms, the traceback walkers */
  int64_t dir_bytes;       /* rows path: direction-record bytes written by the wavefront */
} ta_stats;

/* ---- library / device ---------------------------------------------------- */
const char* ta_last_error(void);
const char* ta_version(void);
int ta_device_count(int* count);

/* ---- one-shot batch: the body of run_batch / align / oracle_align --------
 * Replaces: trioalign::run_batch (dispatch.hpp:58-59) per worker,
 *           trioalign::align (tiled.hpp:34-35) for n = 1,
 *           trioalign::oracle_align(with_rows) (oracle.hpp:42-43).
 * seqs: concatenated ASCII residues; offsets: 3n+1 entries, triplet t has
 * s0 = seqs[offsets[3t] .. offsets[3t+1]), s1 = [3t+1 .. 3t+2), s2 = [3t+2 .. 3t+3).
 * Host buffers in, host buffers out; H2D / D2H happen inside.  stream may be
 * NULL (library stream). */
int ta_align_batch(int device, const char* seqs, const int64_t* offsets, int64_t n,
                   const ta_scheme* scheme, const ta_options* opt, ta_results* out,
                   void* stream);

/* ---- device-resident batch (bench / pipelined callers) -------------------
 * create: validates + uploads + 2-bit packs on device (inputs then live in HBM);
 * run:    kernels only (results stay on device);
 * fetch:  D2H of per-triplet results. */
typedef struct ta_batch ta_batch;
int ta_batch_create(int device, const char* seqs, const int64_t* offsets, int64_t n,
                    ta_batch** out, void* stream);
int ta_batch_run(ta_batch* b, const ta_scheme* scheme, const ta_options* opt, void* stream);
int ta_batch_fetch(ta_batch* b, ta_results* out, void* stream);
int ta_batch_stats(const ta_batch* b, ta_stats* out);
/* statistics of the last ta_align_batch call on a device (its internal batch) */
int ta_last_stats(int device, ta_stats* out);
void ta_batch_destroy(ta_batch* b);

/* ---- host-side helpers with reference semantics (no GPU needed) ---------- */
/* packed_score_bound / packed_bound_ok (tiled.cpp:23-33) */
int64_t ta_packed_score_bound(int64_t a, int64_t b, int64_t c, const ta_scheme* scheme);
/* derive_team_width (tiled.cpp:17-21) */
int32_t ta_derive_team_width(int32_t tile_size, int32_t b, int32_t c);
/* ScoringScheme::validate (core.cpp:10-18): TA_OK or TA_ERR_INVALID_ARGUMENT */
int ta_validate_scheme(const ta_scheme* scheme);
/* EngineConfig::validate (tiled.cpp:8-15): TA_OK or TA_ERR_CONFIG */
int ta_validate_options(const ta_options* opt);
/* plan_partition (dispatch.cpp:29-60): strategy 0 blocked, 1 interleaved,
 * 2 dynamic; assignment receives n worker indices. */
int ta_plan_partition(const uint64_t* cell_counts, int64_t n, int32_t strategy,
                      int32_t workers, int32_t* assignment);

/* ---- seeded synthetic datasets (support for `generate` / `bench --spec`) --
 * generate_dataset (dataset.cpp:121-211) + DatasetSpec::parse (dataset.cpp:87-119),
 * bit-identical, parallel over triplets.  *seqs / *offsets (3n+1) are malloc'd:
 * release with ta_free.  Errors: TA_ERR_PARSE (message via ta_generate_error). */
int ta_generate(const char* spec, double mutation, double indel, uint64_t seed, int threads,
                char** seqs, int64_t** offsets, int64_t* n);
/* Triplets [begin, end) of the same dataset (per-rank shards); end < 0 = all. */
int ta_generate_slice(const char* spec, double mutation, double indel, uint64_t seed,
                      int64_t begin, int64_t end, int threads, char** seqs, int64_t** offsets,
                      int64_t* n);
/* The recorded true alignment rows (generate --ref-out): triplet t's rows are
 * ref[ref_off[t] + d*ref_len[t] ...] for d = 0..2; ref_len[t] < 0 = none. */
int ta_generate_reference(const char* spec, double mutation, double indel, uint64_t seed,
                          char** ref, int64_t** ref_off, int64_t** ref_len, int64_t* n);
const char* ta_generate_error(void);
void ta_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* TRIOALIGN_CAPI_H */
