// ref_driver.cpp — extern "C" entry points over the UNMODIFIED reference
// sources (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libtrioref.so.
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY.  It lets the Python tests generate
// golden fixtures from the reference itself and lets bench.py time the
// reference's own CPU path (run_batch over the tiled engine,
// dispatch.cpp:119-162) on the GPU box's host cores.  Nothing in the product
// (paper_2605_28400_b200/) links or loads it.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "trioalign/core.hpp"
#include "trioalign/dataset.hpp"
#include "trioalign/dispatch.hpp"
#include "trioalign/errors.hpp"
#include "trioalign/oracle.hpp"
#include "trioalign/tiled.hpp"

using namespace trioalign;

namespace {

thread_local std::string g_err;

// status codes shared with include/trioalign_capi.h
int classify(const std::exception& e) {
  if (dynamic_cast<const ParseError*>(&e)) return 1;
  if (dynamic_cast<const CapacityError*>(&e)) return 2;
  if (dynamic_cast<const ConfigError*>(&e)) return 3;
  if (dynamic_cast<const ShapeMismatchError*>(&e)) return 4;
  if (dynamic_cast<const LaneOverflowError*>(&e)) return 5;
  if (dynamic_cast<const MalformedAlignmentError*>(&e)) return 6;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 7;
  if (dynamic_cast<const std::logic_error*>(&e)) return 8;
  return 11;
}

std::vector<Triplet> to_triplets(const char* seqs, const int64_t* off, int64_t n) {
  std::vector<Triplet> out(static_cast<size_t>(n));
  for (int64_t t = 0; t < n; ++t) {
    out[t].id = "t" + std::to_string(t);
    out[t].s0.assign(seqs + off[3 * t], seqs + off[3 * t + 1]);
    out[t].s1.assign(seqs + off[3 * t + 1], seqs + off[3 * t + 2]);
    out[t].s2.assign(seqs + off[3 * t + 2], seqs + off[3 * t + 3]);
  }
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

// generate_dataset (dataset.cpp:121-211) for a CLI-grammar spec.  Returns the
// triplet count (>= 0) or -status on error; *seqs/*offsets are malloc'd
// (3n+1 offsets).
int64_t ref_generate(const char* spec, double mutation, double indel, uint64_t seed,
                     char** seqs_out, int64_t** offsets_out) {
  try {
    DatasetSpec sp = DatasetSpec::parse(spec);
    sp.mutation_rate = mutation;
    sp.indel_rate = indel;
    sp.seed = seed;
    sp.validate();
    const GeneratedDataset data = generate_dataset(sp);
    size_t total = 0;
    for (const auto& t : data.triplets) total += t.s0.size() + t.s1.size() + t.s2.size();
    char* seqs = static_cast<char*>(std::malloc(total + 1));
    int64_t* off = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (3 * data.triplets.size() + 1)));
    size_t pos = 0;
    for (size_t t = 0; t < data.triplets.size(); ++t) {
      const std::string* s[3] = {&data.triplets[t].s0, &data.triplets[t].s1, &data.triplets[t].s2};
      for (int d = 0; d < 3; ++d) {
        off[3 * t + d] = int64_t(pos);
        std::memcpy(seqs + pos, s[d]->data(), s[d]->size());
        pos += s[d]->size();
      }
    }
    off[3 * data.triplets.size()] = int64_t(pos);
    *seqs_out = seqs;
    *offsets_out = off;
    return int64_t(data.triplets.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -classify(e);
  }
}

// The reference batch path: plan_partition + run_batch (dispatch.cpp:29-162)
// over the tiled engine.  strategy 0 blocked / 1 interleaved / 2 dynamic.
// Per-triplet status 0 = ok, else the reference error class (message dropped).
int ref_run_batch(const char* seqs, const int64_t* offsets, int64_t n, int32_t match,
                  int32_t mismatch, int32_t gap, int mode, int32_t tile_size, int32_t workers,
                  int strategy, int packed, uint64_t cell_budget, int32_t* scores, int32_t* ends,
                  int32_t* status, double* wall_seconds) {
  try {
    const std::vector<Triplet> data = to_triplets(seqs, offsets, n);
    std::vector<uint64_t> cells;
    cells.reserve(data.size());
    for (const auto& t : data) cells.push_back(t.cell_count());
    const PartitionPlan plan = plan_partition(cells, Strategy(strategy), workers);
    EngineConfig cfg;
    cfg.tile_size = tile_size;
    cfg.lane_mode = packed ? LaneMode::PackedDual16 : LaneMode::Single32;
    cfg.cell_budget = cell_budget;
    const ScoringScheme scheme = make_scheme(match, mismatch, gap);
    const BatchReport rep = run_batch(data, scheme, AlignmentMode(mode), cfg, plan);
    for (int64_t t = 0; t < n; ++t) {
      const auto& o = rep.per_triplet[size_t(t)];
      scores[t] = o.ok ? o.score : 0;
      ends[3 * t] = o.end.i;
      ends[3 * t + 1] = o.end.j;
      ends[3 * t + 2] = o.end.k;
      status[t] = o.ok ? 0 : (o.error.find("budget") != std::string::npos ? 2 : 11);
    }
    *wall_seconds = rep.wall_seconds;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Single-triplet tiled engine call (tiled.cpp:62-71).
int ref_align(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2, int32_t c,
              int32_t match, int32_t mismatch, int32_t gap, int mode, int32_t tile_size,
              int32_t team_threads, uint64_t cell_budget, int32_t* score, int32_t* end) {
  try {
    Triplet t{"t", std::string(s0, size_t(a)), std::string(s1, size_t(b)), std::string(s2, size_t(c))};
    EngineConfig cfg;
    cfg.tile_size = tile_size;
    cfg.team_threads = team_threads;
    cfg.cell_budget = cell_budget;
    const AlignmentResult r = align(t, make_scheme(match, mismatch, gap), AlignmentMode(mode), cfg);
    *score = r.score;
    end[0] = r.end.i;
    end[1] = r.end.j;
    end[2] = r.end.k;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// oracle_align with rows (oracle.cpp:182-190).  rows must hold a+b+c+1 bytes
// each; res = {score, end i,j,k, begin i,j,k, row_len}.
int ref_oracle_align(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2,
                     int32_t c, int32_t match, int32_t mismatch, int32_t gap, int mode,
                     int with_rows, uint64_t cell_budget, int32_t* res, char* row0, char* row1,
                     char* row2) {
  try {
    Triplet t{"t", std::string(s0, size_t(a)), std::string(s1, size_t(b)), std::string(s2, size_t(c))};
    const AlignmentResult r = oracle_align(t, make_scheme(match, mismatch, gap),
                                           AlignmentMode(mode), with_rows != 0, cell_budget);
    res[0] = r.score;
    res[1] = r.end.i;
    res[2] = r.end.j;
    res[3] = r.end.k;
    res[4] = r.begin.i;
    res[5] = r.begin.j;
    res[6] = r.begin.k;
    res[7] = int32_t(r.rows[0].size());
    if (with_rows) {
      std::memcpy(row0, r.rows[0].data(), r.rows[0].size());
      std::memcpy(row1, r.rows[1].data(), r.rows[1].size());
      std::memcpy(row2, r.rows[2].data(), r.rows[2].size());
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

int ref_packed_bound_ok(const char* s0, int32_t a, const char* s1, int32_t b, const char* s2,
                        int32_t c, int32_t match, int32_t mismatch, int32_t gap) {
  Triplet t{"t", std::string(s0, size_t(a)), std::string(s1, size_t(b)), std::string(s2, size_t(c))};
  return packed_bound_ok(t, ScoringScheme{match, mismatch, gap}) ? 1 : 0;
}

}  // extern "C"
