#include <chrono>
#include <cstdio>
#include <cstdlib>
// Engine entry points over the C-ABI (reference: proj/src/tiled.cpp:8-98,
// proj/src/oracle.cpp:182-190, proj/src/metrics.cpp:11-14).  Every alignment
// is computed by the sm_100a kernels; error classes and messages follow the
// reference so callers (and the CLI's CSV error column) see the same text.
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine_internal.hpp"
#include "trioalign/errors.hpp"
#include "trioalign/metrics.hpp"
#include "trioalign/oracle.hpp"
#include "trioalign/tiled.hpp"
#include "trioalign_capi.h"

namespace trioalign {

void EngineConfig::validate() const {
  if (tile_size < 1 || tile_size > 4096) {
    throw ConfigError("tile size must be in [1, 4096], got " + std::to_string(tile_size));
  }
  if (team_width < 0) throw ConfigError("team width must be >= 0");
  if (team_threads < 1) throw ConfigError("team threads must be >= 1");
  if (cell_budget == 0) throw ConfigError("cell budget must be positive");
}

int32_t derive_team_width(int32_t tile_size, int32_t b, int32_t c) {
  return ta_derive_team_width(tile_size, b, c);
}

int64_t packed_score_bound(const Triplet& t, const ScoringScheme& scheme) {
  const ta_scheme s{scheme.match, scheme.mismatch, scheme.gap, scheme.gap_open};
  return ta_packed_score_bound(int64_t(t.s0.size()), int64_t(t.s1.size()), int64_t(t.s2.size()), &s);
}

bool packed_bound_ok(const Triplet& t, const ScoringScheme& scheme) {
  return packed_score_bound(t, scheme) <= 32767;
}

double tcups(uint64_t cells, double seconds) {
  if (seconds <= 0) throw std::domain_error("tcups: runtime must be positive");
  return double(cells) / (seconds * 1e12);
}

namespace detail {

std::string error_message(int status, const Triplet& t, const EngineConfig& cfg, bool rows_path,
                          uint64_t rows_budget) {
  switch (status) {
    case TA_ERR_CAPACITY:
      if (rows_path) {
        const uint64_t total = uint64_t(t.s0.size() + 1) * uint64_t(t.s1.size() + 1) * uint64_t(t.s2.size() + 1);
        return "tensor of " + std::to_string(total) + " cells exceeds the budget of " +
               std::to_string(rows_budget) + " (triplet '" + t.id + "')";
      }
      return "triplet '" + t.id + "' has " + std::to_string(t.cell_count()) + " cells, over the budget of " +
             std::to_string(cfg.cell_budget);
    case TA_ERR_CONFIG: {
      try {
        cfg.validate();
      } catch (const ConfigError& e) {
        return e.what();
      }
      const int32_t n = cfg.tile_size;
      const int32_t w = cfg.team_width > 0 ? cfg.team_width
                                           : derive_team_width(n, int32_t(t.s1.size()), int32_t(t.s2.size()));
      return "tile grid " + std::to_string(n) + "x" + std::to_string(w) + " cannot cover sequence lengths (" +
             std::to_string(t.s1.size()) + ", " + std::to_string(t.s2.size()) + ")";
    }
    case TA_ERR_PARSE:
      for (const std::string* seq : {&t.s0, &t.s1, &t.s2}) {
        for (char ch : *seq) {
          if (!is_residue(ch)) {
            return "triplet '" + t.id + "': invalid character '" + std::string(1, ch) +
                   "' (alphabet is ACGT, gaps are not allowed in inputs)";
          }
        }
      }
      return "triplet '" + t.id + "': invalid input";
    case TA_ERR_LOGIC:
      return "traceback: no predecessor reproduces a cell value (triplet '" + t.id + "')";
    default:
      return std::string("triplet '") + t.id + "': " + ta_last_error();
  }
}

BatchOut run_engine(const std::vector<const Triplet*>& ts, const ScoringScheme& scheme, AlignmentMode mode,
                    const EngineConfig& cfg, bool rows, uint64_t rows_budget, int device) {
  const size_t n = ts.size();
  BatchOut out;
  out.score.assign(n, 0);
  out.end.assign(3 * n, 0);
  out.status.assign(n, 0);
  std::string seqs;
  std::vector<int64_t> offs;
  offs.reserve(3 * n + 1);
  size_t total = 0;
  for (const Triplet* t : ts) total += t->s0.size() + t->s1.size() + t->s2.size();
  seqs.reserve(total + 1);
  for (const Triplet* t : ts) {
    for (const std::string* s : {&t->s0, &t->s1, &t->s2}) {
      offs.push_back(int64_t(seqs.size()));
      seqs += *s;
    }
  }
  offs.push_back(int64_t(seqs.size()));
  const ta_scheme sch{scheme.match, scheme.mismatch, scheme.gap, scheme.gap_open};
  ta_options opt{};
  opt.mode = int32_t(mode);
  opt.with_rows = rows ? 1 : 0;
  opt.tile_size = cfg.tile_size;
  opt.team_width = cfg.team_width;
  opt.team_threads = cfg.team_threads;
  opt.lane_mode = cfg.lane_mode == LaneMode::PackedDual16 ? 1 : 0;
  opt.cell_budget = rows ? rows_budget : cfg.cell_budget;
  opt.gap_model = cfg.gap_model;
  ta_results res{};
  res.scores = out.score.data();
  res.ends = out.end.data();
  res.status = out.status.data();
  std::vector<int64_t> row_off;
  if (rows) {
    out.begin.assign(3 * n, 0);
    out.row_len.assign(n, 0);
    row_off.resize(n);
    int64_t cap = 0;
    for (size_t t = 0; t < n; ++t) {
      row_off[t] = cap;
      cap += int64_t(ts[t]->s0.size() + ts[t]->s1.size() + ts[t]->s2.size());
    }
    for (auto& r : out.rows) r.assign(size_t(cap) + 1, '\0');
    out.row_off = row_off;
    res.begins = out.begin.data();
    res.rows0 = out.rows[0].data();
    res.rows1 = out.rows[1].data();
    res.rows2 = out.rows[2].data();
    res.row_offsets = out.row_off.data();
    res.row_lens = out.row_len.data();
  }
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = ta_align_batch(device, seqs.data(), offs.data(), int64_t(n), &sch, &opt, &res, nullptr);
  if (std::getenv("TA_PROFILE_CLI"))
    std::fprintf(stderr, "[engine] ta_align_batch %.1f ms (%zu triplets)\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), n);
  if (rc != TA_OK) throw_status(rc, ta_last_error());
  return out;
}

}  // namespace detail

AlignmentResult align(const Triplet& t, const ScoringScheme& scheme, AlignmentMode mode,
                      const EngineConfig& cfg) {
  cfg.validate();
  const detail::BatchOut out = detail::run_engine({&t}, scheme, mode, cfg, false, 0, cfg.device);
  if (out.status[0] != TA_OK) throw_status(out.status[0], detail::error_message(out.status[0], t, cfg, false, 0));
  AlignmentResult r;
  r.score = out.score[0];
  r.mode = mode;
  r.end = Coords{out.end[0], out.end[1], out.end[2]};
  return r;
}

std::pair<AlignmentResult, AlignmentResult> align_packed(const Triplet& t1, const Triplet& t2,
                                                         const ScoringScheme& scheme, AlignmentMode mode,
                                                         const EngineConfig& cfg) {
  if (t1.s0.size() != t2.s0.size() || t1.s1.size() != t2.s1.size() || t1.s2.size() != t2.s2.size()) {
    throw ShapeMismatchError("packed alignment requires identical sequence lengths ('" + t1.id + "' vs '" +
                             t2.id + "')");
  }
  const int64_t bound = packed_score_bound(t1, scheme);
  if (bound > 32767) {
    throw LaneOverflowError("score bound " + std::to_string(bound) + " does not fit a signed 16-bit lane");
  }
  cfg.validate();
  const detail::BatchOut out = detail::run_engine({&t1, &t2}, scheme, mode, cfg, false, 0, cfg.device);
  AlignmentResult r[2];
  const Triplet* ts[2] = {&t1, &t2};
  for (int x = 0; x < 2; ++x) {
    if (out.status[size_t(x)] != TA_OK)
      throw_status(out.status[size_t(x)], detail::error_message(out.status[size_t(x)], *ts[x], cfg, false, 0));
    r[x].score = out.score[size_t(x)];
    r[x].mode = mode;
    r[x].end = Coords{out.end[size_t(3 * x)], out.end[size_t(3 * x + 1)], out.end[size_t(3 * x + 2)]};
  }
  return {r[0], r[1]};
}

std::vector<RowsOutcome> oracle_align_batch(const std::vector<Triplet>& ts, const ScoringScheme& scheme,
                                            AlignmentMode mode, uint64_t cell_budget, int device) {
  std::vector<RowsOutcome> outc(ts.size());
  if (ts.empty()) return outc;
  std::vector<const Triplet*> ptrs;
  ptrs.reserve(ts.size());
  for (const auto& t : ts) ptrs.push_back(&t);
  EngineConfig cfg;
  const detail::BatchOut out = detail::run_engine(ptrs, scheme, mode, cfg, true, cell_budget, device);
  for (size_t t = 0; t < ts.size(); ++t) {
    RowsOutcome& o = outc[t];
    if (out.status[t] != TA_OK) {
      o.ok = false;
      o.status = out.status[t];
      o.error = detail::error_message(out.status[t], ts[t], cfg, true, cell_budget);
      continue;
    }
    o.ok = true;
    AlignmentResult& r = o.result;
    r.score = out.score[t];
    r.mode = mode;
    r.end = Coords{out.end[3 * t], out.end[3 * t + 1], out.end[3 * t + 2]};
    r.begin = Coords{out.begin[3 * t], out.begin[3 * t + 1], out.begin[3 * t + 2]};
    r.has_rows = true;
    for (int d = 0; d < 3; ++d) r.rows[size_t(d)].assign(out.rows[size_t(d)].data() + out.row_off[t], size_t(out.row_len[t]));
  }
  return outc;
}

AlignmentResult oracle_align(const Triplet& t, const ScoringScheme& scheme, AlignmentMode mode, bool with_rows,
                             uint64_t cell_budget) {
  const uint64_t total = uint64_t(t.s0.size() + 1) * uint64_t(t.s1.size() + 1) * uint64_t(t.s2.size() + 1);
  if (total > cell_budget) {
    throw CapacityError("tensor of " + std::to_string(total) + " cells exceeds the budget of " +
                        std::to_string(cell_budget) + " (triplet '" + t.id + "')");
  }
  std::vector<RowsOutcome> o = oracle_align_batch({t}, scheme, mode, cell_budget, 0);
  // the reference class of the failure (ParseError for a non-ACGT residue:
  // the GPU engine packs 2-bit codes, so it is stricter than the reference's
  // fill_tensor, which scores any character - INTEGRATION.md)
  if (!o[0].ok) throw_status(o[0].status, o[0].error);
  AlignmentResult r = o[0].result;
  if (!with_rows) {
    r.has_rows = false;
    r.begin = Coords{};
    r.rows = {};
  }
  return r;
}

}  // namespace trioalign
