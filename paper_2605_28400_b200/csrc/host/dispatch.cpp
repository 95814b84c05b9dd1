// Batch dispatch (reference: proj/src/dispatch.cpp:12-162), GPU workers.
//
// plan_partition keeps the reference's pure partition rules.  run_batch keeps
// one host thread per worker (dispatch.cpp:146-153) but a worker is a GPU:
// worker w drives device w mod #devices and submits ALL of its triplets as one
// batched kernel call instead of aligning them one at a time.  Results are
// written in input order; per-triplet failures are recorded, never fatal;
// failed cells are excluded from TCUPS (dispatch.cpp:157-160).
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "engine_internal.hpp"
#include "trioalign/dispatch.hpp"
#include "trioalign/errors.hpp"
#include "trioalign/metrics.hpp"
#include "trioalign_capi.h"

namespace trioalign {

std::string_view strategy_name(Strategy s) {
  switch (s) {
    case Strategy::Blocked: return "blocked";
    case Strategy::Interleaved: return "interleaved";
    case Strategy::Dynamic: return "dynamic";
  }
  return "?";
}

Strategy strategy_from_name(std::string_view name) {
  if (name == "blocked") return Strategy::Blocked;
  if (name == "interleaved") return Strategy::Interleaved;
  if (name == "dynamic") return Strategy::Dynamic;
  throw ParseError("unknown partition strategy '" + std::string(name) +
                   "' (expected blocked, interleaved, or dynamic)");
}

PartitionPlan plan_partition(const std::vector<uint64_t>& cell_counts, Strategy strategy, int32_t worker_count) {
  PartitionPlan plan{strategy, worker_count, std::vector<int32_t>(cell_counts.size(), 0)};
  const int rc = ta_plan_partition(cell_counts.data(), int64_t(cell_counts.size()), int32_t(strategy), worker_count,
                                   plan.assignment.data());
  if (rc != TA_OK) throw_status(rc, ta_last_error());
  return plan;
}

BatchReport run_batch(const std::vector<Triplet>& dataset, const ScoringScheme& scheme, AlignmentMode mode,
                      const EngineConfig& cfg, const PartitionPlan& plan) {
  if (plan.assignment.size() != dataset.size()) {
    throw ConfigError("partition plan covers " + std::to_string(plan.assignment.size()) + " triplets, dataset has " +
                      std::to_string(dataset.size()));
  }
  const int32_t workers = plan.worker_count;
  for (int32_t w : plan.assignment) {
    if (w < 0 || w >= workers) throw ConfigError("partition plan names an out-of-range worker");
  }
  BatchReport report;
  report.per_triplet.resize(dataset.size());
  report.per_worker.resize(size_t(workers));
  std::vector<std::vector<size_t>> by_worker(static_cast<size_t>(workers));
  for (size_t i = 0; i < dataset.size(); ++i) {
    const int32_t w = plan.assignment[i];
    by_worker[size_t(w)].push_back(i);
    report.per_triplet[i].id = dataset[i].id;
    report.per_triplet[i].worker = w;
    report.per_triplet[i].cells = dataset[i].cell_count();
    report.per_worker[size_t(w)].assigned += 1;
    report.per_worker[size_t(w)].cells += dataset[i].cell_count();
  }
  int devices = 0;
  ta_device_count(&devices);
  if (devices < 1) devices = 1;  // the call below then fails loudly (no CPU fallback)

  std::vector<std::exception_ptr> errors(static_cast<size_t>(workers));
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  pool.reserve(size_t(workers));
  for (int32_t w = 0; w < workers; ++w) {
    pool.emplace_back([&, w] {
      const auto w0 = std::chrono::steady_clock::now();
      const auto& idx = by_worker[size_t(w)];
      try {
        if (!idx.empty()) {
          std::vector<const Triplet*> ts;
          ts.reserve(idx.size());
          for (size_t i : idx) ts.push_back(&dataset[i]);
          // configuration errors are per triplet in the reference (make_layout)
          bool cfg_ok = true;
          std::string cfg_err;
          try {
            cfg.validate();
          } catch (const std::exception& e) {
            cfg_ok = false;
            cfg_err = e.what();
          }
          if (!cfg_ok) {
            for (size_t i : idx) report.per_triplet[i].error = cfg_err;
          } else {
            const detail::BatchOut out = detail::run_engine(ts, scheme, mode, cfg, false, 0, w % devices);
            for (size_t x = 0; x < idx.size(); ++x) {
              TripletOutcome& o = report.per_triplet[idx[x]];
              if (out.status[x] == TA_OK) {
                o.ok = true;
                o.score = out.score[x];
                o.end = Coords{out.end[3 * x], out.end[3 * x + 1], out.end[3 * x + 2]};
              } else {
                o.ok = false;
                o.error = detail::error_message(out.status[x], *ts[x], cfg, false, 0);
              }
            }
          }
        }
      } catch (...) {
        errors[size_t(w)] = std::current_exception();
      }
      report.per_worker[size_t(w)].seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    });
  }
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);  // device failure: no silent fallback
  report.wall_seconds = std::chrono::duration<double>(t1 - t0).count();
  for (const auto& o : report.per_triplet)
    if (o.ok) report.scored_cells += o.cells;
  report.tcups = report.wall_seconds > 0 ? tcups(report.scored_cells, report.wall_seconds) : 0.0;
  return report;
}

}  // namespace trioalign
