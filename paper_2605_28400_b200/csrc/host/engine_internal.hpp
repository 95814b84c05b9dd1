#pragma once
// Shared glue between the C++ API and the C-ABI.
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "trioalign/core.hpp"
#include "trioalign/tiled.hpp"

namespace trioalign::detail {

struct BatchOut {
  std::vector<int32_t> score, end, status, begin, row_len;
  std::vector<int64_t> row_off;
  std::array<std::string, 3> rows;
};

BatchOut run_engine(const std::vector<const Triplet*>& ts, const ScoringScheme& scheme, AlignmentMode mode,
                    const EngineConfig& cfg, bool rows, uint64_t rows_budget, int device);

std::string error_message(int status, const Triplet& t, const EngineConfig& cfg, bool rows_path,
                          uint64_t rows_budget);

}  // namespace trioalign::detail
