#pragma once
// Rows-producing alignment (reference: proj/include/trioalign/oracle.hpp:42-43).
// oracle_align keeps its name, budget rule and results, but is computed on the
// GPU (direction cube + walker).  The reference's full-tensor Tensor3 /
// fill_tensor / traceback(Tensor3) are CPU-oracle internals and live only in
// the test oracle (oracle/), not in this product.
#include <cstdint>
#include <string>
#include <vector>

#include "trioalign/core.hpp"

namespace trioalign {

inline constexpr uint64_t kOracleCellBudget = uint64_t{1} << 27;

AlignmentResult oracle_align(const Triplet& t, const ScoringScheme& scheme, AlignmentMode mode,
                             bool with_rows = false, uint64_t cell_budget = kOracleCellBudget);

// Batched form used by the CLI `oracle` subcommand (one GPU call).
struct RowsOutcome {
  bool ok = false;
  AlignmentResult result;
  std::string error;
  int status = 0;  // ta_status of a failure (maps onto the reference exception class)
};
std::vector<RowsOutcome> oracle_align_batch(const std::vector<Triplet>& ts, const ScoringScheme& scheme,
                                            AlignmentMode mode, uint64_t cell_budget = kOracleCellBudget,
                                            int device = 0);

}  // namespace trioalign
