#pragma once
// Engine entry points (reference: proj/include/trioalign/tiled.hpp:18-50).
// The reference's CPU tile machinery (TileState, tile_step, run_team, lanes::*)
// is replaced by the sm_100a wavefront kernels behind the C-ABI; the public
// contract - results, errors, knobs - is unchanged.
#include <cstdint>
#include <utility>

#include "trioalign/core.hpp"
#include "trioalign/errors.hpp"

namespace trioalign {

enum class LaneMode { Single32, PackedDual16 };

struct EngineConfig {
  int32_t tile_size = 8;                     // N (validated; GPU geometry is per bucket)
  int32_t team_width = 0;                    // 0 = derive; forced width must cover (ConfigError)
  LaneMode lane_mode = LaneMode::Single32;   // results identical either way
  uint64_t cell_budget = uint64_t{1} << 31;  // max a*b*c per triplet (CapacityError)
  int32_t team_threads = 1;
  int32_t device = 0;                        // CUDA device (B200 extension)
  int32_t gap_model = 0;                     // 1: always the affine kernels (B200 extension)
  void validate() const;                     // ConfigError (tiled.cpp:8-15)
};

AlignmentResult align(const Triplet& t, const ScoringScheme& scheme, AlignmentMode mode,
                      const EngineConfig& cfg);

std::pair<AlignmentResult, AlignmentResult> align_packed(const Triplet& t1, const Triplet& t2,
                                                         const ScoringScheme& scheme,
                                                         AlignmentMode mode,
                                                         const EngineConfig& cfg);

int64_t packed_score_bound(const Triplet& t, const ScoringScheme& scheme);
bool packed_bound_ok(const Triplet& t, const ScoringScheme& scheme);
int32_t derive_team_width(int32_t tile_size, int32_t b, int32_t c);

}  // namespace trioalign
