#pragma once
// Command-line entry point (reference: proj/include/trioalign/cli.hpp:10-15).
// Exit codes: 0 success, 1 usage/other, 2 parse/malformed, 3 capacity.
#include <cstdint>
#include <string>
#include <vector>

namespace trioalign {

int cli_main(std::vector<std::string> args);
int32_t auto_tile_size();

}  // namespace trioalign
