// Force-included ahead of the UNMODIFIED reference proj/src/dispatch.cpp when
// oracle/Makefile builds oracle/_ref.  dispatch.cpp:134 reads
//   std::vector<std::vector<size_t>> by_worker(size_t(workers));
// which g++ 13 parses as a function declaration (most vexing parse, SURVEY
// §0.5).  Every header dispatch.cpp includes is pulled in first (include
// guards make its own #includes no-ops), then `size_t(x)` is turned into an
// explicit cast expression for the rest of that one translation unit only.
#pragma once
#include <chrono>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "trioalign/dispatch.hpp"
#include "trioalign/errors.hpp"
#include "trioalign/metrics.hpp"

#define size_t(x) (static_cast<std::size_t>(x))
