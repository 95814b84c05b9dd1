// Re-hosts the reference's public-API test cases (proj/tests/test_tiled.cpp,
// test_oracle.cpp, test_dispatch.cpp) against the B200 library
// (paper_2605_28400_b200/libtrioalign.so), with the C oracle
// (oracle/trio_oracle.c) as the independent checker.  Built and run by
// tests/test_cpp_api.py (-m gpu).
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>
#include <vector>

#include "../../oracle/trio_oracle.h"
#include "trioalign/dataset.hpp"
#include "trioalign/dispatch.hpp"
#include "trioalign/errors.hpp"
#include "trioalign/oracle.hpp"
#include "trioalign/tiled.hpp"

using namespace trioalign;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::fprintf(stderr, "%s:%d: FAILED: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, type)        \
  do {                                     \
    bool ok_ = false;                      \
    try {                                  \
      (void)(expr);                        \
    } catch (const type&) {                \
      ok_ = true;                          \
    } catch (...) {                        \
    }                                      \
    CHECK(ok_ && #type);                   \
  } while (0)

namespace {

struct Rng {  // rng.hpp CounterRng (stream-compatible) for corpora
  uint64_t key, counter = 0;
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  Rng(uint64_t seed, uint64_t stream) : key(mix(seed ^ 0x9e3779b97f4a7c15ull) ^ mix(stream ^ 0xbf58476d1ce4e5b9ull)) {}
  uint64_t next() { return mix(key + (++counter) * 0x9e3779b97f4a7c15ull); }
  uint64_t below(uint64_t n) { return n ? uint64_t((static_cast<unsigned __int128>(next()) * n) >> 64) : 0; }
  char base() { return "ACGT"[below(4)]; }
};

Triplet random_triplet(Rng& rng, int max_len) {
  Triplet t;
  t.id = "r";
  for (auto* s : {&t.s0, &t.s1, &t.s2}) {
    const int len = int(rng.below(uint64_t(max_len) + 1));
    for (int p = 0; p < len; ++p) s->push_back(rng.base());
  }
  return t;
}

to_result oracle(const Triplet& t, const ScoringScheme& s, AlignmentMode m, bool rows, std::string out[3]) {
  to_result r{};
  std::vector<char> b0(t.s0.size() + t.s1.size() + t.s2.size() + 1), b1(b0.size()), b2(b0.size());
  to_oracle_align(t.s0.data(), int(t.s0.size()), t.s1.data(), int(t.s1.size()), t.s2.data(), int(t.s2.size()),
                  to_scheme{s.match, s.mismatch, s.gap}, int(m), uint64_t(1) << 40, &r, rows ? b0.data() : nullptr,
                  rows ? b1.data() : nullptr, rows ? b2.data() : nullptr);
  if (rows) {
    out[0].assign(b0.data(), size_t(r.row_len));
    out[1].assign(b1.data(), size_t(r.row_len));
    out[2].assign(b2.data(), size_t(r.row_len));
  }
  return r;
}

EngineConfig cfg_with(int n, int threads = 1) {
  EngineConfig c;
  c.tile_size = n;
  c.team_threads = threads;
  return c;
}

const AlignmentMode kModes[] = {AlignmentMode::Global, AlignmentMode::SemiGlobal, AlignmentMode::Local};

}  // namespace

int main() {
  const ScoringScheme kScheme{1, -1, -2};
  // test_tiled.cpp:97-110
  {
    const AlignmentResult r = align(Triplet{"id", "ACG", "ACG", "ACG"}, ScoringScheme{2, -1, -2},
                                    AlignmentMode::Global, cfg_with(2));
    CHECK(r.score == 18);
    CHECK((r.end == Coords{3, 3, 3}));
    for (auto m : kModes) CHECK(align(Triplet{"e", "", "", ""}, kScheme, m, cfg_with(4)).score == 0);
  }
  // test_tiled.cpp:112-132: engine == oracle on a random corpus (score + end)
  {
    Rng rng(314159, 1);
    for (int rep = 0; rep < 40; ++rep) {
      const Triplet t = random_triplet(rng, 24);
      const ScoringScheme sch{int32_t(1 + rng.below(5)), -int32_t(rng.below(6)), -int32_t(rng.below(6))};
      for (auto m : kModes) {
        std::string rows[3];
        const to_result want = oracle(t, sch, m, false, rows);
        for (int n : {1, 2, 3, 4, 8}) {
          const AlignmentResult got = align(t, sch, m, cfg_with(n));
          CHECK(got.score == want.score);
          CHECK((got.end == Coords{want.end_i, want.end_j, want.end_k}));
        }
      }
    }
  }
  // test_tiled.cpp:134-149: invariance across tile size and team threads
  {
    Rng rng(777, 2);
    for (int rep = 0; rep < 6; ++rep) {
      const Triplet t = random_triplet(rng, 32);
      for (auto m : kModes) {
        const AlignmentResult base = align(t, kScheme, m, cfg_with(4));
        for (int n : {1, 2, 5, 8, 16, 64})
          for (int th : {1, 2, 3}) {
            const AlignmentResult r = align(t, kScheme, m, cfg_with(n, th));
            CHECK(r.score == base.score);
            CHECK(r.end == base.end);
          }
      }
    }
  }
  // test_tiled.cpp:203-244: packed == single
  {
    Rng rng(4321, 5);
    for (int rep = 0; rep < 12; ++rep) {
      Triplet t1{"p1", "", "", ""}, t2{"p2", "", "", ""};
      for (auto [a, b] : {std::pair{&t1.s0, &t2.s0}, std::pair{&t1.s1, &t2.s1}, std::pair{&t1.s2, &t2.s2}}) {
        const int len = int(rng.below(25));
        for (int p = 0; p < len; ++p) {
          a->push_back(rng.base());
          b->push_back(rng.base());
        }
      }
      const ScoringScheme sch{int32_t(1 + rng.below(5)), -int32_t(rng.below(6)), -int32_t(rng.below(6))};
      for (auto m : kModes) {
        const auto [r1, r2] = align_packed(t1, t2, sch, m, cfg_with(8));
        const AlignmentResult w1 = align(t1, sch, m, cfg_with(8)), w2 = align(t2, sch, m, cfg_with(8));
        CHECK(r1.score == w1.score && r1.end == w1.end);
        CHECK(r2.score == w2.score && r2.end == w2.end);
      }
    }
  }
  // test_tiled.cpp:246-275: errors
  {
    CHECK_THROWS_AS(align_packed(Triplet{"a", "ACGT", "AC", "G"}, Triplet{"b", "ACG", "AC", "G"}, kScheme,
                                 AlignmentMode::Global, cfg_with(4)),
                    ShapeMismatchError);
    const std::string ls(32, 'A');
    const Triplet big{"big", ls, ls, ls};
    CHECK_THROWS_AS(align_packed(big, big, ScoringScheme{5, -1, -300}, AlignmentMode::Global, cfg_with(4)),
                    LaneOverflowError);
    const Triplet t{"t", "ACGTACGT", "ACGTACGT", "ACGTACGT"};
    EngineConfig tiny = cfg_with(4);
    tiny.cell_budget = 10;
    CHECK_THROWS_AS(align(t, kScheme, AlignmentMode::Global, tiny), CapacityError);
    EngineConfig narrow = cfg_with(2);
    narrow.team_width = 2;
    CHECK_THROWS_AS(align(t, kScheme, AlignmentMode::Global, narrow), ConfigError);
    CHECK_THROWS_AS(cfg_with(0).validate(), ConfigError);
    CHECK(packed_score_bound(Triplet{"t", "ACGT", "ACG", "AC"}, ScoringScheme{1, -1, -300}) == 9 * 600);
  }
  // test_oracle.cpp:195-244: rows (oracle_align with_rows on the GPU)
  {
    const AlignmentResult r = oracle_align(Triplet{"m", "A", "A", "A"}, kScheme, AlignmentMode::Global, true);
    CHECK(r.score == 3 && r.rows[0] == "A" && r.rows[1] == "A" && r.rows[2] == "A");
    const AlignmentResult b = oracle_align(Triplet{"b", "A", "", ""}, kScheme, AlignmentMode::Global, true);
    CHECK(b.score == -4 && b.rows[0] == "A" && b.rows[1] == "-" && b.rows[2] == "-");
    const AlignmentResult n = oracle_align(Triplet{"neg", "AAA", "CCC", "GGG"}, kScheme, AlignmentMode::Local, true);
    CHECK(n.score == 0 && n.rows[0].empty());
    CHECK_THROWS_AS(oracle_align(Triplet{"big", "ACGTACGT", "ACGTACGT", "ACGTACGT"}, kScheme, AlignmentMode::Global,
                                 true, 100),
                    CapacityError);
    Rng rng(5150, 1);
    for (int rep = 0; rep < 30; ++rep) {
      const Triplet t = random_triplet(rng, 8);
      const ScoringScheme sch{int32_t(1 + rng.below(4)), -int32_t(rng.below(4)), -int32_t(rng.below(4))};
      for (auto m : kModes) {
        std::string rows[3];
        const to_result want = oracle(t, sch, m, true, rows);
        const AlignmentResult got = oracle_align(t, sch, m, true);
        CHECK(got.score == want.score);
        CHECK((got.begin == Coords{want.begin_i, want.begin_j, want.begin_k}));
        CHECK(got.rows[0] == rows[0] && got.rows[1] == rows[1] && got.rows[2] == rows[2]);
      }
    }
  }
  // test_dispatch.cpp:117-249: run_batch
  {
    const auto data = generate_dataset("uniform:1:12:20", 0.2, 0.0, 11).triplets;
    std::vector<uint64_t> cells;
    for (const auto& t : data) cells.push_back(t.cell_count());
    std::vector<int32_t> baseline;
    bool first = true;
    for (auto st : {Strategy::Blocked, Strategy::Interleaved, Strategy::Dynamic})
      for (int w : {1, 2, 4}) {
        const auto rep = run_batch(data, kScheme, AlignmentMode::SemiGlobal, cfg_with(4), plan_partition(cells, st, w));
        std::vector<int32_t> scores;
        for (const auto& o : rep.per_triplet) {
          CHECK(o.ok);
          scores.push_back(o.score);
        }
        if (first) {
          baseline = scores;
          first = false;
        } else {
          CHECK(scores == baseline);
        }
      }
    auto fixed = generate_dataset("fixed:4:4:4:3", 0.0, 0.0, 9).triplets;
    Triplet big;
    big.id = "too-big";
    big.s0 = big.s1 = big.s2 = std::string(40, 'A');
    fixed.insert(fixed.begin() + 1, big);
    std::vector<uint64_t> fc;
    for (const auto& t : fixed) fc.push_back(t.cell_count());
    EngineConfig c4 = cfg_with(4);
    c4.cell_budget = 10000;
    const auto rep = run_batch(fixed, kScheme, AlignmentMode::Global, c4, plan_partition(fc, Strategy::Interleaved, 2));
    CHECK(rep.per_triplet[0].ok && !rep.per_triplet[1].ok && rep.per_triplet[2].ok && rep.per_triplet[3].ok);
    CHECK(rep.per_triplet[1].error == "triplet 'too-big' has 64000 cells, over the budget of 10000");
    uint64_t okc = 0;
    for (const auto& o : rep.per_triplet)
      if (o.ok) okc += o.cells;
    CHECK(rep.scored_cells == okc);
  }
  std::printf("[cpp-api] checks: %d | failed: %d\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
