// dataset.cpp — seeded synthetic triplet generator, parallel over triplets.
//
// Same outputs, bit for bit, as the reference generate_dataset
// (/root/reference/proj/src/dataset.cpp:121-211) with its counter-based RNG
// (proj/include/trioalign/rng.hpp:12-43) and spec grammar
// (dataset.cpp:87-119).  Every triplet draws from its own stream
// (seed, index + 1), so triplets are generated independently on all host
// cores and concatenated in index order.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "../../../include/trioalign_capi.h"

namespace {

thread_local std::string g_gen_err;

struct Rng {
  uint64_t key, counter = 0;
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  Rng(uint64_t seed, uint64_t stream)
      : key(mix(seed ^ 0x9e3779b97f4a7c15ull) ^ mix(stream ^ 0xbf58476d1ce4e5b9ull)) {}
  uint64_t next() { return mix(key + (++counter) * 0x9e3779b97f4a7c15ull); }
  uint64_t below(uint64_t n) {
    return n == 0 ? 0 : uint64_t((static_cast<unsigned __int128>(next()) * n) >> 64);
  }
  double unit() { return double(next() >> 11) * 0x1.0p-53; }
  char base() { return "ACGT"[below(4)]; }
};

enum class Model { Uniform, Blocked, Cycle, Fixed };

struct Spec {
  Model model = Model::Uniform;
  int64_t count = 1;
  int64_t min_len = 1, max_len = 1;
  std::vector<int64_t> lengths;
  int64_t fa = 0, fb = 0, fc = 0;
};

bool parse_int(std::string_view s, int64_t* out) {
  int64_t v = 0;
  const auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc{} || p != s.data() + s.size()) return false;
  *out = v;
  return true;
}

std::vector<std::string_view> split(std::string_view s, char sep) {
  std::vector<std::string_view> out;
  size_t start = 0;
  for (;;) {
    const size_t p = s.find(sep, start);
    if (p == std::string_view::npos) {
      out.push_back(s.substr(start));
      return out;
    }
    out.push_back(s.substr(start, p - start));
    start = p + 1;
  }
}

// DatasetSpec::parse + validate (dataset.cpp:56-119); messages match.
int parse_spec(std::string_view text, double mut, double indel, Spec* sp) {
  const auto parts = split(text, ':');
  auto bad = [&](const std::string& what, std::string_view v) {
    g_gen_err = "dataset spec: bad " + what + " '" + std::string(v) + "'";
    return TA_ERR_PARSE;
  };
  const std::string_view kind = parts[0];
  if (kind == "uniform") {
    if (parts.size() != 4) return g_gen_err = "dataset spec: expected uniform:MIN:MAX:COUNT", TA_ERR_PARSE;
    sp->model = Model::Uniform;
    if (!parse_int(parts[1], &sp->min_len)) return bad("min length", parts[1]);
    if (!parse_int(parts[2], &sp->max_len)) return bad("max length", parts[2]);
    if (!parse_int(parts[3], &sp->count)) return bad("count", parts[3]);
  } else if (kind == "fixed") {
    if (parts.size() != 4 && parts.size() != 5)
      return g_gen_err = "dataset spec: expected fixed:A:B:C[:COUNT]", TA_ERR_PARSE;
    sp->model = Model::Fixed;
    if (!parse_int(parts[1], &sp->fa)) return bad("length", parts[1]);
    if (!parse_int(parts[2], &sp->fb)) return bad("length", parts[2]);
    if (!parse_int(parts[3], &sp->fc)) return bad("length", parts[3]);
    sp->count = 1;
    if (parts.size() == 5 && !parse_int(parts[4], &sp->count)) return bad("count", parts[4]);
  } else if (kind == "blocked" || kind == "cycle") {
    if (parts.size() != 3) {
      g_gen_err = "dataset spec: expected " + std::string(kind) + ":L1,L2,...:COUNT";
      return TA_ERR_PARSE;
    }
    sp->model = kind == "blocked" ? Model::Blocked : Model::Cycle;
    for (const auto part : split(parts[1], ',')) {
      int64_t v = 0;
      if (!parse_int(part, &v)) return bad("length", part);
      sp->lengths.push_back(v);
    }
    if (!parse_int(parts[2], &sp->count)) return bad("count", parts[2]);
  } else {
    g_gen_err = "dataset spec: unknown model '" + std::string(kind) +
                "' (expected uniform, fixed, blocked, or cycle)";
    return TA_ERR_PARSE;
  }
  // validate
  if (sp->count < 1) return g_gen_err = "dataset spec: count must be >= 1", TA_ERR_PARSE;
  if (!(mut >= 0 && mut <= 1 && indel >= 0 && indel <= 1))
    return g_gen_err = "dataset spec: rates must be within [0, 1]", TA_ERR_PARSE;
  switch (sp->model) {
    case Model::Uniform:
      if (sp->min_len < 0 || sp->max_len < sp->min_len)
        return g_gen_err = "dataset spec: uniform needs 0 <= min <= max", TA_ERR_PARSE;
      break;
    case Model::Blocked:
    case Model::Cycle:
      if (sp->lengths.empty()) return g_gen_err = "dataset spec: length list must not be empty", TA_ERR_PARSE;
      for (int64_t v : sp->lengths)
        if (v < 0) return g_gen_err = "dataset spec: lengths must be >= 0", TA_ERR_PARSE;
      break;
    case Model::Fixed:
      if (sp->fa < 0 || sp->fb < 0 || sp->fc < 0)
        return g_gen_err = "dataset spec: fixed lengths must be >= 0", TA_ERR_PARSE;
      if ((sp->fa != sp->fb || sp->fb != sp->fc) && (mut > 0 || indel > 0))
        return g_gen_err = "dataset spec: fixed with unequal lengths has no common ancestor; rates must be 0",
               TA_ERR_PARSE;
      break;
  }
  return TA_OK;
}

char other_base(char base, uint64_t pick) {
  for (char b : {'A', 'C', 'G', 'T'}) {
    if (b == base) continue;
    if (pick == 0) return b;
    --pick;
  }
  return 'A';
}

// One triplet: appends s0, s1, s2 to `out` and their lengths to `lens`;
// optionally appends the three true-alignment rows to `ref`.
void gen_one(const Spec& sp, double mut, double indel, uint64_t seed, int64_t idx,
             std::string* out, int64_t lens[3], std::string* ref, int64_t* ref_len) {
  Rng rng(seed, uint64_t(idx) + 1);
  if (sp.model == Model::Fixed && (sp.fa != sp.fb || sp.fb != sp.fc)) {
    const int64_t L[3] = {sp.fa, sp.fb, sp.fc};
    for (int d = 0; d < 3; ++d) {
      for (int64_t p = 0; p < L[d]; ++p) out->push_back(rng.base());
      lens[d] = L[d];
    }
    if (ref_len) *ref_len = -1;
    return;
  }
  int64_t len = 0;
  switch (sp.model) {
    case Model::Uniform:
      len = sp.min_len + int64_t(rng.below(uint64_t(sp.max_len - sp.min_len + 1)));
      break;
    case Model::Blocked: {
      const size_t groups = sp.lengths.size();
      const size_t group = std::min(groups - 1, size_t(idx) * groups / size_t(sp.count));
      len = sp.lengths[group];
      break;
    }
    case Model::Cycle:
      len = sp.lengths[size_t(idx) % sp.lengths.size()];
      break;
    case Model::Fixed:
      len = sp.fa;
      break;
  }
  std::string anc(size_t(len), 'A');
  for (auto& ch : anc) ch = rng.base();
  std::string rows[3];
  for (int64_t site = 0; site < len; ++site) {
    char col[3] = {anc[size_t(site)], anc[size_t(site)], anc[size_t(site)]};
    for (int d = 0; d < 3; ++d) {
      if (mut > 0 && rng.unit() < mut) col[d] = other_base(col[d], rng.below(3));
    }
    char ins[3][3];
    int nins = 0;
    for (int d = 0; d < 3; ++d) {
      if (indel > 0 && rng.unit() < indel) {
        if (rng.below(2) == 0) {
          col[d] = '-';
        } else {
          ins[nins][0] = ins[nins][1] = ins[nins][2] = '-';
          ins[nins][d] = rng.base();
          ++nins;
        }
      }
    }
    if (col[0] != '-' || col[1] != '-' || col[2] != '-') {
      for (int d = 0; d < 3; ++d) rows[d].push_back(col[d]);
    }
    for (int e = 0; e < nins; ++e) {
      for (int d = 0; d < 3; ++d) rows[d].push_back(ins[e][d]);
    }
  }
  for (int d = 0; d < 3; ++d) {
    const size_t before = out->size();
    for (char ch : rows[d])
      if (ch != '-') out->push_back(ch);
    lens[d] = int64_t(out->size() - before);
  }
  if (ref) {
    for (int d = 0; d < 3; ++d) ref->append(rows[d]);
    *ref_len = int64_t(rows[0].size());
  }
}

}  // namespace

extern "C" {

const char* ta_generate_error(void) { return g_gen_err.c_str(); }

void ta_free(void* p) { std::free(p); }

int ta_generate_slice(const char* spec, double mutation, double indel, uint64_t seed,
                      int64_t begin, int64_t end, int threads, char** seqs_out,
                      int64_t** offsets_out, int64_t* n_out) {
  *seqs_out = nullptr;
  *offsets_out = nullptr;
  *n_out = 0;
  Spec sp;
  if (int rc = parse_spec(spec ? spec : "", mutation, indel, &sp)) return rc;
  if (end < 0 || end > sp.count) end = sp.count;
  if (begin < 0) begin = 0;
  if (begin > end) begin = end;
  const int64_t n = end - begin;
  if (threads < 1) threads = int(std::max(1u, std::thread::hardware_concurrency()));
  threads = int(std::min<int64_t>(threads, std::max<int64_t>(1, n / 64)));
  std::vector<std::string> chunk(static_cast<size_t>(threads));
  std::vector<int64_t> lens(static_cast<size_t>(3 * n));
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) {
    pool.emplace_back([&, w] {
      const int64_t lo = n * w / threads, hi = n * (w + 1) / threads;
      for (int64_t t = lo; t < hi; ++t)
        gen_one(sp, mutation, indel, seed, begin + t, &chunk[size_t(w)], &lens[size_t(3 * t)], nullptr, nullptr);
    });
  }
  for (auto& th : pool) th.join();
  size_t total = 0;
  for (const auto& c : chunk) total += c.size();
  char* seqs = static_cast<char*>(std::malloc(total + 1));
  int64_t* offs = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * size_t(3 * n + 1)));
  if (!seqs || !offs) {
    std::free(seqs);
    std::free(offs);
    g_gen_err = "out of host memory";
    return TA_ERR_NOMEM;
  }
  size_t pos = 0;
  for (const auto& c : chunk) {
    std::memcpy(seqs + pos, c.data(), c.size());
    pos += c.size();
  }
  int64_t o = 0;
  for (int64_t i = 0; i < 3 * n; ++i) {
    offs[i] = o;
    o += lens[size_t(i)];
  }
  offs[3 * n] = o;
  *seqs_out = seqs;
  *offsets_out = offs;
  *n_out = n;
  return TA_OK;
}

int ta_generate(const char* spec, double mutation, double indel, uint64_t seed, int threads,
                char** seqs_out, int64_t** offsets_out, int64_t* n_out) {
  return ta_generate_slice(spec, mutation, indel, seed, 0, -1, threads, seqs_out, offsets_out, n_out);
}

// Reference rows of a generated dataset (the `generate --ref-out` payload):
// rows of triplet t are ref[ref_off[t] .. ) as three consecutive rows of
// length ref_len[t]; ref_len < 0 when the spec records no alignment.
int ta_generate_reference(const char* spec, double mutation, double indel, uint64_t seed,
                          char** ref_out, int64_t** ref_off_out, int64_t** ref_len_out,
                          int64_t* n_out) {
  *ref_out = nullptr;
  *ref_off_out = nullptr;
  *ref_len_out = nullptr;
  Spec sp;
  if (int rc = parse_spec(spec ? spec : "", mutation, indel, &sp)) return rc;
  const int64_t n = sp.count;
  std::string all, scratch;
  std::vector<int64_t> off(static_cast<size_t>(n)), rl(static_cast<size_t>(n));
  int64_t lens[3];
  for (int64_t t = 0; t < n; ++t) {
    off[size_t(t)] = int64_t(all.size());
    scratch.clear();
    gen_one(sp, mutation, indel, seed, t, &scratch, lens, &all, &rl[size_t(t)]);
  }
  char* ref = static_cast<char*>(std::malloc(all.size() + 1));
  int64_t* o = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * size_t(n)));
  int64_t* l = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * size_t(n)));
  std::memcpy(ref, all.data(), all.size());
  std::memcpy(o, off.data(), sizeof(int64_t) * size_t(n));
  std::memcpy(l, rl.data(), sizeof(int64_t) * size_t(n));
  *ref_out = ref;
  *ref_off_out = o;
  *ref_len_out = l;
  *n_out = n;
  return TA_OK;
}

}  // extern "C"
