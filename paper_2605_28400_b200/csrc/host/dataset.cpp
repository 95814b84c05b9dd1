// Synthetic datasets: the reference's DatasetSpec API (proj/src/dataset.cpp:
// 56-119 grammar and validation, same ParseError messages) over the engine
// library's parallel generator (csrc/core/dataset.cpp, bit-identical to
// proj/src/dataset.cpp:121-211, pinned by tests/golden/gen_hashes.json).
#include <charconv>
#include <cstring>
#include <string_view>

#include "trioalign/dataset.hpp"
#include "trioalign/errors.hpp"
#include "trioalign_capi.h"

namespace trioalign {

namespace {

int32_t to_int(std::string_view text, const char* what) {
  int64_t v = 0;
  const auto [p, ec] = std::from_chars(text.data(), text.data() + text.size(), v);
  if (ec != std::errc{} || p != text.data() + text.size())
    throw ParseError("dataset spec: bad " + std::string(what) + " '" + std::string(text) + "'");
  return int32_t(v);
}

std::vector<std::string_view> fields(std::string_view text, char sep) {
  std::vector<std::string_view> out;
  for (size_t start = 0;;) {
    const size_t at = text.find(sep, start);
    out.push_back(text.substr(start, at == std::string_view::npos ? std::string_view::npos : at - start));
    if (at == std::string_view::npos) return out;
    start = at + 1;
  }
}

}  // namespace

void DatasetSpec::validate() const {
  if (count < 1) throw ParseError("dataset spec: count must be >= 1");
  if (!(mutation_rate >= 0 && mutation_rate <= 1 && indel_rate >= 0 && indel_rate <= 1))
    throw ParseError("dataset spec: rates must be within [0, 1]");
  switch (model) {
    case LengthModel::Uniform:
      if (min_len < 0 || max_len < min_len) throw ParseError("dataset spec: uniform needs 0 <= min <= max");
      break;
    case LengthModel::Blocked:
    case LengthModel::InterleavedCycle:
      if (lengths.empty()) throw ParseError("dataset spec: length list must not be empty");
      for (int32_t len : lengths)
        if (len < 0) throw ParseError("dataset spec: lengths must be >= 0");
      break;
    case LengthModel::Fixed:
      if (fixed_a < 0 || fixed_b < 0 || fixed_c < 0) throw ParseError("dataset spec: fixed lengths must be >= 0");
      if ((fixed_a != fixed_b || fixed_b != fixed_c) && (mutation_rate > 0 || indel_rate > 0))
        throw ParseError("dataset spec: fixed with unequal lengths has no common ancestor; rates must be 0");
      break;
  }
}

DatasetSpec DatasetSpec::parse(const std::string& text) {
  const auto f = fields(text, ':');
  DatasetSpec spec;
  const std::string_view kind = f[0];
  if (kind == "uniform") {
    if (f.size() != 4) throw ParseError("dataset spec: expected uniform:MIN:MAX:COUNT");
    spec.model = LengthModel::Uniform;
    spec.min_len = to_int(f[1], "min length");
    spec.max_len = to_int(f[2], "max length");
    spec.count = to_int(f[3], "count");
  } else if (kind == "fixed") {
    if (f.size() != 4 && f.size() != 5) throw ParseError("dataset spec: expected fixed:A:B:C[:COUNT]");
    spec.model = LengthModel::Fixed;
    spec.fixed_a = to_int(f[1], "length");
    spec.fixed_b = to_int(f[2], "length");
    spec.fixed_c = to_int(f[3], "length");
    spec.count = f.size() == 5 ? to_int(f[4], "count") : 1;
  } else if (kind == "blocked" || kind == "cycle") {
    if (f.size() != 3) throw ParseError("dataset spec: expected " + std::string(kind) + ":L1,L2,...:COUNT");
    spec.model = kind == "blocked" ? LengthModel::Blocked : LengthModel::InterleavedCycle;
    for (const auto part : fields(f[1], ',')) spec.lengths.push_back(to_int(part, "length"));
    spec.count = to_int(f[2], "count");
  } else {
    throw ParseError("dataset spec: unknown model '" + std::string(kind) +
                     "' (expected uniform, fixed, blocked, or cycle)");
  }
  spec.validate();
  return spec;
}

std::string DatasetSpec::to_string() const {
  auto list = [&] {
    std::string s;
    for (size_t i = 0; i < lengths.size(); ++i) s += (i ? "," : "") + std::to_string(lengths[i]);
    return s;
  };
  switch (model) {
    case LengthModel::Uniform:
      return "uniform:" + std::to_string(min_len) + ":" + std::to_string(max_len) + ":" + std::to_string(count);
    case LengthModel::Blocked:
      return "blocked:" + list() + ":" + std::to_string(count);
    case LengthModel::InterleavedCycle:
      return "cycle:" + list() + ":" + std::to_string(count);
    case LengthModel::Fixed:
      break;
  }
  return "fixed:" + std::to_string(fixed_a) + ":" + std::to_string(fixed_b) + ":" + std::to_string(fixed_c) + ":" +
         std::to_string(count);
}

GeneratedDataset generate_dataset(const DatasetSpec& spec) {
  spec.validate();
  const bool independent = spec.model == DatasetSpec::LengthModel::Fixed &&
                           (spec.fixed_a != spec.fixed_b || spec.fixed_b != spec.fixed_c);
  return generate_dataset(spec.to_string(), spec.mutation_rate, spec.indel_rate, spec.seed, !independent);
}

GeneratedDataset generate_dataset(const std::string& spec, double mutation_rate, double indel_rate, uint64_t seed,
                                  bool with_references) {
  char* seqs = nullptr;
  int64_t* offs = nullptr;
  int64_t n = 0;
  int rc = ta_generate(spec.c_str(), mutation_rate, indel_rate, seed, 0, &seqs, &offs, &n);
  if (rc != TA_OK) throw_status(rc, ta_generate_error());
  GeneratedDataset out;
  out.triplets.resize(size_t(n));
  for (int64_t t = 0; t < n; ++t) {
    Triplet& tr = out.triplets[size_t(t)];
    tr.id = "t" + std::to_string(t);
    tr.s0.assign(seqs + offs[3 * t], seqs + offs[3 * t + 1]);
    tr.s1.assign(seqs + offs[3 * t + 1], seqs + offs[3 * t + 2]);
    tr.s2.assign(seqs + offs[3 * t + 2], seqs + offs[3 * t + 3]);
  }
  ta_free(seqs);
  ta_free(offs);
  if (with_references) {
    char* ref = nullptr;
    int64_t *roff = nullptr, *rlen = nullptr, rn = 0;
    rc = ta_generate_reference(spec.c_str(), mutation_rate, indel_rate, seed, &ref, &roff, &rlen, &rn);
    if (rc != TA_OK) throw_status(rc, ta_generate_error());
    out.has_references = rn == 0 || rlen[0] >= 0;
    if (out.has_references) {
      out.references.resize(size_t(rn));
      for (int64_t t = 0; t < rn; ++t)
        for (int d = 0; d < 3; ++d)
          out.references[size_t(t)][size_t(d)].assign(ref + roff[t] + d * rlen[t], size_t(rlen[t]));
    }
    ta_free(ref);
    ta_free(roff);
    ta_free(rlen);
  }
  return out;
}

}  // namespace trioalign
