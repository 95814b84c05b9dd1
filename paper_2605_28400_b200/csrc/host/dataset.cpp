// Synthetic datasets through the engine library's parallel generator
// (csrc/core/dataset.cpp, bit-identical to proj/src/dataset.cpp:121-211).
#include <cstring>

#include "trioalign/dataset.hpp"
#include "trioalign/errors.hpp"
#include "trioalign_capi.h"

namespace trioalign {

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
