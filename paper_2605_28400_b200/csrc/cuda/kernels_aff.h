// kernels_aff.h — instantiation table of the affine-gap wavefront kernel
// (affine.cuh): one 16 x 16 grid of 5 x 5 tiles (80-cell block side).
#pragma once

#include <cstddef>

#include "affine.cuh"

namespace ta {

constexpr int kAffG = 16;
constexpr int kAffExtent = kAffG * kAffN;
constexpr int kAffSmallN = 4;  // block items in 64-wide blocks (16 x 16 tiles of 4 x 4)

using AffFn = void (*)(AffArgs);

struct AffEntry {
  AffFn fn = nullptr;
  size_t smem = 0;
  int threads = 0;
};

// trace requires lanes == 1; blk: 0 single block, 1 sequential block items,
// 2 wave mode (no trace)
AffEntry affine_kernel_single(int lanes, int mode, bool trace);
AffEntry affine_kernel_blocks(int lanes, int mode, bool trace);
AffEntry affine_kernel_wave(int lanes, int mode, bool trace);
// 4 x 4 tiles, block items only (no trace): long triplets whose extents pad
// less in 64-wide blocks than in 80-wide ones
AffEntry affine_kernel_blocks4(int lanes, int mode);
// the same 4 x 4 tiles in wave mode (few long triplets, score only): 16
// instead of 25 cells per latency-bound wave step
AffEntry affine_kernel_wave4(int lanes, int mode);

inline AffEntry lookup_affine(int lanes, int mode, bool trace, int blk) {
  if (blk == 2) return affine_kernel_wave(lanes, mode, trace);
  return blk ? affine_kernel_blocks(lanes, mode, trace) : affine_kernel_single(lanes, mode, trace);
}

}  // namespace ta

#define TA_AFF_ENTRY(L, M, TR, BL) \
  AffEntry{&affine_kernel<kAffN, kAffG, L, M, TR, BL>, AffSmem<kAffN, kAffG, L, BL>::bytes, kAffG * kAffG}

#define TA_DEFINE_AFF_TABLE(NAME, BL)                          \
  namespace ta {                                               \
  AffEntry NAME(int lanes, int mode, bool trace) {             \
    if (trace) {                                               \
      if (lanes != 1) return {};                               \
      switch (mode) {                                          \
        case kGlobal: return TA_AFF_ENTRY(1, kGlobal, true, BL); \
        case kSemi: return TA_AFF_ENTRY(1, kSemi, true, BL);     \
        case kLocal: return TA_AFF_ENTRY(1, kLocal, true, BL);   \
      }                                                        \
      return {};                                               \
    }                                                          \
    if (lanes == 1) {                                          \
      switch (mode) {                                          \
        case kGlobal: return TA_AFF_ENTRY(1, kGlobal, false, BL); \
        case kSemi: return TA_AFF_ENTRY(1, kSemi, false, BL);     \
        case kLocal: return TA_AFF_ENTRY(1, kLocal, false, BL);   \
      }                                                        \
    } else {                                                   \
      switch (mode) {                                          \
        case kGlobal: return TA_AFF_ENTRY(2, kGlobal, false, BL); \
        case kSemi: return TA_AFF_ENTRY(2, kSemi, false, BL);     \
        case kLocal: return TA_AFF_ENTRY(2, kLocal, false, BL);   \
      }                                                        \
    }                                                          \
    return {};                                                 \
  }                                                            \
  }

#define TA_AFF4_ENTRY(L, M) \
  AffEntry{&affine_kernel<kAffSmallN, kAffG, L, M, false, 1>, AffSmem<kAffSmallN, kAffG, L, 1>::bytes, kAffG * kAffG}

#define TA_DEFINE_AFF4_TABLE()                          \
  namespace ta {                                        \
  AffEntry affine_kernel_blocks4(int lanes, int mode) { \
    if (lanes == 1) {                                   \
      switch (mode) {                                   \
        case kGlobal: return TA_AFF4_ENTRY(1, kGlobal); \
        case kSemi: return TA_AFF4_ENTRY(1, kSemi);     \
        case kLocal: return TA_AFF4_ENTRY(1, kLocal);   \
      }                                                 \
    } else {                                            \
      switch (mode) {                                   \
        case kGlobal: return TA_AFF4_ENTRY(2, kGlobal); \
        case kSemi: return TA_AFF4_ENTRY(2, kSemi);     \
        case kLocal: return TA_AFF4_ENTRY(2, kLocal);   \
      }                                                 \
    }                                                   \
    return {};                                          \
  }                                                     \
  }

#define TA_AFF4W_ENTRY(L, M) \
  AffEntry{&affine_kernel<kAffSmallN, kAffG, L, M, false, 2>, AffSmem<kAffSmallN, kAffG, L, 2>::bytes, kAffG * kAffG}

#define TA_DEFINE_AFF4W_TABLE()                          \
  namespace ta {                                         \
  AffEntry affine_kernel_wave4(int lanes, int mode) {    \
    if (lanes == 1) {                                    \
      switch (mode) {                                    \
        case kGlobal: return TA_AFF4W_ENTRY(1, kGlobal); \
        case kSemi: return TA_AFF4W_ENTRY(1, kSemi);     \
        case kLocal: return TA_AFF4W_ENTRY(1, kLocal);   \
      }                                                  \
    } else {                                             \
      switch (mode) {                                    \
        case kGlobal: return TA_AFF4W_ENTRY(2, kGlobal); \
        case kSemi: return TA_AFF4W_ENTRY(2, kSemi);     \
        case kLocal: return TA_AFF4W_ENTRY(2, kLocal);   \
      }                                                  \
    }                                                    \
    return {};                                           \
  }                                                      \
  }
