// kernels.h — instantiation table of the wavefront kernel family.
// Each tile-grid size G lives in its own translation unit (kernels_gXX.cu)
// so the heavy unrolled instantiations compile in parallel.
#pragma once

#include <cstddef>

#include "wavefront.cuh"

namespace ta {

constexpr int kTileN = 10;                 // cells per tile side
constexpr int kGridSizes[] = {4, 8, 12, 16};  // tile-grid sides (plane extent G*N)
constexpr int kNumGrid = sizeof(kGridSizes) / sizeof(kGridSizes[0]);
constexpr int kMaxExtent = 16 * kTileN;    // largest single-block plane side
constexpr int kSmallTileN = 8;             // multi-block items in 128-wide blocks (16 x 16 tiles of 8 x 8)

using WaveFn = void (*)(WaveArgs);

struct KernelEntry {
  WaveFn fn = nullptr;
  size_t smem = 0;
  int threads = 0;
  int grid = 0;
};

// lanes in {1, 2}; mode in {kGlobal, kSemi, kLocal}; trace with either lane width;
// blk: 0 single-plane, 1 sequential multi-block items, 2 wave (multi-CTA)
// blocks; blk > 0 exists for the largest grid only.
KernelEntry kernel_g4(int lanes, int mode, bool trace, int blk);
KernelEntry kernel_g8(int lanes, int mode, bool trace, int blk);
KernelEntry kernel_g12(int lanes, int mode, bool trace, int blk);
KernelEntry kernel_g16(int lanes, int mode, bool trace, int blk);
KernelEntry kernel_g16_wave(int lanes, int mode);
// wave mode with direction records (traceback of a few long triplets)
KernelEntry kernel_g16_wave_trace(int lanes, int mode);
// 16 x 16 grid of 8 x 8 tiles, multi-block items only (blk 1, no trace): long
// triplets whose extents pad less in 128-wide blocks than in 160-wide ones
KernelEntry kernel_g16_t8(int lanes, int mode);
// the same 8 x 8 tiles in wave mode (few long triplets, score only): a wave
// step is latency bound per thread, so 64 instead of 100 cells per tile-step
// shortens every step of the triplet's critical path
KernelEntry kernel_g16_t8_wave(int lanes, int mode);

inline KernelEntry lookup_kernel(int grid, int lanes, int mode, bool trace, int blk) {
  if (blk == 2) return grid != 16 ? KernelEntry{} : trace ? kernel_g16_wave_trace(lanes, mode) : kernel_g16_wave(lanes, mode);
  switch (grid) {
    case 4: return kernel_g4(lanes, mode, trace, blk);
    case 8: return kernel_g8(lanes, mode, trace, blk);
    case 12: return kernel_g12(lanes, mode, trace, blk);
    case 16: return kernel_g16(lanes, mode, trace, blk);
  }
  return {};
}

}  // namespace ta

#define TA_KERNEL_ENTRY(G, L, M, TR, BL) \
  KernelEntry{&wavefront_kernel<kTileN, G, L, M, TR, BL>, WaveSmem<kTileN, G, L, BL>::bytes, G * G, G}

#define TA_DEFINE_KERNEL_TABLE(G, WITH_BLOCKS)                                         \
  namespace ta {                                                                       \
  template <int BL>                                                                    \
  static KernelEntry pick_##G(int lanes, int mode, bool trace) {                       \
    if (trace) {                                                                       \
      if (lanes == 1) {                                                                \
        switch (mode) {                                                                \
          case kGlobal: return TA_KERNEL_ENTRY(G, 1, kGlobal, true, BL);               \
          case kSemi: return TA_KERNEL_ENTRY(G, 1, kSemi, true, BL);                   \
          case kLocal: return TA_KERNEL_ENTRY(G, 1, kLocal, true, BL);                 \
        }                                                                              \
      } else {                                                                         \
        switch (mode) {                                                                \
          case kGlobal: return TA_KERNEL_ENTRY(G, 2, kGlobal, true, BL);               \
          case kSemi: return TA_KERNEL_ENTRY(G, 2, kSemi, true, BL);                   \
          case kLocal: return TA_KERNEL_ENTRY(G, 2, kLocal, true, BL);                 \
        }                                                                              \
      }                                                                                \
      return {};                                                                       \
    }                                                                                  \
    if (lanes == 1) {                                                                  \
      switch (mode) {                                                                  \
        case kGlobal: return TA_KERNEL_ENTRY(G, 1, kGlobal, false, BL);                \
        case kSemi: return TA_KERNEL_ENTRY(G, 1, kSemi, false, BL);                    \
        case kLocal: return TA_KERNEL_ENTRY(G, 1, kLocal, false, BL);                  \
      }                                                                                \
    } else {                                                                           \
      switch (mode) {                                                                  \
        case kGlobal: return TA_KERNEL_ENTRY(G, 2, kGlobal, false, BL);                \
        case kSemi: return TA_KERNEL_ENTRY(G, 2, kSemi, false, BL);                    \
        case kLocal: return TA_KERNEL_ENTRY(G, 2, kLocal, false, BL);                  \
      }                                                                                \
    }                                                                                  \
    return {};                                                                         \
  }                                                                                    \
  KernelEntry kernel_g##G(int lanes, int mode, bool trace, int blk) {                  \
    if (blk == 1) {                                                                    \
      if constexpr (WITH_BLOCKS) return pick_##G<1>(lanes, mode, trace);               \
      return {};                                                                       \
    }                                                                                  \
    if (blk != 0) return {};                                                           \
    return pick_##G<0>(lanes, mode, trace);                                            \
  }                                                                                    \
  }

#define TA_DEFINE_T8_TABLE()                                                                       \
  namespace ta {                                                                                   \
  KernelEntry kernel_g16_t8(int lanes, int mode) {                                                 \
    constexpr int N8 = kSmallTileN;                                                                \
    if (lanes == 1) {                                                                              \
      switch (mode) {                                                                              \
        case kGlobal: return {&wavefront_kernel<N8, 16, 1, kGlobal, false, 1>, WaveSmem<N8, 16, 1, 1>::bytes, 256, 16}; \
        case kSemi: return {&wavefront_kernel<N8, 16, 1, kSemi, false, 1>, WaveSmem<N8, 16, 1, 1>::bytes, 256, 16};     \
        case kLocal: return {&wavefront_kernel<N8, 16, 1, kLocal, false, 1>, WaveSmem<N8, 16, 1, 1>::bytes, 256, 16};   \
      }                                                                                            \
    } else {                                                                                       \
      switch (mode) {                                                                              \
        case kGlobal: return {&wavefront_kernel<N8, 16, 2, kGlobal, false, 1>, WaveSmem<N8, 16, 2, 1>::bytes, 256, 16}; \
        case kSemi: return {&wavefront_kernel<N8, 16, 2, kSemi, false, 1>, WaveSmem<N8, 16, 2, 1>::bytes, 256, 16};     \
        case kLocal: return {&wavefront_kernel<N8, 16, 2, kLocal, false, 1>, WaveSmem<N8, 16, 2, 1>::bytes, 256, 16};   \
      }                                                                                            \
    }                                                                                              \
    return {};                                                                                     \
  }                                                                                                \
  }

#define TA_DEFINE_WAVE_TABLE(G, NAME, TR)                                              \
  namespace ta {                                                                       \
  KernelEntry NAME(int lanes, int mode) {                                              \
    if (lanes == 1) {                                                                  \
      switch (mode) {                                                                  \
        case kGlobal: return TA_KERNEL_ENTRY(G, 1, kGlobal, TR, 2);                    \
        case kSemi: return TA_KERNEL_ENTRY(G, 1, kSemi, TR, 2);                        \
        case kLocal: return TA_KERNEL_ENTRY(G, 1, kLocal, TR, 2);                      \
      }                                                                                \
    } else {                                                                           \
      switch (mode) {                                                                  \
        case kGlobal: return TA_KERNEL_ENTRY(G, 2, kGlobal, TR, 2);                    \
        case kSemi: return TA_KERNEL_ENTRY(G, 2, kSemi, TR, 2);                        \
        case kLocal: return TA_KERNEL_ENTRY(G, 2, kLocal, TR, 2);                      \
      }                                                                                \
    }                                                                                  \
    return {};                                                                         \
  }                                                                                    \
  }

#define TA_DEFINE_T8_WAVE_TABLE()                                                                  \
  namespace ta {                                                                                   \
  KernelEntry kernel_g16_t8_wave(int lanes, int mode) {                                            \
    constexpr int N8 = kSmallTileN;                                                                \
    if (lanes == 1) {                                                                              \
      switch (mode) {                                                                              \
        case kGlobal: return {&wavefront_kernel<N8, 16, 1, kGlobal, false, 2>, WaveSmem<N8, 16, 1, 2>::bytes, 256, 16}; \
        case kSemi: return {&wavefront_kernel<N8, 16, 1, kSemi, false, 2>, WaveSmem<N8, 16, 1, 2>::bytes, 256, 16};     \
        case kLocal: return {&wavefront_kernel<N8, 16, 1, kLocal, false, 2>, WaveSmem<N8, 16, 1, 2>::bytes, 256, 16};   \
      }                                                                                            \
    } else {                                                                                       \
      switch (mode) {                                                                              \
        case kGlobal: return {&wavefront_kernel<N8, 16, 2, kGlobal, false, 2>, WaveSmem<N8, 16, 2, 2>::bytes, 256, 16}; \
        case kSemi: return {&wavefront_kernel<N8, 16, 2, kSemi, false, 2>, WaveSmem<N8, 16, 2, 2>::bytes, 256, 16};     \
        case kLocal: return {&wavefront_kernel<N8, 16, 2, kLocal, false, 2>, WaveSmem<N8, 16, 2, 2>::bytes, 256, 16};   \
      }                                                                                            \
    }                                                                                              \
    return {};                                                                                     \
  }                                                                                                \
  }
