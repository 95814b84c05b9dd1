// Wave-mode (multi-CTA long triplet) instantiations of the 16x16 tile grid.
#include "kernels.h"
TA_DEFINE_WAVE_TABLE(16, kernel_g16_wave, false)
#ifdef TA_WAVE_CLOCK
extern "C" int ta_debug_wave_clock(unsigned long long* out, size_t bytes) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, ta::g_wave_clock, bytes));
}
#endif
