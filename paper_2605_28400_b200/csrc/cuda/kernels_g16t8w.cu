// Wave-mode (multi-CTA long triplet) instantiations of the 16x16 grid of 8x8
// tiles, score only (kernels.h: kernel_g16_t8_wave).
#include "kernels.h"
TA_DEFINE_T8_WAVE_TABLE()
