// Wave-mode (multi-CTA long triplet) instantiations of the 16x16 tile grid.
#include "kernels.h"
TA_DEFINE_WAVE_TABLE(16, kernel_g16_wave, false)
