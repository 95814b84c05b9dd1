// Wave-mode instantiations with direction records (traceback of few long
// triplets spread over all CTAs), 16x16 tile grid.
#include "kernels.h"
TA_DEFINE_WAVE_TABLE(16, kernel_g16_wave_trace, true)
