// Affine-gap wave-mode (multi-CTA long triplet) kernels with 4 x 4 tiles,
// score only (kernels_aff.h: affine_kernel_wave4).
#include "kernels_aff.h"
TA_DEFINE_AFF4W_TABLE()
