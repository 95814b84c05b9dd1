// Affine-gap kernels, wave mode (blocks of few long triplets spread over all CTAs).
#include "kernels_aff.h"
TA_DEFINE_AFF_TABLE(affine_kernel_wave, 2)
