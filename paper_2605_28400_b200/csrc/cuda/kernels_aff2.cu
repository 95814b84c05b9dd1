// Affine-gap kernels, multi-block (long) triplets.
#include "kernels_aff.h"
TA_DEFINE_AFF_TABLE(affine_kernel_blocks, 1)
