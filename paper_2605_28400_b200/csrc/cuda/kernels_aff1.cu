// Affine-gap kernels, single-block planes.
#include "kernels_aff.h"
TA_DEFINE_AFF_TABLE(affine_kernel_single, 0)
