// Affine-gap kernels with 4 x 4 tiles (64-wide blocks) for long triplets
// whose extents waste less padding at 64 than at 80.
#include "kernels_aff.h"
TA_DEFINE_AFF4_TABLE()
