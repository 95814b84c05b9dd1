// Multi-block instantiations of the 16x16 tile grid with 8x8 tiles (128-wide
// blocks): long triplets whose extents waste less padding at 128 than at 160.
#include "kernels.h"
TA_DEFINE_T8_TABLE()
