// Instantiations of the wavefront kernel for a 8x8 tile grid.
#include "kernels.h"
TA_DEFINE_KERNEL_TABLE(8, false)
