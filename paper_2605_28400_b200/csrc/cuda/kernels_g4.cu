// Instantiations of the wavefront kernel for a 4x4 tile grid.
#include "kernels.h"
TA_DEFINE_KERNEL_TABLE(4, false)
