// Instantiations of the wavefront kernel for a 16x16 tile grid.
#include "kernels.h"
TA_DEFINE_KERNEL_TABLE(16, true)
