// Instantiations of the wavefront kernel for a 12x12 tile grid.
#include "kernels.h"
TA_DEFINE_KERNEL_TABLE(12, false)
