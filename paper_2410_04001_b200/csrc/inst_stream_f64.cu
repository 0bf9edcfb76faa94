// Kernel instantiations (see instances.h).
#define LRNR_INSTANTIATING 1
#include "instances.h"

LRNR_V1_F64(LRNR_V1_INST)
