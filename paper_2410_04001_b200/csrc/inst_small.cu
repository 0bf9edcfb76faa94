// Kernel instantiations (see instances.h).
#define LRNR_INSTANTIATING 1
#include "instances.h"

LRNR_SMALL(LRNR_SMALL_INST)
