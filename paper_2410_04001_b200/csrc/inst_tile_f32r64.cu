// Kernel instantiations (see instances.h).
#define LRNR_INSTANTIATING 1
#include "instances.h"

LRNR_TILE_F32R64(LRNR_TILE_INST)
