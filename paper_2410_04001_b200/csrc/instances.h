// Explicit-instantiation registry: every kernel variant is compiled in exactly
// one of the inst_*.cu translation units (built in parallel); lrnr_gpu.cu only
// sees extern declarations.
#pragma once

#include "internal.h"

// streaming kernel v1: (T, TPP, RMAX, ACT, MODE)
#define LRNR_V1_F64(X) \
    X(double, 4, 16, 0, 0) X(double, 4, 32, 0, 0) X(double, 4, 64, 0, 0) \
    X(double, 4, 16, 1, 0) X(double, 4, 32, 1, 0) X(double, 4, 64, 1, 0) \
    X(double, 4, 16, 0, 1) X(double, 4, 32, 0, 1) X(double, 4, 64, 0, 1) \
    X(double, 4, 16, 1, 1) X(double, 4, 32, 1, 1) X(double, 4, 64, 1, 1)
#define LRNR_V1_F32(X) \
    X(float, 4, 16, 0, 0) X(float, 4, 32, 0, 0) X(float, 4, 64, 0, 0) \
    X(float, 4, 16, 1, 0) X(float, 4, 32, 1, 0) X(float, 4, 64, 1, 0) \
    X(float, 4, 16, 0, 1) X(float, 4, 32, 0, 1) X(float, 4, 64, 0, 1) \
    X(float, 4, 16, 1, 1) X(float, 4, 32, 1, 1) X(float, 4, 64, 1, 1)

// tile kernel: (T, P, PT1, NG, RPMAX, ACT, FAST)
#define LRNR_TILE_F32(X) \
    X(float, 64, 2, 16, 32, 1, false) X(float, 64, 2, 16, 32, 1, true) X(float, 64, 2, 16, 32, 0, false) \
    X(float, 64, 1, 8, 32, 1, false) X(float, 64, 1, 8, 32, 1, true) X(float, 64, 1, 8, 32, 0, false) \
    X(float, 32, 2, 16, 32, 1, false) X(float, 32, 2, 16, 32, 1, true) X(float, 32, 2, 16, 32, 0, false) \
    X(float, 32, 1, 8, 32, 1, false) X(float, 32, 1, 8, 32, 1, true) X(float, 32, 1, 8, 32, 0, false)
#define LRNR_TILE_F32R64(X) \
    X(float, 32, 2, 16, 64, 1, false) X(float, 32, 2, 16, 64, 1, true) X(float, 32, 2, 16, 64, 0, false)
#define LRNR_TILE_F64(X) X(double, 32, 1, 8, 32, 0, false) X(double, 32, 1, 8, 32, 1, false)

#define LRNR_V1_EXTERN(T, TPP, RM, ACT, MODE)                                                            \
    extern template void lrnr_b200::detail::launch_pinn<T, TPP, RM, ACT, MODE>(                           \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);
#define LRNR_V1_INST(T, TPP, RM, ACT, MODE)                                                              \
    template void lrnr_b200::detail::launch_pinn<T, TPP, RM, ACT, MODE>(                                  \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);
#define LRNR_TILE_EXTERN(T, P, PT1, NG, RP, ACT, FAST)                                                   \
    extern template void lrnr_b200::detail::launch_v2<T, P, PT1, NG, RP, ACT, FAST, false>(               \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);
#define LRNR_TILE_INST(T, P, PT1, NG, RP, ACT, FAST)                                                     \
    template void lrnr_b200::detail::launch_v2<T, P, PT1, NG, RP, ACT, FAST, false>(                      \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);
// meta (dU/dV/db) variants of the tile kernel: (T, ACT, RPMAX); P = 32, KC = 32
#define LRNR_META(X) X(float, 1, 64) X(float, 1, 32) X(float, 0, 64) X(float, 0, 32) X(double, 0, 32) X(double, 1, 32)
#define LRNR_META_EXTERN(T, ACT, RP)                                                                    \
    extern template void lrnr_b200::detail::launch_v2<T, 32, 1, 8, RP, ACT, false, true>(                  \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);
#define LRNR_META_INST(T, ACT, RP)                                                                      \
    template void lrnr_b200::detail::launch_v2<T, 32, 1, 8, RP, ACT, false, true>(                         \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);



// small-batch latency kernel: (T, ACT, MODE)
#define LRNR_SMALL(X) \
    X(float, 0, 0) X(float, 1, 0) X(float, 0, 1) X(float, 1, 1) \
    X(double, 0, 0) X(double, 1, 0) X(double, 0, 1) X(double, 1, 1)
#define LRNR_SMALL_EXTERN(T, ACT, MODE)                                                                   \
    extern template void lrnr_b200::detail::launch_small<T, ACT, MODE>(                                    \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);
#define LRNR_SMALL_INST(T, ACT, MODE)                                                                     \
    template void lrnr_b200::detail::launch_small<T, ACT, MODE>(                                           \
        lrnr_gpu_ctx*, const lrnr_b200::detail::Model&, const double*, const double*, double, double*, double*);

#ifndef LRNR_INSTANTIATING
LRNR_V1_F64(LRNR_V1_EXTERN)
LRNR_V1_F32(LRNR_V1_EXTERN)
LRNR_TILE_F32(LRNR_TILE_EXTERN)
LRNR_TILE_F32R64(LRNR_TILE_EXTERN)
LRNR_TILE_F64(LRNR_TILE_EXTERN)
LRNR_META(LRNR_META_EXTERN)
LRNR_SMALL(LRNR_SMALL_EXTERN)
#endif
