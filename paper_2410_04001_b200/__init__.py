"""B200-native LRNR / FastLRNR physics-informed residual + gradient path.

Native code: paper_2410_04001_b200/liblrnr_gpu.so (C ABI in include/lrnr_gpu.h,
CUDA sm_100a kernels in csrc/).  This package is the ctypes binding used by the
tests and bench; C++ callers use include/lrnr_gpu_adapter.hpp.
"""
from .api import (  # noqa: F401
    ACT_SIN, ACT_TANH, Checkpoint, F32, F64, MODEL_FAST, MODEL_LRNR, FastParams, GpuContext, HyperParams, LrnrGpuError,
    LrnrParams, NonFiniteError, algorithmic_flops_per_point, build_fast, build_fast_qdeim, build_fastparams, qdeim, config0, config1, config2, config3,
    config4, fast_flops_per_point, make_baseline_model, make_hyper_params, hyper_forward, c3_hyper, sample_collocation, eim_greedy, harvest_points, uniform_grid,
    KERNEL_AUTO, KERNEL_FMA_TILE, KERNEL_NARROW, KERNEL_SMALL, KERNEL_STREAM, KERNEL_TC, OBJ_ABS, OBJ_SQUARED, OPT_FAST_SINCOS, OPT_KERNEL, OPT_META_PREC, OPT_SOLVE,
    OPT_TILE_P,
)
