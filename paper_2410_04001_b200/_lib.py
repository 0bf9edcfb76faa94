"""Loader for the in-tree native library ``liblrnr_gpu.so`` (include/lrnr_gpu.h).

The product path has no fallback: if the library is missing the import fails
loudly (build it with ``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LRNR_GPU_LIB") or os.path.join(PKG, "liblrnr_gpu.so")

# every symbol include/lrnr_gpu.h declares
EXPORTS = (
    "lrnr_gpu_create", "lrnr_gpu_destroy", "lrnr_gpu_last_error", "lrnr_gpu_last_layer_tag",
    "lrnr_gpu_set_stream", "lrnr_gpu_set_option", "lrnr_gpu_launch_count", "lrnr_gpu_set_lrnr", "lrnr_gpu_set_fast",
    "lrnr_gpu_set_hyper", "lrnr_gpu_set_points", "lrnr_gpu_set_points_device", "lrnr_gpu_stage_points",
    "lrnr_gpu_use_staged_points", "lrnr_gpu_loss_grad_s",
    "lrnr_gpu_set_boundary", "lrnr_gpu_terms_grad", "lrnr_gpu_meta_terms_grad", "lrnr_gpu_set_meta_boundary", "lrnr_gpu_fine_tune",
    "lrnr_gpu_fast_solve", "lrnr_host_epoch_seed", "lrnr_host_sample_batch", "lrnr_gpu_l1_error",
    "lrnr_ckpt_last_error", "lrnr_ckpt_create", "lrnr_ckpt_load", "lrnr_ckpt_save", "lrnr_ckpt_free",
    "lrnr_ckpt_get_lrnr", "lrnr_ckpt_put_lrnr", "lrnr_ckpt_get_hyper", "lrnr_ckpt_put_hyper", "lrnr_ckpt_has_fast",
    "lrnr_ckpt_get_fast", "lrnr_ckpt_put_fast", "lrnr_ckpt_get_sampling", "lrnr_ckpt_put_sampling",
    "lrnr_gpu_loss_grad_s_multi", "lrnr_gpu_hyper_loss_grad", "lrnr_gpu_meta_loss_grad", "lrnr_gpu_jets",
    "lrnr_gpu_loss", "lrnr_gpu_upload_coeffs", "lrnr_gpu_run", "lrnr_gpu_check", "lrnr_gpu_download",
    "lrnr_gpu_fma_peak",
    "lrnr_host_make_baseline_model", "lrnr_host_make_hyper_params", "lrnr_host_sample_collocation",
    "lrnr_host_build_fast", "lrnr_host_harvest_points", "lrnr_host_uniform_grid", "lrnr_host_eim_greedy", "lrnr_host_build_fastparams",
    "lrnr_gpu_eim_greedy", "lrnr_gpu_build_fast", "lrnr_gpu_harvest_snapshots",
    "lrnr_gpu_comm_unique_id", "lrnr_gpu_comm_init", "lrnr_gpu_set_comm", "lrnr_gpu_comm_info", "lrnr_gpu_allreduce",
    "lrnr_gpu_values", "lrnr_gpu_loss_tune", "lrnr_gpu_loss_fast", "lrnr_gpu_loss_meta", "lrnr_host_hyper_forward",
    "lrnr_host_qdeim", "lrnr_host_build_fast_qdeim",
)

LRNR_OK, LRNR_EINVAL, LRNR_ENONFINITE, LRNR_ECUDA, LRNR_ENOMEM, LRNR_ESTATE, LRNR_ENCCL = range(7)
ACT_TANH, ACT_SIN = 0, 1
F64, F32 = 0, 1
MODEL_LRNR, MODEL_FAST = 0, 1
OPT_FAST_SINCOS, OPT_KERNEL, OPT_TILE_P, OPT_SOLVE, OPT_META_PREC = 1, 2, 3, 4, 5
# LRNR_OPT_KERNEL values
KERNEL_AUTO, KERNEL_STREAM, KERNEL_TC, KERNEL_FMA_TILE, KERNEL_SMALL, KERNEL_NARROW = 0, 1, 2, 3, 4, 5
# lrnr_gpu_terms_grad objectives
OBJ_SQUARED, OBJ_ABS = 0, 1

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, dp, ip = C.c_void_p, C.c_int64, C.c_void_p, C.c_int
    lib.lrnr_gpu_create.argtypes = [ip, C.POINTER(vp)]
    lib.lrnr_gpu_destroy.argtypes = [vp]
    lib.lrnr_gpu_last_error.argtypes = [vp]
    lib.lrnr_gpu_last_error.restype = C.c_char_p
    lib.lrnr_gpu_last_layer_tag.argtypes = [vp]
    lib.lrnr_gpu_set_stream.argtypes = [vp, vp]
    lib.lrnr_gpu_set_option.argtypes = [vp, ip, ip]
    lib.lrnr_gpu_launch_count.argtypes = [vp]
    lib.lrnr_gpu_launch_count.restype = i64
    lib.lrnr_gpu_set_lrnr.argtypes = [vp, ip, dp, dp, dp, ip, ip]
    lib.lrnr_gpu_set_fast.argtypes = [vp, ip, dp, dp, i64, i64, dp, ip, ip]
    lib.lrnr_gpu_set_hyper.argtypes = [vp, ip, dp, dp, dp, dp]
    lib.lrnr_gpu_set_points.argtypes = [vp, dp, i64, i64]
    lib.lrnr_gpu_set_points_device.argtypes = [vp, vp, i64, i64]
    lib.lrnr_gpu_stage_points.argtypes = [vp, dp, i64, i64]
    lib.lrnr_gpu_use_staged_points.argtypes = [vp]
    lib.lrnr_gpu_loss_grad_s.argtypes = [vp, ip, dp, dp, C.c_double, dp, dp, dp]
    lib.lrnr_gpu_set_boundary.argtypes = [vp, dp, i64, dp, i64]
    lib.lrnr_gpu_terms_grad.argtypes = [vp, ip, dp, dp, ip, C.c_double, C.c_double, C.c_double, dp, C.c_double,
                                        dp, dp, dp]
    lib.lrnr_gpu_fine_tune.argtypes = [vp, dp, dp, C.c_double, i64, i64, i64, i64, C.c_uint64, dp, dp, dp, dp, dp, dp]
    lib.lrnr_gpu_fast_solve.argtypes = [vp, dp, dp, dp, i64, C.c_double, C.c_double, i64, dp, dp, dp, dp, dp, dp]
    lib.lrnr_host_epoch_seed.argtypes = [C.c_uint64, i64]
    lib.lrnr_host_epoch_seed.restype = C.c_uint64
    lib.lrnr_host_sample_batch.argtypes = [C.c_uint64, i64, i64, i64, dp, dp, dp]
    lib.lrnr_gpu_l1_error.argtypes = [vp, ip, dp, dp, i64, i64, dp]
    lib.lrnr_ckpt_last_error.restype = C.c_char_p
    lib.lrnr_ckpt_create.argtypes = [C.POINTER(vp)]
    lib.lrnr_ckpt_load.argtypes = [C.c_char_p, C.POINTER(vp)]
    lib.lrnr_ckpt_save.argtypes = [vp, C.c_char_p]
    lib.lrnr_ckpt_free.argtypes = [vp]
    lib.lrnr_ckpt_free.restype = None
    lib.lrnr_ckpt_get_lrnr.argtypes = [vp, C.POINTER(C.c_int), dp, dp, C.POINTER(i64), dp]
    lib.lrnr_ckpt_put_lrnr.argtypes = [vp, ip, dp, dp, dp]
    lib.lrnr_ckpt_get_hyper.argtypes = [vp, C.POINTER(C.c_int), dp, C.POINTER(i64), dp, dp, dp]
    lib.lrnr_ckpt_put_hyper.argtypes = [vp, ip, dp, dp, ip, dp, dp, dp]
    lib.lrnr_ckpt_has_fast.argtypes = [vp]
    lib.lrnr_ckpt_get_fast.argtypes = [vp, C.POINTER(C.c_int), dp, dp, C.POINTER(i64), dp]
    lib.lrnr_ckpt_put_fast.argtypes = [vp, ip, dp, dp, i64, i64, dp]
    lib.lrnr_ckpt_get_sampling.argtypes = [vp, C.POINTER(i64), dp]
    lib.lrnr_ckpt_put_sampling.argtypes = [vp, i64, dp]
    lib.lrnr_gpu_loss_grad_s_multi.argtypes = [vp, ip, dp, dp, C.c_double, dp, dp]
    lib.lrnr_gpu_hyper_loss_grad.argtypes = [vp, ip, dp, C.c_double, dp, dp, dp]
    lib.lrnr_gpu_meta_loss_grad.argtypes = [vp, dp, C.c_double, dp, dp]
    lib.lrnr_gpu_set_meta_boundary.argtypes = [vp, i64, dp, i64, dp, i64]
    lib.lrnr_gpu_meta_terms_grad.argtypes = [vp, dp, C.c_double, C.c_double, C.c_double, C.c_double, dp, dp, dp, dp]
    lib.lrnr_gpu_jets.argtypes = [vp, ip, dp, dp]
    lib.lrnr_gpu_loss.argtypes = [vp, ip, dp, dp, C.c_double, dp]
    lib.lrnr_gpu_upload_coeffs.argtypes = [vp, dp, dp, i64]
    lib.lrnr_gpu_run.argtypes = [vp, ip, C.c_double, vp]
    lib.lrnr_gpu_check.argtypes = [vp]
    lib.lrnr_gpu_download.argtypes = [vp, dp, i64]
    lib.lrnr_gpu_fma_peak.argtypes = [vp, ip, dp]
    lib.lrnr_host_make_baseline_model.argtypes = [ip, dp, dp, C.c_uint64, dp, dp]
    lib.lrnr_host_make_hyper_params.argtypes = [ip, dp, ip, ip, C.c_uint64, C.c_double, C.c_double, dp]
    lib.lrnr_host_sample_collocation.argtypes = [C.c_uint64, i64, dp, dp, ip, dp, dp]
    lib.lrnr_host_build_fast.argtypes = [ip, dp, dp, dp, ip, dp, i64, i64, i64, i64, C.c_double, C.c_uint64, i64,
                                         dp, dp, dp, dp]
    lib.lrnr_host_uniform_grid.argtypes = [i64, i64, dp]
    lib.lrnr_host_harvest_points.argtypes = [dp, i64, i64, i64, C.c_double, C.c_uint64, dp]
    lib.lrnr_host_eim_greedy.argtypes = [i64, i64, dp, i64, dp, dp, dp, dp]
    lib.lrnr_host_build_fastparams.argtypes = [ip, dp, dp, dp, ip, i64, dp, dp, dp, dp]
    lib.lrnr_host_qdeim.argtypes = [i64, i64, dp, dp, dp]
    lib.lrnr_host_build_fast_qdeim.argtypes = [ip, dp, dp, dp, ip, i64, dp, dp, dp]
    lib.lrnr_gpu_eim_greedy.argtypes = [vp, i64, i64, dp, i64, dp, dp, dp, dp]
    lib.lrnr_gpu_harvest_snapshots.argtypes = [vp, ip, dp, dp, dp, ip, dp, i64, dp, i64, i64, C.c_double,
                                               C.c_uint64, dp]
    lib.lrnr_gpu_build_fast.argtypes = [vp, ip, dp, dp, dp, ip, dp, i64, i64, i64, i64, C.c_double, C.c_uint64, i64,
                                        dp, dp, dp, dp]
    lib.lrnr_host_hyper_forward.argtypes = [ip, dp, dp, dp, dp, i64, dp, dp]
    lib.lrnr_gpu_comm_unique_id.argtypes = [vp, C.c_size_t]
    lib.lrnr_gpu_comm_init.argtypes = [vp, ip, ip, vp, C.c_size_t]
    lib.lrnr_gpu_set_comm.argtypes = [vp, vp]
    lib.lrnr_gpu_comm_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.lrnr_gpu_allreduce.argtypes = [vp, vp, i64]
    lib.lrnr_gpu_values.argtypes = [vp, ip, dp, dp, i64, dp]
    lib.lrnr_gpu_loss_tune.argtypes = [vp, ip, dp, dp, dp]
    lib.lrnr_gpu_loss_fast.argtypes = [vp, ip, dp, dp, dp, i64, dp]
    lib.lrnr_gpu_loss_meta.argtypes = [vp, dp, dp]
    _lib = lib
    return lib
