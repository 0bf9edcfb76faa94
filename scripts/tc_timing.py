"""Per-phase cycle breakdown of the tensor-core kernel, CTA 0 (dev aid).
LRNR_GPU_LIB=scripts/liblrnr_gpu_timing.so python scripts/tc_timing.py"""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
lib = _lib.load()
n = 148 * 128 * 4
model_fast = len(sys.argv) > 2 and sys.argv[2] == "fast"
c = pkg.config2(n_points=n, with_fast=model_fast)
ctx = pkg.GpuContext(0)
ctx.set_option(_lib.OPT_KERNEL, 2)
ctx.set_option(_lib.OPT_FAST_SINCOS, int(sys.argv[1]) if len(sys.argv) > 1 else 0)
if model_fast:
    ctx.set_fast(c['fast'], pkg.F32)
else:
    ctx.set_lrnr(c['model'], pkg.F32)
ctx.set_points(c['pts'])
MODEL = pkg.MODEL_FAST if model_fast else pkg.MODEL_LRNR
ctx.loss_grad_s(MODEL, c['s'], c['mu'])
out = (C.c_ulonglong * 16)()
lib.lrnr_dev_tc_timing(out)
ctx.loss_grad_s(MODEL, c['s'], c['mu'])
lib.lrnr_dev_tc_timing(out)
names = ["fwd: wait P2(ch-1) + add_y", "fwd: chunk top", "fwd: wait P1", "fwd: epilogue act jet + Z split",
         "fwd: Z store + signal", "fwd: trans end (Y, exchange)", "fwd: trans end (SY / output layer)",
         "bwd: chunk top", "bwd: wait A / DZ", "bwd: epilogue VJP + G split", "bwd: wait P2r(ch-1) + add_t",
         "bwd: G store + signal", "bwd: trans end: syncs + reduce_points", "fwd: trans end: wait P2 + add_y",
         "bwd: trans end: wait P2r + add_t", "bwd: trans end: ds, y loads, exchange, ST / SY"]
tot = sum(out[:16])
tiles = 4
for i in range(16):
    print(f"{names[i]:40s} {out[i]/tiles:12.0f} cycles/tile  {out[i]/tot*100:5.1f}%")
print("total cycles per tile", tot / tiles)
import time
import torch
for _ in range(2): ctx.loss_grad_s(MODEL, c['s'], c['mu'])
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): ctx.loss_grad_s(MODEL, c['s'], c['mu'])
print(f"host-timed per call (n={n}): {(time.perf_counter()-t0)/5*1e3:.3f} ms")
