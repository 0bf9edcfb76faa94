"""Dev aid: median fine_tune ms/epoch (c2 LRNR FP32, 1024 + 256 + 256 points,
100 epochs) over several runs, for A/B builds selected with LRNR_GPU_LIB
(e.g. scripts/build_timing.sh -D<switch> for the B side)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_04001_b200 as pkg  # noqa: E402

c = pkg.config2(n_points=0, act=pkg.ACT_TANH, with_fast=False)
ctx = pkg.GpuContext(0)
ctx.set_lrnr(c["model"], pkg.F32)
mu = np.array([20.0, 0.01, 5.0])
ts = []
for rep in range(7):
    t0 = time.perf_counter()
    r = ctx.fine_tune(c["s"], mu, lr=1e-2, epochs=100, n_int=1024, n_ic=256, n_bc=256, seed=1234)
    ts.append((time.perf_counter() - t0) / 100 * 1e3)
print(os.environ.get("LRNR_GPU_LIB", "default"), "fine_tune ms/epoch median %.3f" % np.median(ts[1:]),
      "all", ["%.3f" % t for t in ts], "best", r["best_loss"])
