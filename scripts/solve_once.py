"""One fast_solve (persistent solver) and 3 fine_tune epochs (small kernel) on c2, for ncu (dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg
c = pkg.config2(n_points=0, act=pkg.ACT_TANH)
X = np.array([(2 * np.pi * i / 3.0, j / 2.0) for j in range(3) for i in range(4)])
ctx = pkg.GpuContext(0)
ctx.set_lrnr(c["model"], pkg.F32)
ctx.set_fast(c["fast"], pkg.F32)
r = ctx.fast_solve(c["s"], c["mu"], X, 1e-2, 1e-2, 400)
q = ctx.fine_tune(c["s"], c["mu"], 1e-2, 3)
print("ok", r["best_loss"], q["best_loss"])
