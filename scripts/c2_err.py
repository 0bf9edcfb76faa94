import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2410_04001_b200 as pkg
from oracle.oracle import Oracle
O = Oracle()
for n in (8192, 65536):
    c2 = pkg.config2(n_points=n, with_fast=False)
    ctx = pkg.GpuContext(0)
    ctx.set_lrnr(c2["model"], pkg.F32); ctx.set_points(c2["pts"])
    got = ctx.loss_grad_s(pkg.MODEL_LRNR, c2["s"], c2["mu"])
    m = c2["model"]
    want = O.lrnr_grad(m.widths, m.ranks, m.params, c2["s"], c2["mu"], c2["pts"], act=pkg.ACT_SIN)
    e = np.linalg.norm(got["grad_s"] - want["grad_s"]) / np.linalg.norm(want["grad_s"])
    print(os.environ.get("LRNR_GPU_LIB", "default"), n, f"dL/ds normwise {e:.2e} loss rel {abs(got['value'] - want['value']) / want['value']:.2e}")
    ctx.close()
