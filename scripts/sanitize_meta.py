"""Dev aid: one small meta step on each tensor-core meta kernel (run under compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg
c = pkg.config4(n_inst=2, pts_per_inst=200)
ctx = pkg.GpuContext(0)
ctx.set_lrnr(c["model"], pkg.F32)
ctx.set_hyper(c["hyper"])
ctx.set_points(c["pts"], n_inst=2)
for prec in (1, 2):
    ctx.set_option(pkg.OPT_META_PREC, prec)
    r = ctx.meta_loss_grad(c["mus"], c["model"].params.size)
    print(prec, r["value"], float(np.linalg.norm(r["grad"])))
