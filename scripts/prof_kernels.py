"""One launch each of the dominant kernels for an ncu --set full capture (dev aid):
pinn_tc_kernel (c2 LRNR and FastLRNR r_hat 32, 1M points each; c3 FastLRNR 64 mu x 16,384 points),
meta_tc2_kernel (c4 meta, 2 instances x 1M points), pinn_tile_kernel (c0 LRNR FP64, 4096 points).
  python scripts/prof_kernels.py [which...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg

which = sys.argv[1:] or ["c2", "c3", "c4", "c0"]
ctx = pkg.GpuContext(0)
if "c2" in which:
    c = pkg.config2()
    ctx.set_lrnr(c["model"], pkg.F32)
    ctx.set_fast(c["fast"], pkg.F32)
    ctx.set_points(c["pts"])
    for model in (pkg.MODEL_LRNR, pkg.MODEL_FAST):
        r = ctx.loss_grad_s(model, c["s"], c["mu"])
        print("c2", model, r["value"])
if "c3" in which:
    c = pkg.config3(n_inst=64, pts_per_inst=16384)
    ctx.set_fast(c["fast"], pkg.F32)
    ctx.set_hyper(c["hyper"])
    ctx.set_points(c["pts"], n_inst=64)
    r = ctx.hyper_loss_grad(pkg.MODEL_FAST, c["mus"], 1.0 / len(c["pts"]))
    print("c3", r["value"])
if "c4" in which:
    c = pkg.config4(n_inst=2, pts_per_inst=1 << 20)
    ctx.set_option(pkg.OPT_META_PREC, 1)
    ctx.set_lrnr(c["model"], pkg.F32)
    ctx.set_hyper(c["hyper"])
    ctx.set_points(c["pts"], n_inst=2)
    r = ctx.meta_loss_grad(c["mus"], c["model"].params.size)
    print("c4", r["value"])
if "c0" in which:
    c = pkg.config1()
    ctx.set_lrnr(c["model"], pkg.F64)
    ctx.set_fast(c["fast"], pkg.F64)
    ctx.set_points(c["pts"])
    for model in (pkg.MODEL_LRNR, pkg.MODEL_FAST):
        r = ctx.loss_grad_s(model, c["s"], c["mu"])
        print("c0/c1", model, r["value"])
ctx.close()
