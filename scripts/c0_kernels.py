import sys, time, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2410_04001_b200 as pkg
c = pkg.config1()
ctx = pkg.GpuContext(0)
ctx.set_lrnr(c["model"], pkg.F64); ctx.set_fast(c["fast"], pkg.F64); ctx.set_points(c["pts"])
for name, model in (("c0", pkg.MODEL_LRNR), ("c1", pkg.MODEL_FAST)):
    for k in (0, 1, 3, 4):
        ctx.set_option(pkg.OPT_KERNEL, k)
        for _ in range(5): r = ctx.loss_grad_s(model, c["s"], c["mu"])
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(100): r = ctx.loss_grad_s(model, c["s"], c["mu"])
        dt = (time.perf_counter() - t0) / 100
        print(name, "kernel", k, f"{dt*1e6:.1f} us", r["value"])
