"""Dev aid: c4 meta step throughput, BF16 tensor-core kernel vs the FP32 FMA path.
usage: python scripts/meta_tc_time.py [n_inst] [pts_per_inst] [fp32: 0/1]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_04001_b200 as pkg

n_inst = int(sys.argv[1]) if len(sys.argv) > 1 else 2
per = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
with_fp32 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = pkg.config4(n_inst=n_inst, pts_per_inst=per)
m, h = c["model"], c["hyper"]
fl = pkg.algorithmic_flops_per_point(m.widths, m.ranks, meta=True)
ctx = pkg.GpuContext(0)
ctx.set_lrnr(m, pkg.F32)
ctx.set_hyper(h)
ctx.set_points(c["pts"], n_inst=n_inst)
out = {}
for prec in ([1, 0] if with_fp32 else [1]):
    ctx.set_option(pkg.OPT_META_PREC, prec)
    r = ctx.meta_loss_grad(c["mus"], m.params.size)
    torch.cuda.synchronize()
    K = 3 if prec else 1
    t0 = time.perf_counter()
    for _ in range(K):
        r = ctx.meta_loss_grad(c["mus"], m.params.size)
    dt = (time.perf_counter() - t0) / K
    n = n_inst * per
    out[{1: "bf16_tc_v2", 0: "fp32_fma"}[prec]] = dict(ms=dt * 1e3, point_evals_per_s=n / dt, tflops=fl * n / dt / 1e12,
                                                 loss=r["value"], gnorm=float(np.linalg.norm(r["grad"])))
print(json.dumps(out))
