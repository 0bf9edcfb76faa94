"""Dev aid: c4 meta step time on the BF16 tensor-core kernel for A/B of builds (LRNR_GPU_LIB).
usage: python scripts/c4_ab.py [n_inst] [pts_per_inst]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_04001_b200 as pkg

n_inst = int(sys.argv[1]) if len(sys.argv) > 1 else 2
per = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
c = pkg.config4(n_inst=n_inst, pts_per_inst=per)
m, h = c["model"], c["hyper"]
fl = pkg.algorithmic_flops_per_point(m.widths, m.ranks, meta=True)
ctx = pkg.GpuContext(0)
ctx.set_lrnr(m, pkg.F32)
ctx.set_hyper(h)
ctx.set_points(c["pts"], n_inst=n_inst)
ctx.set_option(pkg.OPT_META_PREC, 1)
r = ctx.meta_loss_grad(c["mus"], m.params.size)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    r = ctx.meta_loss_grad(c["mus"], m.params.size)
    ts.append(time.perf_counter() - t0)
ts.sort()
dt = ts[2]
n = n_inst * per
print(json.dumps(dict(lib=os.environ.get("LRNR_GPU_LIB", "default"), ms=dt * 1e3, tflops=fl * n / dt / 1e12, loss=r["value"],
                      gnorm=float(np.linalg.norm(r["grad"])))))
