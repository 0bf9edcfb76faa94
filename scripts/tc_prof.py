"""Run the tensor-core kernel on config 2 (for ncu; dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
c = pkg.config2(n_points=n, with_fast=False)
ctx = pkg.GpuContext(0)
ctx.set_option(_lib.OPT_KERNEL, 2)
ctx.set_lrnr(c['model'], pkg.F32); ctx.set_points(c['pts'])
for _ in range(2):
    r = ctx.loss_grad_s(pkg.MODEL_LRNR, c['s'], c['mu'])
print("ok", r['value'])
