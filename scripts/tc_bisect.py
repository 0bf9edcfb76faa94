"""Bisect the tensor-core kernel error vs the FP64 oracle over shapes (dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
from oracle.oracle import Oracle
O = Oracle()
ctx = pkg.GpuContext(0)
def run(widths, ranks, n, act=1, seed=5):
    m, s = pkg.make_baseline_model(widths, ranks, seed, act)
    pts = pkg.sample_collocation(seed + 1, n)
    mu = np.array([20.0, 0.01, 5.0])
    want = O.lrnr_grad(m.widths, m.ranks, m.params, s, mu, pts, act=act)
    ctx.set_lrnr(m, pkg.F32); ctx.set_points(pts)
    res = []
    for k in (0, 2):
        ctx.set_option(_lib.OPT_KERNEL, k)
        g = ctx.loss_grad_s(pkg.MODEL_LRNR, s, mu)
        res.append((abs(g['value'] - want['value']) / abs(want['value']), np.linalg.norm(g['grad_s'] - want['grad_s']) / np.linalg.norm(want['grad_s'])))
    print(f"{str(widths):40s} {str(ranks):28s} n={n:5d}  FMA loss {res[0][0]:.1e} grad {res[0][1]:.1e} | TC loss {res[1][0]:.1e} grad {res[1][1]:.1e}", flush=True)
run([2, 32, 1], [2, 1], 128)
run([2, 64, 1], [2, 1], 128)
run([2, 256, 1], [2, 1], 128)
run([2, 32, 32, 1], [2, 32, 1], 128)
run([2, 64, 64, 1], [2, 32, 1], 128)
run([2, 256, 256, 1], [2, 32, 1], 128)
run([2, 32, 32, 32, 1], [2, 32, 32, 1], 128)
run([2, 256, 256, 256, 1], [2, 32, 32, 1], 128)
run([2] + [256] * 6 + [1], [2] + [32] * 5 + [1], 128)
run([2] + [256] * 6 + [1], [2] + [32] * 5 + [1], 128, act=0)
run([2, 256, 256, 1], [2, 32, 1], 1)
print("---")
W, R = [2] + [256] * 6 + [1], [2] + [32] * 5 + [1]
for n in (128, 256, 1024, 2048):
    run(W, R, n, act=1, seed=2411)
run(W, R, 2048, act=1, seed=5)
def run_c2(n):
    c = pkg.config2(n_points=n, act=1, with_fast=False)
    m, s, pts, mu = c['model'], c['s'], c['pts'], c['mu']
    want = O.lrnr_grad(m.widths, m.ranks, m.params, s, mu, pts, act=1)
    ctx.set_lrnr(m, pkg.F32); ctx.set_points(pts)
    for k in (0, 2):
        ctx.set_option(_lib.OPT_KERNEL, k)
        g = ctx.loss_grad_s(pkg.MODEL_LRNR, s, mu)
        print(f"config2 n={n} kernel={k}: loss rel {abs(g['value']-want['value'])/want['value']:.2e} grad {np.linalg.norm(g['grad_s']-want['grad_s'])/np.linalg.norm(want['grad_s']):.2e}", flush=True)
run_c2(128); run_c2(2048)
