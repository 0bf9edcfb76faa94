"""Tensor-core (option KERNEL=2) vs FMA tile kernel vs FP64 oracle on config 2 (dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
from oracle.oracle import Oracle
O = Oracle()
def nw(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for act in (1, 0):
    c = pkg.config2(n_points=2048, act=act)
    m, f = c['model'], c['fast']
    ctx = pkg.GpuContext(0)
    ctx.set_lrnr(m, pkg.F32); ctx.set_fast(f, pkg.F32); ctx.set_points(c['pts'])
    want = O.lrnr_grad(m.widths, m.ranks, m.params, c['s'], c['mu'], c['pts'], act=act)
    wantf = O.fast_grad(f.ranks, f.red_ranks, f.fparams, c['s'], c['mu'], c['pts'], act=act)
    for kern, fs in ((0, 0), (2, 0), (2, 1)):
        ctx.set_option(_lib.OPT_KERNEL, kern); ctx.set_option(_lib.OPT_FAST_SINCOS, fs)
        g = ctx.loss_grad_s(pkg.MODEL_LRNR, c['s'], c['mu'])
        gf = ctx.loss_grad_s(pkg.MODEL_FAST, c['s'], c['mu'])
        print(f"act={act} kernel={kern} fast={fs}: LRNR loss rel {abs(g['value']-want['value'])/want['value']:.2e} grad nw {nw(g['grad_s'], want['grad_s']):.2e} | "
              f"Fast loss rel {abs(gf['value']-wantf['value'])/wantf['value']:.2e} grad nw {nw(gf['grad_s'], wantf['grad_s']):.2e}", flush=True)
    ctx.close()
n = 1 << 20
c = pkg.config2(n_points=n)
m = c['model']
ctx = pkg.GpuContext(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
ctx.set_lrnr(m, pkg.F32); ctx.set_fast(c['fast'], pkg.F32); ctx.set_points(c['pts']); ctx.upload_coeffs(c['s'], c['mu'])
for kern, fs in ((0, 0), (2, 0), (2, 1)):
    ctx.set_option(_lib.OPT_KERNEL, kern); ctx.set_option(_lib.OPT_FAST_SINCOS, fs)
    for model, name, flops in ((pkg.MODEL_LRNR, 'lrnr', pkg.algorithmic_flops_per_point(m.widths, m.ranks)),
                               (pkg.MODEL_FAST, 'fast', pkg.fast_flops_per_point(c['fast'].ranks, c['fast'].red_ranks))):
        for _ in range(2): ctx.run(model)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): ctx.run(model)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out = ctx.download(1 + m.r_total)
        print(f"kernel={kern} fast={fs} {name}: {ms:.3f} ms  {flops*n/ms/1e9:.2f} TFLOP/s ({flops*n/ms/1e9/74.45*100:.1f}% of FP32 FMA)  loss={out[0]:.9e}", flush=True)
ctx.check()
