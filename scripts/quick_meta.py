"""Quick device timing of the meta (c4) step (dev aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg
n_inst, per = int(sys.argv[1]), int(sys.argv[2])
c = pkg.config4(n_inst=n_inst, pts_per_inst=per)
ctx = pkg.GpuContext(0)
ctx.set_lrnr(c['model'], pkg.F32); ctx.set_hyper(c['hyper']); ctx.set_points(c['pts'], n_inst=n_inst)
r = ctx.meta_loss_grad(c['mus'], c['model'].params.size)
t0 = time.perf_counter(); K = 3
for _ in range(K): r = ctx.meta_loss_grad(c['mus'], c['model'].params.size)
dt = (time.perf_counter() - t0) / K
n = n_inst * per
fl = pkg.algorithmic_flops_per_point(c['model'].widths, c['model'].ranks, meta=True)
print(f"meta c4 {n_inst}x{per}: {dt*1e3:.1f} ms/step {n/dt:.3e} pt/s {fl*n/dt/1e12:.2f} TFLOP/s loss={r['value']:.6e} |g|={np.linalg.norm(r['grad']):.4e}")
