"""Wall time of the solve loops on the device vs the reference CPU loops (dev aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg
from oracle.oracle import Reference, reference_available
c = pkg.config2(n_points=0, act=pkg.ACT_TANH)
m, f = c["model"], c["fast"]
X = np.array([(2 * np.pi * i / 3.0, j / 2.0) for j in range(3) for i in range(4)])
ctx = pkg.GpuContext(0)
for dt in (pkg.F32, pkg.F64):
    ctx.set_lrnr(m, dt); ctx.set_fast(f, dt)
    ctx.fast_solve(c["s"], c["mu"], X, 1e-2, 1e-2, 5)
    t = time.perf_counter(); r = ctx.fast_solve(c["s"], c["mu"], X, 1e-2, 1e-2, 400); tf = time.perf_counter() - t
    ctx.fine_tune(c["s"], c["mu"], 1e-2, 3)
    t = time.perf_counter(); q = ctx.fine_tune(c["s"], c["mu"], 1e-2, 400); tt = time.perf_counter() - t
    print(f"device {'f32' if dt == pkg.F32 else 'f64'}: fast_solve 400 ep {tf*1e3:.1f} ms ({tf/400*1e6:.1f} us/epoch), "
          f"fine_tune 400 ep x (1024+256+256) {tt*1e3:.1f} ms ({tt/400*1e6:.1f} us/epoch); best {r['best_loss']:.6g} {q['best_loss']:.6g}")
if reference_available():
    R = Reference()
    th = os.cpu_count()
    t = time.perf_counter(); a = R.fast_solve(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], X, 1e-2, 1e-2, 400, threads=th)
    tf = time.perf_counter() - t
    t = time.perf_counter(); b = R.fine_tune(m.widths, m.ranks, m.params, c["s"], c["mu"], 1e-2, 20, 1024, 256, 256, 1234, threads=th)
    tt = (time.perf_counter() - t) * 20
    print(f"reference ({th} threads, f64 tanh): fast_solve 400 ep {tf*1e3:.1f} ms; fine_tune 400 ep ~{tt*1e3:.0f} ms (20-epoch sample x20); best {a['best_loss']:.6g}")
