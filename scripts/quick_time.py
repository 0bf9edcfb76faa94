"""Quick device timing of the fused kernels on BASELINE config 2 (dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20)
c = pkg.config2(n_points=n)
ctx = pkg.GpuContext(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
ctx.set_lrnr(c['model'], pkg.F32); ctx.set_fast(c['fast'], pkg.F32); ctx.set_points(c['pts'])
ctx.upload_coeffs(c['s'], c['mu'])
m = c['model']
for kern, tp in ((0, 64), (0, 32)):
    for fast in (0, 1):
        ctx.set_option(_lib.OPT_KERNEL, kern); ctx.set_option(_lib.OPT_FAST_SINCOS, fast); ctx.set_option(_lib.OPT_TILE_P, tp)
        for model, name, flops in ((pkg.MODEL_LRNR, 'lrnr', pkg.algorithmic_flops_per_point(m.widths, m.ranks)),
                                   (pkg.MODEL_FAST, 'fast', pkg.fast_flops_per_point(c['fast'].ranks, c['fast'].red_ranks))):
            for _ in range(2): ctx.run(model)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 3 if kern == 1 else 10
            e0.record()
            for _ in range(K): ctx.run(model)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
            out = ctx.download(1 + m.r_total)
            print(f"tile P={tp} fastsin={fast} {name}: {ms:.3f} ms/step  {n/ms*1e3:.3e} pt/s  {flops*n/ms/1e9:.2f} TFLOP/s ({flops*n/ms/1e9/74.45*100:.1f}% of FP32)  loss={out[0]:.9e} g0={out[1]:.6e}")
ctx.check()
