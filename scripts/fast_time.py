"""Time the FastLRNR sweep (c2, 1M points) under each LRNR_OPT_KERNEL (dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_04001_b200 as pkg
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20)
c = pkg.config2(n_points=n)
ctx = pkg.GpuContext(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
ctx.set_fast(c['fast'], pkg.F32); ctx.set_points(c['pts']); ctx.upload_coeffs(c['s'], c['mu'])
fl = pkg.fast_flops_per_point(c['fast'].ranks, c['fast'].red_ranks)
for kern, tp in ((pkg.KERNEL_NARROW, 64), (pkg.KERNEL_FMA_TILE, 64), (pkg.KERNEL_TC, 64)):
    ctx.set_option(pkg.OPT_KERNEL, kern)
    ctx.set_option(pkg.OPT_TILE_P, tp)
    ctx.set_fast(c['fast'], pkg.F32)
    for _ in range(2): ctx.run(pkg.MODEL_FAST)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 5
    e0.record(st)
    for _ in range(K): ctx.run(pkg.MODEL_FAST)
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    out = ctx.download(1 + c['model'].r_total)
    print(f"kernel={kern} tile_p={tp} fast: {ms:.3f} ms  {fl*n/ms/1e9:.2f} TFLOP/s ({fl*n/ms/1e9/74.45*100:.1f}%)  loss={out[0]:.9e}")
ctx.check()
