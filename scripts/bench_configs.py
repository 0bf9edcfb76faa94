"""Throughput of the non-headline BASELINE configs on one GPU (measurement record):
c3 = hypernetwork -> FastLRNR per instance + hypernet VJP (1024 mu x 16,384 pts),
c4 = meta step (U, V, b, theta gradients; 64 mu x 1,048,576 pts per step on the BF16 tensor-core kernel, 2 of them on the FP32 FMA path).
Device time with CUDA events around the host-buffer call (points resident)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_04001_b200 as pkg

PEAK = 74.45
out = {}
# c0 / c1 (FP64, 4096 points): one gradient call each, device time over 200 calls
# (launch-latency bound at this size; FP64 FMA peak = half the FP32 one)
c = pkg.config1()
ctx = pkg.GpuContext(0)
ctx.set_lrnr(c["model"], pkg.F64)
ctx.set_fast(c["fast"], pkg.F64)
ctx.set_points(c["pts"])
for key, model, fl in (("c0", pkg.MODEL_LRNR, pkg.algorithmic_flops_per_point(c["model"].widths, c["model"].ranks)),
                       ("c1", pkg.MODEL_FAST, pkg.fast_flops_per_point(c["fast"].ranks, c["fast"].red_ranks))):
    for _ in range(5):
        ctx.loss_grad_s(model, c["s"], c["mu"])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        r = ctx.loss_grad_s(model, c["s"], c["mu"])
    dt = (time.perf_counter() - t0) / 200
    n = len(c["pts"])
    out[key] = {"us_per_call": dt * 1e6, "point_evals_per_s": n / dt, "tflops": fl * n / dt / 1e12,
                "frac_fp64_fma": fl * n / dt / 1e12 / (PEAK / 2), "flop_per_point": fl, "points": n,
                "loss": r["value"], "path": "lrnr_gpu_loss_grad_s (host buffers in / out), FP64"}
ctx.close()
# c3
c = pkg.config3(n_inst=1024, pts_per_inst=16384)
ctx = pkg.GpuContext(0)
ctx.set_fast(c["fast"], pkg.F32)
ctx.set_hyper(c["hyper"])
ctx.set_points(c["pts"], n_inst=1024)
ctx.hyper_loss_grad(pkg.MODEL_FAST, c["mus"])
torch.cuda.synchronize()
t0 = time.perf_counter()
K = 3
for _ in range(K):
    r = ctx.hyper_loss_grad(pkg.MODEL_FAST, c["mus"])
dt = (time.perf_counter() - t0) / K
n = 1024 * 16384
fl = pkg.fast_flops_per_point(c["fast"].ranks, c["fast"].red_ranks)
out["c3"] = {"ms_per_step": dt * 1e3, "point_evals_per_s": n / dt, "tflops": fl * n / dt / 1e12,
             "frac_fp32_fma": fl * n / dt / 1e12 / PEAK, "flop_per_point": fl, "points": n,
             "kernel": "narrow-network kernel (FastLRNR, auto) + FP64 hypernetwork fwd/VJP", "loss": r["value"]}
ctx.close()
# c4: the full meta step (64 instances x 1,048,576 points) on the tcgen05 meta kernel
# (BF16 operands, FP32 accumulate), and 2 of the 64 instances on the FP32 FMA tile kernel
for prec, n_inst in ((1, 64), (0, 2)):
    per = 1 << 20
    c = pkg.config4(n_inst=n_inst, pts_per_inst=per)
    ctx = pkg.GpuContext(0)
    ctx.set_option(pkg.OPT_META_PREC, prec)
    ctx.set_lrnr(c["model"], pkg.F32)
    ctx.set_hyper(c["hyper"])
    ctx.set_points(c["pts"], n_inst=n_inst)
    ctx.meta_loss_grad(c["mus"], c["model"].params.size)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ctx.meta_loss_grad(c["mus"], c["model"].params.size)
    dt = time.perf_counter() - t0
    n = n_inst * per
    fl = pkg.algorithmic_flops_per_point(c["model"].widths, c["model"].ranks, meta=True)
    key = "c4_bf16_tc" if prec else "c4_fp32_fma"
    out[key] = {"instances": n_inst, "ms_per_step": dt * 1e3, "point_evals_per_s": n / dt, "tflops": fl * n / dt / 1e12,
                "frac_fp32_fma": fl * n / dt / 1e12 / PEAK, "frac_bf16_sustained": fl * n / dt / 1e12 / 1398.4,
                "flop_per_point": fl, "points": n, "loss": r["value"],
                "kernel": "meta_tc2_kernel (tcgen05, BF16 operands, FP32 accumulate) + FP64 hypernetwork" if prec else
                "FMA tile (META phase 3, FP32) + FP64 hypernetwork"}
    ctx.close()
print(json.dumps(out))
