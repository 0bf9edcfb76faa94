"""Dev aid: c2 FastLRNR sweep (1M points, resident) on each FP32 kernel choice, with its
error against the FP64 oracle on a 16K-point subset."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_04001_b200 as pkg
from oracle.oracle import Oracle

c = pkg.config2(with_fast=True)
small = pkg.config2(n_points=16384, with_fast=True)
O = Oracle()
f = small["fast"]
want = O.fast_grad(f.ranks, f.red_ranks, f.fparams, small["s"], small["mu"], small["pts"], act=pkg.ACT_SIN)
for kern in (pkg.KERNEL_AUTO, 2):
    ctx = pkg.GpuContext(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s.cuda_stream)
    ctx.set_option(pkg.OPT_KERNEL, kern)
    ctx.set_fast(c["fast"], pkg.F32)
    fs = c["fast"]
    ctx.set_points(c["pts"])
    ctx.upload_coeffs(c["s"], c["mu"])
    for _ in range(3):
        ctx.run(pkg.MODEL_FAST, 1.0 / len(c["pts"]))
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); ctx.run(pkg.MODEL_FAST, 1.0 / len(c["pts"])); e1.record(s); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ctx.set_fast(small["fast"], pkg.F32)
    ctx.set_points(small["pts"])
    got = ctx.loss_grad_s(pkg.MODEL_FAST, small["s"], small["mu"])
    err = None
    if want is not None:
        err = float(np.linalg.norm(got["grad_s"] - want["grad_s"]) / np.linalg.norm(want["grad_s"]))
    print(json.dumps({"kernel": kern, "median_ms": ts[5], "grad_rel_err": err}))
    ctx.close()
