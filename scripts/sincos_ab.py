"""Dev aid: c2 LRNR on the tensor-core kernel with polynomial vs SFU sin/cos (LRNR_OPT_FAST_SINCOS): time and error vs the FP64 oracle."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
from oracle.oracle import Oracle
O = Oracle()
c = pkg.config2(with_fast=False)
ce = pkg.config2(n_points=65536, with_fast=False)
m = ce["model"]
want = O.lrnr_grad(m.widths, m.ranks, m.params, ce["s"], ce["mu"], ce["pts"], act=pkg.ACT_SIN)
for fs in (0, 1):
    ctx = pkg.GpuContext(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s.cuda_stream)
    ctx.set_option(_lib.OPT_FAST_SINCOS, fs)
    ctx.set_lrnr(ce["model"], pkg.F32); ctx.set_points(ce["pts"])
    got = ctx.loss_grad_s(pkg.MODEL_LRNR, ce["s"], ce["mu"])
    e = np.linalg.norm(got["grad_s"] - want["grad_s"]) / np.linalg.norm(want["grad_s"])
    le = abs(got["value"] - want["value"]) / want["value"]
    ctx.set_points(c["pts"]); ctx.upload_coeffs(c["s"], c["mu"])
    for _ in range(3):
        ctx.run(pkg.MODEL_LRNR, 1.0 / len(c["pts"]))
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); ctx.run(pkg.MODEL_LRNR, 1.0 / len(c["pts"])); e1.record(s); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"fast_sincos": fs, "median_ms": ts[5], "dlds_normwise": e, "loss_rel": le}))
    ctx.close()
