"""Dev aid: why bench.py's LRNR kernel time differs from lrnr_ab.py's (stream, points path,
output pointer, per-step FastLRNR interleave), c2, 1M points, L2 flushed, CUDA events."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_04001_b200 as pkg


def run(side_stream, dev_points, out_ptr, with_fast, n=10):
    c = pkg.config2(with_fast=with_fast)
    s = torch.cuda.Stream() if side_stream else torch.cuda.current_stream()
    torch.cuda.set_stream(s)
    ctx = pkg.GpuContext(0)
    ctx.set_stream(s.cuda_stream)
    ctx.set_lrnr(c["model"], pkg.F32)
    if with_fast:
        ctx.set_fast(c["fast"], pkg.F32)
    if dev_points:
        pd = torch.from_numpy(np.ascontiguousarray(c["pts"])).to("cuda")
        ctx.set_points_device(pd.data_ptr(), len(c["pts"]))
    else:
        ctx.set_points(c["pts"])
    ctx.upload_coeffs(c["s"], c["mu"])
    R1 = 1 + int(np.sum(c["model"].ranks))
    out = torch.zeros(R1, dtype=torch.float64, device="cuda")
    w = 1.0 / len(c["pts"])
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")

    def go():
        ctx.run(pkg.MODEL_LRNR, w, out.data_ptr() if out_ptr else 0)
    for _ in range(3):
        go()
        if with_fast:
            ctx.run(pkg.MODEL_FAST, w, 0)
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); go(); e1.record(s)
        if with_fast:
            ctx.run(pkg.MODEL_FAST, w, 0)
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 3))
    ctx.close()
    torch.cuda.set_stream(torch.cuda.default_stream())
    print(json.dumps(dict(side=side_stream, dev_pts=dev_points, out=out_ptr, fast=with_fast,
                          mean=round(sum(ts) / n, 3), ts=ts)))


run(0, 0, 0, 0)
run(1, 0, 0, 0)
run(0, 1, 0, 0)
run(0, 0, 1, 0)
run(0, 0, 0, 1)
run(1, 1, 1, 1)
