"""Dev aid: c2 LRNR sweep time (CUDA events, 1M points, points resident) for A/B of builds."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_04001_b200 as pkg
c = pkg.config2(with_fast=False)
ctx = pkg.GpuContext(0)
s = torch.cuda.current_stream()
ctx.set_stream(s.cuda_stream)
ctx.set_lrnr(c["model"], pkg.F32)
ctx.set_points(c["pts"])
ctx.upload_coeffs(c["s"], c["mu"])
for _ in range(3):
    ctx.run(pkg.MODEL_LRNR, 1.0 / len(c["pts"]))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB > L2
for fl in (0, 1):
    ts = []
    for _ in range(10):
        if fl:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); ctx.run(pkg.MODEL_LRNR, 1.0 / len(c["pts"])); e1.record(s); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"lib": os.environ.get("LRNR_GPU_LIB", "default"), "l2_flush": fl, "median_ms": ts[5],
                      "min_ms": ts[0]}))
