"""Dev aid: device time of the c0 / c1 FP64 gradient sweeps per kernel choice (LRNR_OPT_KERNEL)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
c = pkg.config1()
for kern in (0, 1, 3, 4):
    ctx = pkg.GpuContext(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s.cuda_stream)
    ctx.set_option(_lib.OPT_KERNEL, kern)
    ctx.set_lrnr(c["model"], pkg.F64)
    ctx.set_fast(c["fast"], pkg.F64)
    ctx.set_points(c["pts"])
    ctx.upload_coeffs(c["s"], c["mu"])
    for name, model in (("c0", pkg.MODEL_LRNR), ("c1", pkg.MODEL_FAST)):
        for _ in range(5):
            ctx.run(model, 1.0 / len(c["pts"]))
        ts = []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); ctx.run(model, 1.0 / len(c["pts"])); e1.record(s); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(json.dumps({"kernel_opt": kern, "config": name, "median_us": round(ts[25] * 1e3, 1)}))
    ctx.close()
