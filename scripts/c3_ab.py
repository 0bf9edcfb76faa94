"""Dev aid: c3 (1024 mu x 16,384 points, hypernetwork -> FastLRNR -> VJP) step time per FP32 kernel choice."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_04001_b200 as pkg
N_INST, PER = 1024, 16384
c = pkg.config3(n_inst=N_INST, pts_per_inst=0)
pts = np.concatenate([pkg.sample_collocation(5000 + i, PER) for i in range(N_INST)])
pts_dev = torch.from_numpy(pts).to("cuda")
for kern in (pkg.KERNEL_AUTO, 2):
    ctx = pkg.GpuContext(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s.cuda_stream)
    ctx.set_option(pkg.OPT_KERNEL, kern)
    ctx.set_fast(c["fast"], pkg.F32)
    ctx.set_hyper(c["hyper"])
    ctx.set_points_device(pts_dev.data_ptr(), len(pts), n_inst=N_INST)
    w = 1.0 / (N_INST * PER)
    for _ in range(2):
        r = ctx.hyper_loss_grad(pkg.MODEL_FAST, c["mus"], w)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); r = ctx.hyper_loss_grad(pkg.MODEL_FAST, c["mus"], w); e1.record(s); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"kernel": kern, "median_ms": ts[2], "loss": float(r["value"])}))
    ctx.close()
