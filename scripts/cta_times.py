"""Dev aid: per-CTA start/end of the c2 LRNR tensor-core sweep (a -DTC_CTA_TIMES build that
printf's globaltimer per CTA): is the 22..25 ms run-to-run spread load imbalance?"""
import os, sys, subprocess, collections
if len(sys.argv) > 1:
    lines = [l.split() for l in open(sys.argv[1]) if l.startswith("CTA ")]
    runs = [lines[i:i + 148] for i in range(0, len(lines), 148)]
    for r in runs:
        t0 = min(int(x[3]) for x in r)
        s = min(int(x[3]) for x in r) - t0
        ends = sorted((int(x[4]) - t0) / 1e6 for x in r)
        starts = sorted((int(x[3]) - t0) / 1e6 for x in r)
        durs = sorted((int(x[4]) - int(x[3])) / 1e6 for x in r)
        slow = sorted(r, key=lambda x: int(x[3]) - int(x[4]))[:3]
        print(f"end max {ends[-1]:.2f} min {ends[0]:.2f} med {ends[74]:.2f} | start max {starts[-1]:.3f} | dur min {durs[0]:.2f} max {durs[-1]:.2f}"
              f" | slowest sm {[x[2] for x in slow]} tiles {[x[5] for x in slow]}")
    sys.exit()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_04001_b200 as pkg
c = pkg.config2(with_fast=False)
ctx = pkg.GpuContext(0)
ctx.set_lrnr(c["model"], pkg.F32)
ctx.set_points(c["pts"])
ctx.upload_coeffs(c["s"], c["mu"])
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(8):
    flush.zero_()
    ctx.run(pkg.MODEL_LRNR, 1.0 / len(c["pts"]))
    torch.cuda.synchronize()
