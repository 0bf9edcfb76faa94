"""Dev aid: per-phase cycle counters of the meta tensor-core kernel (CTA 0).
scripts/build_meta_variant.sh timing -DMTC_TIMING && LRNR_GPU_LIB=scripts/liblrnr_gpu_timing.so python scripts/meta_tc_timing.py"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib
per = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
c = pkg.config4(n_inst=1, pts_per_inst=per)
ctx = pkg.GpuContext(0)
ctx.set_option(pkg.OPT_META_PREC, int(os.environ.get("META_PREC", "1")))
ctx.set_lrnr(c["model"], pkg.F32); ctx.set_hyper(c["hyper"]); ctx.set_points(c["pts"], n_inst=1)
lib = _lib.load()
buf = (C.c_ulonglong * 32)()
ctx.meta_loss_grad(c["mus"], c["model"].params.size)
lib.lrnr_mtc_timing(buf)
ctx.meta_loss_grad(c["mus"], c["model"].params.size)
lib.lrnr_mtc_timing(buf)
names = {0: "epi fwd wait p1full", 1: "epi fwd wait zgfree", 2: "epi fwd wait tdone", 4: "epi rev wait p1full",
         5: "epi rev wait zgfree", 6: "epi rev flush (total)", 7: "epi rev wait tdone", 8: "epi rev wait dready",
         9: "epi input layer", 10: "epi fwd chunk loops", 3: "epi tdone waits", 11: "epi fwd transition ends",
         12: "epi output layer + SY rebuild", 13: "epi rev chunk loops (incl flush)", 14: "epi rev end: ds + ST",
         25: "epi rev end: SY rebuild", 15: "epi TOTAL", 16: "iss wait sready", 17: "iss wait full", 18: "iss wait p1empty", 19: "iss wait zgfull",
         20: "iss wait dfree", 21: "iss fwd p1 (v1)", 22: "iss rev p1 (v1)", 23: "iss fwd P2 step (v2)",
         24: "iss rev P2r/dU/dV step (v2)", 31: "iss TOTAL"}
tiles = (per + 63) // 64
tpc = -(-tiles // 148)
print(f"tiles on CTA 0: ~{tpc}")
for k, v in names.items():
    print(f"{v:32s} {buf[k] / 1e6:10.2f} Mcyc  {buf[k] / max(buf[15], 1) * 100:6.1f} %")
