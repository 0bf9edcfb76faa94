"""Dev aid: BF16 meta tensor-core kernel vs FP64 oracle and vs the bf16 numpy reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2410_04001_b200 as pkg
from oracle.oracle import Oracle
from bf16_meta_ref import meta_grad
o = Oracle()
nrm = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for act, per in [(pkg.ACT_SIN, 96), (pkg.ACT_SIN, 300), (pkg.ACT_TANH, 300)]:
    n_inst = 2
    c = pkg.config4(n_inst=n_inst, pts_per_inst=per, act=act)
    m, h = c["model"], c["hyper"]
    ctx = pkg.GpuContext(0)
    ctx.set_option(pkg.OPT_META_PREC, 1)
    ctx.set_lrnr(m, pkg.F32); ctx.set_hyper(h); ctx.set_points(c["pts"], n_inst=n_inst)
    got = ctx.meta_loss_grad(c["mus"], m.params.size)
    ctx.set_option(pkg.OPT_META_PREC, 0)
    f32 = ctx.meta_loss_grad(c["mus"], m.params.size)
    nP = m.params.size
    for fmt in ("f64", "bf16"):
        val, want = 0.0, np.zeros(nP + h.n_params)
        for i in range(n_inst):
            s = o.hyper_forward(h.hw, h.params, h.lo, h.hi, c["mus"][i])
            l, ds, g = meta_grad(m, s, c["mus"][i], c["pts"][i * per:(i + 1) * per], fmt, act)
            val += l / n_inst
            want[:nP] += g / n_inst
            o.hyper_vjp(h.hw, h.params, h.lo, h.hi, c["mus"][i], ds / n_inst, out=want[nP:])
        print(f"act {act} per {per} vs {fmt}: loss rel {abs(got['value'] - val) / val:.2e} grad {nrm(got['grad'], want):.2e} "
              f"factors {nrm(got['grad'][:nP], want[:nP]):.2e} hyper {nrm(got['grad'][nP:], want[nP:]):.2e} | fp32 path: "
              f"loss {abs(f32['value'] - val) / val:.2e} grad {nrm(f32['grad'], want):.2e}")
    ctx.close()
