"""B200: the tensor-core kernel's FP16 two-term split with power-of-two scales
(csrc/pinn_tc.cuh: SY / ST rows scaled by their exact norms, Z / G rows by
Cauchy-Schwarz bounds, factors per matrix) on inputs that stress the scaling:
zero and tiny coefficients s, factors scaled by 1e2 / 1e-2, points far outside
the domain, tanh saturation, odd widths and ranks.  Every case against the FP64
oracle (the restated emit_lrnr_jet + run_batch_gradient) at the FP32 tolerance."""
import numpy as np
import pytest

import paper_2410_04001_b200 as pkg
from conftest import normwise

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _run_tc(gpu, m, s, mu, pts):
    gpu.set_option(pkg.OPT_KERNEL, pkg.KERNEL_TC)
    try:
        gpu.set_lrnr(m, pkg.F32)
        gpu.set_points(pts)
        return gpu.loss_grad_s(pkg.MODEL_LRNR, s, mu)
    finally:
        gpu.set_option(pkg.OPT_KERNEL, pkg.KERNEL_AUTO)


def _check(gpu, oracle, m, s, mu, pts):
    got = _run_tc(gpu, m, s, mu, pts)
    want = oracle.lrnr_grad(m.widths, m.ranks, m.params, s, mu, pts, act=m.act)
    assert np.isfinite(got["value"]) and np.all(np.isfinite(got["grad_s"]))
    assert abs(got["value"] - want["value"]) <= TOL * abs(want["value"])
    assert normwise(got["grad_s"], want["grad_s"]) <= TOL


def _c2(n=1500, act=pkg.ACT_SIN):
    c = pkg.config2(n_points=n, act=act, with_fast=False)
    return c["model"], np.array(c["s"], dtype=np.float64), c["mu"], c["pts"]


def _scale_factors(m, fac):
    """U_l and V_l of transition l multiplied by fac[l] (biases unchanged)."""
    p = np.array(m.params, dtype=np.float64)
    offs, _ = m.offsets()
    for l, (oU, oV, ob) in enumerate(offs):
        p[oU:oV] *= fac[l % len(fac)]
        p[oV:ob] *= fac[l % len(fac)]
    return pkg.LrnrParams(m.widths, m.ranks, p, m.act)


def test_zero_and_tiny_coefficients(gpu, oracle):
    m, s, mu, pts = _c2()
    rng = np.random.default_rng(5)
    idx = rng.permutation(len(s))
    s[idx[:len(s) // 8]] = 0.0           # truncated modes: all-zero SY rank columns
    s[idx[len(s) // 8:len(s) // 4]] *= 1e-6
    _check(gpu, oracle, m, s, mu, pts)


def test_factors_scaled_up_and_down(gpu, oracle):
    m, s, mu, pts = _c2()
    _check(gpu, oracle, _scale_factors(m, [4.0, 0.25]), s, mu, pts)
    _check(gpu, oracle, _scale_factors(m, [1e-2]), s, mu, pts)


def test_points_far_outside_the_domain(gpu, oracle):
    m, s, mu, _ = _c2()
    rng = np.random.default_rng(6)
    pts = np.column_stack([rng.uniform(-40.0, 40.0, 1500), rng.uniform(-6.0, 6.0, 1500)])
    _check(gpu, oracle, m, s, mu, pts)


def test_tanh_saturation(gpu, oracle):
    m, s, mu, pts = _c2(act=pkg.ACT_TANH)
    _check(gpu, oracle, _scale_factors(m, [3.0]), s, mu, pts)


@pytest.mark.parametrize("act", [pkg.ACT_SIN, pkg.ACT_TANH])
def test_odd_widths_and_ranks(gpu, oracle, act):
    widths, ranks = [2, 70, 45, 33, 1], [2, 13, 9, 1]
    m, s = pkg.make_baseline_model(widths, ranks, 91, act)
    pts = pkg.sample_collocation(92, 777)
    _check(gpu, oracle, m, np.array(s, dtype=np.float64), np.array([7.0, 0.02, 1.5]), pts)
