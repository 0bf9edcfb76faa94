"""B200: FastLRNR construction on the device.

lrnr_gpu_eim_greedy must select the same interpolation indices and produce the
same basis columns as reduction::eim_greedy BIT-FOR-BIT (golden fixtures made by
the reference; larger / NaN / tie cases against the host restatement, itself
pinned to the reference in tests/test_host.py). lrnr_gpu_build_fast harvests on
the device with the reference's own tanh (glibc's fdlibm tanh/expm1, restated in
eim.cu) and the reference build's rounding, so for tanh networks the whole
FastLRNR construction is bit-identical to the reference: c2's deep layers exhaust
the EIM budget, where even one-ulp snapshot differences reach the late basis
columns (1e-3 in the gradient), so nothing weaker would pin it. The sin
activation (this build's extension) uses CUDA's sin: tolerance there.
"""
import numpy as np
import pytest

import paper_2410_04001_b200 as pkg
from conftest import floor_rel

pytestmark = pytest.mark.gpu

EIM_TAGS = ["a", "b", "c", "d"]


def maxnorm_rel(got, want):
    return float(np.abs(got - want).max() / np.abs(want).max())


@pytest.mark.parametrize("tag", EIM_TAGS)
def test_eim_greedy_bit_exact(gpu, golden, tag):
    e = gpu.eim_greedy(golden[f"eim_{tag}_S"], int(golden[f"eim_{tag}_rhat"][0]))
    assert np.array_equal(e["indices"], golden[f"eim_{tag}_idx"])
    assert np.array_equal(e["xi"], golden[f"eim_{tag}_xi"])
    assert e["exhausted"] == bool(golden[f"eim_{tag}_exh"][0])


@pytest.mark.parametrize("shape,r_hat", [((32, 20000), 24), ((7, 129), 7), ((40, 3000), 64)])
def test_eim_greedy_matches_host_at_size(gpu, shape, r_hat):
    rng = np.random.default_rng(shape[1])
    S = np.tanh(rng.normal(0, 1, (shape[0], 6)) @ rng.normal(0, 1, (6, shape[1])) +
                0.05 * rng.normal(0, 1, shape))
    want = pkg.eim_greedy(S, r_hat)
    got = gpu.eim_greedy(S, r_hat)
    assert np.array_equal(got["indices"], want["indices"])
    assert np.array_equal(got["xi"], want["xi"])
    assert got["exhausted"] == want["exhausted"]


def test_eim_greedy_nan_and_ties_follow_cpu(gpu):
    """A NaN residual is skipped by the max-norm (std::max), ties go to the first column."""
    rng = np.random.default_rng(5)
    S = np.repeat(rng.normal(0, 1, (12, 30)), 3, axis=1)
    S[4, 7] = np.nan
    want = pkg.eim_greedy(S, 10)
    got = gpu.eim_greedy(S, 10)
    assert np.array_equal(got["indices"], want["indices"])
    assert np.array_equal(got["xi"], want["xi"], equal_nan=True)


def test_eim_greedy_errors(gpu):
    with pytest.raises(ValueError):
        gpu.eim_greedy(np.ones((4, 3)), 0)
    with pytest.raises(ValueError):
        gpu.eim_greedy(np.zeros((4, 3)), 2)  # no basis vector selected
    with pytest.raises(ValueError):
        gpu.eim_greedy(np.ones((80, 3)), 65)  # device budget cap


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_build_fast_matches_reference(gpu, golden, cfg):
    src, r_hat = ("c0", 10) if cfg == "c1" else ("c2", 32)
    m = pkg.LrnrParams(golden[f"{src}_widths"], golden[f"{src}_ranks"], golden[f"{src}_params"], pkg.ACT_TANH)
    f = gpu.build_fast(m, golden[f"{src}_s"], nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=r_hat)
    assert np.array_equal(f.indices, golden[f"{cfg}_indices"])
    assert np.array_equal(f.red_ranks, golden[f"{cfg}_red_ranks"])
    assert np.array_equal(f.fparams, golden[f"{cfg}_fparams"])
    # the FastLRNR built on the device gives the reference FastLRNR's FP64 gradient
    pts, grad_key, val_key = ("c0_pts", "c1_grad_s", "c1_value") if cfg == "c1" else \
        ("c2_pts", "c2_fast_grad_s", "c2_fast_value")
    gpu.set_fast(f, pkg.F64)
    gpu.set_points(golden[pts])
    r = gpu.loss_grad_s(pkg.MODEL_FAST, golden[f"{src}_s"], golden[f"{src}_mu"])
    print(cfg, "value rel", abs(r["value"] / golden[val_key][0] - 1), "grad floor_rel",
          floor_rel(r["grad_s"], golden[grad_key]))
    assert abs(r["value"] - golden[val_key][0]) <= 1e-12 * abs(golden[val_key][0])
    assert floor_rel(r["grad_s"], golden[grad_key]) <= 1e-10


@pytest.mark.parametrize("act", [pkg.ACT_TANH, pkg.ACT_SIN])
def test_build_fast_many_mu_matches_host(gpu, golden, act):
    """n_mu coefficient vectors (the hyper_forward outputs of a mu grid), c2 widths."""
    m = pkg.LrnrParams(golden["c2_widths"], golden["c2_ranks"], golden["c2_params"], act)
    rng = np.random.default_rng(3)
    s = golden["c2_s"][None, :] * rng.uniform(0.5, 1.5, (24, m.r_total))
    want = pkg.build_fast(m, s, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=99, r_hat=20)
    got = gpu.build_fast(m, s, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=99, r_hat=20)
    assert np.array_equal(got.indices, want.indices)
    assert np.array_equal(got.exhausted, want.exhausted)
    if act == pkg.ACT_TANH:
        assert np.array_equal(got.fparams, want.fparams)
    else:
        assert maxnorm_rel(got.fparams, want.fparams) <= 1e-6
    # exact composition: the device build == host EIM + host assembly on the device snapshots
    snaps = gpu.harvest_snapshots(m, s, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=99)
    exact = pkg.build_fastparams(m, [pkg.eim_greedy(S, 20) for S in snaps], r_hat=20)
    assert np.array_equal(got.indices, exact.indices)
    assert np.array_equal(got.fparams, exact.fparams)


@pytest.mark.parametrize("act", [pkg.ACT_TANH, pkg.ACT_SIN])
def test_harvest_snapshots_match_numpy(gpu, golden, act):
    """Device hidden states vs an FP64 numpy forward (model.cpp:407-428) at the harvest points."""
    m = pkg.LrnrParams(golden["c2_widths"], golden["c2_ranks"], golden["c2_params"], act)
    s = np.stack([golden["c2_s"], 0.7 * golden["c2_s"]])
    snaps = gpu.harvest_snapshots(m, s, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=5)
    X = pkg.harvest_points(2, 4, 3, 8, 0.05, 5)
    offs, _ = m.offsets()
    for mi in range(2):
        z, so = X[mi * 108:(mi + 1) * 108].T, 0
        for l in range(m.depth - 1):
            w0, w1, r = int(m.widths[l]), int(m.widths[l + 1]), int(m.ranks[l])
            oU, oV, ob = offs[l]
            U, V, b = (m.params[oU:oU + w1 * r].reshape(w1, r), m.params[oV:oV + w0 * r].reshape(w0, r),
                       m.params[ob:ob + w1])
            a = U @ ((V.T @ z) * s[mi, so:so + r, None]) + b[:, None]
            z = np.sin(a) if act == pkg.ACT_SIN else np.tanh(a)
            so += r
            assert np.abs(snaps[l][:, mi * 108:(mi + 1) * 108] - z).max() <= 1e-13


def test_glibc_tanh_restatement_matches_host_libm(gpu):
    """The device tanh used by the harvest == the host's libm tanh (math.tanh) bit for bit.
    A (2, 1, 1) rank-1 net with V^0 = (1, 0), s = 1 makes the pre-activation exactly
    U*x + b (IEEE, no fusion: a one-term ref_dot is one rounded product), so the
    harvested column for grid point x is tanh(U*x + b)."""
    import math

    nx = 2000
    xs = pkg.harvest_points(1, nx, 1, 0, 0.05, 0)[:, 0]
    for U, b in [(5.0, -15.0), (30.0, -100.0), (1e-3, -3e-3), (0.7, -2.2), (1e-17, 0.0), (-3.0, 9.0)]:
        m = pkg.LrnrParams(np.array([2, 1, 1]), np.array([1, 1]), np.array([U, 1.0, 0.0, b, 1.0, 1.0, 0.0]))
        S = gpu.harvest_snapshots(m, np.ones(2), nx=nx, nt=1, n_perturb=0)[0][0]
        want = np.array([math.tanh(U * x + b) for x in xs])
        assert np.array_equal(S, want), (U, b, int(np.sum(S != want)))
