"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the C oracle, on seeded inputs; size-independent properties at
BASELINE.json's full sizes.

Tolerances (BASELINE.json north_star / SURVEY 8(c1)):
  FP64 (configs 0, 1): floor-relative <= 1e-10 on dL/ds, loss <= 1e-12 relative.
  FP32 (configs 2, 3): normwise <= 1e-4 on dL/ds (and dL/dtheta); loss <= 1e-4 relative.
"""
import numpy as np
import pytest

import paper_2410_04001_b200 as pkg
from conftest import floor_rel, normwise

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32_NORM = 1e-4
TOL32_LOSS = 1e-4


# FP32 kernel choices (LRNR_OPT_KERNEL): auto = tcgen05 (LRNR and FastLRNR, ranks <= 32);
# forced tcgen05; FMA tile; per-point streaming; small-batch; forced narrow-network FMA kernel
FP32_KERNELS = [pkg.KERNEL_AUTO, pkg.KERNEL_TC, pkg.KERNEL_FMA_TILE, pkg.KERNEL_STREAM, pkg.KERNEL_SMALL,
                pkg.KERNEL_NARROW]


@pytest.fixture
def opts(gpu):
    """Set context options for one test; restore the defaults afterwards."""

    def apply(kernel=pkg.KERNEL_AUTO, fast_sincos=0):
        gpu.set_option(pkg.OPT_KERNEL, kernel)
        gpu.set_option(pkg.OPT_FAST_SINCOS, fast_sincos)

    yield apply
    apply()


def lrnr_from_golden(g, prefix, act=pkg.ACT_TANH):
    return pkg.LrnrParams(g[prefix + "_widths"], g[prefix + "_ranks"], g[prefix + "_params"], act)


# ----------------------------------------------------------------------------
# config 0 / 1 (FP64) against the reference's own outputs
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("kernel", [pkg.KERNEL_AUTO, pkg.KERNEL_SMALL, pkg.KERNEL_STREAM])
def test_c0_lrnr_fp64_matches_reference(gpu, golden, opts, kernel):
    opts(kernel)
    m = lrnr_from_golden(golden, "c0")
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(golden["c0_pts"])
    r = gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c0_s"], golden["c0_mu"])
    assert abs(r["value"] - golden["c0_value"][0]) <= 1e-12 * abs(golden["c0_value"][0])
    assert floor_rel(r["grad_s"], golden["c0_grad_s"]) <= TOL64
    np.testing.assert_allclose(r["comps"], golden["c0_comps"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("kernel", [pkg.KERNEL_AUTO, pkg.KERNEL_SMALL, pkg.KERNEL_STREAM])
def test_c1_fast_fp64_matches_reference(gpu, golden, opts, kernel):
    opts(kernel)
    f = pkg.FastParams(golden["c0_ranks"], golden["c1_red_ranks"], golden["c1_fparams"], pkg.ACT_TANH)
    gpu.set_fast(f, pkg.F64)
    gpu.set_points(golden["c0_pts"])
    r = gpu.loss_grad_s(pkg.MODEL_FAST, golden["c0_s"], golden["c0_mu"])
    assert abs(r["value"] - golden["c1_value"][0]) <= 1e-12 * abs(golden["c1_value"][0])
    assert floor_rel(r["grad_s"], golden["c1_grad_s"]) <= TOL64
    # the paper's approximation metric: FastLRNR vs full-LRNR gradient
    rel = normwise(r["grad_s"], golden["c0_grad_s"])
    assert 0.0 < rel < 1.0


@pytest.mark.parametrize("kernel", [pkg.KERNEL_AUTO, pkg.KERNEL_STREAM])
def test_c0_jets_match_reference(gpu, golden, opts, kernel):
    opts(kernel)
    m = lrnr_from_golden(golden, "c0")
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(golden["c0_pts"][:256])
    j = gpu.jets(pkg.MODEL_LRNR, golden["c0_s"])
    np.testing.assert_allclose(j, golden["c0_jets"], rtol=1e-12, atol=1e-13)
    f = pkg.FastParams(golden["c0_ranks"], golden["c1_red_ranks"], golden["c1_fparams"], pkg.ACT_TANH)
    gpu.set_fast(f, pkg.F64)
    jf = gpu.jets(pkg.MODEL_FAST, golden["c0_s"])
    np.testing.assert_allclose(jf, golden["c1_jets"], rtol=1e-12, atol=1e-13)


def test_c0_loss_only_matches_loss_tune(gpu, golden):
    m = lrnr_from_golden(golden, "c0")
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(golden["c0_pts"])
    v = gpu.loss(pkg.MODEL_LRNR, golden["c0_s"], golden["c0_mu"])
    assert abs(v - golden["c0_loss_tune"][0]) <= 1e-12 * abs(golden["c0_loss_tune"][0])


def test_identity_reduction_equals_lrnr(gpu, golden):
    """FastLRNR == LRNR under the identity reduction (test_model.cpp:298-315)."""
    m = lrnr_from_golden(golden, "c0")
    f = pkg.FastParams(golden["c0_ranks"], golden["c0_identity_red"], golden["c0_identity_fparams"], pkg.ACT_TANH)
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_fast(f, pkg.F64)
    gpu.set_points(golden["c0_pts"][:512])
    a = gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c0_s"], golden["c0_mu"])
    b = gpu.loss_grad_s(pkg.MODEL_FAST, golden["c0_s"], golden["c0_mu"])
    assert abs(a["value"] - b["value"]) <= 1e-12 * abs(a["value"])
    assert floor_rel(b["grad_s"], a["grad_s"]) <= 1e-10


# ----------------------------------------------------------------------------
# config 2 shapes (FP32): tanh against the reference, sin against the oracle
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("kernel", FP32_KERNELS)
def test_c2_tanh_fp32_matches_reference(gpu, golden, opts, kernel):
    opts(kernel)
    m = lrnr_from_golden(golden, "c2")
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_points(golden["c2_pts"])
    r = gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c2_s"], golden["c2_mu"])
    assert abs(r["value"] - golden["c2_value"][0]) <= TOL32_LOSS * abs(golden["c2_value"][0])
    assert normwise(r["grad_s"], golden["c2_grad_s"]) <= TOL32_NORM
    f = pkg.FastParams(golden["c2_ranks"], golden["c2_red_ranks"], golden["c2_fparams"], pkg.ACT_TANH)
    gpu.set_fast(f, pkg.F32)
    rf = gpu.loss_grad_s(pkg.MODEL_FAST, golden["c2_s"], golden["c2_mu"])
    # the EIM interpolation blocks amplify FP32 rounding (V_hat = (P^T Xi)^-T ...): loss to 1e-4
    assert abs(rf["value"] - golden["c2_fast_value"][0]) <= TOL32_LOSS * abs(golden["c2_fast_value"][0])
    assert normwise(rf["grad_s"], golden["c2_fast_grad_s"]) <= TOL32_NORM


@pytest.mark.parametrize(
    "dtype,kernel,fast_sincos",
    [(pkg.F64, pkg.KERNEL_AUTO, 0)] + [(pkg.F32, k, fs) for k in FP32_KERNELS for fs in (0, 1)],
)
def test_c2_sin_matches_oracle(gpu, oracle, opts, dtype, kernel, fast_sincos):
    opts(kernel, fast_sincos)
    c = pkg.config2(n_points=2048, act=pkg.ACT_SIN)
    m, f = c["model"], c["fast"]
    gpu.set_lrnr(m, dtype)
    gpu.set_fast(f, dtype)
    gpu.set_points(c["pts"])
    want = oracle.lrnr_grad(m.widths, m.ranks, m.params, c["s"], c["mu"], c["pts"], act=pkg.ACT_SIN)
    got = gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"])
    wantf = oracle.fast_grad(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], c["pts"], act=pkg.ACT_SIN)
    gotf = gpu.loss_grad_s(pkg.MODEL_FAST, c["s"], c["mu"])
    if dtype == pkg.F64:
        assert abs(got["value"] - want["value"]) <= 1e-12 * abs(want["value"])
        assert floor_rel(got["grad_s"], want["grad_s"]) <= TOL64
        assert floor_rel(gotf["grad_s"], wantf["grad_s"]) <= TOL64
    else:
        assert abs(got["value"] - want["value"]) <= TOL32_LOSS * abs(want["value"])
        assert normwise(got["grad_s"], want["grad_s"]) <= TOL32_NORM
        assert normwise(gotf["grad_s"], wantf["grad_s"]) <= TOL32_NORM


# ----------------------------------------------------------------------------
# config 3: hypernetwork -> FastLRNR per instance + hypernet VJP
# ----------------------------------------------------------------------------
def test_c3_hyper_fast_matches_oracle(gpu, oracle):
    n_inst, per = 6, 333
    c = pkg.config3(n_inst=n_inst, pts_per_inst=per, act=pkg.ACT_SIN)
    f, h = c["fast"], c["hyper"]
    gpu.set_fast(f, pkg.F32)
    gpu.set_hyper(h)
    gpu.set_points(c["pts"], n_inst=n_inst)
    got = gpu.hyper_loss_grad(pkg.MODEL_FAST, c["mus"])
    w = 1.0 / (n_inst * per)
    val = 0.0
    gth = np.zeros(h.n_params)
    for i in range(n_inst):
        s_i = oracle.hyper_forward(h.hw, h.params, h.lo, h.hi, c["mus"][i])
        r = oracle.fast_grad(f.ranks, f.red_ranks, f.fparams, s_i, c["mus"][i], c["pts"][i * per:(i + 1) * per], w=w,
                             act=pkg.ACT_SIN)
        val += r["value"]
        assert normwise(got["grad_s"][i], r["grad_s"]) <= TOL32_NORM
        oracle.hyper_vjp(h.hw, h.params, h.lo, h.hi, c["mus"][i], r["grad_s"], out=gth)
    assert abs(got["value"] - val) <= TOL32_LOSS * abs(val)
    assert normwise(got["grad_theta"], gth) <= TOL32_NORM


def test_c3_full_points_per_instance_matches_oracle(gpu, oracle):
    """c3 at BASELINE's 16,384 points per instance, on three of the 1024 mu (first, middle, last),
    against the FP64 oracle per instance (points sampled exactly as bench.py does)."""
    per = 16384
    c = pkg.config3(n_inst=1024, pts_per_inst=0, act=pkg.ACT_SIN)
    f, h = c["fast"], c["hyper"]
    idx = [0, 511, 1023]
    pts = np.concatenate([pkg.sample_collocation(5000 + i, per) for i in idx])
    mus = np.ascontiguousarray(c["mus"][idx])
    gpu.set_fast(f, pkg.F32)
    gpu.set_hyper(h)
    gpu.set_points(pts, n_inst=len(idx))
    w = 1.0 / (1024 * per)
    got = gpu.hyper_loss_grad(pkg.MODEL_FAST, mus, w)
    for k, i in enumerate(idx):
        s_i = oracle.hyper_forward(h.hw, h.params, h.lo, h.hi, mus[k])
        r = oracle.fast_grad(f.ranks, f.red_ranks, f.fparams, s_i, mus[k], pts[k * per:(k + 1) * per], w=w,
                             act=pkg.ACT_SIN)
        assert normwise(got["grad_s"][k], r["grad_s"]) <= TOL32_NORM


def test_c3_full_config_shard_invariant(gpu):
    """The full c3 step (1024 mu x 16,384 points): each instance's dL/ds row is the same when the
    instances run in two halves (what a 2-GPU shard computes; only the tile grouping of the FP32
    partial sums differs), and dL/dtheta is the sum of the halves' (a size-independent property at
    BASELINE's size)."""
    import torch
    per, n = 16384, 1024
    c = pkg.config3(n_inst=n, pts_per_inst=0, act=pkg.ACT_SIN)
    pts = np.concatenate([pkg.sample_collocation(5000 + i, per) for i in range(n)])
    pts_dev = torch.from_numpy(pts).to("cuda")
    gpu.set_fast(c["fast"], pkg.F32)
    gpu.set_hyper(c["hyper"])
    w = 1.0 / (n * per)
    gpu.set_points_device(pts_dev.data_ptr(), n * per, n_inst=n)
    full = gpu.hyper_loss_grad(pkg.MODEL_FAST, c["mus"], w)
    halves = []
    for a, b in ((0, n // 2), (n // 2, n)):
        sub = pts_dev[a * per:b * per]
        gpu.set_points_device(sub.data_ptr(), (b - a) * per, n_inst=b - a)
        halves.append(gpu.hyper_loss_grad(pkg.MODEL_FAST, np.ascontiguousarray(c["mus"][a:b]), w))
    assert np.isfinite(full["value"]) and np.all(np.isfinite(full["grad_theta"]))
    cat = np.concatenate([hh["grad_s"] for hh in halves])
    assert max(normwise(full["grad_s"][i], cat[i]) for i in range(n)) <= 1e-5
    th = halves[0]["grad_theta"] + halves[1]["grad_theta"]
    assert normwise(full["grad_theta"], th) <= 1e-5
    assert abs(full["value"] - (halves[0]["value"] + halves[1]["value"])) <= 1e-5 * abs(full["value"])


def test_staged_points_double_buffer(gpu):
    """lrnr_gpu_stage_points / lrnr_gpu_use_staged_points (the double-buffered host upload of a
    training loop): alternating batches, each staged while the previous one is in use, give
    bitwise the results of lrnr_gpu_set_points; the staged host buffer may then be reused."""
    c = pkg.config2(n_points=0, act=pkg.ACT_SIN, with_fast=False)
    gpu.set_lrnr(c["model"], pkg.F32)
    batches = [pkg.sample_collocation(300 + k, 5000 + 700 * k) for k in range(3)]
    want = []
    for b in batches:
        gpu.set_points(b)
        want.append(gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"]))
    buf = np.array(batches[0])
    gpu.stage_points(buf)
    for k in range(len(batches)):
        gpu.use_staged_points()
        if k + 1 < len(batches):
            buf = np.array(batches[k + 1])  # a new host buffer each step
            gpu.stage_points(buf)
        got = gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"])
        assert got["value"] == want[k]["value"]
        assert np.array_equal(got["grad_s"], want[k]["grad_s"])
    with pytest.raises(ValueError):
        gpu.use_staged_points()  # nothing staged (LRNR_EINVAL)


def test_hyper_forward_vjp_match_reference(gpu, golden):
    """Hypernetwork forward + VJP (c3 shape) against the reference (FP64 path)."""
    split = golden["c2_ranks"]
    h = pkg.HyperParams(golden["c3_hw"], golden["c3_hparams"], golden["c3_lo"], golden["c3_hi"])
    # identity-like use: a FastLRNR whose gradient we replace is not needed; check through the c3 call with a
    # constant-residual-free probe: compare s via jets of a 1-point problem is indirect, so use loss_grad with
    # the identity of hyper_forward through the multi path instead.
    f = pkg.FastParams(golden["c2_ranks"], golden["c2_red_ranks"], golden["c2_fparams"], pkg.ACT_TANH)
    gpu.set_fast(f, pkg.F64)
    gpu.set_hyper(h)
    mus = golden["c3_mu"]
    pts = np.tile(golden["c2_pts"][:64], (len(mus), 1))
    gpu.set_points(pts, n_inst=len(mus))
    got = gpu.hyper_loss_grad(pkg.MODEL_FAST, mus)
    # per-instance s must equal the reference's hyper_forward: check via the multi path with those s
    gm = gpu.loss_grad_s_multi(pkg.MODEL_FAST, golden["c3_s"], mus)
    np.testing.assert_allclose(got["grad_s"], gm["grad_s"], rtol=1e-12, atol=1e-15)
    assert abs(got["value"] - gm["value"]) <= 1e-13 * abs(gm["value"])
    assert split.sum() == golden["c3_s"].shape[1]


# ----------------------------------------------------------------------------
# edge cases (empty / ragged / single point / non-finite), determinism
# ----------------------------------------------------------------------------
def test_empty_batch_returns_zeros(gpu, golden):
    m = lrnr_from_golden(golden, "c0")
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(np.zeros((0, 2)))
    r = gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c0_s"], golden["c0_mu"])
    assert r["value"] == 0.0 and not r["grad_s"].any()


@pytest.mark.parametrize("n", [1, 31, 33, 97, 1000])
def test_ragged_sizes_match_oracle(gpu, oracle, golden, n):
    m = lrnr_from_golden(golden, "c0")
    gpu.set_lrnr(m, pkg.F64)
    pts = golden["c0_pts"][:n]
    gpu.set_points(pts)
    got = gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c0_s"], golden["c0_mu"])
    want = oracle.lrnr_grad(m.widths, m.ranks, m.params, golden["c0_s"], golden["c0_mu"], pts)
    assert abs(got["value"] - want["value"]) <= 1e-12 * abs(want["value"])
    assert floor_rel(got["grad_s"], want["grad_s"]) <= TOL64


def test_nonfinite_maps_to_nonfinite_error(gpu, golden):
    m = lrnr_from_golden(golden, "c0")
    P = m.params.copy()
    widths, ranks = m.widths, m.ranks
    # poison the layer-2 bias (b_1): a_2 becomes inf -> AffineFactoredJet tag 2 ... but b leaves come first
    # in tape order, so the reference reports -1 (leaf); poison U_1 instead -> first bad node is layer 2.
    o = 0
    for l in range(1):
        o += widths[l + 1] * ranks[l] + widths[l] * ranks[l] + widths[l + 1]
    P[o] = np.inf  # U_1[0,0]
    gpu.set_lrnr(pkg.LrnrParams(widths, ranks, P), pkg.F64)
    gpu.set_points(golden["c0_pts"][:64])
    with pytest.raises(pkg.NonFiniteError) as ei:
        gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c0_s"], golden["c0_mu"])
    assert ei.value.layer_tag == 2


def test_nonfinite_leaf_reports_minus_one(gpu, golden):
    m = lrnr_from_golden(golden, "c0")
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(golden["c0_pts"][:64])
    s = golden["c0_s"].copy()
    s[3] = np.nan
    with pytest.raises(pkg.NonFiniteError) as ei:
        gpu.loss_grad_s(pkg.MODEL_LRNR, s, golden["c0_mu"])
    assert ei.value.layer_tag == -1


def test_bitwise_deterministic(gpu, golden):
    m = lrnr_from_golden(golden, "c2")
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_points(golden["c2_pts"])
    a = gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c2_s"], golden["c2_mu"])
    b = gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c2_s"], golden["c2_mu"])
    assert a["value"] == b["value"] and np.array_equal(a["grad_s"], b["grad_s"])


@pytest.mark.parametrize("kernel", [pkg.KERNEL_TC, pkg.KERNEL_FMA_TILE, pkg.KERNEL_SMALL])
@pytest.mark.parametrize("n", [1, 127, 129, 1000])
def test_c2_fp32_ragged_tiles_match_oracle(gpu, oracle, opts, kernel, n):
    """Partial point tiles (128-point TMEM tiles / 64-point FMA tiles) on the FP32 kernels."""
    opts(kernel)
    c = pkg.config2(n_points=n, act=pkg.ACT_SIN, with_fast=False)
    m = c["model"]
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_points(c["pts"])
    got = gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"])
    want = oracle.lrnr_grad(m.widths, m.ranks, m.params, c["s"], c["mu"], c["pts"], act=pkg.ACT_SIN)
    assert abs(got["value"] - want["value"]) <= TOL32_LOSS * abs(want["value"])
    assert normwise(got["grad_s"], want["grad_s"]) <= TOL32_NORM


@pytest.mark.parametrize("kernel", [pkg.KERNEL_TC, pkg.KERNEL_FMA_TILE, pkg.KERNEL_SMALL])
def test_c2_fp32_multi_instance_matches_oracle(gpu, oracle, opts, kernel):
    """Several PDE instances (own s, mu, ragged point counts padded per instance)."""
    opts(kernel)
    c = pkg.config2(n_points=0, act=pkg.ACT_SIN, with_fast=False)
    m = c["model"]
    n_inst, n_per = 3, 300
    pts = pkg.sample_collocation(91, n_inst * n_per)
    rng = np.random.default_rng(5)
    S = np.stack([c["s"] * (1.0 + 0.1 * rng.standard_normal(c["s"].shape)) for _ in range(n_inst)])
    MU = np.array([[20.0, 0.01, 5.0], [5.0, 0.05, 1.0], [35.0, 0.002, 8.0]])
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_points(pts, n_inst=n_inst)
    got = gpu.loss_grad_s_multi(pkg.MODEL_LRNR, S, MU, w=1.0 / n_per)  # oracle weight: 1 / n per instance
    total = 0.0
    for i in range(n_inst):
        sl = pts[i * n_per:(i + 1) * n_per]
        want = oracle.lrnr_grad(m.widths, m.ranks, m.params, S[i], MU[i], sl, act=pkg.ACT_SIN)
        total += want["value"]
        assert normwise(got["grad_s"][i], want["grad_s"]) <= TOL32_NORM
    assert abs(got["value"] - total) <= TOL32_LOSS * abs(total)


def test_c2_fp32_tc_dynamic_claims_deterministic(gpu, opts):
    """The tensor-core sweep claims single-tile units from a global counter and reduces the
    per-unit rows in two fixed-order levels (> 128 units per instance): 5 instances x 40000
    points (1565 units on 148 CTAs) are bitwise reproducible across runs, whatever CTA ran
    each unit, and agree per instance with the statically scheduled FMA tile kernel."""
    c = pkg.config2(n_points=0, act=pkg.ACT_SIN, with_fast=False)
    m = c["model"]
    n_inst, n_per = 5, 40000
    pts = pkg.sample_collocation(93, n_inst * n_per)
    rng = np.random.default_rng(9)
    S = np.stack([c["s"] * (1.0 + 0.1 * rng.standard_normal(c["s"].shape)) for _ in range(n_inst)])
    MU = np.tile(c["mu"], (n_inst, 1))
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_points(pts, n_inst=n_inst)
    opts(pkg.KERNEL_TC)
    runs = [gpu.loss_grad_s_multi(pkg.MODEL_LRNR, S, MU, w=1.0 / n_per) for _ in range(3)]
    for r in runs[1:]:
        assert r["value"] == runs[0]["value"] and np.array_equal(r["grad_s"], runs[0]["grad_s"])
    opts(pkg.KERNEL_FMA_TILE)
    ref = gpu.loss_grad_s_multi(pkg.MODEL_LRNR, S, MU, w=1.0 / n_per)
    assert abs(runs[0]["value"] - ref["value"]) <= TOL32_LOSS * abs(ref["value"])
    for i in range(n_inst):
        assert normwise(runs[0]["grad_s"][i], ref["grad_s"][i]) <= TOL32_NORM


def test_c2_fp32_tc_nonfinite_tag(gpu, golden, opts):
    """The tensor-core path reports the reference's NonFiniteError layer tag."""
    opts(pkg.KERNEL_TC)
    m = lrnr_from_golden(golden, "c2")
    P = m.params.copy()
    widths, ranks = m.widths, m.ranks
    o = widths[1] * ranks[0] + widths[0] * ranks[0] + widths[1]
    P[o] = np.inf  # U_1[0,0] -> first non-finite node is layer 2
    gpu.set_lrnr(pkg.LrnrParams(widths, ranks, P), pkg.F32)
    gpu.set_points(golden["c2_pts"][:256])
    with pytest.raises(pkg.NonFiniteError) as ei:
        gpu.loss_grad_s(pkg.MODEL_LRNR, golden["c2_s"], golden["c2_mu"])
    assert ei.value.layer_tag == 2


def test_invalid_shapes_raise_value_error(gpu):
    bad = pkg.LrnrParams(np.array([2, 4, 1]), np.array([3, 1]), np.zeros(100))
    with pytest.raises(ValueError):
        gpu.set_lrnr(bad, pkg.F64)


# ----------------------------------------------------------------------------
# full BASELINE size (config 2, 1M points): size-independent properties
# ----------------------------------------------------------------------------
@pytest.mark.slow
def test_c2_full_size_linearity_and_subsample(gpu, oracle):
    c = pkg.config2(n_points=1 << 20, act=pkg.ACT_SIN, with_fast=False)
    m = c["model"]
    n = c["pts"].shape[0]
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_points(c["pts"])
    full = gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"], w=1.0 / n)
    # linearity over a disjoint split: L(all) = L(A) + L(B), grad likewise (same weight 1/n)
    h = n // 2
    gpu.set_points(c["pts"][:h])
    a = gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"], w=1.0 / n)
    gpu.set_points(c["pts"][h:])
    b = gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"], w=1.0 / n)
    assert abs(full["value"] - (a["value"] + b["value"])) <= 1e-6 * abs(full["value"])
    assert normwise(full["grad_s"], a["grad_s"] + b["grad_s"]) <= 1e-5
    # a strided 1/256 subsample of the full batch against the FP64 oracle
    sub = c["pts"][::256]
    gpu.set_points(sub)
    got = gpu.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"])
    want = oracle.lrnr_grad(m.widths, m.ranks, m.params, c["s"], c["mu"], sub, act=pkg.ACT_SIN)
    assert normwise(got["grad_s"], want["grad_s"]) <= TOL32_NORM


# ----------------------------------------------------------------------------
# config 4 (meta): bases, biases and hypernetwork, ParamPacker order
# ----------------------------------------------------------------------------
def test_meta_fp64_matches_reference(gpu, golden):
    g = golden
    m = pkg.LrnrParams(g["c4_widths"], g["c4_ranks"], g["c4_params"], pkg.ACT_TANH)
    h = pkg.HyperParams(g["c4_hw"], g["c4_hparams"], g["c3_lo"], g["c3_hi"])
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_hyper(h)
    mus = g["c4_mus"]
    uniq = [mus[0], mus[-1]]
    assert np.array_equal(np.concatenate([np.tile(uniq[0], (48, 1)), np.tile(uniq[1], (48, 1))]), mus)
    gpu.set_points(g["c4_pts"], n_inst=2)
    r = gpu.meta_loss_grad(np.array(uniq), m.params.size)
    assert abs(r["value"] - g["c4_value"][0]) <= 1e-12 * g["c4_value"][0]
    assert normwise(r["grad"], g["c4_grad"]) <= 1e-10
    assert floor_rel(r["grad"], g["c4_grad"], floor=1e-6) <= 1e-8


@pytest.mark.parametrize("act", [pkg.ACT_SIN, pkg.ACT_TANH])
def test_meta_c4_shape_fp32_matches_oracle(gpu, oracle, act):
    n_inst, per = 2, 96
    c = pkg.config4(n_inst=n_inst, pts_per_inst=per, act=act)
    m, h = c["model"], c["hyper"]
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_hyper(h)
    gpu.set_points(c["pts"], n_inst=n_inst)
    got = gpu.meta_loss_grad(c["mus"], m.params.size)
    w = 1.0 / (n_inst * per)
    nP = m.params.size
    want = np.zeros(nP + h.n_params)
    val = 0.0
    for i in range(n_inst):
        s_i = oracle.hyper_forward(h.hw, h.params, h.lo, h.hi, c["mus"][i])
        r = oracle.lrnr_grad(m.widths, m.ranks, m.params, s_i, c["mus"][i], c["pts"][i * per:(i + 1) * per], w=w,
                             act=act, params_grad=True)
        val += r["value"]
        want[:nP] += r["grad_params"]
        oracle.hyper_vjp(h.hw, h.params, h.lo, h.hi, c["mus"][i], r["grad_s"], out=want[nP:])
    assert abs(got["value"] - val) <= TOL32_LOSS * abs(val)
    assert normwise(got["grad"], want) <= TOL32_NORM
    assert normwise(got["grad"][nP:], want[nP:]) <= TOL32_NORM


def test_meta_regularizers_fp64_match_reference(gpu, golden):
    """meta_train's step with lambda_sparse banded decay and lambda_ortho Gram penalties."""
    g = golden
    lam_sp, gamma, lam_o = g["c4_reg"]
    m = pkg.LrnrParams(g["c4_widths"], g["c4_ranks"], g["c4_reg_params"], pkg.ACT_TANH)
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_hyper(pkg.HyperParams(g["c4_hw"], g["c4_hparams"], g["c3_lo"], g["c3_hi"]))
    gpu.set_points(g["c4_pts"], n_inst=2)
    r = gpu.meta_terms_grad(np.array([g["c4_mus"][0], g["c4_mus"][-1]]), m.params.size, lam_sp, gamma, lam_o)
    assert abs(r["value"] - g["c4_reg_value"][0]) <= 1e-12 * g["c4_reg_value"][0]
    np.testing.assert_allclose(r["comps"], g["c4_reg_comps"], rtol=1e-12, atol=0)
    assert abs(r["ortho"] - g["c4_reg_ortho"][0]) <= 1e-12 * g["c4_reg_ortho"][0]
    assert normwise(r["grad"], g["c4_reg_grad"]) <= 1e-10


@pytest.mark.parametrize("act", [pkg.ACT_SIN, pkg.ACT_TANH])
def test_meta_regularizers_c4_shape_fp32_match_oracle(gpu, oracle, act):
    n_inst, per = 2, 96
    c = pkg.config4(n_inst=n_inst, pts_per_inst=per, act=act)
    m, h = c["model"], c["hyper"]
    P = m.params * 1.05  # off the Stiefel manifold: non-trivial Gram penalty
    m = pkg.LrnrParams(m.widths, m.ranks, P, act)
    lam = (1e-2, 1.5, 1e-4)
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_hyper(h)
    gpu.set_points(c["pts"], n_inst=n_inst)
    got = gpu.meta_terms_grad(c["mus"], m.params.size, *lam)
    w = 1.0 / (n_inst * per)
    nP = m.params.size
    S = np.stack([oracle.hyper_forward(h.hw, h.params, h.lo, h.hi, mu) for mu in c["mus"]])
    regs = oracle.meta_regs(m.widths, m.ranks, P, S, per, w, *lam)
    want = np.zeros(nP + h.n_params)
    val = 0.0
    for i in range(n_inst):
        r = oracle.lrnr_grad(m.widths, m.ranks, P, S[i], c["mus"][i], c["pts"][i * per:(i + 1) * per], w=w, act=act,
                             params_grad=True)
        val += r["value"]
        want[:nP] += r["grad_params"]
        oracle.hyper_vjp(h.hw, h.params, h.lo, h.hi, c["mus"][i], r["grad_s"] + regs["ds"][i], out=want[nP:])
    want[:nP] += regs["grad_params"]
    assert abs(got["comps"][0] - val) <= TOL32_LOSS * abs(val)
    assert abs(got["comps"][2] - regs["sparse"]) <= 1e-6 * abs(regs["sparse"])  # FP64 on the device
    assert abs(got["ortho"] - regs["ortho"]) <= 1e-10 * abs(regs["ortho"])
    assert normwise(got["grad"], want) <= TOL32_NORM
    assert normwise(got["grad"][nP:], want[nP:]) <= TOL32_NORM


@pytest.mark.parametrize("dtype", [pkg.F64, pkg.F32])
def test_meta_full_emitter_matches_reference(gpu, golden, dtype):
    """meta_train's full step: interior (+ sparse), initial and periodic terms per instance, + ortho."""
    g = golden
    lam_sp, gamma, lam_o = g["c4_reg"]
    m = pkg.LrnrParams(g["c4_widths"], g["c4_ranks"], g["c4_reg_params"], pkg.ACT_TANH)
    gpu.set_lrnr(m, dtype)
    gpu.set_hyper(pkg.HyperParams(g["c4_hw"], g["c4_hparams"], g["c3_lo"], g["c3_hi"]))
    gpu.set_points(g["c4_pts"], n_inst=2)
    gpu.set_meta_boundary(2, g["c4_full_ic_x"], g["c4_full_per_t"])
    try:
        r = gpu.meta_terms_grad(np.array([g["c4_mus"][0], g["c4_mus"][-1]]), m.params.size, lam_sp, gamma, lam_o)
    finally:
        gpu.set_meta_boundary(0)
    tol_v, tol_g = (1e-12, 1e-10) if dtype == pkg.F64 else (TOL32_LOSS, TOL32_NORM)
    assert abs(r["value"] - g["c4_full_value"][0]) <= tol_v * g["c4_full_value"][0]
    np.testing.assert_allclose(r["comps"], g["c4_full_comps"], rtol=tol_v, atol=1e-14)
    assert normwise(r["grad"], g["c4_full_grad"]) <= tol_g


def test_cpp_adapter_drop_in_against_reference():
    """include/lrnr_gpu_adapter.hpp compiled against the reference's own headers and
    objects (oracle/_ref/adapter_test): same fine-tune / FastLRNR gradient as
    run_batch_gradient, NonFiniteError mapping."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "adapter_test")
    # built by __graft_entry__.build() in the build container (it needs /root/reference) and shipped with
    # the snapshot: a GPU run without it is a packaging failure, not a skip
    assert os.path.exists(exe), "oracle/_ref/adapter_test missing: run __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER PARITY OK" in r.stdout


# ----------------------------------------------------------------------------
# full solve-step term set (boundary terms, fast-phase l1 objective + locality)
# ----------------------------------------------------------------------------
def classify_phase_points(X):
    two_pi = 6.283185307179586476925286766559
    pts, ic, pt = [], [], []
    for x, t in X:
        if t == 0.0:
            ic.append(x)
        elif x == 0.0 or x == two_pi:
            pt.append(t)
        else:
            pts.append((x, t))
    return np.array(pts).reshape(-1, 2), np.array(ic), np.array(pt)


def test_full_tune_terms_fp64_match_reference(gpu, golden):
    """Interior + initial + periodic PinnTermEmitter terms on the device (training.cpp:286-327)."""
    g = golden
    gpu.set_lrnr(lrnr_from_golden(g, "c0"), pkg.F64)
    gpu.set_points(g["c0_full_pts"])
    gpu.set_boundary(g["c0_full_ic_x"], g["c0_full_per_t"])
    try:
        r = gpu.terms_grad(pkg.MODEL_LRNR, g["c0_s"], g["c0_mu"])
    finally:
        gpu.set_boundary()
    assert abs(r["value"] - g["c0_full_value"][0]) <= 1e-12 * abs(g["c0_full_value"][0])
    np.testing.assert_allclose(r["comps"], g["c0_full_comps"], rtol=1e-12, atol=0)
    assert floor_rel(r["grad_s"], g["c0_full_grad_s"]) <= TOL64


def test_fast_phase_objective_fp64_matches_reference(gpu, golden):
    """The fast-phase emitter on the device: |N|, |u - sin x|, |u(0,t) - u(2pi,t)|, lambda ||s - s0||_1."""
    g = golden
    pts, ic, pt = classify_phase_points(g["c1_phase_x"])
    gpu.set_fast(pkg.FastParams(g["c0_ranks"], g["c1_red_ranks"], g["c1_fparams"], pkg.ACT_TANH), pkg.F64)
    gpu.set_points(pts)
    gpu.set_boundary(ic, pt)
    try:
        r = gpu.terms_grad(pkg.MODEL_FAST, g["c1_phase_s"], g["c0_mu"], objective=pkg.OBJ_ABS, w_int=1.0, w_ic=1.0,
                           w_bc=1.0, s_init=g["c0_s"], lambda_local=1e-2)
    finally:
        gpu.set_boundary()
    assert abs(r["value"] - g["c1_phase_value"][0]) <= 1e-12 * abs(g["c1_phase_value"][0])
    np.testing.assert_allclose(r["comps"], g["c1_phase_comps"], rtol=1e-12, atol=1e-300)
    assert floor_rel(r["grad_s"], g["c1_phase_grad_s"]) <= TOL64


@pytest.mark.parametrize("objective", [pkg.OBJ_SQUARED, pkg.OBJ_ABS])
@pytest.mark.parametrize("model", [pkg.MODEL_LRNR, pkg.MODEL_FAST])
def test_c2_fp32_terms_match_oracle(gpu, oracle, model, objective):
    """FP32 c2 shapes (sin): every term kind, both models, both objectives against the FP64 oracle."""
    c = pkg.config2(n_points=1024, act=pkg.ACT_SIN)
    m, f = c["model"], c["fast"]
    rng = np.random.default_rng(11)
    ic, pt = rng.uniform(0, 2 * np.pi, 200), rng.uniform(0, 1, 150)
    if model == pkg.MODEL_LRNR:
        gpu.set_lrnr(m, pkg.F32)
        dims, P = (m.widths, m.ranks), m.params
    else:
        gpu.set_fast(f, pkg.F32)
        dims, P = (f.ranks, f.red_ranks), f.fparams
    s_init = c["s"] * 1.05
    gpu.set_points(c["pts"])
    gpu.set_boundary(ic, pt)
    try:
        got = gpu.terms_grad(model, c["s"], c["mu"], objective=objective, s_init=s_init, lambda_local=1e-3)
    finally:
        gpu.set_boundary()
    want = oracle.terms_grad(0 if model == pkg.MODEL_LRNR else 1, dims, P, c["s"], c["mu"], c["pts"], ic, pt,
                             objective=objective, s_init=s_init, lambda_local=1e-3, act=pkg.ACT_SIN)
    assert abs(got["value"] - want["value"]) <= TOL32_LOSS * abs(want["value"])
    np.testing.assert_allclose(got["comps"], want["comps"], rtol=TOL32_LOSS, atol=1e-12)
    assert normwise(got["grad_s"], want["grad_s"]) <= TOL32_NORM


def test_boundary_only_terms(gpu, golden, oracle):
    """No interior points: only the initial / periodic terms contribute."""
    g = golden
    m = lrnr_from_golden(g, "c0")
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(np.zeros((0, 2)))
    gpu.set_boundary(g["c0_full_ic_x"][:17], g["c0_full_per_t"][:9])
    try:
        r = gpu.terms_grad(pkg.MODEL_LRNR, g["c0_s"], g["c0_mu"])
    finally:
        gpu.set_boundary()
    want = oracle.terms_grad(0, (m.widths, m.ranks), m.params, g["c0_s"], g["c0_mu"], np.zeros((0, 2)),
                             g["c0_full_ic_x"][:17], g["c0_full_per_t"][:9])
    assert r["comps"][0] == 0.0
    assert abs(r["value"] - want["value"]) <= 1e-12 * abs(want["value"])
    assert floor_rel(r["grad_s"], want["grad_s"]) <= TOL64


def test_boundary_nonfinite_maps_to_nonfinite_error(gpu, golden):
    """A non-finite s leaf seen only through the boundary terms -> NonFiniteError(-1)."""
    g = golden
    gpu.set_lrnr(lrnr_from_golden(g, "c0"), pkg.F64)
    gpu.set_points(np.zeros((0, 2)))
    gpu.set_boundary(np.array([0.5, 1.5]), np.array([0.25]))
    s = g["c0_s"].copy()
    s[5] = np.nan
    try:
        with pytest.raises(pkg.NonFiniteError) as ei:
            gpu.terms_grad(pkg.MODEL_LRNR, s, g["c0_mu"])
    finally:
        gpu.set_boundary()
    assert ei.value.layer_tag == -1


# ----------------------------------------------------------------------------
# solve loops on the device: fine_tune, fast_solve (CUDA graph)
# ----------------------------------------------------------------------------
def test_fine_tune_fp64_matches_reference(gpu, golden):
    g = golden
    lr, ep, ni, nc, nb, seed = g["c0_ft_cfg"]
    gpu.set_lrnr(lrnr_from_golden(g, "c0"), pkg.F64)
    r = gpu.fine_tune(g["c0_s"], g["c0_mu"], lr, int(ep), int(ni), int(nc), int(nb), int(seed))
    np.testing.assert_allclose(r["losses"], g["c0_ft_losses"], rtol=1e-10, atol=0)
    np.testing.assert_allclose(r["s"], g["c0_ft_s"], rtol=0, atol=1e-10)
    assert r["best_epoch"] == g["c0_ft_best"][1] and not r["aborted"]


@pytest.fixture
def solve_path(gpu):
    def apply(path):
        gpu.set_option(pkg.OPT_SOLVE, path)

    yield apply
    apply(0)


@pytest.mark.parametrize("path", [0, 1])  # 0: persistent single-CTA solver, 1: graph path
@pytest.mark.parametrize("tag", ["a", "b"])
def test_fast_solve_fp64_matches_reference(gpu, golden, solve_path, tag, path):
    solve_path(path)
    g = golden
    lam, lr, ep = g[f"c1_fs{tag}_cfg"]
    gpu.set_fast(pkg.FastParams(g["c0_ranks"], g["c1_red_ranks"], g["c1_fparams"], pkg.ACT_TANH), pkg.F64)
    r = gpu.fast_solve(g["c0_s"], g["c0_mu"], g["c1_phase_x"], lam, lr, int(ep))
    np.testing.assert_allclose(r["losses"], g[f"c1_fs{tag}_losses"], rtol=1e-10, atol=0)
    np.testing.assert_allclose(r["s"], g[f"c1_fs{tag}_s"], rtol=0, atol=1e-10)
    assert r["best_epoch"] == g[f"c1_fs{tag}_best"][1] and not r["diverged"]


@pytest.mark.parametrize("path", [0, 1])
def test_fast_solve_nonfinite_start_aborts(gpu, golden, solve_path, path):
    solve_path(path)
    g = golden
    gpu.set_fast(pkg.FastParams(g["c0_ranks"], g["c1_red_ranks"], g["c1_fparams"], pkg.ACT_TANH), pkg.F64)
    s = g["c0_s"].copy()
    s[2] = np.nan
    r = gpu.fast_solve(s, g["c0_mu"], g["c1_phase_x"], 1e-2, 1e-2, 5)
    assert r["aborted"] and r["diverged"] and len(r["losses"]) == 0 and r["best_epoch"] == 0


@pytest.mark.parametrize("path", [0, 1])
def test_fast_solve_fp32_c2_tracks_oracle(gpu, oracle, solve_path, path):
    """FP32 sin c2 FastLRNR: the device fast phase tracks the FP64 oracle loop."""
    solve_path(path)
    c = pkg.config2(n_points=0, act=pkg.ACT_SIN)
    f = c["fast"]
    X = np.array([(2 * np.pi * i / 3.0, j / 2.0) for j in range(3) for i in range(4)])
    gpu.set_fast(f, pkg.F32)
    r = gpu.fast_solve(c["s"], c["mu"], X, 1e-2, 1e-2, 30)
    want = oracle.fast_solve(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], X, 1e-2, 1e-2, 30, act=pkg.ACT_SIN)
    np.testing.assert_allclose(r["losses"], want["losses"], rtol=1e-3, atol=0)
    assert normwise(r["s"], want["s"]) <= 1e-4


def test_fine_tune_fp32_c2_shape_tracks_oracle(gpu, oracle):
    """FP32 sin c2 shape: the device loop (tensor-core interior kernel) tracks the FP64 oracle loop."""
    c = pkg.config2(n_points=0, act=pkg.ACT_SIN, with_fast=False)
    m = c["model"]
    gpu.set_lrnr(m, pkg.F32)
    r = gpu.fine_tune(c["s"], c["mu"], 1e-2, 8, 512, 128, 128, 99)
    want = oracle.fine_tune(m.widths, m.ranks, m.params, c["s"], c["mu"], 1e-2, 8, 512, 128, 128, 99,
                            act=pkg.ACT_SIN)
    np.testing.assert_allclose(r["losses"], want["losses"], rtol=1e-3, atol=0)
    assert normwise(r["s"], want["s"]) <= 1e-4


# ----------------------------------------------------------------------------
# evaluation and checkpoint-loaded models
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [pkg.F64, pkg.F32])
def test_l1_relative_error_matches_reference(gpu, golden, dtype):
    g = golden
    gpu.set_lrnr(lrnr_from_golden(g, "c0"), dtype)
    field = g["l1_field"]
    got = gpu.l1_error(pkg.MODEL_LRNR, g["c0_s"], field, field.shape[1], field.shape[0] - 1)
    tol = 1e-12 if dtype == pkg.F64 else 1e-5
    assert abs(got - g["l1_value"][0]) <= tol * g["l1_value"][0]


def test_model_from_reference_checkpoint_runs(gpu, golden):
    """A model loaded from a reference-written checkpoint gives the reference's gradient."""
    import os
    g = golden
    ck = pkg.Checkpoint(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_checkpoint.lrnr"))
    gpu.set_lrnr(ck.lrnr(), pkg.F64)
    gpu.set_fast(ck.fast(), pkg.F64)
    gpu.set_points(g["c0_pts"])
    r = gpu.loss_grad_s(pkg.MODEL_LRNR, g["c0_s"], g["c0_mu"])
    assert floor_rel(r["grad_s"], g["c0_grad_s"]) <= TOL64
    rf = gpu.loss_grad_s(pkg.MODEL_FAST, g["c0_s"], g["c0_mu"])
    assert floor_rel(rf["grad_s"], g["c1_grad_s"]) <= TOL64


@pytest.mark.parametrize("kernel", FP32_KERNELS)
@pytest.mark.parametrize("act", [pkg.ACT_SIN, pkg.ACT_TANH])
def test_unaligned_shapes_fp32_match_oracle(gpu, oracle, opts, kernel, act):
    """Width 100 (not a multiple of the 32-neuron chunk), ranks 2 / 10 / 1 (padded MMA K / N,
    rank classes): every FP32 kernel against the FP64 oracle."""
    opts(kernel)
    m, s = pkg.make_baseline_model([2, 100, 100, 100, 1], [2, 10, 10, 1], 2410, act)
    pts = pkg.sample_collocation(4001, 700)
    mu = np.array([5.0, 0.01, 1.0])
    gpu.set_lrnr(m, pkg.F32)
    gpu.set_points(pts)
    got = gpu.loss_grad_s(pkg.MODEL_LRNR, s, mu)
    want = oracle.lrnr_grad(m.widths, m.ranks, m.params, s, mu, pts, act=act)
    assert abs(got["value"] - want["value"]) <= TOL32_LOSS * abs(want["value"])
    assert normwise(got["grad_s"], want["grad_s"]) <= TOL32_NORM


@pytest.mark.parametrize("act", [pkg.ACT_TANH, pkg.ACT_SIN])
@pytest.mark.parametrize("ranks", [[2, 5, 16, 1], [2, 17, 4, 1], [2, 16, 32, 1], [2, 12, 9, 1]])
def test_fp64_rank_classes_match_oracle(gpu, oracle, ranks, act):
    """FP64 FMA tile kernel over its rank classes (4 / 16 / 32: ranks 5..16 pad to 16) with ragged
    widths and a partial last tile; tanh runs the sigma stash (derivatives from the value)."""
    m, s = pkg.make_baseline_model([2, 70, 33, 100, 1], ranks, 77, act)
    pts = pkg.sample_collocation(4003, 1000)
    mu = np.array([12.0, 0.03, 2.0])
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(pts)
    got = gpu.loss_grad_s(pkg.MODEL_LRNR, s, mu)
    want = oracle.lrnr_grad(m.widths, m.ranks, m.params, s, mu, pts, act=act)
    assert abs(got["value"] - want["value"]) <= 1e-12 * abs(want["value"])
    assert floor_rel(got["grad_s"], want["grad_s"]) <= TOL64


def test_context_lifecycle_does_not_leak(golden):
    """create -> every feature -> destroy, repeated: device memory returns to its baseline."""
    import torch
    g = golden
    m = lrnr_from_golden(g, "c0")
    f = pkg.FastParams(g["c0_ranks"], g["c1_red_ranks"], g["c1_fparams"], pkg.ACT_TANH)

    def cycle():
        ctx = pkg.GpuContext(0)
        ctx.set_lrnr(m, pkg.F64)
        ctx.set_fast(f, pkg.F64)
        ctx.set_points(g["c0_pts"][:512])
        ctx.loss_grad_s(pkg.MODEL_LRNR, g["c0_s"], g["c0_mu"])
        ctx.set_boundary(g["c0_full_ic_x"][:8], g["c0_full_per_t"][:8])
        ctx.terms_grad(pkg.MODEL_LRNR, g["c0_s"], g["c0_mu"])
        ctx.fast_solve(g["c0_s"], g["c0_mu"], g["c1_phase_x"], 1e-2, 1e-2, 3)
        ctx.fine_tune(g["c0_s"], g["c0_mu"], 1e-2, 2, 64, 16, 16)
        ctx.close()

    cycle()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        cycle()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 8 << 20, f"{(free0 - free1) / 2**20:.1f} MiB not returned"
