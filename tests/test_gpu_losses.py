"""GPU: the forward-only surface (value-only forward, loss_tune / loss_fast /
loss_meta) against the UNMODIFIED reference (oracle/_ref) on the same seeded
inputs, the per-model non-finite flags, and the NCCL communicator plumbing of
the C ABI at one rank.

Tolerances: FP64 relative 1e-12 on losses and values (the reference sums in a
different order); FP32 against the reference's FP64 at 1e-5
relative on values and 1e-4 on losses."""
import numpy as np
import pytest

import paper_2410_04001_b200 as pkg

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def c1():
    return pkg.config1(n_points=2048)


@pytest.mark.parametrize("dtype,tol", [(pkg.F64, 1e-12), (pkg.F32, 1e-5)])
def test_values_match_reference(gpu, reference, c1, dtype, tol):
    m, f = c1["model"], c1["fast"]
    gpu.set_lrnr(m, dtype)
    gpu.set_fast(f, dtype)
    pts = np.concatenate([c1["pts"][:1000], [[0.0, 0.0], [pkg.api.TWO_PI, 0.5], [1.0, 0.0]]])
    u = gpu.values(pkg.MODEL_LRNR, c1["s"], pts)
    uf = gpu.values(pkg.MODEL_FAST, c1["s"], pts)
    assert rel(u, reference.values(0, m.widths, m.ranks, m.params, None, None, c1["s"], pts)) <= tol
    assert rel(uf, reference.values(1, None, f.ranks, None, f.red_ranks, f.fparams, c1["s"], pts)) <= tol
    # u is the value slot of the 4-slot jets
    gpu.set_points(pts)
    np.testing.assert_allclose(u, gpu.jets(pkg.MODEL_LRNR, c1["s"])[:, 0], rtol=0, atol=1e-12 if dtype == pkg.F64 else 1e-5)


def test_values_c2_shape_sin_fp32_matches_oracle_jets(gpu, oracle):
    c = pkg.config2(n_points=4096, with_fast=False)
    m = c["model"]
    gpu.set_lrnr(m, pkg.F32)
    u = gpu.values(pkg.MODEL_LRNR, c["s"], c["pts"])
    want = oracle.lrnr_jets(m.widths, m.ranks, m.params, c["s"], c["pts"], act=pkg.ACT_SIN)[:, 0]
    assert rel(u, want) <= 1e-4  # FP32 vs FP64 (|u| ~ 6e-4 here: the error scale is the summands')


@pytest.mark.parametrize("n_ic,n_bc", [(0, 0), (37, 0), (0, 19), (64, 33)])
@pytest.mark.parametrize("model", [pkg.MODEL_LRNR, pkg.MODEL_FAST])
def test_loss_tune_fp64_matches_reference(gpu, reference, c1, n_ic, n_bc, model):
    m, f = c1["model"], c1["fast"]
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_fast(f, pkg.F64)
    pts = c1["pts"][:777]
    rng = np.random.default_rng(5)
    icx = rng.uniform(0, pkg.api.TWO_PI, n_ic)
    pt = rng.uniform(0, 1, n_bc)
    gpu.set_points(pts)
    gpu.set_boundary(icx, pt)
    got = gpu.loss_tune(model, c1["s"], c1["mu"])
    if model == pkg.MODEL_LRNR:
        want = reference.loss_tune(m.widths, m.ranks, m.params, c1["s"], c1["mu"], pts, icx, pt)
    else:  # loss_tune's terms on the FastLRNR: reference jets / values, the same means
        jets = reference.fast_jets(f.ranks, f.red_ranks, f.fparams, c1["s"], pts)
        mu = c1["mu"]
        N = jets[:, 2] + mu[0] * jets[:, 1] - mu[1] * jets[:, 3] - mu[2] * jets[:, 0] * (1 - jets[:, 0])
        val = lambda xt: reference.values(1, None, f.ranks, None, f.red_ranks, f.fparams, c1["s"], xt)
        b = 0.0
        if n_ic:
            b += np.mean((val(np.stack([icx, 0 * icx], 1)) - np.sin(icx)) ** 2)
        if n_bc:
            b += np.mean((val(np.stack([0 * pt, pt], 1)) - val(np.stack([0 * pt + pkg.api.TWO_PI, pt], 1))) ** 2)
        want = np.array([np.mean(N ** 2) + b, np.mean(N ** 2), b])
    np.testing.assert_allclose([got["total"], got["residual"], got["boundary"]], want, rtol=1e-12, atol=1e-300)
    gpu.set_boundary([], [])


@pytest.mark.parametrize("nx,nt", [(4, 3), (7, 5), (1, 1)])
def test_loss_fast_fp64_matches_reference(gpu, reference, c1, nx, nt):
    f = c1["fast"]
    gpu.set_fast(f, pkg.F64)
    X = pkg.uniform_grid(nx, nt)
    got = gpu.loss_fast(pkg.MODEL_FAST, c1["s"], c1["mu"], X)
    want = reference.loss_fast(f.ranks, f.red_ranks, f.fparams, c1["s"], c1["mu"], X)
    np.testing.assert_allclose([got["total"], got["residual"], got["boundary"]], want, rtol=1e-12, atol=1e-300)


def test_loss_fast_c2_fp32_tanh_matches_reference(gpu, reference):
    c = pkg.config2(n_points=0, act=pkg.ACT_TANH)
    f = c["fast"]
    gpu.set_fast(f, pkg.F32)
    X = pkg.uniform_grid(4, 3)
    got = gpu.loss_fast(pkg.MODEL_FAST, c["s"], c["mu"], X)
    want = reference.loss_fast(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], X)
    np.testing.assert_allclose([got["total"], got["residual"], got["boundary"]], want, rtol=1e-4)


@pytest.mark.parametrize("dtype,tol", [(pkg.F64, 1e-12), (pkg.F32, 1e-4)])
@pytest.mark.parametrize("with_bnd", [False, True])
def test_loss_meta_matches_reference(gpu, reference, dtype, tol, with_bnd):
    n_inst, per, n_ic, n_bc = 3, 40, 5, 4
    m, _ = pkg.make_baseline_model([2, 48, 48, 1], [2, 8, 1], 99, pkg.ACT_TANH)
    h = pkg.make_hyper_params(m.ranks, 2, 16, 98, pkg.api.C3_LO, pkg.api.C3_HI, 0.01, 0.5)
    _, mus = pkg.sample_collocation(97, n_inst, pkg.api.C3_LO, pkg.api.C3_HI, with_mu=True)
    pts = pkg.sample_collocation(96, n_inst * per)
    rng = np.random.default_rng(3)
    icx = rng.uniform(0, pkg.api.TWO_PI, (n_inst, n_ic)) if with_bnd else np.zeros((n_inst, 0))
    pt = rng.uniform(0, 1, (n_inst, n_bc)) if with_bnd else np.zeros((n_inst, 0))
    gpu.set_lrnr(m, dtype)
    gpu.set_hyper(h)
    gpu.set_points(pts, n_inst=n_inst)
    gpu.set_meta_boundary(n_inst, icx.reshape(-1), pt.reshape(-1))
    got = gpu.loss_meta(mus)
    want = reference.loss_meta(m.widths, m.ranks, m.params, h.hw, h.params, h.lo, h.hi, pts,
                               np.repeat(mus, per, axis=0), icx.reshape(-1), np.repeat(mus, icx.shape[1], axis=0),
                               pt.reshape(-1), np.repeat(mus, pt.shape[1], axis=0))
    np.testing.assert_allclose([got["total"], got["residual"], got["boundary"]], want, rtol=tol, atol=1e-300)
    gpu.set_meta_boundary(n_inst)


def test_loss_nonfinite_raises_tag_minus_one(gpu, c1):
    m = c1["model"]
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_points(c1["pts"][:64])
    gpu.set_boundary([0.5], [])
    s = c1["s"].copy()
    s[3] = np.nan
    with pytest.raises(pkg.NonFiniteError) as e:
        gpu.loss_tune(pkg.MODEL_LRNR, s, c1["mu"])
    assert e.value.layer_tag == -1
    gpu.set_boundary([], [])
    # the context stays usable and clean
    r = gpu.loss_tune(pkg.MODEL_LRNR, c1["s"], c1["mu"])
    assert np.isfinite(r["total"])


def test_nonfinite_flag_is_per_model(gpu, c1):
    """A FastLRNR failure queued before a clean LRNR step is neither lost nor blamed on the LRNR
    (one flag per model slot, cleared only when read)."""
    m, f = c1["model"], c1["fast"]
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_fast(f, pkg.F64)
    gpu.set_points(c1["pts"][:256])
    bad_s = c1["s"].copy()
    bad_s[0] = np.inf
    gpu.upload_coeffs(bad_s, c1["mu"])
    gpu.run(pkg.MODEL_FAST)              # asynchronous, not checked yet
    r = gpu.loss_grad_s(pkg.MODEL_LRNR, c1["s"], c1["mu"])  # clean LRNR step: no error
    assert np.isfinite(r["value"])
    with pytest.raises(pkg.NonFiniteError):
        gpu.check()                      # the FastLRNR's failure is still reported
    gpu.check()                          # and cleared once read
    with pytest.raises(pkg.NonFiniteError):
        gpu.loss_grad_s(pkg.MODEL_FAST, bad_s, c1["mu"])
    r = gpu.loss_grad_s(pkg.MODEL_FAST, c1["s"], c1["mu"])
    assert np.isfinite(r["value"])


def test_nccl_comm_single_rank_is_identity(golden):
    """The C ABI's NCCL communicator at nranks = 1 (a 2-rank NCCL needs two GPUs): attaching
    it leaves every result unchanged (the all-reduce runs on the context stream)."""
    c = pkg.config1(n_points=1024)
    ctx = pkg.GpuContext(0)
    try:
        ctx.set_lrnr(c["model"], pkg.F64)
        ctx.set_fast(c["fast"], pkg.F64)
        ctx.set_points(c["pts"])
        before = ctx.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"])
        beforef = ctx.loss_grad_s(pkg.MODEL_FAST, c["s"], c["mu"])
        ctx.comm_init(1, 0, pkg.GpuContext.comm_unique_id())
        assert ctx.comm_info() == (1, 0)
        after = ctx.loss_grad_s(pkg.MODEL_LRNR, c["s"], c["mu"])
        afterf = ctx.loss_grad_s(pkg.MODEL_FAST, c["s"], c["mu"])
        assert after["value"] == before["value"] and np.array_equal(after["grad_s"], before["grad_s"])
        assert afterf["value"] == beforef["value"] and np.array_equal(afterf["grad_s"], beforef["grad_s"])
        lt = ctx.loss_tune(pkg.MODEL_LRNR, c["s"], c["mu"])
        assert abs(lt["residual"] - before["value"]) <= 1e-12 * before["value"]
        ctx.set_comm(None)
        assert ctx.comm_info() == (1, 0)
    finally:
        ctx.close()


# ---------------------------------------------------------------------------
# against the committed reference fixtures (tests/golden/make_golden_r2.py)
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def g2():
    import os
    return dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden_r2.npz")))


def c0_model(g2):
    return pkg.LrnrParams(np.array(pkg.api.C0_WIDTHS), np.array(pkg.api.C0_RANKS), g2["c0_params"], pkg.ACT_TANH)


def test_golden_values_loss_tune_loss_fast(gpu, g2):
    m = c0_model(g2)
    f = pkg.FastParams(np.array(pkg.api.C0_RANKS), g2["c1_red"], g2["c1_fparams"], pkg.ACT_TANH)
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_fast(f, pkg.F64)
    s, mu = g2["c0_s"], np.array([30.0, 0.0, 0.0])
    assert rel(gpu.values(pkg.MODEL_LRNR, s, g2["val_pts"]), g2["val_lrnr"]) <= 1e-12
    assert rel(gpu.values(pkg.MODEL_FAST, s, g2["val_pts"]), g2["val_fast"]) <= 1e-12
    gpu.set_points(g2["lt_pts"])
    gpu.set_boundary(g2["lt_icx"], g2["lt_pert"])
    lt = gpu.loss_tune(pkg.MODEL_LRNR, s, mu)
    np.testing.assert_allclose([lt["total"], lt["residual"], lt["boundary"]], g2["lt_out"], rtol=1e-12)
    gpu.set_boundary([], [])
    for k in ("4x3", "7x5"):
        lf = gpu.loss_fast(pkg.MODEL_FAST, s, mu, g2[f"lf_{k}_X"])
        np.testing.assert_allclose([lf["total"], lf["residual"], lf["boundary"]], g2[f"lf_{k}_out"], rtol=1e-12)


def test_golden_loss_meta_per_sample_mu(gpu, g2):
    """loss_meta with a different mu for every sample: one instance per sample (the adapter's mapping)."""
    m = c0_model(g2)
    h = pkg.HyperParams(np.array([3, 16, 16, 23]), g2["lm_hparams"], np.array(pkg.api.C3_LO), np.array(pkg.api.C3_HI))
    gpu.set_lrnr(m, pkg.F64)
    gpu.set_hyper(h)
    parts = []
    gpu.set_points(g2["lm_pts"], n_inst=len(g2["lm_pts"]))
    gpu.set_meta_boundary(len(g2["lm_pts"]))
    parts.append(gpu.loss_meta(g2["lm_mu"]))
    gpu.set_points(np.zeros((0, 2)), n_inst=len(g2["lm_icx"]))
    gpu.set_meta_boundary(len(g2["lm_icx"]), g2["lm_icx"], [])
    parts.append(gpu.loss_meta(g2["lm_icmu"]))
    gpu.set_points(np.zeros((0, 2)), n_inst=len(g2["lm_pert"]))
    gpu.set_meta_boundary(len(g2["lm_pert"]), [], g2["lm_pert"])
    parts.append(gpu.loss_meta(g2["lm_permu"]))
    gpu.set_meta_boundary(len(g2["lm_pert"]))
    residual = parts[0]["residual"]
    boundary = parts[1]["boundary"] + parts[2]["boundary"]
    np.testing.assert_allclose([residual + boundary, residual, boundary], g2["lm_out"], rtol=1e-12)


def test_mu_grid_fastlrnr_c2_fp32_gradient_matches_oracle(gpu, oracle, g2):
    """The bench's c2 FastLRNR (mu-grid recipe, r_hat 32) on the narrow-network kernel vs the FP64 oracle."""
    m, s = pkg.make_baseline_model(pkg.api.C2_WIDTHS, pkg.api.C2_RANKS, 2411, pkg.ACT_TANH)
    f = pkg.FastParams(m.ranks, g2["c2grid_red"], g2["c2grid_fparams"], pkg.ACT_TANH)
    pts = pkg.sample_collocation(4002, 20000)
    mu = np.array([20.0, 0.01, 5.0])
    gpu.set_fast(f, pkg.F32)
    gpu.set_points(pts)
    r = gpu.loss_grad_s(pkg.MODEL_FAST, s, mu)
    want = oracle.fast_grad(f.ranks, f.red_ranks, f.fparams, s, mu, pts)
    assert np.linalg.norm(r["grad_s"] - want["grad_s"]) / np.linalg.norm(want["grad_s"]) <= 1e-4
    assert abs(r["value"] - want["value"]) <= 1e-4 * abs(want["value"])
