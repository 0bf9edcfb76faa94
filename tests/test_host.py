"""CPU: host-side setup of the product library (generators, FastLRNR EIM
construction) bit-exact against the reference's golden vectors, and the C ABI
surface (every symbol include/lrnr_gpu.h declares is exported; errors map to
the reference's exception types).  No GPU compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2410_04001_b200 as pkg
from paper_2410_04001_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_generators_bit_exact(golden):
    m, s = pkg.make_baseline_model(golden["c0_widths"], golden["c0_ranks"], 2410)
    assert np.array_equal(m.params, golden["c0_params"]) and np.array_equal(s, golden["c0_s"])
    m2, s2 = pkg.make_baseline_model(golden["c2_widths"], golden["c2_ranks"], 2411)
    assert np.array_equal(m2.params, golden["c2_params"]) and np.array_equal(s2, golden["c2_s"])
    assert np.array_equal(pkg.sample_collocation(4001, 4096), golden["c0_pts"])
    assert np.array_equal(pkg.sample_collocation(4002, 1024), golden["c2_pts"])
    h = pkg.make_hyper_params(golden["c2_ranks"], 2, 64, 4003, golden["c3_lo"], golden["c3_hi"], 0.01, 0.5)
    assert np.array_equal(h.hw, golden["c3_hw"]) and np.array_equal(h.params, golden["c3_hparams"])


def test_eim_reduction_bit_exact_c1(golden):
    """harvest_snapshots + eim_greedy + build_fastparams: index selection bit-for-bit."""
    m = pkg.LrnrParams(golden["c0_widths"], golden["c0_ranks"], golden["c0_params"], pkg.ACT_TANH)
    f = pkg.build_fast(m, golden["c0_s"], nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=10)
    assert np.array_equal(f.indices, golden["c1_indices"])
    assert np.array_equal(f.red_ranks, golden["c1_red_ranks"])
    assert np.array_equal(f.fparams, golden["c1_fparams"])


def test_eim_reduction_bit_exact_c2(golden):
    m = pkg.LrnrParams(golden["c2_widths"], golden["c2_ranks"], golden["c2_params"], pkg.ACT_TANH)
    f = pkg.build_fast(m, golden["c2_s"], nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=32)
    assert np.array_equal(f.indices, golden["c2_indices"])
    assert np.array_equal(f.red_ranks, golden["c2_red_ranks"])
    assert np.array_equal(f.fparams, golden["c2_fparams"])


EIM_TAGS = ["a", "b", "c", "d"]


@pytest.mark.parametrize("tag", EIM_TAGS)
def test_host_eim_greedy_bit_exact(golden, tag):
    """lrnr_host_eim_greedy == reduction::eim_greedy bit-for-bit (indices, basis columns,
    exhaustion) on the golden snapshot sets: tanh features, rank-deficient (exhausts the
    budget), duplicated columns (argmax ties), 64 rows with r_hat = 64."""
    e = pkg.eim_greedy(golden[f"eim_{tag}_S"], int(golden[f"eim_{tag}_rhat"][0]))
    assert np.array_equal(e["indices"], golden[f"eim_{tag}_idx"])
    assert np.array_equal(e["xi"], golden[f"eim_{tag}_xi"])
    assert e["exhausted"] == bool(golden[f"eim_{tag}_exh"][0])


def test_eim_greedy_rejects_bad_input():
    with pytest.raises(ValueError):
        pkg.eim_greedy(np.ones((4, 3)), 0)
    with pytest.raises(ValueError):
        pkg.eim_greedy(np.zeros((4, 0)), 2)
    with pytest.raises(ValueError):
        pkg.eim_greedy(np.zeros((4, 3)), 2)  # all-zero snapshots: no basis vector selected


def numpy_hidden_states(m, s, pts):
    """hidden_states (model.cpp:407-428) for many points at once, FP64 numpy."""
    offs, _ = m.offsets()
    P, z, so, out = m.params, pts.T, 0, []
    for l in range(m.depth - 1):
        w0, w1, r = int(m.widths[l]), int(m.widths[l + 1]), int(m.ranks[l])
        oU, oV, ob = offs[l]
        U, V, b = P[oU:oU + w1 * r].reshape(w1, r), P[oV:oV + w0 * r].reshape(w0, r), P[ob:ob + w1]
        y = (V.T @ z) * s[so:so + r, None]
        z = np.tanh(U @ y + b[:, None])
        out.append(z)
        so += r
    return out


def test_harvest_points_and_build_fastparams_compose(golden):
    """harvest_points -> hidden states -> eim_greedy per layer -> build_fastparams reproduces
    build_fast (and so the reference's c1 reduction): the pieces the device path uses."""
    m = pkg.LrnrParams(golden["c0_widths"], golden["c0_ranks"], golden["c0_params"], pkg.ACT_TANH)
    X = pkg.harvest_points(1, 4, 3, 8, 0.05, 777)
    assert X.shape == (108, 2)
    assert np.all((X[:, 0] >= 0) & (X[:, 0] <= 2 * np.pi) & (X[:, 1] >= 0) & (X[:, 1] <= 1))
    assert np.array_equal(X[::9, 0], np.tile(2 * np.pi * np.arange(4) / 3, 3))
    bases = [pkg.eim_greedy(S, 10) for S in numpy_hidden_states(m, golden["c0_s"], X)]
    f = pkg.build_fastparams(m, bases, r_hat=10)
    assert np.array_equal(f.indices, golden["c1_indices"])
    assert np.allclose(f.fparams, golden["c1_fparams"], rtol=1e-9, atol=1e-12)


def test_eim_rejects_bad_shapes():
    m = pkg.LrnrParams(np.array([2, 4, 1]), np.array([3, 1]), np.zeros(64))
    with pytest.raises(ValueError):
        pkg.build_fast(m, np.ones(4))


def test_flop_model_matches_survey():
    """68,880 / 1,323,088 / 7,364,688 FLOP per point; meta 11,047,032."""
    assert pkg.algorithmic_flops_per_point([2, 100, 100, 100, 1], [2, 10, 10, 1]) == 68880
    assert pkg.algorithmic_flops_per_point([2] + [256] * 6 + [1], [2] + [32] * 5 + [1]) == 1323088
    assert pkg.algorithmic_flops_per_point([2] + [512] * 8 + [1], [2] + [64] * 7 + [1]) == 7364688
    assert pkg.algorithmic_flops_per_point([2] + [512] * 8 + [1], [2] + [64] * 7 + [1], meta=True) == 11047032
    assert pkg.fast_flops_per_point([2, 10, 10, 1], [10, 10, 10]) == 6960
    assert pkg.fast_flops_per_point([2] + [32] * 5 + [1], [32] * 6) == 165456


def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "lrnr_gpu.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(lrnr_(?:gpu|host|ckpt)_\w+)\s*\(", header, re.M))
    assert len(declared) >= 25
    lib = C.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTS)


def test_abi_context_errors_without_a_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.LrnrGpuError):
        pkg.GpuContext(0)


def test_abi_null_and_bad_arguments_are_einval():
    lib = _lib.load()
    assert lib.lrnr_gpu_create(0, None) == _lib.LRNR_EINVAL
    assert lib.lrnr_gpu_destroy(None) == _lib.LRNR_OK
    assert lib.lrnr_gpu_set_points(None, None, 1, 1) == _lib.LRNR_EINVAL
    assert lib.lrnr_gpu_last_layer_tag(None) == -1
    w = np.array([2, 4, 1], np.int64)
    r = np.array([3, 1], np.int64)  # rank exceeds min(M_l, M_{l-1})
    P = np.zeros(64)
    s = np.zeros(4)
    rc = lib.lrnr_host_make_baseline_model(2, w.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p),
                                           C.c_uint64(1), P.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p))
    assert rc == _lib.LRNR_EINVAL


def test_dist_shard_ranges_cover_exactly():
    from paper_2410_04001_b200.dist import shard_range

    for n in (0, 1, 7, 1 << 20, 1000003):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, k) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[k][1] == spans[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


# ----------------------------------------------------------------------------
# checkpoint interop (proj/src/checkpoint.cpp format)
# ----------------------------------------------------------------------------
CKPT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_checkpoint.lrnr")


def test_reads_reference_written_checkpoint(golden):
    g = golden
    ck = pkg.Checkpoint(CKPT)
    m = ck.lrnr()
    assert list(m.widths) == list(g["c0_widths"]) and list(m.ranks) == list(g["c0_ranks"])
    assert np.array_equal(m.params, g["c0_params"])
    h = ck.hyper()
    assert list(h.hw) == list(g["ck_hw"]) and np.array_equal(h.params, g["ck_hparams"])
    assert np.array_equal(h.lo, g["c3_lo"]) and np.array_equal(h.hi, g["c3_hi"])
    assert ck.has_fast()
    f = ck.fast()
    assert list(f.red_ranks) == list(g["c1_red_ranks"]) and np.array_equal(f.fparams, g["c1_fparams"])
    assert np.array_equal(ck.sampling(), g["c1_phase_x"])


def test_checkpoint_round_trip(tmp_path, golden):
    g = golden
    src = pkg.Checkpoint(CKPT)
    out = pkg.Checkpoint()
    out.put_lrnr(src.lrnr())
    out.put_hyper(src.hyper(), g["c0_ranks"])
    out.put_fast(src.fast())
    out.put_sampling(src.sampling())
    path = tmp_path / "ours.lrnr"
    out.save(path)
    back = pkg.Checkpoint(path)
    assert np.array_equal(back.lrnr().params, g["c0_params"])
    assert np.array_equal(back.hyper().params, g["ck_hparams"])
    assert np.array_equal(back.fast().fparams, g["c1_fparams"])
    assert np.array_equal(back.sampling(), g["c1_phase_x"])


def test_checkpoint_written_here_loads_in_the_reference(tmp_path, golden):
    from oracle.oracle import ReferenceCheckpoint, reference_ckpt_available
    if not reference_ckpt_available():
        pytest.skip("reference checkpoint library not built (needs /root/reference and its json header)")
    g = golden
    out = pkg.Checkpoint()
    m = pkg.LrnrParams(g["c0_widths"], g["c0_ranks"], g["c0_params"])
    out.put_lrnr(m)
    out.put_hyper(pkg.HyperParams(g["ck_hw"], g["ck_hparams"], g["c3_lo"], g["c3_hi"]), g["c0_ranks"])
    out.put_sampling(g["c1_phase_x"])
    path = tmp_path / "ours.lrnr"
    out.save(path)
    P, H = ReferenceCheckpoint().read(path, m.params.size, g["ck_hparams"].size)
    assert np.array_equal(P, g["c0_params"]) and np.array_equal(H, g["ck_hparams"])


def test_checkpoint_rejects_bad_files(tmp_path):
    bad = tmp_path / "bad.lrnr"
    bad.write_bytes(b"NOPE\x01\x00\x00\x00")
    with pytest.raises(ValueError):
        pkg.Checkpoint(bad)
    trunc = tmp_path / "trunc.lrnr"
    trunc.write_bytes(open(CKPT, "rb").read()[:1000])
    with pytest.raises(ValueError):
        pkg.Checkpoint(trunc)


@pytest.fixture(scope="module")
def golden_r2():
    return dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden_r2.npz")))


def test_host_hyper_forward_bit_exact(golden_r2):
    """hyper_forward (model.cpp:294-318) of the c3 hypernetwork on the mu grid, bit for bit."""
    h = pkg.c3_hyper()
    assert np.array_equal(h.params, golden_r2["c3_hparams"])
    S = pkg.hyper_forward(h, golden_r2["mu_grid"])
    assert np.array_equal(S, golden_r2["grid_s"])


def test_mu_grid_fast_construction_bit_exact(golden_r2):
    """The c2 FastLRNR from snapshots over the mu grid (harvest_snapshots with mu_grid, eim_greedy,
    build_fastparams; reduction.cpp:111-283): indices and reduced matrices equal the reference's, and
    the budget of 32 is reached in every inner layer (tanh, the reference's activation)."""
    m, _ = pkg.make_baseline_model(pkg.api.C2_WIDTHS, pkg.api.C2_RANKS, 2411, pkg.ACT_TANH)
    f = pkg.build_fast(m, golden_r2["grid_s"], nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=32)
    assert list(f.red_ranks) == list(golden_r2["c2grid_red"]) == [32] * 6
    assert np.array_equal(f.indices, golden_r2["c2grid_idx"])
    assert np.array_equal(f.fparams, golden_r2["c2grid_fparams"])
    c = pkg.config2(n_points=0, act=pkg.ACT_TANH)  # the bench's / tests' c2 builder uses this recipe
    assert np.array_equal(c["fast"].fparams, golden_r2["c2grid_fparams"])


def test_hyper_forward_rejects_bad_shapes():
    h = pkg.c3_hyper()
    bad = pkg.HyperParams(np.array([2, 64, 163]), h.params[:10], h.lo, h.hi)
    with pytest.raises(ValueError):
        pkg.hyper_forward(bad, [[1.0, 0.0, 0.0]])
