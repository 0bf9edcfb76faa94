"""Python binding of the C ABI (include/lrnr_gpu.h) used by the tests and bench.

The drop-in for the reference's C++ callers is include/lrnr_gpu_adapter.hpp
(C++ over the same ABI); this module is the ctypes view of that ABI plus the
BASELINE-config builders.  Errors map to the reference's exception types:
LRNR_EINVAL -> ValueError (std::invalid_argument), LRNR_ENONFINITE ->
NonFiniteError(layer_tag) (autodiff.hpp:28-34).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import ACT_SIN, ACT_TANH, F32, F64, MODEL_FAST, MODEL_LRNR  # noqa: F401
from ._lib import (  # noqa: F401
    KERNEL_AUTO, KERNEL_FMA_TILE, KERNEL_NARROW, KERNEL_SMALL, KERNEL_STREAM, KERNEL_TC, OBJ_ABS, OBJ_SQUARED, OPT_FAST_SINCOS, OPT_KERNEL, OPT_META_PREC, OPT_SOLVE,
    OPT_TILE_P,
)

TWO_PI = 6.283185307179586476925286766559


class NonFiniteError(FloatingPointError):
    """Mirror of lrnr::NonFiniteError (autodiff.hpp:28-34)."""

    def __init__(self, layer_tag: int, msg: str = ""):
        super().__init__(msg or f"non-finite value in recorded computation, layer tag {layer_tag}")
        self.layer_tag = layer_tag


class LrnrGpuError(RuntimeError):
    pass


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# parameter containers (flat layouts of include/lrnr_gpu.h)
# ---------------------------------------------------------------------------
@dataclass
class LrnrParams:
    """LrnrParams (model.hpp:38-49) as widths, ranks and the flat U,V,b array."""
    widths: np.ndarray
    ranks: np.ndarray
    params: np.ndarray
    act: int = ACT_TANH

    @property
    def depth(self) -> int:
        return len(self.ranks)

    @property
    def r_total(self) -> int:
        return int(np.sum(self.ranks))

    def offsets(self):
        o, out = 0, []
        for l in range(self.depth):
            w0, w1, r = int(self.widths[l]), int(self.widths[l + 1]), int(self.ranks[l])
            oU = o
            o += w1 * r
            oV = o
            o += w0 * r
            ob = o
            o += w1
            out.append((oU, oV, ob))
        return out, o


@dataclass
class FastParams:
    """FastParams (model.hpp:65-78), flat layout of include/lrnr_gpu.h."""
    ranks: np.ndarray
    red_ranks: np.ndarray
    fparams: np.ndarray
    act: int = ACT_TANH
    indices: Optional[np.ndarray] = None
    exhausted: Optional[np.ndarray] = None

    @property
    def r_total(self) -> int:
        return int(np.sum(self.ranks))


@dataclass
class HyperParams:
    """HyperParams (model.hpp:83-95): widths hw (3, ..., r_total), flat W,b, box."""
    hw: np.ndarray
    params: np.ndarray
    lo: np.ndarray = field(default_factory=lambda: np.zeros(3))
    hi: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def n_params(self) -> int:
        return int(sum(self.hw[k + 1] * self.hw[k] + self.hw[k + 1] for k in range(len(self.hw) - 1)))


# ---------------------------------------------------------------------------
# host-side generators and FastLRNR construction (CPU, inside the native lib)
# ---------------------------------------------------------------------------
def make_baseline_model(widths, ranks, seed, act=ACT_TANH):
    lib = _lib.load()
    w, r = _i64(widths), _i64(ranks)
    n = int(sum(w[l + 1] * r[l] + w[l] * r[l] + w[l + 1] for l in range(len(r))))
    P, s = np.zeros(n), np.zeros(int(r.sum()))
    rc = lib.lrnr_host_make_baseline_model(len(r), _p(w), _p(r), C.c_uint64(seed), _p(P), _p(s))
    if rc != 0:
        raise ValueError("make_baseline_model: invalid shapes")
    return LrnrParams(w, r, P, act), s


def make_hyper_params(split, hidden_depth, hidden_width, seed, lo, hi, out_w_scale=0.01, out_bias=0.5):
    lib = _lib.load()
    sp = _i64(split)
    hw = np.array([3] + [hidden_width] * hidden_depth + [int(sp.sum())], np.int64)
    n = int(sum(hw[k + 1] * hw[k] + hw[k + 1] for k in range(len(hw) - 1)))
    H = np.zeros(n)
    rc = lib.lrnr_host_make_hyper_params(len(sp), _p(sp), hidden_depth, hidden_width, C.c_uint64(seed),
                                         C.c_double(out_w_scale), C.c_double(out_bias), _p(H))
    if rc != 0:
        raise ValueError("make_hyper_params failed")
    return HyperParams(hw, H, _f64(lo), _f64(hi))


def hyper_forward(h: HyperParams, mus):
    """hyper_forward (model.cpp:294-318) on the host for each row of mus (n, 3) -> (n, r_total); the same
    roundings as the reference build (host C++, lrnr_host_hyper_forward)."""
    mus = _f64(mus).reshape(-1, 3)
    hw = _i64(h.hw)
    out = np.zeros((mus.shape[0], int(hw[-1])))
    rc = _lib.load().lrnr_host_hyper_forward(len(hw) - 1, _p(hw), _p(_f64(h.params)), _p(_f64(h.lo)), _p(_f64(h.hi)),
                                             mus.shape[0], _p(mus), _p(out))
    if rc != 0:
        raise ValueError("hyper_forward: bad shapes")
    return out


def sample_collocation(seed, n_interior, lo=(0.0, 0.0, 0.0), hi=(0.0, 0.0, 0.0), with_mu=False):
    lib = _lib.load()
    xt = np.zeros(2 * n_interior + 2)
    mu = np.zeros(3 * n_interior + 3)
    rc = lib.lrnr_host_sample_collocation(C.c_uint64(seed), n_interior, _p(_f64(lo)), _p(_f64(hi)), int(with_mu),
                                          _p(xt), _p(mu))
    if rc != 0:
        raise ValueError("sample_collocation failed")
    xt = xt[:2 * n_interior].reshape(n_interior, 2)
    return (xt, mu[:3 * n_interior].reshape(n_interior, 3)) if with_mu else xt


def _fast_buffers(model: LrnrParams, r_hat):
    L = model.depth
    nF = 2 * int(model.ranks[0])
    for l in range(L - 1):
        nF += r_hat * int(model.ranks[l]) + r_hat + r_hat * int(model.ranks[l + 1])
    nF += int(model.ranks[-1]) + 1
    return np.zeros(L - 1, np.int64), np.zeros((L - 1) * r_hat, np.int64), np.zeros(nF), np.zeros(L - 1, np.int32)


def _fast_result(model: LrnrParams, r_hat, red, idx, F, exh) -> FastParams:
    L = model.depth
    used = 2 * int(model.ranks[0])
    for l in range(L - 1):
        used += int(red[l]) * (int(model.ranks[l]) + 1 + int(model.ranks[l + 1]))
    used += int(model.ranks[-1]) + 1
    return FastParams(model.ranks.copy(), red, F[:used], model.act, idx.reshape(L - 1, r_hat), exh)


def build_fast(model: LrnrParams, s, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=10) -> FastParams:
    """harvest_snapshots + eim_greedy + build_fastparams (reduction.cpp:111-283), on the host.
    GpuContext.build_fast is the device path."""
    lib = _lib.load()
    S = _f64(s).reshape(-1, model.r_total)
    red, idx, F, exh = _fast_buffers(model, r_hat)
    rc = lib.lrnr_host_build_fast(model.depth, _p(model.widths), _p(model.ranks), _p(_f64(model.params)), model.act,
                                  _p(S), S.shape[0], nx, nt, n_perturb, C.c_double(sigma), C.c_uint64(seed), r_hat,
                                  _p(red), _p(idx), _p(F), exh.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise ValueError("build_fast: reduction failed (shape error or singular interpolation block)")
    return _fast_result(model, r_hat, red, idx, F, exh)


def uniform_grid(nx=4, nt=3):
    """SamplingSetX::uniform_grid (reduction.cpp:10-25): (nx*nt, 2) points, x fastest."""
    out = np.zeros(2 * nx * nt)
    if _lib.load().lrnr_host_uniform_grid(nx, nt, _p(out)) != 0:
        raise ValueError("uniform_grid: bad sizes")
    return out.reshape(-1, 2)


def harvest_points(n_mu=1, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, X=None):
    """The (x, t) columns harvest_snapshots evaluates (reduction.cpp:111-148) for the sampling
    set X (default: uniform_grid(nx, nt)), (n_mu * len(X) * (1 + n_perturb), 2)."""
    X = uniform_grid(nx, nt) if X is None else _f64(X).reshape(-1, 2)
    n = n_mu * X.shape[0] * (1 + n_perturb)
    out = np.zeros(2 * n)
    rc = _lib.load().lrnr_host_harvest_points(_p(X), X.shape[0], n_mu, n_perturb, C.c_double(sigma),
                                              C.c_uint64(seed), _p(out))
    if rc != 0:
        raise ValueError("harvest_points: bad arguments")
    return out.reshape(n, 2)


def _eim_call(fn, lead, S, r_hat, what):
    S = _f64(S)
    if S.ndim != 2:
        raise ValueError(what + ": snapshots must be a 2-D (M x n_cols) array")
    m, n = S.shape
    idx = np.zeros(max(r_hat, 1), np.int64)
    xi = np.zeros((m, max(r_hat, 1)))
    cnt, ex = C.c_int64(0), C.c_int(0)
    rc = fn(*lead, m, n, _p(S), r_hat, _p(idx), _p(xi), C.byref(cnt), C.byref(ex))
    return rc, dict(indices=idx[:cnt.value].copy(), xi=xi[:, :cnt.value].copy(), exhausted=bool(ex.value))


def eim_greedy(S, r_hat):
    """reduction::eim_greedy (reduction.cpp:150-238) on the host: dict(indices, xi (M x r), exhausted)."""
    rc, out = _eim_call(_lib.load().lrnr_host_eim_greedy, (), S, r_hat, "eim_greedy")
    if rc != 0:
        raise ValueError("eim_greedy: bad snapshots/budget or singular interpolation block")
    return out


def build_fastparams(model: LrnrParams, bases, r_hat=None) -> FastParams:
    """reduction::build_fastparams (reduction.cpp:240-283) from per-inner-layer EIM bases
    (dicts with 'indices' and 'xi', as eim_greedy returns)."""
    L = model.depth
    if len(bases) != L - 1:
        raise ValueError("build_fastparams: one basis per inner layer")
    r_hat = r_hat or max(len(b["indices"]) for b in bases)
    red, idx, F, exh = _fast_buffers(model, r_hat)
    xi = []
    for l, b in enumerate(bases):
        k = len(b["indices"])
        red[l] = k
        idx[l * r_hat:l * r_hat + k] = b["indices"]
        idx[l * r_hat + k:(l + 1) * r_hat] = -1
        x = np.zeros((int(model.widths[l + 1]), r_hat))
        x[:, :k] = _f64(b["xi"])[:, :k]
        xi.append(x.reshape(-1))
        exh[l] = int(b.get("exhausted", False))
    rc = _lib.load().lrnr_host_build_fastparams(L, _p(model.widths), _p(model.ranks), _p(_f64(model.params)),
                                                model.act, r_hat, _p(red), _p(idx), _p(np.concatenate(xi)), _p(F))
    if rc != 0:
        raise ValueError("build_fastparams: bad bases or singular interpolation block")
    return _fast_result(model, r_hat, red, idx, F, exh)


def qdeim(xi):
    """Q-DEIM rows of the basis xi (M x r): the rows a column-pivoted QR of xi^T picks, in
    selection order (BASELINE configs[1] wording; no reference counterpart)."""
    X = _f64(xi)
    if X.ndim != 2:
        raise ValueError("qdeim: xi must be a 2-D (M x r) array")
    m, r = X.shape
    idx = np.zeros(max(r, 1), np.int64)
    cnt = C.c_int64(0)
    if _lib.load().lrnr_host_qdeim(m, r, _p(X), _p(idx), C.byref(cnt)) != 0:
        raise ValueError("qdeim: bad sizes")
    return idx[:cnt.value].copy()


def build_fast_qdeim(model: LrnrParams) -> FastParams:
    """FastLRNR with Q-DEIM indices: per inner layer EimBasis{xi = U^l, indices = qdeim(U^l)},
    r_hat_l = r_l, then the reference's build_fastparams (reduction.cpp:240-283)."""
    r_hat = int(max(model.ranks[:-1]))
    red, idx, F, exh = _fast_buffers(model, r_hat)
    rc = _lib.load().lrnr_host_build_fast_qdeim(model.depth, _p(model.widths), _p(model.ranks),
                                                _p(_f64(model.params)), model.act, r_hat, _p(red), _p(idx), _p(F))
    if rc != 0:
        raise ValueError("build_fast_qdeim: rank-deficient U^l or singular interpolation block")
    return _fast_result(model, r_hat, red, idx, F, exh)


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
class GpuContext:
    """One device + one stream (lrnr_gpu_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.lrnr_gpu_create(device, C.byref(h))
        if rc != 0:
            raise LrnrGpuError(f"lrnr_gpu_create({device}) failed with code {rc} (no usable CUDA device)")
        self.h = h
        self.r_total = {}
        self.hyper_n = 0
        self.n_points = 0
        self.n_inst = 0

    def close(self):
        if self.h:
            self.lib.lrnr_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _rc(self, rc, what):
        if rc == _lib.LRNR_OK:
            return
        msg = self.lib.lrnr_gpu_last_error(self.h).decode()
        if rc == _lib.LRNR_ENONFINITE:
            raise NonFiniteError(self.lib.lrnr_gpu_last_layer_tag(self.h), msg)
        if rc == _lib.LRNR_EINVAL:
            raise ValueError(f"{what}: {msg}")
        raise LrnrGpuError(f"{what}: code {rc}: {msg}")

    @property
    def launches(self) -> int:
        return int(self.lib.lrnr_gpu_launch_count(self.h))

    def set_stream(self, stream_handle: int | None):
        """Launch on a caller stream (e.g. torch.cuda.current_stream().cuda_stream).

        Handle 0 is the legacy default stream and is passed as cudaStreamLegacy;
        None restores the context's own stream."""
        h = None if stream_handle is None else (stream_handle if stream_handle != 0 else 1)
        self._rc(self.lib.lrnr_gpu_set_stream(self.h, C.c_void_p(h)), "set_stream")

    def set_lrnr(self, m: LrnrParams, dtype=F64):
        self._rc(self.lib.lrnr_gpu_set_lrnr(self.h, m.depth, _p(_i64(m.widths)), _p(_i64(m.ranks)),
                                            _p(_f64(m.params)), m.act, dtype), "set_lrnr")
        self.r_total[MODEL_LRNR] = m.r_total

    def set_fast(self, f: FastParams, dtype=F64):
        self._rc(self.lib.lrnr_gpu_set_fast(self.h, len(f.ranks), _p(_i64(f.ranks)), _p(_i64(f.red_ranks)), 2, 1,
                                            _p(_f64(f.fparams)), f.act, dtype), "set_fast")
        self.r_total[MODEL_FAST] = f.r_total

    def set_hyper(self, h: HyperParams):
        hw = _i64(h.hw)
        self._rc(self.lib.lrnr_gpu_set_hyper(self.h, len(hw) - 1, _p(hw), _p(_f64(h.params)), _p(_f64(h.lo)),
                                             _p(_f64(h.hi))), "set_hyper")
        self.hyper_n = h.n_params

    def set_points(self, xt, n_inst: int = 1):
        xt = _f64(xt).reshape(-1, 2)
        n = xt.shape[0]
        if n % n_inst:
            raise ValueError("points not divisible into instances")
        self._keep_pts = xt
        self._rc(self.lib.lrnr_gpu_set_points(self.h, _p(xt), n_inst, n // n_inst), "set_points")
        self.n_points, self.n_inst = n, n_inst

    def stage_points(self, xt, n_inst: int = 1):
        """Copy the NEXT batch asynchronously (lrnr_gpu_stage_points); keep xt unmodified until
        use_staged_points() returns (pinned memory makes the copy overlap current work)."""
        xt = _f64(xt).reshape(-1, 2)
        n = xt.shape[0]
        if n % n_inst:
            raise ValueError("points not divisible into instances")
        self._keep_stage = xt
        self._rc(self.lib.lrnr_gpu_stage_points(self.h, _p(xt), n_inst, n // n_inst), "stage_points")
        self._stage_counts = (n, n_inst)

    def use_staged_points(self):
        self._rc(self.lib.lrnr_gpu_use_staged_points(self.h), "use_staged_points")
        self._keep_pts, self._keep_stage = self._keep_stage, None
        self.n_points, self.n_inst = self._stage_counts

    def set_points_device(self, ptr: int, n_points: int, n_inst: int = 1):
        self._rc(self.lib.lrnr_gpu_set_points_device(self.h, C.c_void_p(ptr), n_inst, n_points // n_inst),
                 "set_points_device")
        self.n_points, self.n_inst = n_points, n_inst

    # --- per-step calls (host buffers) ---
    def loss_grad_s(self, model, s, mu, w=0.0):
        R = self.r_total[model]
        g = np.zeros(R)
        comps = np.zeros(4)
        v = C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_loss_grad_s(self.h, model, _p(_f64(s)), _p(_f64(mu)), C.c_double(w), C.byref(v),
                                               _p(comps), _p(g)), "loss_grad_s")
        return dict(value=v.value, comps=comps, grad_s=g)

    def set_boundary(self, initial_x=(), periodic_t=()):
        """Boundary points (CollocationBatch::initial_x / periodic_t) for terms_grad."""
        ic, pt = _f64(initial_x).reshape(-1), _f64(periodic_t).reshape(-1)
        self._rc(self.lib.lrnr_gpu_set_boundary(self.h, _p(ic), ic.shape[0], _p(pt), pt.shape[0]), "set_boundary")
        self.n_ic, self.n_bc = ic.shape[0], pt.shape[0]

    def terms_grad(self, model, s, mu, objective=OBJ_SQUARED, w_int=0.0, w_ic=0.0, w_bc=0.0, s_init=None,
                   lambda_local=0.0):
        """One solve step over interior + initial + periodic (+ locality) terms."""
        g = np.zeros(self.r_total[model])
        comps = np.zeros(4)
        v = C.c_double(0.0)
        si = None if s_init is None else _f64(s_init)
        self._rc(self.lib.lrnr_gpu_terms_grad(self.h, model, _p(_f64(s)), _p(_f64(mu)), objective, C.c_double(w_int),
                                              C.c_double(w_ic), C.c_double(w_bc), _p(si), C.c_double(lambda_local),
                                              C.byref(v), _p(comps), _p(g)), "terms_grad")
        return dict(value=v.value, comps=comps, grad_s=g)

    def loss_grad_s_multi(self, model, s, mu, w=0.0):
        R = self.r_total[model]
        g = np.zeros((self.n_inst, R))
        v = C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_loss_grad_s_multi(self.h, model, _p(_f64(s)), _p(_f64(mu)), C.c_double(w),
                                                     C.byref(v), _p(g)), "loss_grad_s_multi")
        return dict(value=v.value, grad_s=g)

    def hyper_loss_grad(self, model, mus, w=0.0):
        R = self.r_total[model]
        g = np.zeros((self.n_inst, R))
        gt = np.zeros(self.hyper_n)
        v = C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_hyper_loss_grad(self.h, model, _p(_f64(mus)), C.c_double(w), C.byref(v), _p(g),
                                                   _p(gt)), "hyper_loss_grad")
        return dict(value=v.value, grad_s=g, grad_theta=gt)

    def meta_loss_grad(self, mus, n_lrnr_params, w=0.0):
        g = np.zeros(n_lrnr_params + self.hyper_n)
        v = C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_meta_loss_grad(self.h, _p(_f64(mus)), C.c_double(w), C.byref(v), _p(g)),
                 "meta_loss_grad")
        return dict(value=v.value, grad=g)

    def set_meta_boundary(self, n_inst, initial_x=(), periodic_t=()):
        """Meta boundary points per instance: initial_x (n_inst x n_ic), periodic_t (n_inst x n_bc)."""
        ic = _f64(initial_x).reshape(n_inst, -1) if len(initial_x) else np.zeros((n_inst, 0))
        pt = _f64(periodic_t).reshape(n_inst, -1) if len(periodic_t) else np.zeros((n_inst, 0))
        ic, pt = np.ascontiguousarray(ic), np.ascontiguousarray(pt)
        self._rc(self.lib.lrnr_gpu_set_meta_boundary(self.h, n_inst, _p(ic), ic.shape[1], _p(pt), pt.shape[1]),
                 "set_meta_boundary")

    def meta_terms_grad(self, mus, n_lrnr_params, lambda_sparse=0.0, gamma=1.5, lambda_ortho=0.0, w=0.0):
        """meta_train's step: interior terms + sparse (banded decay) + ortho (Gram) regularizers."""
        g = np.zeros(n_lrnr_params + self.hyper_n)
        comps = np.zeros(4)
        v, ro = C.c_double(0.0), C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_meta_terms_grad(self.h, _p(_f64(mus)), C.c_double(w), C.c_double(lambda_sparse),
                                                   C.c_double(gamma), C.c_double(lambda_ortho), C.byref(v),
                                                   _p(comps), C.byref(ro), _p(g)), "meta_terms_grad")
        return dict(value=v.value, comps=comps, ortho=ro.value, grad=g)

    def fine_tune(self, s_init, mu, lr=1e-2, epochs=400, n_int=1024, n_ic=256, n_bc=256, seed=1234):
        """fine_tune (training.cpp:428-496) on the device for the bound LRNR."""
        return self._solve(self.lib.lrnr_gpu_fine_tune, self.r_total[MODEL_LRNR], epochs, _p(_f64(s_init)),
                           _p(_f64(mu)), C.c_double(lr), epochs, n_int, n_ic, n_bc, C.c_uint64(seed))

    def fast_solve(self, s_init, mu, X, lambda_local=1e-2, lr=1e-2, epochs=400):
        """fast_solve (training.cpp:498-607) on the device for the bound FastLRNR (one CUDA graph per epoch)."""
        X = _f64(X).reshape(-1, 2)
        return self._solve(self.lib.lrnr_gpu_fast_solve, self.r_total[MODEL_FAST], epochs, _p(_f64(s_init)),
                           _p(_f64(mu)), _p(X), X.shape[0], C.c_double(lambda_local), C.c_double(lr), epochs)

    def _solve(self, fn, G, epochs, *args):
        s = np.zeros(G)
        losses = np.zeros(max(1, epochs))
        bl, be, nr, fl = C.c_double(0.0), C.c_int64(0), C.c_int64(0), C.c_int(0)
        self._rc(fn(self.h, *args, _p(s), C.byref(bl), C.byref(be), _p(losses), C.byref(nr), C.byref(fl)), "solve")
        return dict(s=s, best_loss=bl.value, best_epoch=be.value, losses=losses[:nr.value], aborted=bool(fl.value & 1),
                    diverged=bool(fl.value & 2))

    def eim_greedy(self, S, r_hat):
        """reduction::eim_greedy (reduction.cpp:150-238) on the device; bit-identical to eim_greedy()."""
        rc, out = _eim_call(self.lib.lrnr_gpu_eim_greedy, (self.h,), S, r_hat, "eim_greedy")
        self._rc(rc, "eim_greedy")
        return out

    def harvest_snapshots(self, model: LrnrParams, s, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, X=None):
        """reduction::harvest_snapshots (reduction.cpp:111-148) on the device for the sampling set X
        (default uniform_grid(nx, nt)): one M_l x n_cols array per inner layer."""
        S = _f64(s).reshape(-1, model.r_total)
        X = uniform_grid(nx, nt) if X is None else _f64(X).reshape(-1, 2)
        n = S.shape[0] * X.shape[0] * (1 + n_perturb)
        rows = [int(w) for w in model.widths[1:-1]]
        out = np.zeros(sum(rows) * n)
        self._rc(self.lib.lrnr_gpu_harvest_snapshots(self.h, model.depth, _p(model.widths), _p(model.ranks),
                                                     _p(_f64(model.params)), model.act, _p(S), S.shape[0], _p(X),
                                                     X.shape[0], n_perturb, C.c_double(sigma), C.c_uint64(seed),
                                                     _p(out)),
                 "harvest_snapshots")
        blocks, o = [], 0
        for m in rows:
            blocks.append(out[o:o + m * n].reshape(m, n))
            o += m * n
        return blocks

    def build_fast(self, model: LrnrParams, s, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=10) -> FastParams:
        """harvest_snapshots + eim_greedy on the device, build_fastparams on the host (reduction.cpp:111-283)."""
        S = _f64(s).reshape(-1, model.r_total)
        red, idx, F, exh = _fast_buffers(model, r_hat)
        self._rc(self.lib.lrnr_gpu_build_fast(self.h, model.depth, _p(model.widths), _p(model.ranks),
                                              _p(_f64(model.params)), model.act, _p(S), S.shape[0], nx, nt, n_perturb,
                                              C.c_double(sigma), C.c_uint64(seed), r_hat, _p(red), _p(idx), _p(F),
                                              exh.ctypes.data_as(C.c_void_p)), "build_fast")
        return _fast_result(model, r_hat, red, idx, F, exh)

    def l1_error(self, model, s, ref_values, n_x, n_t):
        """l1_relative_error (pde.cpp:166-178) of the model against a GridField ((n_t+1) x n_x)."""
        v = C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_l1_error(self.h, model, _p(_f64(s)), _p(_f64(ref_values).reshape(-1)), n_x, n_t,
                                            C.byref(v)), "l1_error")
        return v.value

    def jets(self, model, s):
        out = np.zeros((self.n_points, 4))
        self._rc(self.lib.lrnr_gpu_jets(self.h, model, _p(_f64(s)), _p(out)), "jets")
        return out

    def loss(self, model, s, mu, w=0.0):
        v = C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_loss(self.h, model, _p(_f64(s)), _p(_f64(mu)), C.c_double(w), C.byref(v)),
                 "loss")
        return v.value

    # --- plain losses / values, forward only (training.cpp:76-189, model.cpp:260-292) ---
    def values(self, model, s, xt):
        """u only (lrnr_forward / fast_forward) at (n, 2) points, on the value-only kernel."""
        xt = _f64(xt).reshape(-1, 2)
        out = np.zeros(xt.shape[0])
        self._rc(self.lib.lrnr_gpu_values(self.h, model, _p(_f64(s)), _p(xt), xt.shape[0], _p(out)), "values")
        return out

    def loss_tune(self, model, s, mu):
        """loss_tune: LossBreakdown dict(total, residual, boundary) over the resident interior points and the
        boundary points of set_boundary."""
        o = np.zeros(3)
        self._rc(self.lib.lrnr_gpu_loss_tune(self.h, model, _p(_f64(s)), _p(_f64(mu)), _p(o)), "loss_tune")
        return dict(total=o[0], residual=o[1], boundary=o[2])

    def loss_fast(self, model, s, mu, X):
        """loss_fast: l1 sums over the classified sampling set X ((n, 2) points)."""
        X = _f64(X).reshape(-1, 2)
        o = np.zeros(3)
        self._rc(self.lib.lrnr_gpu_loss_fast(self.h, model, _p(_f64(s)), _p(_f64(mu)), _p(X), X.shape[0], _p(o)),
                 "loss_fast")
        return dict(total=o[0], residual=o[1], boundary=o[2])

    def loss_meta(self, mus):
        """loss_meta: per-instance mu through the hypernetwork; resident points + meta boundary points."""
        o = np.zeros(3)
        self._rc(self.lib.lrnr_gpu_loss_meta(self.h, _p(_f64(mus)), _p(o)), "loss_meta")
        return dict(total=o[0], residual=o[1], boundary=o[2])

    # --- NCCL communicator (multi-GPU, one process per GPU) ---
    @staticmethod
    def _map_nccl():
        """The library dlopens libnccl.so.2 by soname: map torch's NCCL first so both share one."""
        try:
            import torch  # noqa: F401  (libtorch_cuda links the NCCL torch.distributed uses)
        except ImportError:
            pass

    @staticmethod
    def comm_unique_id() -> bytes:
        GpuContext._map_nccl()
        buf = C.create_string_buffer(128)
        rc = _lib.load().lrnr_gpu_comm_unique_id(C.cast(buf, C.c_void_p), 128)
        if rc != 0:
            raise LrnrGpuError(f"lrnr_gpu_comm_unique_id failed with code {rc} (libnccl.so.2 not loadable?)")
        return buf.raw

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """ncclCommInitRank on this context's device; results are then summed over the ranks."""
        self._map_nccl()
        buf = C.create_string_buffer(bytes(uid), 128)
        self._rc(self.lib.lrnr_gpu_comm_init(self.h, nranks, rank, C.cast(buf, C.c_void_p), 128), "comm_init")

    def set_comm(self, nccl_comm_ptr: int | None):
        self._map_nccl()
        self._rc(self.lib.lrnr_gpu_set_comm(self.h, C.c_void_p(nccl_comm_ptr or 0)), "set_comm")

    def comm_info(self):
        n, r = C.c_int(0), C.c_int(0)
        self._rc(self.lib.lrnr_gpu_comm_info(self.h, C.byref(n), C.byref(r)), "comm_info")
        return n.value, r.value

    def allreduce(self, dev_ptr: int, n: int):
        self._rc(self.lib.lrnr_gpu_allreduce(self.h, C.c_void_p(dev_ptr), n), "allreduce")

    def set_option(self, opt: int, value: int):
        self._rc(self.lib.lrnr_gpu_set_option(self.h, opt, value), "set_option")

    def fma_peak_tflops(self, dtype=F32):
        v = C.c_double(0.0)
        self._rc(self.lib.lrnr_gpu_fma_peak(self.h, dtype, C.byref(v)), "fma_peak")
        return v.value

    # --- device-resident step ---
    def upload_coeffs(self, s, mu, n_inst=1):
        self._rc(self.lib.lrnr_gpu_upload_coeffs(self.h, _p(_f64(s)), _p(_f64(mu)), n_inst), "upload_coeffs")

    def run(self, model, w=0.0, dev_out: int | None = None):
        self._rc(self.lib.lrnr_gpu_run(self.h, model, C.c_double(w), C.c_void_p(dev_out or 0)), "run")

    def check(self):
        self._rc(self.lib.lrnr_gpu_check(self.h), "check")

    def download(self, n):
        out = np.zeros(n)
        self._rc(self.lib.lrnr_gpu_download(self.h, _p(out), n), "download")
        return out


# ---------------------------------------------------------------------------
# BASELINE.json configurations (seeded synthetic inputs)
# ---------------------------------------------------------------------------
C0_WIDTHS, C0_RANKS = [2, 100, 100, 100, 1], [2, 10, 10, 1]
C2_WIDTHS, C2_RANKS = [2] + [256] * 6 + [1], [2, 32, 32, 32, 32, 32, 1]
C4_WIDTHS, C4_RANKS = [2] + [512] * 8 + [1], [2] + [64] * 7 + [1]
C3_LO, C3_HI = (1.0, 0.0, 0.0), (40.0, 0.1, 10.0)


def config0(n_points=4096):
    """c0: LRNR 2-100x3-1, r (2,10,10,1), FP64, tanh, mu=(30,0,0), 4096 pts."""
    m, s = make_baseline_model(C0_WIDTHS, C0_RANKS, 2410, ACT_TANH)
    pts = sample_collocation(4001, n_points)
    return dict(model=m, s=s, pts=pts, mu=np.array([30.0, 0.0, 0.0]), dtype=F64)


def config1(n_points=4096):
    """c1: FastLRNR of c0 with rhat=10 from the reference EIM recipe."""
    c = config0(n_points)
    c["fast"] = build_fast(c["model"], c["s"], nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=10)
    return c


# The FastLRNR of the c2 / c3 base network: snapshots harvested over a mu grid (the 8 corners of the
# c3 parameter box) through the c3 hypernetwork, as harvest_snapshots does with a mu_grid
# (reduction.cpp:111-148; the cli's build_reduction).  At one fixed s the reference recipe exhausts
# its 108 snapshot columns at the 1e-12 residual floor before the budget (r_hat 16-29 on c2); over
# the grid's 8 x 108 columns the greedy EIM reaches the budget of 32.
C2_FAST_MU_GRID = np.array([(a, b, c) for a in (C3_LO[0], C3_HI[0]) for b in (C3_LO[1], C3_HI[1])
                            for c in (C3_LO[2], C3_HI[2])])


def c3_hyper():
    """c3 hypernetwork 3-64-64-163 (tanh, Xavier-uniform hidden layers) on the c2 base network."""
    return make_hyper_params(C2_RANKS, 2, 64, 4003, C3_LO, C3_HI, 0.01, 0.5)


def config2(n_points=1 << 20, act=ACT_SIN, with_fast=True):
    """c2: LRNR 2-256x6-1, r (2,32x5,1), FP32, sin, mu=(20,0.01,5); FastLRNR r_hat 32 (mu-grid snapshots)."""
    m, s = make_baseline_model(C2_WIDTHS, C2_RANKS, 2411, act)
    pts = sample_collocation(4002, n_points)
    out = dict(model=m, s=s, pts=pts, mu=np.array([20.0, 0.01, 5.0]), dtype=F32)
    if with_fast:
        S = hyper_forward(c3_hyper(), C2_FAST_MU_GRID)
        out["fast"] = build_fast(m, S, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=32)
    return out


def config3(n_inst=1024, pts_per_inst=16384, act=ACT_SIN):
    """c3: 1024 mu ~ U[1,40]xU[0,0.1]xU[0,10]; hypernet 3-64-64-163 on the c2 base; FastLRNR."""
    c = config2(n_points=0, act=act, with_fast=True)
    hyper = c3_hyper()
    _, mus = sample_collocation(4004, n_inst, C3_LO, C3_HI, with_mu=True)
    pts = np.concatenate([sample_collocation(5000 + i, pts_per_inst) for i in range(n_inst)]) if pts_per_inst else \
        np.zeros((0, 2))
    c.update(hyper=hyper, mus=mus, pts=pts, n_inst=n_inst)
    return c


def config4(n_inst=64, pts_per_inst=1 << 20, act=ACT_SIN):
    """c4: meta step, 2-512x8-1, r (2,64x7,1), hypernet 3-64-64-451, 64 mu x 1M pts."""
    m, _ = make_baseline_model(C4_WIDTHS, C4_RANKS, 2412, act)
    hyper = make_hyper_params(C4_RANKS, 2, 64, 4005, C3_LO, C3_HI, 0.01, 0.5)
    _, mus = sample_collocation(4006, n_inst, C3_LO, C3_HI, with_mu=True)
    pts = np.concatenate([sample_collocation(6000 + i, pts_per_inst) for i in range(n_inst)]) if pts_per_inst else \
        np.zeros((0, 2))
    return dict(model=m, hyper=hyper, mus=mus, pts=pts, n_inst=n_inst, dtype=F32)


def algorithmic_flops_per_point(widths: Sequence[int], ranks: Sequence[int], meta: bool = False) -> int:
    """LRNR coefficient-only 8*S FMA, meta 12*S; FLOP = 2*FMA."""
    S = sum(int(ranks[l]) * (int(widths[l]) + int(widths[l + 1])) for l in range(len(ranks)))
    return 2 * (12 if meta else 8) * S


def fast_flops_per_point(ranks: Sequence[int], red: Sequence[int], m_in=2, m_out=1) -> int:
    """SURVEY Appendix B FastLRNR: fwd 4*(M0 r1 + sum rhat(r_l + r_{l+1}) + r_L M_L) FMA, bwd = fwd."""
    L = len(ranks)
    fwd = m_in * int(ranks[0]) + sum(int(red[l]) * (int(ranks[l]) + int(ranks[l + 1])) for l in range(L - 1)) + \
        int(ranks[-1]) * m_out
    return 2 * 2 * 4 * fwd


# ---------------------------------------------------------------------------
# checkpoint interop (lrnr_ckpt_*, proj/src/checkpoint.cpp format)
# ---------------------------------------------------------------------------
class Checkpoint:
    """The reference's LRNR v1 checkpoint, read / written by the package's host C++."""

    def __init__(self, path: str | None = None):
        self.lib = _lib.load()
        self.h = C.c_void_p()
        if path is None:
            rc = self.lib.lrnr_ckpt_create(C.byref(self.h))
        else:
            rc = self.lib.lrnr_ckpt_load(str(path).encode(), C.byref(self.h))
        self._rc(rc)

    def _rc(self, rc):
        if rc != 0:
            msg = self.lib.lrnr_ckpt_last_error().decode()
            raise (ValueError if rc == 1 else LrnrGpuError)(f"checkpoint: {msg}")

    def close(self):
        if self.h:
            self.lib.lrnr_ckpt_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def save(self, path):
        self._rc(self.lib.lrnr_ckpt_save(self.h, str(path).encode()))

    def lrnr(self, act=ACT_TANH) -> LrnrParams:
        L, n = C.c_int(0), C.c_int64(0)
        self._rc(self.lib.lrnr_ckpt_get_lrnr(self.h, C.byref(L), None, None, C.byref(n), None))
        w, r, P = np.zeros(L.value + 1, np.int64), np.zeros(L.value, np.int64), np.zeros(n.value)
        self._rc(self.lib.lrnr_ckpt_get_lrnr(self.h, C.byref(L), _p(w), _p(r), C.byref(n), _p(P)))
        return LrnrParams(w, r, P, act)

    def put_lrnr(self, m: LrnrParams):
        w, r = _i64(m.widths), _i64(m.ranks)
        self._rc(self.lib.lrnr_ckpt_put_lrnr(self.h, len(r), _p(w), _p(r), _p(_f64(m.params))))

    def hyper(self) -> HyperParams:
        K, n = C.c_int(0), C.c_int64(0)
        self._rc(self.lib.lrnr_ckpt_get_hyper(self.h, C.byref(K), None, C.byref(n), None, None, None))
        hw, H, lo, hi = np.zeros(K.value + 1, np.int64), np.zeros(n.value), np.zeros(3), np.zeros(3)
        self._rc(self.lib.lrnr_ckpt_get_hyper(self.h, C.byref(K), _p(hw), C.byref(n), _p(H), _p(lo), _p(hi)))
        return HyperParams(hw, H, lo, hi)

    def put_hyper(self, h: HyperParams, split):
        hw, sp = _i64(h.hw), _i64(split)
        self._rc(self.lib.lrnr_ckpt_put_hyper(self.h, len(hw) - 1, _p(hw), _p(_f64(h.params)), len(sp), _p(sp),
                                              _p(_f64(h.lo)), _p(_f64(h.hi))))

    def has_fast(self) -> bool:
        return bool(self.lib.lrnr_ckpt_has_fast(self.h))

    def fast(self, act=ACT_TANH) -> FastParams:
        L, n = C.c_int(0), C.c_int64(0)
        self._rc(self.lib.lrnr_ckpt_get_fast(self.h, C.byref(L), None, None, C.byref(n), None))
        r, rh, F = np.zeros(L.value, np.int64), np.zeros(L.value - 1, np.int64), np.zeros(n.value)
        self._rc(self.lib.lrnr_ckpt_get_fast(self.h, C.byref(L), _p(r), _p(rh), C.byref(n), _p(F)))
        return FastParams(r, rh, F, act)

    def put_fast(self, f: FastParams):
        r, rh = _i64(f.ranks), _i64(f.red_ranks)
        self._rc(self.lib.lrnr_ckpt_put_fast(self.h, len(r), _p(r), _p(rh), 2, 1, _p(_f64(f.fparams))))

    def sampling(self):
        n = C.c_int64(0)
        self._rc(self.lib.lrnr_ckpt_get_sampling(self.h, C.byref(n), None))
        X = np.zeros((n.value, 2))
        self._rc(self.lib.lrnr_ckpt_get_sampling(self.h, C.byref(n), _p(X)))
        return X

    def put_sampling(self, X):
        X = _f64(X).reshape(-1, 2)
        self._rc(self.lib.lrnr_ckpt_put_sampling(self.h, X.shape[0], _p(X)))
