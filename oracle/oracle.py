"""TEST INFRASTRUCTURE ONLY -- ctypes front-end to the two CPU checkers.

* ``Oracle``    -> oracle/liblrnr_oracle.so : the plain-C FP64 restatement of the
  reference hot path (oracle/lrnr_oracle.c), tanh + the sin extension.
* ``Reference`` -> oracle/_ref/liblrnr_ref.so : the UNMODIFIED reference
  (/root/reference/proj/src, compiled in place) driven through its public API by
  oracle/ref_harness.cpp.  Present only where the reference compiled (built in
  the build container; the built .so travels to the GPU box with gpurun).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  The product package
(paper_2410_04001_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblrnr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblrnr_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _ensure_built():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    pass


def lrnr_param_count(widths, ranks):
    return int(sum(widths[l + 1] * ranks[l] + widths[l] * ranks[l] + widths[l + 1]
                   for l in range(len(ranks))))


def hyper_param_count(hw):
    return int(sum(hw[k + 1] * hw[k] + hw[k + 1] for k in range(len(hw) - 1)))


def fast_param_count(ranks, red, m_in=2, m_out=1):
    L = len(ranks)
    n = m_in * ranks[0]
    for l in range(L - 1):
        n += red[l] * ranks[l] + red[l] + red[l] * ranks[l + 1]
    return int(n + m_out * ranks[-1] + m_out)


class Oracle:
    """The C restatement (always available: gcc builds it anywhere)."""

    def __init__(self, path: str = ORACLE_SO):
        _ensure_built()
        self.lib = C.CDLL(path)
        self.lib.orc_lrnr_grad.restype = C.c_int
        self.lib.orc_fast_grad.restype = C.c_int

    # --- construction ---
    def rng_stream(self, seed, n, kind):
        out = np.zeros(n, np.float64)
        raw = np.zeros(n, np.uint64)
        self.lib.orc_rng_stream(C.c_uint64(seed), C.c_int64(n), C.c_int(kind), _ptr(out), _ptr(raw))
        return raw if kind == 2 else out

    def make_baseline_model(self, widths, ranks, seed):
        w, r = _i64(widths), _i64(ranks)
        P = np.zeros(lrnr_param_count(w, r))
        s = np.zeros(int(r.sum()))
        self.lib.orc_make_baseline_model(C.c_int(len(r)), _ptr(w), _ptr(r), C.c_uint64(seed), _ptr(P), _ptr(s))
        return P, s

    def make_lrnr_params(self, widths, ranks, seed, orthonormal=True, bias_scale=0.5):
        w, r = _i64(widths), _i64(ranks)
        P = np.zeros(lrnr_param_count(w, r))
        self.lib.orc_make_lrnr_params(C.c_int(len(r)), _ptr(w), _ptr(r), C.c_uint64(seed),
                                      C.c_int(int(orthonormal)), C.c_double(bias_scale), _ptr(P))
        return P

    def make_hyper_params(self, split, depth, width, seed, out_w_scale=0.01, out_bias=0.5):
        sp = _i64(split)
        hw = [3] + [width] * depth + [int(sp.sum())]
        P = np.zeros(hyper_param_count(hw))
        self.lib.orc_make_hyper_params(C.c_int(len(sp)), _ptr(sp), C.c_int(depth), C.c_int(width),
                                       C.c_uint64(seed), C.c_double(out_w_scale), C.c_double(out_bias), _ptr(P))
        return np.array(hw, np.int64), P

    def sample_collocation(self, seed, n_int, n_ic=0, n_per=0, lo=(0, 0, 0), hi=(0, 0, 0), with_mu=False):
        pi = np.zeros(2 * n_int + 1)
        pic = np.zeros(n_ic + 1)
        pper = np.zeros(n_per + 1)
        mi, mic, mp = np.zeros(3 * n_int + 1), np.zeros(3 * n_ic + 1), np.zeros(3 * n_per + 1)
        self.lib.orc_sample_collocation(C.c_uint64(seed), C.c_int64(n_int), C.c_int64(n_ic), C.c_int64(n_per),
                                        _ptr(_f64(lo)), _ptr(_f64(hi)), C.c_int(int(with_mu)),
                                        _ptr(pi), _ptr(pic), _ptr(pper), _ptr(mi), _ptr(mic), _ptr(mp))
        out = dict(interior=pi[:2 * n_int].reshape(n_int, 2), initial_x=pic[:n_ic], periodic_t=pper[:n_per])
        if with_mu:
            out.update(interior_mu=mi[:3 * n_int].reshape(n_int, 3), initial_mu=mic[:3 * n_ic].reshape(n_ic, 3),
                       periodic_mu=mp[:3 * n_per].reshape(n_per, 3))
        return out

    # --- hot path ---
    def lrnr_grad(self, widths, ranks, P, s, mu, pts, w=None, act=0, chunk=64, params_grad=False,
                  terms=False):
        wv, rv = _i64(widths), _i64(ranks)
        pts = _f64(pts).reshape(-1, 2)
        n = pts.shape[0]
        w = (1.0 / n if n else 0.0) if w is None else w
        gs = np.zeros(int(rv.sum()))
        gp = np.zeros(lrnr_param_count(wv, rv)) if params_grad else None
        tv = np.zeros(max(n, 1)) if terms else None
        val = C.c_double(0.0)
        rc = self.lib.orc_lrnr_grad(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), C.c_int(act),
                                    _ptr(_f64(s)), _ptr(_f64(mu)), _ptr(pts), C.c_int64(n), C.c_double(w),
                                    C.c_int64(chunk), C.byref(val), _ptr(gs), _ptr(gp), _ptr(tv))
        if rc == 1:
            raise OracleError("orc_lrnr_grad: invalid arguments")
        out = dict(value=val.value, grad_s=gs, nonfinite=(rc == 2))
        if params_grad:
            out["grad_params"] = gp
        if terms:
            out["terms"] = tv[:n]
        return out

    def lrnr_jets(self, widths, ranks, P, s, pts, act=0):
        wv, rv = _i64(widths), _i64(ranks)
        pts = _f64(pts).reshape(-1, 2)
        out = np.zeros((pts.shape[0], 4))
        self.lib.orc_lrnr_jets(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), C.c_int(act),
                               _ptr(_f64(s)), _ptr(pts), C.c_int64(pts.shape[0]), _ptr(out))
        return out

    def fast_grad(self, ranks, red, F, s, mu, pts, w=None, act=0, chunk=64, terms=False):
        rv, hv = _i64(ranks), _i64(red)
        pts = _f64(pts).reshape(-1, 2)
        n = pts.shape[0]
        w = (1.0 / n if n else 0.0) if w is None else w
        gs = np.zeros(int(rv.sum()))
        tv = np.zeros(max(n, 1)) if terms else None
        val = C.c_double(0.0)
        rc = self.lib.orc_fast_grad(C.c_int(len(rv)), _ptr(rv), _ptr(hv), C.c_int64(2), C.c_int64(1),
                                    _ptr(_f64(F)), C.c_int(act), _ptr(_f64(s)), _ptr(_f64(mu)), _ptr(pts),
                                    C.c_int64(n), C.c_double(w), C.c_int64(chunk), C.byref(val), _ptr(gs),
                                    _ptr(tv))
        if rc == 1:
            raise OracleError("orc_fast_grad: invalid arguments")
        out = dict(value=val.value, grad_s=gs, nonfinite=(rc == 2))
        if terms:
            out["terms"] = tv[:n]
        return out

    def terms_grad(self, model, dims, P, s, mu, pts=(), ic_x=(), per_t=(), w_int=None, w_ic=None, w_bc=None,
                   objective=0, s_init=None, lambda_local=0.0, act=0, chunk=64, params_grad=False):
        """Full solve-step term set (orc_terms_grad): model 0 = LRNR with dims = (widths, ranks),
        1 = FastLRNR with dims = (ranks, red_ranks); weights default to 1/n of each kind
        (training.cpp:364-366); objective 0 = squared, 1 = abs."""
        pts = _f64(pts).reshape(-1, 2)
        icx, pt = _f64(ic_x).reshape(-1), _f64(per_t).reshape(-1)
        inv = lambda n: 1.0 / n if n else 0.0  # noqa: E731
        w_int = inv(pts.shape[0]) if w_int is None else w_int
        w_ic = inv(icx.shape[0]) if w_ic is None else w_ic
        w_bc = inv(pt.shape[0]) if w_bc is None else w_bc
        if model == 0:
            wv, rv = _i64(dims[0]), _i64(dims[1])
            L, rh = len(rv), None
        else:
            rv, hv = _i64(dims[0]), _i64(dims[1])
            wv, L, rh = _i64([2, 1]), len(rv), hv
        gs = np.zeros(int(rv.sum()))
        comps = np.zeros(4)
        val = C.c_double(0.0)
        si = None if s_init is None else _f64(s_init)
        gp = np.zeros(lrnr_param_count(dims[0], dims[1])) if params_grad else None
        rc = self.lib.orc_terms_grad(C.c_int(model), C.c_int(L), _ptr(wv), _ptr(rv), _ptr(rh), _ptr(_f64(P)),
                                     C.c_int(act), _ptr(_f64(s)), _ptr(_f64(mu)), _ptr(pts), C.c_int64(pts.shape[0]),
                                     _ptr(icx), C.c_int64(icx.shape[0]), _ptr(pt), C.c_int64(pt.shape[0]),
                                     C.c_double(w_int), C.c_double(w_ic), C.c_double(w_bc), C.c_int(objective),
                                     _ptr(si), C.c_double(lambda_local), C.c_int64(chunk), C.byref(val),
                                     _ptr(comps), _ptr(gs), _ptr(gp))
        if rc == 1:
            raise OracleError("orc_terms_grad: invalid arguments")
        out = dict(value=val.value, comps=comps, grad_s=gs, nonfinite=(rc == 2))
        if params_grad:
            out["grad_params"] = gp
        return out

    def meta_regs(self, widths, ranks, P, s_inst, n_per, w, lambda_sparse, gamma, lambda_ortho):
        """meta_train's regularizers for points grouped by instance (s_inst: n_inst x r_total):
        sparse = sum_i n_per * lambda * w * sum_l banded(s_l(mu_i)) with its dL/ds_i rows, and
        ortho = lambda_o * sum_l (gram(U_l) + gram(V_l)) with its dL/dparams (ParamPacker order)."""
        self.lib.orc_banded_decay.restype = C.c_double
        self.lib.orc_gram_penalty.restype = C.c_double
        wv, rv = _i64(widths), _i64(ranks)
        s_inst = np.atleast_2d(_f64(s_inst))
        ds = np.zeros_like(s_inst)
        coef = lambda_sparse * w * n_per
        sparse = 0.0
        offs = np.concatenate([[0], np.cumsum(rv)])
        for i in range(s_inst.shape[0]):
            acc = 0.0
            for l in range(len(rv)):
                f = np.ascontiguousarray(s_inst[i, offs[l]:offs[l + 1]])
                g = np.zeros_like(f)
                acc += self.lib.orc_banded_decay(_ptr(f), C.c_int64(f.size), C.c_double(gamma), C.c_double(coef),
                                                 _ptr(g))
                ds[i, offs[l]:offs[l + 1]] += g
            sparse += coef * acc
        P = _f64(P)
        gP = np.zeros_like(P)
        ortho, o = 0.0, 0
        for l in range(len(rv)):
            for rows in (wv[l + 1], wv[l]):
                A = np.ascontiguousarray(P[o:o + rows * rv[l]])
                g = np.zeros_like(A)
                ortho += lambda_ortho * self.lib.orc_gram_penalty(_ptr(A), C.c_int64(rows), C.c_int64(rv[l]),
                                                                  C.c_double(lambda_ortho), _ptr(g))
                gP[o:o + rows * rv[l]] += g
                o += rows * rv[l]
            o += wv[l + 1]
        return dict(sparse=sparse, ds=ds, ortho=ortho, grad_params=gP)

    def fine_tune(self, widths, ranks, P, s_init, mu, lr, epochs, n_int, n_ic, n_bc, seed, act=0, chunk=64):
        """fine_tune (training.cpp:428-496) from s_init = hyper_forward(mu)."""
        wv, rv = _i64(widths), _i64(ranks)
        return self._solve(self.lib.orc_fine_tune, int(rv.sum()), epochs, C.c_int(len(rv)), _ptr(wv), _ptr(rv),
                           _ptr(_f64(P)), C.c_int(act), _ptr(_f64(s_init)), _ptr(_f64(mu)), C.c_double(lr),
                           C.c_int64(epochs), C.c_int64(n_int), C.c_int64(n_ic), C.c_int64(n_bc), C.c_uint64(seed),
                           C.c_int64(chunk))

    def fast_solve(self, ranks, red, F, s_init, mu, X, lambda_local, lr, epochs, act=0, chunk=64):
        """fast_solve (training.cpp:498-607) on the sampling set X."""
        rv, hv = _i64(ranks), _i64(red)
        X = _f64(X).reshape(-1, 2)
        return self._solve(self.lib.orc_fast_solve, int(rv.sum()), epochs, C.c_int(len(rv)), _ptr(rv), _ptr(hv),
                           _ptr(_f64(F)), C.c_int(act), _ptr(_f64(s_init)), _ptr(_f64(mu)), _ptr(X),
                           C.c_int64(X.shape[0]), C.c_double(lambda_local), C.c_double(lr), C.c_int64(epochs),
                           C.c_int64(chunk))

    def _solve(self, fn, G, epochs, *args):
        s = np.zeros(G)
        losses = np.zeros(max(1, epochs))
        bl, be, nr, fl = C.c_double(0.0), C.c_int64(0), C.c_int64(0), C.c_int(0)
        rc = fn(*args, _ptr(s), C.byref(bl), C.byref(be), _ptr(losses), C.byref(nr), C.byref(fl))
        if rc:
            raise OracleError("solve loop: invalid arguments")
        return dict(s=s, best_loss=bl.value, best_epoch=be.value, losses=losses[:nr.value], aborted=bool(fl.value & 1),
                    diverged=bool(fl.value & 2))

    def fast_jets(self, ranks, red, F, s, pts, act=0):
        rv, hv = _i64(ranks), _i64(red)
        pts = _f64(pts).reshape(-1, 2)
        out = np.zeros((pts.shape[0], 4))
        self.lib.orc_fast_jets(C.c_int(len(rv)), _ptr(rv), _ptr(hv), C.c_int64(2), C.c_int64(1), _ptr(_f64(F)),
                               C.c_int(act), _ptr(_f64(s)), _ptr(pts), C.c_int64(pts.shape[0]), _ptr(out))
        return out

    def hyper_forward(self, hw, H, lo, hi, mu):
        hwv = _i64(hw)
        out = np.zeros(int(hwv[-1]))
        self.lib.orc_hyper_forward(C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)), _ptr(_f64(lo)), _ptr(_f64(hi)),
                                   _ptr(_f64(mu)), _ptr(out))
        return out

    def hyper_vjp(self, hw, H, lo, hi, mu, g_s, out=None):
        hwv = _i64(hw)
        out = np.zeros(hyper_param_count(hwv)) if out is None else out
        self.lib.orc_hyper_vjp(C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)), _ptr(_f64(lo)), _ptr(_f64(hi)),
                               _ptr(_f64(mu)), _ptr(_f64(g_s)), _ptr(out))
        return out

    def meta_train(self, widths, ranks, hyper_depth, hyper_width, init_bias_scale, out_w_scale, out_bias,
                   init_seed, lo, hi, lr, epochs, n_int, n_ic, n_per, seed, lambda_ortho, lambda_sparse, gamma,
                   chunk=64):
        wv, rv = _i64(widths), _i64(ranks)
        best = C.c_double(0.0)
        be = C.c_int64(0)
        losses = np.zeros(epochs)
        self.lib.orc_meta_train(C.c_int(len(rv)), _ptr(wv), _ptr(rv), C.c_int(hyper_depth), C.c_int(hyper_width),
                                C.c_double(init_bias_scale), C.c_double(out_w_scale), C.c_double(out_bias),
                                C.c_uint64(init_seed), _ptr(_f64(lo)), _ptr(_f64(hi)), C.c_double(lr),
                                C.c_int64(epochs), C.c_int64(n_int), C.c_int64(n_ic), C.c_int64(n_per),
                                C.c_uint64(seed), C.c_double(lambda_ortho), C.c_double(lambda_sparse),
                                C.c_double(gamma), C.c_int64(chunk), C.byref(best), C.byref(be), _ptr(losses))
        return best.value, be.value, losses


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference through oracle/ref_harness.cpp (tanh only)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise OracleError("reference library not built: " + path)
        self.lib = C.CDLL(path)

    def _rc(self, rc, what):
        if rc == 2:
            raise FloatingPointError(f"{what}: NonFiniteError layer tag {self.lib.ref_last_tag()}")
        if rc != 0:
            raise OracleError(f"{what}: reference error code {rc}")

    def rng_stream(self, seed, n, kind):
        out = np.zeros(n, np.float64)
        raw = np.zeros(n, np.uint64)
        self._rc(self.lib.ref_rng_stream(C.c_uint64(seed), C.c_int64(n), C.c_int(kind), _ptr(out), _ptr(raw)),
                 "rng")
        return raw if kind == 2 else out

    def make_baseline_model(self, widths, ranks, seed):
        w, r = _i64(widths), _i64(ranks)
        P = np.zeros(lrnr_param_count(w, r))
        s = np.zeros(int(r.sum()))
        self._rc(self.lib.ref_make_baseline_model(C.c_int(len(r)), _ptr(w), _ptr(r), C.c_uint64(seed), _ptr(P),
                                                  _ptr(s)), "make_baseline_model")
        return P, s

    def make_lrnr_params(self, widths, ranks, seed, orthonormal=True, bias_scale=0.5):
        w, r = _i64(widths), _i64(ranks)
        P = np.zeros(lrnr_param_count(w, r))
        self._rc(self.lib.ref_make_lrnr_params(C.c_int(len(r)), _ptr(w), _ptr(r), C.c_uint64(seed),
                                               C.c_int(int(orthonormal)), C.c_double(bias_scale), _ptr(P)),
                 "make_lrnr_params")
        return P

    def make_hyper_params(self, split, depth, width, lo, hi, seed, out_w_scale=0.01, out_bias=0.5):
        sp = _i64(split)
        hw = [3] + [width] * depth + [int(sp.sum())]
        P = np.zeros(hyper_param_count(hw))
        self._rc(self.lib.ref_make_hyper_params(C.c_int(len(sp)), _ptr(sp), C.c_int(depth), C.c_int(width),
                                                _ptr(_f64(lo)), _ptr(_f64(hi)), C.c_uint64(seed),
                                                C.c_double(out_w_scale), C.c_double(out_bias), _ptr(P)),
                 "make_hyper_params")
        return np.array(hw, np.int64), P

    def sample_collocation(self, seed, n_int, n_ic=0, n_per=0, lo=(0, 0, 0), hi=(0, 0, 0), with_mu=False):
        pi = np.zeros(2 * n_int + 1)
        pic = np.zeros(n_ic + 1)
        pper = np.zeros(n_per + 1)
        mi, mic, mp = np.zeros(3 * n_int + 1), np.zeros(3 * n_ic + 1), np.zeros(3 * n_per + 1)
        self._rc(self.lib.ref_sample_collocation(C.c_uint64(seed), C.c_int64(n_int), C.c_int64(n_ic),
                                                 C.c_int64(n_per), _ptr(_f64(lo)), _ptr(_f64(hi)),
                                                 C.c_int(int(with_mu)), _ptr(pi), _ptr(pic), _ptr(pper), _ptr(mi),
                                                 _ptr(mic), _ptr(mp)), "sample_collocation")
        out = dict(interior=pi[:2 * n_int].reshape(n_int, 2), initial_x=pic[:n_ic], periodic_t=pper[:n_per])
        if with_mu:
            out.update(interior_mu=mi[:3 * n_int].reshape(n_int, 3), initial_mu=mic[:3 * n_ic].reshape(n_ic, 3),
                       periodic_mu=mp[:3 * n_per].reshape(n_per, 3))
        return out

    def lrnr_grad(self, widths, ranks, P, s, mu, pts, w=None, threads=1, chunk=64):
        wv, rv = _i64(widths), _i64(ranks)
        pts = _f64(pts).reshape(-1, 2)
        n = pts.shape[0]
        w = (1.0 / n if n else 0.0) if w is None else w
        gs = np.zeros(int(rv.sum()))
        comps = np.zeros(4)
        val = C.c_double(0.0)
        self._rc(self.lib.ref_lrnr_grad(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), _ptr(_f64(s)),
                                        _ptr(_f64(mu)), _ptr(pts), C.c_int64(n), C.c_double(w), C.c_int(threads),
                                        C.c_int(chunk), C.byref(val), _ptr(comps), _ptr(gs)), "lrnr_grad")
        return dict(value=val.value, comps=comps, grad_s=gs)

    def fast_grad(self, ranks, red, F, s, mu, pts, w=None, threads=1, chunk=64):
        rv, hv = _i64(ranks), _i64(red)
        pts = _f64(pts).reshape(-1, 2)
        n = pts.shape[0]
        w = (1.0 / n if n else 0.0) if w is None else w
        gs = np.zeros(int(rv.sum()))
        comps = np.zeros(4)
        val = C.c_double(0.0)
        self._rc(self.lib.ref_fast_grad(C.c_int(len(rv)), _ptr(rv), _ptr(hv), C.c_int64(2), C.c_int64(1),
                                        _ptr(_f64(F)), _ptr(_f64(s)), _ptr(_f64(mu)), _ptr(pts), C.c_int64(n),
                                        C.c_double(w), C.c_int(threads), C.c_int(chunk), C.byref(val), _ptr(comps),
                                        _ptr(gs)), "fast_grad")
        return dict(value=val.value, comps=comps, grad_s=gs)

    def fast_phase_grad(self, ranks, red, F, s, s_init, mu, xpts, lambda_local, threads=1, chunk=64):
        rv, hv = _i64(ranks), _i64(red)
        xpts = _f64(xpts).reshape(-1, 2)
        gs = np.zeros(int(rv.sum()))
        comps = np.zeros(4)
        val = C.c_double(0.0)
        self._rc(self.lib.ref_fast_phase_grad(C.c_int(len(rv)), _ptr(rv), _ptr(hv), C.c_int64(2), C.c_int64(1),
                                              _ptr(_f64(F)), _ptr(_f64(s)), _ptr(_f64(s_init)), _ptr(_f64(mu)),
                                              _ptr(xpts), C.c_int64(xpts.shape[0]), C.c_double(lambda_local),
                                              C.c_int(threads), C.c_int(chunk), C.byref(val), _ptr(comps), _ptr(gs)),
                 "fast_phase_grad")
        return dict(value=val.value, comps=comps, grad_s=gs)

    def tune_grad_full(self, widths, ranks, P, s, mu, pts, ic_x=(), per_t=(), w_int=None, w_ic=None, w_bc=None,
                       threads=1, chunk=64):
        """Fine-tune PinnTermEmitter terms: interior + initial + periodic (training.cpp:286-327)."""
        wv, rv = _i64(widths), _i64(ranks)
        pts = _f64(pts).reshape(-1, 2)
        icx, pt = _f64(ic_x).reshape(-1), _f64(per_t).reshape(-1)
        inv = lambda n: 1.0 / n if n else 0.0  # noqa: E731
        w_int = inv(pts.shape[0]) if w_int is None else w_int
        w_ic = inv(icx.shape[0]) if w_ic is None else w_ic
        w_bc = inv(pt.shape[0]) if w_bc is None else w_bc
        gs = np.zeros(int(rv.sum()))
        comps = np.zeros(4)
        val = C.c_double(0.0)
        self._rc(self.lib.ref_tune_grad_full(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), _ptr(_f64(s)),
                                             _ptr(_f64(mu)), _ptr(pts), C.c_int64(pts.shape[0]), _ptr(icx),
                                             C.c_int64(icx.shape[0]), _ptr(pt), C.c_int64(pt.shape[0]),
                                             C.c_double(w_int), C.c_double(w_ic), C.c_double(w_bc), C.c_int(threads),
                                             C.c_int(chunk), C.byref(val), _ptr(comps), _ptr(gs)), "tune_grad_full")
        return dict(value=val.value, comps=comps, grad_s=gs)

    def fine_tune(self, widths, ranks, P, s_init, mu, lr, epochs, n_int, n_ic, n_bc, seed, threads=2):
        wv, rv = _i64(widths), _i64(ranks)
        return self._solve(self.lib.ref_fine_tune, int(rv.sum()), epochs, C.c_int(len(rv)), _ptr(wv), _ptr(rv),
                           _ptr(_f64(P)), _ptr(_f64(s_init)), _ptr(_f64(mu)), C.c_double(lr), C.c_int64(epochs),
                           C.c_int64(n_int), C.c_int64(n_ic), C.c_int64(n_bc), C.c_uint64(seed), C.c_int(threads))

    def fast_solve(self, ranks, red, F, s_init, mu, X, lambda_local, lr, epochs, threads=2):
        rv, hv = _i64(ranks), _i64(red)
        X = _f64(X).reshape(-1, 2)
        return self._solve(self.lib.ref_fast_solve, int(rv.sum()), epochs, C.c_int(len(rv)), _ptr(rv), _ptr(hv),
                           C.c_int64(2), C.c_int64(1), _ptr(_f64(F)), _ptr(_f64(s_init)), _ptr(_f64(mu)), _ptr(X),
                           C.c_int64(X.shape[0]), C.c_double(lambda_local), C.c_double(lr), C.c_int64(epochs),
                           C.c_int(threads))

    def _solve(self, fn, G, epochs, *args):
        s = np.zeros(G)
        losses = np.zeros(max(1, epochs))
        bl, be, nr, fl = C.c_double(0.0), C.c_int64(0), C.c_int64(0), C.c_int(0)
        self._rc(fn(*args, _ptr(s), C.byref(bl), C.byref(be), _ptr(losses), C.byref(nr), C.byref(fl)), "solve")
        return dict(s=s, best_loss=bl.value, best_epoch=be.value, losses=losses[:nr.value], aborted=bool(fl.value & 1),
                    diverged=bool(fl.value & 2))

    def l1_error(self, widths, ranks, P, s, values, n_x, n_t):
        wv, rv = _i64(widths), _i64(ranks)
        out = C.c_double(0.0)
        self._rc(self.lib.ref_l1_error(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), _ptr(_f64(s)),
                                       _ptr(_f64(values).reshape(-1)), C.c_int64(n_x), C.c_int64(n_t), C.byref(out)),
                 "l1_error")
        return out.value

    def lrnr_jets(self, widths, ranks, P, s, pts):
        wv, rv = _i64(widths), _i64(ranks)
        pts = _f64(pts).reshape(-1, 2)
        out = np.zeros((pts.shape[0], 4))
        self._rc(self.lib.ref_lrnr_jets(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), _ptr(_f64(s)),
                                        _ptr(pts), C.c_int64(pts.shape[0]), _ptr(out)), "lrnr_jets")
        return out

    def fast_jets(self, ranks, red, F, s, pts):
        rv, hv = _i64(ranks), _i64(red)
        pts = _f64(pts).reshape(-1, 2)
        out = np.zeros((pts.shape[0], 4))
        self._rc(self.lib.ref_fast_jets(C.c_int(len(rv)), _ptr(rv), _ptr(hv), C.c_int64(2), C.c_int64(1),
                                        _ptr(_f64(F)), _ptr(_f64(s)), _ptr(pts), C.c_int64(pts.shape[0]), _ptr(out)),
                 "fast_jets")
        return out

    def loss_tune(self, widths, ranks, P, s, mu, pts, ic_x=(), per_t=()):
        wv, rv = _i64(widths), _i64(ranks)
        pts = _f64(pts).reshape(-1, 2)
        icx, pt = _f64(list(ic_x) + [0.0]), _f64(list(per_t) + [0.0])
        out = np.zeros(3)
        self._rc(self.lib.ref_loss_tune(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), _ptr(_f64(s)),
                                        _ptr(_f64(mu)), _ptr(pts), C.c_int64(pts.shape[0]), _ptr(icx),
                                        C.c_int64(len(ic_x)), _ptr(pt), C.c_int64(len(per_t)), _ptr(out)),
                 "loss_tune")
        return out

    def values(self, model, widths, ranks, P, red, F, s, pts):
        """lrnr_forward (model 0) / fast_forward (model 1): u at the points."""
        wv, rv = _i64(widths if widths is not None else [0]), _i64(ranks)
        hv = _i64(red if red is not None else [0])
        pts = _f64(pts).reshape(-1, 2)
        out = np.zeros(pts.shape[0])
        self._rc(self.lib.ref_values(C.c_int(model), C.c_int(len(rv)), _ptr(wv), _ptr(rv),
                                     _ptr(_f64(P if P is not None else [0.0])), _ptr(hv),
                                     _ptr(_f64(F if F is not None else [0.0])), _ptr(_f64(s)), _ptr(pts),
                                     C.c_int64(pts.shape[0]), _ptr(out)), "values")
        return out

    def loss_fast(self, ranks, red, F, s, mu, X):
        rv, hv = _i64(ranks), _i64(red)
        X = _f64(X).reshape(-1, 2)
        out = np.zeros(3)
        self._rc(self.lib.ref_loss_fast(C.c_int(len(rv)), _ptr(rv), _ptr(hv), _ptr(_f64(F)), _ptr(_f64(s)),
                                        _ptr(_f64(mu)), _ptr(X), C.c_int64(X.shape[0]), _ptr(out)), "loss_fast")
        return out

    def loss_meta(self, widths, ranks, P, hw, H, lo, hi, pts, mus, ic_x=(), ic_mu=(), per_t=(), per_mu=()):
        wv, rv, hwv = _i64(widths), _i64(ranks), _i64(hw)
        pts = _f64(pts).reshape(-1, 2)
        mus = _f64(mus).reshape(-1)
        icx, icm = _f64(list(ic_x) + [0.0]), _f64(np.append(_f64(ic_mu).reshape(-1), 0.0))
        pt, pm = _f64(list(per_t) + [0.0]), _f64(np.append(_f64(per_mu).reshape(-1), 0.0))
        out = np.zeros(3)
        self._rc(self.lib.ref_loss_meta(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), C.c_int(len(hwv) - 1),
                                        _ptr(hwv), _ptr(_f64(H)), _ptr(_f64(lo)), _ptr(_f64(hi)), _ptr(pts),
                                        _ptr(mus), C.c_int64(pts.shape[0]), _ptr(icx), _ptr(icm),
                                        C.c_int64(len(ic_x)), _ptr(pt), _ptr(pm), C.c_int64(len(per_t)), _ptr(out)),
                 "loss_meta")
        return out

    def hyper_forward(self, hw, H, split, lo, hi, mu):
        hwv, sp = _i64(hw), _i64(split)
        out = np.zeros(int(hwv[-1]))
        self._rc(self.lib.ref_hyper_forward(C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)), C.c_int(len(sp)),
                                            _ptr(sp), _ptr(_f64(lo)), _ptr(_f64(hi)), _ptr(_f64(mu)), _ptr(out)),
                 "hyper_forward")
        return out

    def hyper_vjp(self, hw, H, split, lo, hi, mu, g_s):
        hwv, sp = _i64(hw), _i64(split)
        out = np.zeros(hyper_param_count(hwv))
        self._rc(self.lib.ref_hyper_vjp(C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)), C.c_int(len(sp)), _ptr(sp),
                                        _ptr(_f64(lo)), _ptr(_f64(hi)), _ptr(_f64(mu)), _ptr(_f64(g_s)), _ptr(out)),
                 "hyper_vjp")
        return out

    def meta_grad(self, widths, ranks, P, hw, H, lo, hi, pts, mus, w=None, threads=1, chunk=64):
        wv, rv, hwv = _i64(widths), _i64(ranks), _i64(hw)
        pts = _f64(pts).reshape(-1, 2)
        n = pts.shape[0]
        w = (1.0 / n if n else 0.0) if w is None else w
        out = np.zeros(lrnr_param_count(wv, rv) + hyper_param_count(hwv))
        val = C.c_double(0.0)
        self._rc(self.lib.ref_meta_grad(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), C.c_int(len(hwv) - 1),
                                        _ptr(hwv), _ptr(_f64(H)), _ptr(_f64(lo)), _ptr(_f64(hi)), _ptr(pts),
                                        _ptr(_f64(mus).reshape(-1)), C.c_int64(n), C.c_double(w), C.c_int(threads),
                                        C.c_int(chunk), C.byref(val), _ptr(out)), "meta_grad")
        return dict(value=val.value, grad=out)

    def meta_grad_full(self, widths, ranks, P, hw, H, lo, hi, pts, mus, ic_x, ic_mu, per_t, per_mu, lambda_sparse,
                       gamma, lambda_ortho, threads=1, chunk=64):
        """meta_train's full emitter: interior (+ sparse), initial, periodic (per-point mu), + ortho."""
        wv, rv, hwv = _i64(widths), _i64(ranks), _i64(hw)
        pts = _f64(pts).reshape(-1, 2)
        out = np.zeros(lrnr_param_count(wv, rv) + hyper_param_count(hwv))
        comps = np.zeros(4)
        val, ortho = C.c_double(0.0), C.c_double(0.0)
        icx, pt = _f64(ic_x).reshape(-1), _f64(per_t).reshape(-1)
        self._rc(self.lib.ref_meta_grad_full(
            C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)),
            _ptr(_f64(lo)), _ptr(_f64(hi)), _ptr(pts), _ptr(_f64(mus).reshape(-1)), C.c_int64(pts.shape[0]),
            _ptr(icx), _ptr(_f64(ic_mu).reshape(-1)), C.c_int64(icx.shape[0]), _ptr(pt),
            _ptr(_f64(per_mu).reshape(-1)), C.c_int64(pt.shape[0]), C.c_double(lambda_sparse), C.c_double(gamma),
            C.c_double(lambda_ortho), C.c_int(threads), C.c_int(chunk), C.byref(val), _ptr(comps), C.byref(ortho),
            _ptr(out)), "meta_grad_full")
        return dict(value=val.value, comps=comps, ortho=ortho.value, grad=out)

    def meta_grad_reg(self, widths, ranks, P, hw, H, lo, hi, pts, mus, lambda_sparse, gamma, lambda_ortho, w=None,
                      threads=1, chunk=64):
        """meta_train's step gradient with the sparse (banded decay) and ortho (Gram) regularizers."""
        wv, rv, hwv = _i64(widths), _i64(ranks), _i64(hw)
        pts = _f64(pts).reshape(-1, 2)
        n = pts.shape[0]
        w = (1.0 / n if n else 0.0) if w is None else w
        out = np.zeros(lrnr_param_count(wv, rv) + hyper_param_count(hwv))
        comps = np.zeros(4)
        val, ortho = C.c_double(0.0), C.c_double(0.0)
        self._rc(self.lib.ref_meta_grad_reg(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)),
                                            C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)), _ptr(_f64(lo)),
                                            _ptr(_f64(hi)), _ptr(pts), _ptr(_f64(mus).reshape(-1)), C.c_int64(n),
                                            C.c_double(w), C.c_double(lambda_sparse), C.c_double(gamma),
                                            C.c_double(lambda_ortho), C.c_int(threads), C.c_int(chunk), C.byref(val),
                                            _ptr(comps), C.byref(ortho), _ptr(out)), "meta_grad_reg")
        return dict(value=val.value, comps=comps, ortho=ortho.value, grad=out)

    def build_fast(self, widths, ranks, P, s, mu=(0.0, 0.0, 0.0), nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777,
                   r_hat=10):
        wv, rv = _i64(widths), _i64(ranks)
        L = len(rv)
        red = np.zeros(L - 1, np.int64)
        idx = np.full((L - 1) * r_hat, -1, np.int64)
        F = np.zeros(fast_param_count(rv, [r_hat] * (L - 1)))
        exh = np.zeros(L - 1, np.int32)
        self._rc(self.lib.ref_build_fast(C.c_int(L), _ptr(wv), _ptr(rv), _ptr(_f64(P)), _ptr(_f64(s)),
                                         C.c_int64(nx), C.c_int64(nt), C.c_int64(n_perturb), C.c_double(sigma),
                                         C.c_uint64(seed), C.c_int64(r_hat), _ptr(_f64(mu)), _ptr(red), _ptr(idx),
                                         _ptr(F), exh.ctypes.data_as(C.c_void_p)), "build_fast")
        F = F[:fast_param_count(rv, red)]
        return dict(red_ranks=red, indices=idx.reshape(L - 1, r_hat), fparams=F, exhausted=exh)

    def build_fast_hyper(self, widths, ranks, P, hw, H, lo, hi, mus, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777,
                         r_hat=32):
        """harvest_snapshots through the hypernetwork over the mu grid `mus`, eim_greedy, build_fastparams."""
        wv, rv, hwv = _i64(widths), _i64(ranks), _i64(hw)
        mus = _f64(mus).reshape(-1, 3)
        L = len(rv)
        red = np.zeros(L - 1, np.int64)
        idx = np.full((L - 1) * r_hat, -1, np.int64)
        F = np.zeros(fast_param_count(rv, [r_hat] * (L - 1)))
        exh = np.zeros(L - 1, np.int32)
        self._rc(self.lib.ref_build_fast_hyper(
            C.c_int(L), _ptr(wv), _ptr(rv), _ptr(_f64(P)), C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)),
            _ptr(_f64(lo)), _ptr(_f64(hi)), _ptr(mus), C.c_int64(mus.shape[0]), C.c_int64(nx), C.c_int64(nt),
            C.c_int64(n_perturb), C.c_double(sigma), C.c_uint64(seed), C.c_int64(r_hat), _ptr(red), _ptr(idx), _ptr(F),
            exh.ctypes.data_as(C.c_void_p)), "build_fast_hyper")
        F = F[:fast_param_count(rv, red)]
        return dict(red_ranks=red, indices=idx.reshape(L - 1, r_hat), fparams=F, exhausted=exh)

    def eim_greedy(self, S, r_hat):
        """reduction::eim_greedy itself on an M x n_cols snapshot matrix."""
        S = _f64(S)
        m, n = S.shape
        idx = np.zeros(r_hat, np.int64)
        xi = np.zeros((m, r_hat))
        cnt, ex = C.c_int64(0), C.c_int(0)
        self._rc(self.lib.ref_eim_greedy(C.c_int64(m), C.c_int64(n), _ptr(S), C.c_int64(r_hat), _ptr(idx), _ptr(xi),
                                         C.byref(cnt), C.byref(ex)), "eim_greedy")
        k = cnt.value
        return dict(indices=idx[:k].copy(), xi=xi[:, :k].copy(), exhausted=bool(ex.value))

    def identity_fast(self, widths, ranks, P):
        wv, rv = _i64(widths), _i64(ranks)
        red = wv[1:-1].copy()
        F = np.zeros(fast_param_count(rv, red))
        self._rc(self.lib.ref_identity_fast(C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)), _ptr(F)),
                 "identity_fast")
        return red, F

    def meta_train(self, widths, ranks, hyper_depth, hyper_width, init_bias_scale, out_w_scale, out_bias, init_seed,
                   lo, hi, lr, epochs, n_int, n_ic, n_per, seed, lambda_ortho, lambda_sparse, gamma, threads=2,
                   chunk=64):
        wv, rv = _i64(widths), _i64(ranks)
        best = C.c_double(0.0)
        be = C.c_int64(0)
        losses = np.zeros(epochs)
        self._rc(self.lib.ref_meta_train(C.c_int(len(rv)), _ptr(wv), _ptr(rv), C.c_int(hyper_depth),
                                         C.c_int(hyper_width), C.c_double(init_bias_scale), C.c_double(out_w_scale),
                                         C.c_double(out_bias), C.c_uint64(init_seed), _ptr(_f64(lo)), _ptr(_f64(hi)),
                                         C.c_double(lr), C.c_int64(epochs), C.c_int64(n_int), C.c_int64(n_ic),
                                         C.c_int64(n_per), C.c_uint64(seed), C.c_double(lambda_ortho),
                                         C.c_double(lambda_sparse), C.c_double(gamma), C.c_int(threads),
                                         C.c_int(chunk), C.byref(best), C.byref(be), _ptr(losses)), "meta_train")
        return best.value, be.value, losses


REF_CKPT_SO = os.path.join(HERE, "_ref", "liblrnr_ref_ckpt.so")


def reference_ckpt_available() -> bool:
    return os.path.exists(REF_CKPT_SO)


class ReferenceCheckpoint:
    """The reference's own checkpoint writer / reader (oracle/ref_ckpt.cpp; build container only)."""

    def __init__(self, path: str = REF_CKPT_SO):
        self.lib = C.CDLL(path)
        self.lib.ref_ckpt_error.restype = C.c_char_p

    def _rc(self, rc, what):
        if rc != 0:
            raise OracleError(f"{what}: {self.lib.ref_ckpt_error().decode()}")

    def write(self, path, widths, ranks, P, hw, H, lo, hi, X, fast=None):
        wv, rv, hwv = _i64(widths), _i64(ranks), _i64(hw)
        X = _f64(X).reshape(-1, 2)
        if fast is not None:
            fr, frh, F = _i64(fast[0]), _i64(fast[1]), _f64(fast[2])
            Lf = len(fr)
        else:
            fr = frh = F = None
            Lf = 0
        self._rc(self.lib.ref_ckpt_write(str(path).encode(), C.c_int(len(rv)), _ptr(wv), _ptr(rv), _ptr(_f64(P)),
                                         C.c_int(len(hwv) - 1), _ptr(hwv), _ptr(_f64(H)), _ptr(_f64(lo)),
                                         _ptr(_f64(hi)), C.c_int(Lf), _ptr(fr), _ptr(frh), _ptr(F), _ptr(X),
                                         C.c_int64(X.shape[0])), "ref_ckpt_write")

    def read(self, path, n_lrnr, n_hyper):
        P, H = np.zeros(n_lrnr + 1), np.zeros(n_hyper + 1)
        npv, nhv = C.c_int64(0), C.c_int64(0)
        self._rc(self.lib.ref_ckpt_read(str(path).encode(), _ptr(P), C.byref(npv), _ptr(H), C.byref(nhv)),
                 "ref_ckpt_read")
        return P[:npv.value], H[:nhv.value]
