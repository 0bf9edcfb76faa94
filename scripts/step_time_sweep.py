"""The reference's step-time benchmark (training.cpp:613-799, benchmark_step_time) beside the
device: per hidden width M, one fine-tune step (PinnTermEmitter terms over 1024 + 256 + 256
points re-sampled per step, Adam, projection) and one fast step (the l1 objective on the 4x3
grid X + locality, Adam, projection). BenchmarkConfig shapes: ranks (1,16,16,16,1), r_hat 5,
tanh, mu (1, 0.5, 0.5); the device uses seeded synthetic parameters of the same shapes.
Writes profiles/r01_step_time_sweep.json."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2410_04001_b200 as pkg

WIDTHS = [int(w) for w in (sys.argv[1].split(",") if len(sys.argv) > 1 else "64,128,256,512,1024".split(","))]
RANKS = [1, 16, 16, 16, 1]
RHAT = 5
MU = np.array([1.0, 0.5, 0.5])
X = np.array([(2 * np.pi * i / 3.0, j / 2.0) for j in range(3) for i in range(4)])
rows = []
ctx = pkg.GpuContext(0)
for m in WIDTHS:
    widths = [2] + [m] * (len(RANKS) - 1) + [1]
    model, s = pkg.make_baseline_model(widths, RANKS, 2024, pkg.ACT_TANH)
    rng = np.random.default_rng(m)
    # FastParams of BenchContext's shapes: v_in = V_0, u_hat / v_hat normal, b_hat 0.1 normal, u_out = U_last
    L = len(RANKS)
    F = []
    o, _ = model.offsets()  # per layer (U, V, b) offsets
    F.extend(model.params[o[0][1]:o[0][1] + 2 * RANKS[0]])
    red = []
    for l in range(L - 1):
        rh = min(RHAT, widths[l + 1])
        red.append(rh)
        F.extend(rng.standard_normal(rh * RANKS[l]))
        F.extend(0.1 * rng.standard_normal(rh))
        F.extend(rng.standard_normal(rh * RANKS[l + 1]))
    F.extend(model.params[o[L - 1][0]:o[L - 1][0] + RANKS[L - 1]])
    F.extend(model.params[o[L - 1][2]:o[L - 1][2] + 1])
    fast = pkg.FastParams(np.array(RANKS), np.array(red), np.array(F), pkg.ACT_TANH)
    for dt, name in ((pkg.F32, "f32"), (pkg.F64, "f64")):
        ctx.set_lrnr(model, dt)
        ctx.set_fast(fast, dt)
        ctx.fine_tune(s, MU, 1e-2, 2)
        n_tune, samples = 20, []
        for _ in range(5):  # median of 5 runs (first-launch effects, host jitter)
            t0 = time.perf_counter()
            ctx.fine_tune(s, MU, 1e-2, n_tune)
            samples.append((time.perf_counter() - t0) / n_tune)
        t_tune = float(np.median(samples))
        ctx.fast_solve(s, MU, X, 1e-2, 1e-2, 5)
        t0 = time.perf_counter()
        n_fast = 400
        ctx.fast_solve(s, MU, X, 1e-2, 1e-2, n_fast)
        t_fast = (time.perf_counter() - t0) / n_fast
        rows.append({"width": m, "dtype": name, "device_tune_step_ms": t_tune * 1e3, "device_fast_step_us": t_fast * 1e6})
        print(rows[-1], flush=True)
ref = None
try:
    from oracle.oracle import reference_available, REF_SO
    if reference_available():
        lib = C.CDLL(REF_SO)
        w = np.array(WIDTHS, dtype=np.int64)
        tt, tf = np.zeros(len(WIDTHS)), np.zeros(len(WIDTHS))
        th = os.cpu_count() or 1
        rc = lib.ref_benchmark_step_time(w.ctypes.data_as(C.c_void_p), C.c_int64(len(WIDTHS)), C.c_int64(5),
                                         C.c_int64(1), C.c_int(th), tt.ctypes.data_as(C.c_void_p),
                                         tf.ctypes.data_as(C.c_void_p))
        if rc == 0:
            ref = {"threads": th, "rows": [{"width": int(a), "tune_step_ms": b * 1e3, "fast_step_us": c * 1e6}
                                           for a, b, c in zip(WIDTHS, tt, tf)]}
            print(ref, flush=True)
except Exception as e:  # reported, never fatal
    ref = {"error": str(e)}
out = {"what": __doc__.split("\n")[0], "device": rows, "reference_benchmark_step_time": ref}
dest = os.environ.get("SWEEP_OUT", os.path.join("profiles", "r01_step_time_sweep.json"))
os.makedirs(os.path.dirname(dest), exist_ok=True)
json.dump(out, open(dest, "w"), indent=1, default=float)
