#!/usr/bin/env python
"""Benchmark of the B200 LRNR / FastLRNR residual+gradient path.

Workload (BASELINE.json configs[2], the FP32 config the headline metric --
"PINN residual+gradient point-evals/sec (LRNR & FastLRNR), % of FP32
roofline" -- is quoted on): per GPU, 1,048,576 seeded collocation points on
[0,2pi]x[0,1]; one step = the LRNR (2-256x6-1, ranks (2,32x5,1), sin) residual
+ dL/ds over all points AND the FastLRNR (reference EIM recipe, budget 32)
residual + dL/ds over the same points; with N>1 GPUs the [loss, dL/ds] rows are
summed over ranks with one NCCL all-reduce per step (weak scaling: every rank
owns its own 1M-point batch).  A point-eval = one point through both networks.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c0|c1|c2|c3]

--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified reference compiled in place; tanh -- the reference has no sin)
on a bounded sample of the same workload, with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PINN residual+gradient point-evals/sec (LRNR & FastLRNR), % of FP32 roofline"
UNIT = "point-evals/s"
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 at clocks.max.sm
NOMINAL_FP64_TFLOPS = NOMINAL_FP32_TFLOPS / 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c0", "c1", "c2", "c3"])
    ap.add_argument("--points", type=int, default=0, help="points per GPU (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solves", action="store_true", help="skip the fine_tune / fast_solve loop timings")
    ap.add_argument("--kernel", type=int, default=0,
                    help="LRNR_OPT_KERNEL: 0 auto (tcgen05 LRNR, FMA tile FastLRNR), 1 streaming, 2 tcgen05, 3 FMA tile")
    ap.add_argument("--fast-sincos", type=int, default=0, help="LRNR_OPT_FAST_SINCOS (SFU sin/cos)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.path = tempfile.mktemp(suffix=".csv")
        self.p = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        if not self.p or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def measured_peak(key, fallback):
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)[key])
    except Exception:
        return fallback


def traffic_per_launch():
    """DRAM bytes (read + write) per launch of the dominant kernel, from the committed
    ncu --set full capture (profiles/traffic.json, written from the .ncu-rep)."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            return json.load(f)["dram_bytes_per_launch"]
    except Exception:
        return None


def build_workload(pkg, cfg, rank, points):
    if cfg == "c2":
        n = points or (1 << 20)
        c = pkg.config2(n_points=n)
        if rank:  # weak scaling: an independent seeded batch per rank
            c["pts"] = pkg.sample_collocation(4002 + 1000 * rank, n)
        m, f = c["model"], c["fast"]
        return dict(c=c, dtype=pkg.F32, n=n, models=[(pkg.MODEL_LRNR, m), (pkg.MODEL_FAST, f)], r_hat=32,
                    flops=[pkg.algorithmic_flops_per_point(m.widths, m.ranks),
                           pkg.fast_flops_per_point(f.ranks, f.red_ranks)],
                    workload=(f"c2: LRNR 2-256x6-1 ranks (2,32x5,1) + FastLRNR rhat {list(map(int, f.red_ranks))} "
                              f"(reference EIM recipe, budget 32), sin, FP32, residual u_t+20u_x-0.01u_xx-5u(1-u), "
                              f"{n} pts/GPU, dL/ds"))
    if cfg in ("c0", "c1"):
        n = points or 4096
        c = pkg.config1(n_points=n)
        m, f = c["model"], c["fast"]
        models = [(pkg.MODEL_LRNR, m), (pkg.MODEL_FAST, f)] if cfg == "c1" else [(pkg.MODEL_LRNR, m)]
        flops = [pkg.algorithmic_flops_per_point(m.widths, m.ranks), pkg.fast_flops_per_point(f.ranks, f.red_ranks)]
        return dict(c=c, dtype=pkg.F64, n=n, models=models, flops=flops[:len(models)], r_hat=10,
                    workload=f"{cfg}: LRNR 2-100x3-1 ranks (2,10,10,1)" + (" + FastLRNR rhat 10" if cfg == "c1" else "")
                    + f", tanh, FP64, mu (30,0,0), {n} pts")
    raise SystemExit("config c3 is a parity/scaling config; the default bench line is c2")


def cpu_baseline_sample(pkg, wl, seconds=10.0):
    """Reference (oracle/_ref) or C port, on a bounded sample of the same workload."""
    from oracle.oracle import Oracle, Reference, reference_available
    c = wl["c"]
    cores = os.cpu_count() or 1
    m = c["model"]
    use_ref = reference_available()
    kind = "reference" if use_ref else "port"
    if use_ref:
        R = Reference()
        # the reference is tanh-only: same shapes/FLOPs with tanh, FastLRNR from its own EIM
        f_ref = R.build_fast(m.widths, m.ranks, m.params, c["s"], mu=c["mu"], r_hat=wl["r_hat"]) \
            if "fast" in c else None

        def run(pts):
            R.lrnr_grad(m.widths, m.ranks, m.params, c["s"], c["mu"], pts, threads=cores)
            if f_ref is not None and len(wl["models"]) > 1:
                R.fast_grad(m.ranks, f_ref["red_ranks"], f_ref["fparams"], c["s"], c["mu"], pts, threads=cores)
    else:
        O = Oracle()
        f = c.get("fast")
        cores = int(os.environ.get("OMP_NUM_THREADS", cores))

        def run(pts):
            O.lrnr_grad(m.widths, m.ranks, m.params, c["s"], c["mu"], pts, act=m.act)
            if f is not None and len(wl["models"]) > 1:
                O.fast_grad(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], pts, act=f.act)

    pts = c["pts"]
    probe = pts[:256]
    t0 = time.perf_counter()
    run(probe)
    dt = max(time.perf_counter() - t0, 1e-6)
    n = int(min(len(pts), max(256, 256 * seconds / dt)))
    n = max(256, (n // 256) * 256)
    t0 = time.perf_counter()
    run(pts[:n])
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"first {n} of the {wl['n']} points, LRNR+FastLRNR residual+dL/ds, FP64"
                      + (", tanh (reference is tanh-only; identical shapes and FLOPs)" if use_ref else "")}, run


def solve_loops(pkg, local, with_reference):
    """The solve loops the model is trained / deployed with (training.cpp:428-607), on
    BASELINE c2 shapes with tanh (the reference's activation): fast_solve of the FastLRNR
    (12-point X grid, lambda 1e-2, 400 epochs) and fine_tune of the LRNR (1024 + 256 + 256
    points re-sampled per epoch, 100 epochs), device ms/epoch; the reference's own loops
    on the host cores beside them (bounded samples)."""
    c = pkg.config2(n_points=0, act=pkg.ACT_TANH)
    m, f = c["model"], c["fast"]
    X = np.array([(2 * np.pi * i / 3.0, j / 2.0) for j in range(3) for i in range(4)])
    ctx = pkg.GpuContext(local)
    ctx.set_lrnr(m, pkg.F32)
    ctx.set_fast(f, pkg.F32)
    ctx.fast_solve(c["s"], c["mu"], X, 1e-2, 1e-2, 4)
    t0 = time.perf_counter()
    fs = ctx.fast_solve(c["s"], c["mu"], X, 1e-2, 1e-2, 400)
    t_fs = (time.perf_counter() - t0) / 400
    ctx.fine_tune(c["s"], c["mu"], 1e-2, 2)
    t0 = time.perf_counter()
    ft = ctx.fine_tune(c["s"], c["mu"], 1e-2, 100)
    t_ft = (time.perf_counter() - t0) / 100
    launches = ctx.launches
    ctx.close()
    out = {"fast_solve": {"ms_per_epoch": t_fs * 1e3, "epochs": 400, "best_loss": fs["best_loss"], "dtype": "f32",
                          "workload": "c2 FastLRNR (tanh), 12-point X (4x3 grid), lambda_local 1e-2, lr 1e-2",
                          "path": "lrnr_gpu_fast_solve (one CUDA graph per epoch)"},
           "fine_tune": {"ms_per_epoch": t_ft * 1e3, "epochs": 100, "best_loss": ft["best_loss"], "dtype": "f32",
                         "workload": "c2 LRNR (tanh), 1024 + 256 + 256 points re-sampled per epoch, lr 1e-2",
                         "path": "lrnr_gpu_fine_tune"},
           "gpu_launches": launches}
    if with_reference:
        from oracle.oracle import Reference, reference_available
        if reference_available():
            R = Reference()
            th = os.cpu_count() or 1
            t0 = time.perf_counter()
            R.fast_solve(f.ranks, f.red_ranks, f.fparams, c["s"], c["mu"], X, 1e-2, 1e-2, 400, threads=th)
            out["fast_solve"]["reference_ms_per_epoch"] = (time.perf_counter() - t0) / 400 * 1e3
            t0 = time.perf_counter()
            R.fine_tune(m.widths, m.ranks, m.params, c["s"], c["mu"], 1e-2, 5, 1024, 256, 256, 1234, threads=th)
            out["fine_tune"]["reference_ms_per_epoch"] = (time.perf_counter() - t0) / 5 * 1e3
            out["reference_cores"] = th
            out["reference_note"] = "unmodified reference training::fast_solve / fine_tune, FP64, all host threads"
    return out


def meta_step(pkg, local, rank=0, world=1, dist=None, n_inst=4, per=1 << 20):
    """BASELINE config 4's meta step (widths 2-512x8-1, ranks (2,64x7,1), hypernetwork
    3-64-64-451, sin): U, V, b and hypernetwork gradients through the tcgen05 meta kernel
    (LRNR_OPT_META_PREC = 1: BF16 operands, FP32 accumulation). Each rank owns n_inst whole
    instances of the 64 (instances 4 rank .. 4 rank + 3, weak scaling) x 1,048,576 points;
    one step = the rank's meta gradient + the sum over ranks of the 498,121-entry gradient
    (NCCL all-reduce). Device time with CUDA events, max over ranks, points resident."""
    import torch
    m, _ = pkg.make_baseline_model(pkg.api.C4_WIDTHS, pkg.api.C4_RANKS, 2412, pkg.ACT_SIN)
    h = pkg.make_hyper_params(pkg.api.C4_RANKS, 2, 64, 4005, pkg.api.C3_LO, pkg.api.C3_HI, 0.01, 0.5)
    _, mus_all = pkg.sample_collocation(4006, max(64, n_inst * world), pkg.api.C3_LO, pkg.api.C3_HI, with_mu=True)
    first = n_inst * rank
    mus = np.ascontiguousarray(mus_all[first:first + n_inst])
    pts = np.concatenate([pkg.sample_collocation(6000 + i, per) for i in range(first, first + n_inst)])
    fl = pkg.algorithmic_flops_per_point(m.widths, m.ranks, meta=True)
    ctx = pkg.GpuContext(local)
    ctx.set_option(pkg.OPT_META_PREC, 1)
    ctx.set_lrnr(m, pkg.F32)
    ctx.set_hyper(h)
    ctx.set_points(pts, n_inst=n_inst)
    stream = torch.cuda.current_stream(local)
    ctx.set_stream(stream.cuda_stream)

    def step():
        r = ctx.meta_loss_grad(mus, m.params.size)
        if dist is not None:
            g = torch.from_numpy(np.concatenate([[r["value"]], r["grad"]])).cuda(local)
            dist.all_reduce(g)
            return g
        return None

    step()
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(local)
    e0.record(stream)
    for _ in range(reps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(local)
    ms = e0.elapsed_time(e1) / reps
    if dist is not None:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctx.close()
    n = n_inst * per * world
    tf = fl * n / (ms * 1e-3) / 1e12
    peak = measured_peak("bf16_tflops_sustained", 1400.0) * world
    return {"workload": f"c4 meta step: {n_inst} mu instances per GPU x {per} points (instances 0..{n_inst * world - 1} "
                        "of the 64), 2-512x8-1, r (2,64x7,1), hypernet 3-64-64-451, sin; grads U, V, b, theta (498,121)",
            "kernel": "meta_tc2_kernel (tcgen05 kind::f16, BF16 operands, FP32 accumulate)",
            "n_gpus": world, "scaling": "weak", "collective": "NCCL all-reduce of [loss, gradient] (498,122 doubles)"
            if world > 1 else None,
            "ms_per_step": ms, "point_evals_per_s": n / ms * 1e3, "flop_per_point": fl, "tflops": tf,
            "tensor_roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16, 4 s) x GPUs"},
            "full_step_64_instances_ms_extrapolated": ms * 64 / (n_inst * world)}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import paper_2410_04001_b200 as pkg
    wl = build_workload(pkg, args.config, 0, args.points)
    base, run = cpu_baseline_sample(pkg, wl, seconds=4.0)
    n = int(base["sample"].split()[1])
    pts = wl["c"]["pts"][:n]
    for _ in range(args.warmup):
        run(pts)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run(pts)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * args.steps / tot
    base["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["workload"] + f" (CPU sample of {n} points per step)", "points_per_step": n},
            "cpu_baseline": base, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2410_04001_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    wl = build_workload(pkg, args.config, rank, args.points)
    c = wl["c"]
    n = wl["n"]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = pkg.GpuContext(local)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_option(pkg.OPT_KERNEL, args.kernel)
    ctx.set_option(pkg.OPT_FAST_SINCOS, args.fast_sincos)
    for model, params in wl["models"]:
        (ctx.set_lrnr if model == pkg.MODEL_LRNR else ctx.set_fast)(params, wl["dtype"])
    # inputs resident in HBM for the device-timed value
    pts_dev = torch.from_numpy(np.ascontiguousarray(c["pts"])).to("cuda")
    ctx.set_points_device(pts_dev.data_ptr(), n)
    ctx.upload_coeffs(c["s"], c["mu"])
    R1 = 1 + int(np.sum(c["model"].ranks))
    outs = [torch.zeros(R1, dtype=torch.float64, device="cuda") for _ in wl["models"]]
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2
    w = 1.0 / n

    def step(ev=None):
        for i, (model, _) in enumerate(wl["models"]):
            if ev is not None:
                ev[2 * i].record(stream)
            ctx.run(model, w, outs[i].data_ptr())
            if ev is not None:
                ev[2 * i + 1].record(stream)
        if dist is not None:
            for o in outs:
                dist.all_reduce(o)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.check()

    nm = len(wl["models"])
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nm + 2)] for _ in range(args.steps)]
    launches0 = ctx.launches
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the step's events)
            evs[k][-2].record(stream)
            step(evs[k])
            evs[k][-1].record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    launches = ctx.launches - launches0
    step_ms = sum(e[-2].elapsed_time(e[-1]) for e in evs)
    kern_ms = [sum(e[2 * i].elapsed_time(e[2 * i + 1]) for e in evs) for i in range(nm)]
    t = torch.tensor([step_ms] + kern_ms, dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, kern_ms = float(t[0]), [float(x) for x in t[1:]]
    ms_per_step = step_ms / args.steps
    value = world * n / (ms_per_step * 1e-3)
    ctx.check()

    # the paper's approximation metric: FastLRNR dL/ds against the full LRNR's on the same points
    approx = None
    if len(outs) == 2:
        g_l, g_f = outs[0].double().cpu().numpy(), outs[1].double().cpu().numpy()
        approx = {"grad_s_rel_l2": float(np.linalg.norm(g_f[1:] - g_l[1:]) / np.linalg.norm(g_l[1:])),
                  "loss_rel": float(abs(g_f[0] - g_l[0]) / abs(g_l[0])),
                  "cosine": float(np.dot(g_f[1:], g_l[1:]) / (np.linalg.norm(g_f[1:]) * np.linalg.norm(g_l[1:]))),
                  "what": "FastLRNR vs full-LRNR residual loss and dL/ds on the step's points (EIM r_hat "
                          f"{list(map(int, wl['models'][1][1].red_ranks))})"}

    # roofline of the dominant kernel (the LRNR sweep): algorithmic FLOPs / its event time
    peak_meas = ctx.fma_peak_tflops(wl["dtype"])
    nominal = NOMINAL_FP32_TFLOPS if wl["dtype"] == pkg.F32 else NOMINAL_FP64_TFLOPS
    peak = max(peak_meas, nominal)
    k_ms = kern_ms[0] / args.steps
    achieved = wl["flops"][0] * n / (k_ms * 1e-3) / 1e12
    lrnr_on_tc = wl["dtype"] == pkg.F32 and args.kernel in (pkg.KERNEL_AUTO, pkg.KERNEL_TC)
    roofline = {"bound": "fp32-fma" if wl["dtype"] == pkg.F32 else "fp64-fma", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic_per_launch(),
                "kernel": ("pinn_tc_kernel (tcgen05 3xTF32 LRNR sweep)" if lrnr_on_tc else
                           "pinn_tile_kernel (FMA LRNR sweep)"),
                "flop_per_point": wl["flops"][0],
                "peak_source": f"max(nominal {nominal:.1f} = 148 SM x {128 if wl['dtype'] == pkg.F32 else 64} lanes "
                               f"x 2 x 1.965 GHz, measured FMA microbenchmark {peak_meas:.1f})"}
    if lrnr_on_tc:
        # the same algorithmic FLOPs against the tensor pipe: 3 TF32 products per FP32
        # multiply-add, TF32 dense = bf16 dense / 2 (MEASURED_PEAKS.json burst figure)
        bf16 = measured_peak("bf16_tflops", 2250.0)
        roofline["tensor_3xtf32"] = {"peak": bf16 / 2 / 3, "frac": achieved / (bf16 / 2 / 3),
                                     "peak_source": f"bf16 dense {bf16:.1f} TFLOP/s / 2 (tf32) / 3 (3xTF32)"}
    per_kernel = {}
    for i, (model, _) in enumerate(wl["models"]):
        kms = kern_ms[i] / args.steps
        name = "lrnr" if model == pkg.MODEL_LRNR else "fast"
        per_kernel[name] = {"ms": kms, "point_evals_per_s": world * n / (kms * 1e-3),
                            "tflops": wl["flops"][i] * n / (kms * 1e-3) / 1e12,
                            "frac_of_peak": wl["flops"][i] * n / (kms * 1e-3) / 1e12 / peak,
                            "flop_per_point": wl["flops"][i]}

    # end to end through the public host-buffer C ABI: H2D of the step's points
    # from pinned memory, both gradient calls, D2H of the results.
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(np.ascontiguousarray(c["pts"])).pin_memory().numpy()
        ctx2 = pkg.GpuContext(local)
        ctx2.set_option(pkg.OPT_KERNEL, args.kernel)
        ctx2.set_option(pkg.OPT_FAST_SINCOS, args.fast_sincos)
        for model, params in wl["models"]:
            (ctx2.set_lrnr if model == pkg.MODEL_LRNR else ctx2.set_fast)(params, wl["dtype"])

        def e2e_step():
            ctx2.set_points(pinned)
            for model, _ in wl["models"]:
                ctx2.loss_grad_s(model, c["s"], c["mu"], w)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        K = max(1, min(args.steps, 5))
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(K):
            e2e_step()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt[0])
        e2e = {"value": world * n * K / dt, "unit": UNIT, "h2d_bytes_per_step": int(n * 16 + nm * (8 * R1 + 24)),
               "d2h_bytes_per_step": int(nm * 8 * R1), "ms_per_step": 1e3 * dt / K,
               "path": "lrnr_gpu_set_points + lrnr_gpu_loss_grad_s per model (host buffers)"}
        ctx2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu, _ = cpu_baseline_sample(pkg, wl, seconds=8.0)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "error": str(e)}

    solves = None
    if rank == 0 and world == 1 and not args.no_solves:  # per-GPU latency figures: N = 1 only
        try:
            solves = solve_loops(pkg, local, world == 1 and not args.no_cpu_baseline)
        except Exception as e:  # reported, never fatal
            solves = {"error": str(e)}

    meta = None
    if not args.no_solves and world <= 16:  # all ranks: instances sharded, gradient all-reduced
        try:
            meta = meta_step(pkg, local, rank, world, dist)
        except Exception as e:  # reported, never fatal
            meta = {"error": str(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32" if wl["dtype"] == pkg.F32 else "f64", "data": "synthetic",
                "config": {"workload": wl["workload"], "points_per_gpu": n,
                           "parallelism": f"dp{world} (points sharded by rank, NCCL all-reduce of [loss, dL/ds])",
                           "l2": "flushed between timed steps (256 MiB write outside the step events)",
                           "kernel_option": args.kernel, "fast_sincos": args.fast_sincos},
                "roofline": roofline, "kernels": per_kernel, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(), "solve_loops": solves,
                "fast_vs_lrnr": approx, "meta_c4": meta}
        print(json.dumps(line))
    ctx.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
