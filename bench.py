#!/usr/bin/env python
"""Benchmark of the B200 LRNR / FastLRNR residual+gradient path (BASELINE.json).

Headline (BASELINE configs[2], the FP32 config the metric "PINN residual+gradient
point-evals/sec (LRNR & FastLRNR), % of FP32 roofline" is quoted on): per GPU
1,048,576 seeded collocation points on [0,2pi]x[0,1]; one step = the LRNR
(2-256x6-1, ranks (2,32x5,1), sin, FP32) residual + dL/ds over all points AND
the FastLRNR (reduced width 32, EIM over a mu grid) residual + dL/ds over the
same points.  A point-eval = one point through both networks.  With N GPUs
every rank owns its own 1M-point batch (weak scaling, the headline) and the
[loss, dL/ds] rows are summed by the contexts' own NCCL communicator
(lrnr_gpu_comm_init; one ncclAllReduce per model per step); "c2_strong" splits
the one 1M batch into N contiguous ranges.

Beside it, each BASELINE config gets its own measured sub-line ("configs"):
  c0  LRNR 2-100x3-1 FP64 tanh, 4096 pts           (single GPU; device time of a CUDA graph + host call)
  c1  its FastLRNR (r_hat 10) FP64                  (single GPU)
  c3  1024 mu x 16,384 pts, hypernetwork -> FastLRNR per instance + hypernet VJP, FP32 (mu sharded)
  c4  meta step, 64 mu x 1,048,576 pts, BF16 tcgen05 operands / FP32 accumulate (mu sharded)
each with a roofline of its dominant kernel, an end-to-end figure through the
public host-buffer C ABI, and the reference CPU implementation timed on the
host cores (oracle/_ref, the unmodified reference compiled in place; tanh --
the reference has no sin -- on a bounded sample).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--configs c0,c1,c3,c4]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
with N ranks.  --impl reference times the reference's own CPU implementation
of the headline workload on the host cores (rank 0 only; it imports nothing
from the product package).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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

# BASELINE shapes; duplicated here so the reference arm needs no product import
C0_WIDTHS, C0_RANKS = [2, 100, 100, 100, 1], [2, 10, 10, 1]
C2_WIDTHS, C2_RANKS = [2] + [256] * 6 + [1], [2, 32, 32, 32, 32, 32, 1]
C3_LO, C3_HI = (1.0, 0.0, 0.0), (40.0, 0.1, 10.0)
C2_MU = (20.0, 0.01, 5.0)
C2_POINTS = 1 << 20
FAST_GRID = np.array([(a, b, c) for a in (C3_LO[0], C3_HI[0]) for b in (C3_LO[1], C3_HI[1])
                      for c in (C3_LO[2], C3_HI[2])])
C2_WORKLOAD = ("c2: LRNR 2-256x6-1 ranks (2,32x5,1) + FastLRNR (EIM budget 32, snapshots over the 8 corners of the "
               "c3 mu box through the c3 hypernetwork), residual u_t+20u_x-0.01u_xx-5u(1-u), dL/ds")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--configs", default="c0,c1,c3,c4", help="sub-lines beside the c2 headline ('' = none)")
    ap.add_argument("--points", type=int, default=0, help="headline points per GPU (default 1,048,576)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solves", action="store_true", help="skip the fine_tune / fast_solve loops and the budget curve")
    ap.add_argument("--kernel", type=int, default=0, help="LRNR_OPT_KERNEL (0 auto)")
    ap.add_argument("--fast-sincos", type=int, default=0, help="LRNR_OPT_FAST_SINCOS (SFU sin/cos)")
    return ap.parse_args()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def measured_peak(key, fallback):
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)[key]), "MEASURED_PEAKS.json " + key
    except Exception:
        return fallback, "fallback (B200_PROFILING.md)"


def traffic_per_launch(kernel, points):
    """DRAM bytes (read + write) per launch of a kernel from the committed ncu --set full capture
    (profiles/traffic.json), scaled to this launch's points when the profiled launch had fewer."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            k = json.load(f).get("kernels", {}).get(kernel, {})
        b = k.get("dram_bytes_per_launch")
        return None if b is None else b * points / k.get("points", points)
    except Exception:
        return None


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
        rows = [[x.strip() for x in line.split(",")] for line in open(self.path)]
        rows = [r for r in rows if len(r) >= 9]
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# the reference CPU implementation (oracle/_ref) on the host cores: imports only oracle/
# ---------------------------------------------------------------------------
class RefWorkloads:
    """The BASELINE workloads built and run through the unmodified reference's public API
    (make_lrnr_params + BASELINE init, sample_collocation, harvest_snapshots / eim_greedy /
    build_fastparams, run_batch_gradient with the PinnTermEmitter / fast emitters, hyper_forward +
    its VJP, the meta emitter).  tanh and FP64: the reference has no other activation or dtype."""

    def __init__(self):
        from oracle.oracle import Reference, reference_available
        if not reference_available():
            raise RuntimeError("oracle/_ref/liblrnr_ref.so missing (reference not compiled in place)")
        self.R = Reference()
        self.cores = os.cpu_count() or 1
        self._c2 = None

    def c2(self):
        if self._c2 is None:
            R = self.R
            P, s = R.make_baseline_model(C2_WIDTHS, C2_RANKS, 2411)
            hw, H = R.make_hyper_params(C2_RANKS, 2, 64, C3_LO, C3_HI, 4003)
            f = R.build_fast_hyper(C2_WIDTHS, C2_RANKS, P, hw, H, C3_LO, C3_HI, FAST_GRID, nx=4, nt=3, n_perturb=8,
                                   sigma=0.05, seed=777, r_hat=32)
            self._c2 = dict(P=P, s=s, hw=hw, H=H, f=f)
        return self._c2

    def run_c2(self, pts):
        c = self.c2()
        self.R.lrnr_grad(C2_WIDTHS, C2_RANKS, c["P"], c["s"], C2_MU, pts, threads=self.cores)
        self.R.fast_grad(C2_RANKS, c["f"]["red_ranks"], c["f"]["fparams"], c["s"], C2_MU, pts, threads=self.cores)

    def c2_points(self, n):
        return self.R.sample_collocation(4002, n)["interior"]  # the first n of the headline's stream

    def sample_rate(self, run, make_pts, unit_pts, seconds):
        """Size a sample to ~seconds of work from a probe, then time it once: (points, s)."""
        probe = unit_pts
        t0 = time.perf_counter()
        run(make_pts(probe))
        dt = max(time.perf_counter() - t0, 1e-6)
        n = max(unit_pts, int(unit_pts * max(1.0, seconds / dt)) // unit_pts * unit_pts)
        pts = make_pts(n)
        t0 = time.perf_counter()
        run(pts)
        return n, time.perf_counter() - t0, pts


def fast_flops(ranks, red, m_in=2, m_out=1):
    """SURVEY Appendix B FastLRNR: fwd 4*(M0 r1 + sum rhat(r_l + r_{l+1}) + r_L M_L) FMA, bwd = fwd."""
    L = len(ranks)
    fwd = m_in * ranks[0] + sum(int(red[l]) * (ranks[l] + ranks[l + 1]) for l in range(L - 1)) + ranks[-1] * m_out
    return 2 * 2 * 4 * fwd


def lrnr_flops(widths, ranks, meta=False):
    S = sum(ranks[l] * (widths[l] + widths[l + 1]) for l in range(len(ranks)))
    return 2 * (12 if meta else 8) * S


def run_reference(args):
    """The reference's own CPU implementation of the headline workload, all host threads."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    W = RefWorkloads()
    c = W.c2()
    red = [int(v) for v in c["f"]["red_ranks"]]
    n, _, pts = W.sample_rate(W.run_c2, W.c2_points, 256, 4.0)
    for _ in range(args.warmup):
        W.run_c2(pts)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        W.run_c2(pts)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * args.steps / tot
    fl = lrnr_flops(C2_WIDTHS, C2_RANKS) + fast_flops(C2_RANKS, red)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "activation": "tanh", "config": {"workload": C2_WORKLOAD, "points_per_gpu": C2_POINTS},
            "r_hat": red, "flop_per_point": fl,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": W.cores, "kind": "reference",
                             "sample": f"first {n} of the headline's {C2_POINTS} points per step; unmodified reference "
                                       f"run_batch_gradient (PinnTermEmitter interior terms, LRNR then FastLRNR), tanh "
                                       f"FP64 (the reference has neither sin nor FP32), FastLRNR r_hat {red} from its own "
                                       f"harvest_snapshots/eim_greedy over the same mu grid; {fl} FLOP/pt"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class Env:
    def __init__(self, args):
        import torch
        self.torch = torch
        self.args = args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != args.gpus:
            raise SystemExit(f"bench.py: WORLD_SIZE {self.world} != --gpus {args.gpus}")
        # LRNR_BENCH_GLOO=1 (tests only): ranks share one GPU, so no NCCL communicator can exist;
        # the process group is gloo and the contexts get none (their rows are not summed). It
        # exercises the launch / sharding / timing orchestration of the N-rank run on one GPU.
        self.gloo = os.environ.get("LRNR_BENCH_GLOO") == "1"
        if self.gloo:
            self.local %= torch.cuda.device_count()
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            if self.gloo:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.dist = dist
        self.stream = torch.cuda.Stream()
        torch.cuda.set_stream(self.stream)
        self.flush_buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, vals):
        t = self.torch.tensor(vals, dtype=self.torch.float64, device="cpu" if self.gloo else "cuda")
        if self.dist is not None:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in t]

    def context(self, comm=True):
        import paper_2410_04001_b200 as pkg
        ctx = pkg.GpuContext(self.local)
        ctx.set_stream(self.stream.cuda_stream)
        if comm and self.world > 1 and not self.gloo:
            from paper_2410_04001_b200.dist import attach_nccl
            attach_nccl(ctx)
        return ctx

    def time_steps(self, step, steps, warmup, flush=True, extra_events=0, single_rank=False):
        """W untimed steps, then K steps bracketed by barrier + synchronize, CUDA events on the
        launching stream per step (L2 flushed between steps outside the events); max over ranks.
        step(evs) may record extra events (per-kernel splits) into evs.  single_rank: a section
        only one rank runs (no collectives: the other ranks are not there)."""
        torch = self.torch
        barrier = (lambda: None) if single_rank else self.barrier
        for _ in range(warmup):
            step(None)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 + 2 * extra_events)] for _ in range(steps)]
        for k in range(steps):
            if flush:
                self.flush_buf.zero_()
            evs[k][0].record(self.stream)
            step(evs[k][2:])
            evs[k][1].record(self.stream)
        torch.cuda.synchronize()
        barrier()
        total = sum(e[0].elapsed_time(e[1]) for e in evs)
        splits = [sum(e[2 + 2 * i].elapsed_time(e[3 + 2 * i]) for e in evs) for i in range(extra_events)]
        vals = [total] + splits if single_rank else self.max_over_ranks([total] + splits)
        return vals[0] / steps, [v / steps for v in vals[1:]]


def fma_peak(ctx, pkg, dtype):
    meas = ctx.fma_peak_tflops(dtype)
    nominal = NOMINAL_FP32_TFLOPS if dtype == pkg.F32 else NOMINAL_FP64_TFLOPS
    lanes = 128 if dtype == pkg.F32 else 64
    return max(meas, nominal), (f"max(nominal {nominal:.1f} = 148 SM x {lanes} lanes x 2 x 1.965 GHz, measured FMA "
                                f"microbenchmark {meas:.1f})")


def cpu_baseline(fn):
    try:
        return fn()
    except Exception as e:  # reported, never fatal
        return {"value": None, "error": str(e)}


def headline(env, pkg, args, ctx):
    """c2: weak scaling (1M points per rank, NCCL sum of the rows by the contexts), then strong."""
    torch = env.torch
    n = args.points or C2_POINTS
    c = pkg.config2(n_points=n)
    if env.rank:  # weak scaling: an independent seeded batch per rank
        c["pts"] = pkg.sample_collocation(4002 + 1000 * env.rank, n)
    m, f = c["model"], c["fast"]
    models = [(pkg.MODEL_LRNR, m), (pkg.MODEL_FAST, f)]
    ctx.set_option(pkg.OPT_KERNEL, args.kernel)
    ctx.set_option(pkg.OPT_FAST_SINCOS, args.fast_sincos)
    ctx.set_lrnr(m, pkg.F32)
    ctx.set_fast(f, pkg.F32)
    pts_dev = torch.from_numpy(np.ascontiguousarray(c["pts"])).to("cuda")
    ctx.set_points_device(pts_dev.data_ptr(), n)
    ctx.upload_coeffs(c["s"], c["mu"])
    R1 = 1 + m.r_total
    outs = [torch.zeros(R1, dtype=torch.float64, device="cuda") for _ in models]
    w = 1.0 / (n * env.world)
    flops = [pkg.algorithmic_flops_per_point(m.widths, m.ranks), pkg.fast_flops_per_point(f.ranks, f.red_ranks)]

    def step(evs):
        for i, (model, _) in enumerate(models):
            if evs is not None:
                evs[2 * i].record(env.stream)
            ctx.run(model, w, outs[i].data_ptr())  # + the ncclAllReduce of the rows when N > 1
            if evs is not None:
                evs[2 * i + 1].record(env.stream)

    step(None)
    torch.cuda.synchronize()
    ctx.check()
    launches0 = ctx.launches
    with ClockSampler(env.local) as clk:
        ms, kern = env.time_steps(step, args.steps, args.warmup, extra_events=2)
    launches = (ctx.launches - launches0) * args.steps // (args.steps + args.warmup)
    ctx.check()
    value = env.world * n / (ms * 1e-3)

    # the paper's approximation metric on the step's points: FastLRNR dL/ds against the full LRNR's
    g_l, g_f = outs[0].cpu().numpy(), outs[1].cpu().numpy()
    approx = {"grad_s_rel_l2": float(np.linalg.norm(g_f[1:] - g_l[1:]) / np.linalg.norm(g_l[1:])),
              "loss_rel": float(abs(g_f[0] - g_l[0]) / abs(g_l[0])),
              "cosine": float(np.dot(g_f[1:], g_l[1:]) / (np.linalg.norm(g_f[1:]) * np.linalg.norm(g_l[1:]))),
              "what": f"FastLRNR (r_hat {list(map(int, f.red_ranks))}) vs full-LRNR loss and dL/ds on the step's points"}

    # roofline of the dominant kernel (the LRNR sweep on the tcgen05 tensor pipe): every
    # FP32-accurate multiply-add is 3 FP16 products (hi*hi + hi*lo + lo*hi) at the f16 rate
    bf16, bf16_src = measured_peak("bf16_tflops", 1590.0)
    fp32_peak, fp32_src = fma_peak(ctx, pkg, pkg.F32)
    k_ms = kern[0]
    achieved = flops[0] * n / (k_ms * 1e-3) / 1e12
    tc_peak = bf16 / 3
    lrnr_on_tc = args.kernel in (pkg.KERNEL_AUTO, pkg.KERNEL_TC)
    if lrnr_on_tc:
        roofline = {"bound": "tensor", "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                    "frac": achieved / tc_peak, "traffic": traffic_per_launch("pinn_tc_kernel", n),
                    "kernel": "pinn_tc_kernel (tcgen05 kind::f16, FP16 two-term split = FP32-accurate products)",
                    "flop_per_point": flops[0], "points_per_launch": n,
                    "peak_source": f"{bf16_src} {bf16:.1f} TFLOP/s (f16 / bf16 dense, burst) / 3 (3 FP16 products "
                                   f"per FP32-accurate multiply-add); the kernel is timed alone per step",
                    "fp32_fma_equivalent": {"peak": fp32_peak, "frac": achieved / fp32_peak,
                                            "peak_source": fp32_src}}
    else:
        roofline = {"bound": "fp32-fma", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "traffic": None, "kernel": f"LRNR_OPT_KERNEL {args.kernel}",
                    "flop_per_point": flops[0], "points_per_launch": n, "peak_source": fp32_src}
    per_kernel = {}
    for i, (model, _) in enumerate(models):
        tf = flops[i] * n / (kern[i] * 1e-3) / 1e12
        per_kernel["lrnr" if model == pkg.MODEL_LRNR else "fast"] = {
            "ms": kern[i], "point_evals_per_s": env.world * n / (kern[i] * 1e-3), "tflops": tf,
            "frac_of_fp32_fma": tf / fp32_peak, "flop_per_point": flops[i],
            "kernel": ("pinn_tc_kernel (tcgen05, FP16 two-term split)" if lrnr_on_tc else
                       f"LRNR_OPT_KERNEL {args.kernel}")}
    if lrnr_on_tc:
        per_kernel["fast"]["roofline"] = {"bound": "tensor", "peak": tc_peak,
                                          "traffic": traffic_per_launch("pinn_tc_kernel_fast", n),
                                          "frac": per_kernel["fast"]["tflops"] / tc_peak}
    else:
        per_kernel["fast"]["roofline"] = {"bound": "fp32-fma", "peak": fp32_peak, "traffic": None,
                                          "frac": per_kernel["fast"]["tflops"] / fp32_peak}

    # end to end through the public host-buffer C ABI: H2D of the step's points from pinned
    # memory, both gradient calls with host outputs (D2H), every step
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(np.ascontiguousarray(c["pts"])).pin_memory().numpy()
        ctx2 = env.context()
        ctx2.set_option(pkg.OPT_KERNEL, args.kernel)
        ctx2.set_option(pkg.OPT_FAST_SINCOS, args.fast_sincos)
        ctx2.set_lrnr(m, pkg.F32)
        ctx2.set_fast(f, pkg.F32)

        # a training loop's double-buffered upload through the C ABI: every step's host batch
        # is copied inside the timed region (lrnr_gpu_stage_points, pinned memory, the context's
        # copy stream), the next step's copy overlapping this step's gradient calls
        def e2e_run(steps):
            ctx2.stage_points(pinned)
            for k in range(steps):
                ctx2.use_staged_points()
                if k + 1 < steps:
                    ctx2.stage_points(pinned)
                for model, _ in models:
                    ctx2.loss_grad_s(model, c["s"], c["mu"], w)

        e2e_run(max(1, args.warmup))
        K = max(1, min(args.steps, 5))
        env.barrier()
        t0 = time.perf_counter()
        e2e_run(K)
        dt = env.max_over_ranks([time.perf_counter() - t0])[0]
        e2e = {"value": env.world * n * K / dt, "unit": UNIT, "h2d_bytes_per_step": int(n * 16 + 2 * (8 * R1 + 24)),
               "d2h_bytes_per_step": int(2 * 8 * R1), "ms_per_step": 1e3 * dt / K,
               "path": "lrnr_gpu_stage_points / lrnr_gpu_use_staged_points (host batch, H2D of step k+1 overlapping "
                       "step k) + lrnr_gpu_loss_grad_s per model (host outputs; NCCL sum inside when N > 1)"}
        ctx2.close()

    # strong scaling: the one 1,048,576-point batch split into N contiguous ranges
    strong = None
    if env.world > 1:
        from paper_2410_04001_b200.dist import shard_range
        full = pkg.sample_collocation(4002, C2_POINTS)
        lo, hi = shard_range(C2_POINTS, env.world, env.rank)
        sh = torch.from_numpy(np.ascontiguousarray(full[lo:hi])).to("cuda")
        ctx.set_points_device(sh.data_ptr(), hi - lo)
        ws = 1.0 / C2_POINTS
        ms_s, _ = env.time_steps(lambda evs: [ctx.run(md, ws, outs[i].data_ptr()) for i, (md, _) in enumerate(models)],
                                 args.steps, args.warmup)
        strong = {"value": C2_POINTS / (ms_s * 1e-3), "unit": UNIT, "ms_per_step": ms_s, "points_total": C2_POINTS,
                  "scaling": "strong", "n_gpus": env.world,
                  "what": "the headline's 1,048,576 points split into contiguous ranges over the ranks"}
        ctx.set_points_device(pts_dev.data_ptr(), n)
    else:
        strong = {"value": value, "unit": UNIT, "ms_per_step": ms, "points_total": n, "scaling": "strong",
                  "n_gpus": 1, "what": "N = 1: identical to the headline"}

    cpu = None
    if env.rank == 0 and not args.no_cpu_baseline:
        def ref_c2():
            W = RefWorkloads()
            nn, dt, _ = W.sample_rate(W.run_c2, W.c2_points, 256, 8.0)
            red = [int(v) for v in W.c2()["f"]["red_ranks"]]
            return {"value": nn / dt, "unit": UNIT, "cores": W.cores, "kind": "reference",
                    "sample": f"first {nn} of the {n} points; unmodified reference run_batch_gradient, LRNR + FastLRNR "
                              f"(r_hat {red}, its own EIM on the same mu grid), tanh FP64 (no sin / FP32 in the "
                              f"reference)"}
        cpu = cpu_baseline(ref_c2)
    return dict(c=c, value=value, ms=ms, launches=launches, clocks=clk.summary(), approx=approx, roofline=roofline,
                kernels=per_kernel, e2e=e2e, strong=strong, cpu=cpu, n=n)


def single_gpu_fp64(env, pkg, args, key):
    """c0 / c1: FP64, 4096 points (launch-latency scale; single GPU). Device time of one gradient
    call replayed from a CUDA graph, the host-buffer call latency beside it."""
    torch = env.torch
    c = pkg.config1(n_points=4096)
    m, f = c["model"], c["fast"]
    model = pkg.MODEL_LRNR if key == "c0" else pkg.MODEL_FAST
    fl = (pkg.algorithmic_flops_per_point(m.widths, m.ranks) if key == "c0" else
          pkg.fast_flops_per_point(f.ranks, f.red_ranks))
    n = len(c["pts"])
    ctx = env.context(comm=False)
    ctx.set_lrnr(m, pkg.F64)
    ctx.set_fast(f, pkg.F64)
    pts_dev = torch.from_numpy(np.ascontiguousarray(c["pts"])).to("cuda")
    ctx.set_points_device(pts_dev.data_ptr(), n)
    ctx.upload_coeffs(c["s"], c["mu"])
    out = torch.zeros(1 + m.r_total, dtype=torch.float64, device="cuda")
    w = 1.0 / n
    ctx.run(model, w, out.data_ptr())
    torch.cuda.synchronize()
    timing = "CUDA graph replay of one gradient call (kernel + fixed-order reduction)"
    graph = None
    try:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=env.stream, capture_error_mode="relaxed"):
            ctx.run(model, w, out.data_ptr())
        graph.replay()
        torch.cuda.synchronize()
    except Exception as e:
        graph = None
        timing = f"stream launch per call (graph capture failed: {e})"
    l0 = ctx.launches
    step = (lambda evs: graph.replay()) if graph is not None else (lambda evs: ctx.run(model, w, out.data_ptr()))
    ms, _ = env.time_steps(step, max(args.steps, 20), args.warmup, single_rank=True)  # rank 0 only
    launches_per_call = ctx.launches - l0 if graph is None else None
    ctx.check()
    value = n / (ms * 1e-3)
    peak, src = fma_peak(ctx, pkg, pkg.F64)
    tf = fl * n / (ms * 1e-3) / 1e12
    line = {"workload": (f"{key}: " + ("LRNR" if key == "c0" else "FastLRNR (r_hat 10, reference EIM recipe) of the") +
                         " 2-100x3-1 ranks (2,10,10,1), tanh, FP64, mu (30,0,0), 4096 pts, residual + dL/ds"),
            "n_gpus": 1, "value": value, "unit": UNIT, "ms_per_step": ms, "dtype": "f64", "timing": timing,
            "roofline": {"bound": "fp64-fma", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "flop_per_point": fl, "points_per_launch": n, "peak_source": src,
                         "kernel": "pinn_tile_kernel (FMA tile GEMM, FP64)" if key == "c0" else
                         "pinn_tile_kernel (FastLRNR, FP64)",
                         "traffic": traffic_per_launch("pinn_tile_kernel" if key == "c0" else "pinn_tile_kernel_c1", n),
                         "note": "4096 points = 28 per SM: latency-bound by construction (SURVEY 7)"},
            "gpu_launches_per_step": launches_per_call}
    if not args.no_e2e:
        pinned = torch.from_numpy(np.ascontiguousarray(c["pts"])).pin_memory().numpy()
        for _ in range(5):
            ctx.set_points(pinned)
            ctx.loss_grad_s(model, c["s"], c["mu"])
        K = 200
        t0 = time.perf_counter()
        for _ in range(K):
            ctx.set_points(pinned)
            r = ctx.loss_grad_s(model, c["s"], c["mu"])
        dt = (time.perf_counter() - t0) / K
        line["e2e"] = {"value": n / dt, "unit": UNIT, "ms_per_step": dt * 1e3, "h2d_bytes_per_step": n * 16 + 8 * 26,
                       "d2h_bytes_per_step": 8 * (1 + len(c["s"])),
                       "path": "lrnr_gpu_set_points + lrnr_gpu_loss_grad_s (host buffers)", "loss": r["value"]}
    ctx.close()
    if not args.no_cpu_baseline:
        def ref():
            W = RefWorkloads()
            R = W.R
            P, s = R.make_baseline_model(C0_WIDTHS, C0_RANKS, 2410)
            pts = R.sample_collocation(4001, 4096)["interior"]
            if key == "c0":
                run = lambda: R.lrnr_grad(C0_WIDTHS, C0_RANKS, P, s, (30.0, 0.0, 0.0), pts, threads=W.cores)
            else:
                fr = R.build_fast(C0_WIDTHS, C0_RANKS, P, s, (30.0, 0.0, 0.0), r_hat=10)
                run = lambda: R.fast_grad(C0_RANKS, fr["red_ranks"], fr["fparams"], s, (30.0, 0.0, 0.0), pts,
                                          threads=W.cores)
            run()
            reps, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < 3.0:
                run()
                reps += 1
            dt = (time.perf_counter() - t0) / reps
            return {"value": 4096 / dt, "unit": UNIT, "cores": W.cores, "kind": "reference",
                    "sample": f"the same 4096 points and model (tanh FP64 = the reference's own), {reps} repetitions"}
        line["cpu_baseline"] = cpu_baseline(ref)
    return line


def config_c3(env, pkg, args):
    """c3: 1024 mu x 16,384 points; hypernetwork -> FastLRNR per instance + hypernetwork VJP, FP32.
    Instances sharded over the ranks (strong scaling), dL/dtheta summed by the contexts' NCCL."""
    torch = env.torch
    from paper_2410_04001_b200.dist import shard_instances
    N_INST, PER = 1024, 16384
    a, b = shard_instances(N_INST, env.world, env.rank)
    c = pkg.config3(n_inst=N_INST, pts_per_inst=0)
    pts = np.concatenate([pkg.sample_collocation(5000 + i, PER) for i in range(a, b)])
    f = c["fast"]
    ctx = env.context()
    ctx.set_fast(f, pkg.F32)
    ctx.set_hyper(c["hyper"])
    pts_dev = torch.from_numpy(pts).to("cuda")
    ctx.set_points_device(pts_dev.data_ptr(), len(pts), n_inst=b - a)
    mus = np.ascontiguousarray(c["mus"][a:b])
    w = 1.0 / (N_INST * PER)
    l0 = ctx.launches
    ms, _ = env.time_steps(lambda evs: ctx.hyper_loss_grad(pkg.MODEL_FAST, mus, w), max(3, args.steps // 3),
                           max(1, args.warmup // 2), flush=False)
    launches = ctx.launches - l0
    fl = pkg.fast_flops_per_point(f.ranks, f.red_ranks)
    peak, src = fma_peak(ctx, pkg, pkg.F32)
    bf16, tsrc = measured_peak("bf16_tflops", 1590.0)
    tpk = bf16 / 3
    n_all = N_INST * PER
    tf = fl * n_all / (ms * 1e-3) / 1e12
    line = {"workload": f"c3: 1024 mu ~ U[1,40]xU[0,0.1]xU[0,10] x 16384 pts, hypernetwork 3-64-64-163 (FP64) -> "
                        f"FastLRNR r_hat {list(map(int, f.red_ranks))} per instance (sin, FP32) + hypernetwork VJP",
            "n_gpus": env.world, "scaling": "strong", "value": n_all / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "dtype": "f32", "instances_per_gpu": b - a,
            "collective": "ncclAllReduce of dL/dtheta (15,011 doubles) + the loss, by the contexts" if env.world > 1
            else None,
            "roofline": {"bound": "tensor", "achieved": tf, "peak": tpk, "unit": "TFLOP/s", "frac": tf / tpk,
                         "flop_per_point": fl, "points_per_launch": (b - a) * PER,
                         "peak_source": f"{tsrc} {bf16:.1f} TFLOP/s (f16 dense) / 3 (FP16 two-term split)",
                         "kernel": "pinn_tc_kernel (tcgen05, FP16 two-term split) + FP64 hypernetwork fwd / VJP",
                         "traffic": traffic_per_launch("pinn_tc_kernel_c3", (b - a) * PER),
                         "fp32_fma_equivalent": {"peak": peak, "frac": tf / peak, "peak_source": src}},
            "gpu_launches": launches,
            "l2": "inputs (268 MB of points) larger than L2; no flush"}
    if not args.no_e2e:
        pinned = torch.from_numpy(pts).pin_memory().numpy()
        ctx2 = env.context()
        ctx2.set_fast(f, pkg.F32)
        ctx2.set_hyper(c["hyper"])
        ctx2.set_points(pinned, n_inst=b - a)
        ctx2.hyper_loss_grad(pkg.MODEL_FAST, mus, w)
        K = 3
        env.barrier()
        t0 = time.perf_counter()
        # every step's 268 MB host batch copied inside the timed region, the next one staged
        # while this one computes (lrnr_gpu_stage_points / lrnr_gpu_use_staged_points)
        ctx2.stage_points(pinned, n_inst=b - a)
        for k in range(K):
            ctx2.use_staged_points()
            if k + 1 < K:
                ctx2.stage_points(pinned, n_inst=b - a)
            ctx2.hyper_loss_grad(pkg.MODEL_FAST, mus, w)
        dt = env.max_over_ranks([time.perf_counter() - t0])[0] / K
        line["e2e"] = {"value": n_all / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
                       "h2d_bytes_per_step": int(pinned.nbytes + mus.nbytes),
                       "d2h_bytes_per_step": int(8 * ((b - a) * (1 + f.r_total) + c["hyper"].n_params)),
                       "path": "lrnr_gpu_stage_points / lrnr_gpu_use_staged_points (host batch, next step's H2D "
                               "overlapping this step) + lrnr_gpu_hyper_loss_grad (host outputs)"}
        ctx2.close()
    ctx.close()
    if env.rank == 0 and not args.no_cpu_baseline:
        def ref():
            W = RefWorkloads()
            R, c2r = W.R, W.c2()
            red = c2r["f"]["red_ranks"]
            k_inst, t0, npts = 0, time.perf_counter(), 0
            while time.perf_counter() - t0 < 6.0 and k_inst < 8:
                mu = c["mus"][k_inst]
                s_i = R.hyper_forward(c2r["hw"], c2r["H"], C2_RANKS, C3_LO, C3_HI, mu)
                p_i = R.sample_collocation(5000 + k_inst, 4096)["interior"]
                g = R.fast_grad(C2_RANKS, red, c2r["f"]["fparams"], s_i, mu, p_i, threads=W.cores)
                R.hyper_vjp(c2r["hw"], c2r["H"], C2_RANKS, C3_LO, C3_HI, mu, g["grad_s"])
                k_inst += 1
                npts += len(p_i)
            dt = time.perf_counter() - t0
            return {"value": npts / dt, "unit": UNIT, "cores": W.cores, "kind": "reference",
                    "sample": f"{k_inst} instances x 4096 of the 16384 points: reference hyper_forward, "
                              f"run_batch_gradient (FastLRNR, its own EIM, tanh FP64), hypernetwork VJP"}
        line["cpu_baseline"] = cpu_baseline(ref)
    return line


def config_c4(env, pkg, args):
    """c4: the meta step, 64 mu x 1,048,576 points, BF16 tcgen05 operands / FP32 accumulate;
    instances sharded over the ranks (64 / N each), the 498,121-entry gradient summed by NCCL."""
    torch = env.torch
    from paper_2410_04001_b200.dist import shard_instances
    N_INST, PER = 64, 1 << 20
    a, b = shard_instances(N_INST, env.world, env.rank)
    c = pkg.config4(n_inst=N_INST, pts_per_inst=0)
    m, h = c["model"], c["hyper"]
    pts = np.concatenate([pkg.sample_collocation(6000 + i, PER) for i in range(a, b)])
    ctx = env.context()
    ctx.set_option(pkg.OPT_META_PREC, 1)
    ctx.set_lrnr(m, pkg.F32)
    ctx.set_hyper(h)
    pts_dev = torch.from_numpy(pts).to("cuda")
    ctx.set_points_device(pts_dev.data_ptr(), len(pts), n_inst=b - a)
    mus = np.ascontiguousarray(c["mus"][a:b])
    w = 1.0 / (N_INST * PER)
    l0 = ctx.launches
    ms, _ = env.time_steps(lambda evs: ctx.meta_loss_grad(mus, m.params.size, w), 2, 1, flush=False)
    launches = (ctx.launches - l0) // 3
    fl = pkg.algorithmic_flops_per_point(m.widths, m.ranks, meta=True)
    n_all = N_INST * PER
    tf = fl * n_all / (ms * 1e-3) / 1e12
    peak, src = measured_peak("bf16_tflops_sustained", 1400.0)
    peak *= env.world
    line = {"workload": "c4: meta step, 64 mu x 1048576 pts, 2-512x8-1 r (2,64x7,1), hypernetwork 3-64-64-451, sin; "
                        "grads U, V, b, theta (498,121, ParamPacker order)",
            "n_gpus": env.world, "scaling": "strong", "value": n_all / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "dtype": "bf16 operands, f32 accumulate", "instances_per_gpu": b - a,
            "collective": "ncclAllReduce of the packed gradient (498,121 doubles) + loss, by the contexts"
            if env.world > 1 else None,
            "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "flop_per_point": fl, "points_per_launch": (b - a) * PER,
                         "peak_source": f"{src} x {env.world} GPU(s) (the kernel runs for seconds under the power cap)",
                         "kernel": "meta_tc2_kernel (tcgen05 kind::f16, BF16 operands, FP32 accumulate)",
                         "traffic": traffic_per_launch("meta_tc2_kernel", (b - a) * PER)},
            "gpu_launches": launches,
            "l2": "inputs (1 GB of points) larger than L2; no flush"}
    if not args.no_e2e:
        pinned = torch.from_numpy(pts).pin_memory().numpy()
        del pts_dev
        ctx.set_points(pinned, n_inst=b - a)
        env.barrier()
        t0 = time.perf_counter()
        K = 1
        for _ in range(K):
            ctx.set_points(pinned, n_inst=b - a)
            ctx.meta_loss_grad(mus, m.params.size, w)
        dt = env.max_over_ranks([time.perf_counter() - t0])[0] / K
        line["e2e"] = {"value": n_all / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
                       "h2d_bytes_per_step": int(pinned.nbytes + mus.nbytes),
                       "d2h_bytes_per_step": int(8 * (m.params.size + h.n_params + 1)),
                       "path": "lrnr_gpu_set_points + lrnr_gpu_meta_loss_grad (host buffers)"}
    ctx.close()
    if env.rank == 0 and not args.no_cpu_baseline:
        def ref():
            W = RefWorkloads()
            R = W.R
            widths, ranks = [2] + [512] * 8 + [1], [2] + [64] * 7 + [1]
            P, _ = R.make_baseline_model(widths, ranks, 2412)
            hw, H = R.make_hyper_params(ranks, 2, 64, C3_LO, C3_HI, 4005, 0.01, 0.5)
            npt = 1024
            p0 = R.sample_collocation(6000, npt)["interior"]
            mu0 = np.repeat(c["mus"][:1], npt, axis=0)
            t0 = time.perf_counter()
            R.meta_grad(widths, ranks, P, hw, H, C3_LO, C3_HI, p0, mu0, threads=W.cores)
            dt = time.perf_counter() - t0
            return {"value": npt / dt, "unit": UNIT, "cores": W.cores, "kind": "reference",
                    "sample": f"instance 0 x {npt} points: reference run_batch_gradient with the meta emitter "
                              "(emit_hyper per point -> emit_lrnr_jet, BasesBiasesAndHyper), tanh FP64"}
        line["cpu_baseline"] = cpu_baseline(ref)
    return line


def budget_curve(env, pkg, c):
    """The paper's FastLRNR accuracy against the reduction budget (Fig. 2's metric, acceptance.cpp:400-453):
    per r_hat, |u_fast - u_lrnr| at the sampling set X and over 65,536 points, and the dL/ds
    approximation (rel. L2, cosine) against the full LRNR, on the c2 model (sin, FP32)."""
    torch = env.torch
    m, s, mu = c["model"], c["s"], c["mu"]
    ctx = env.context(comm=False)
    ctx.set_lrnr(m, pkg.F32)
    X = pkg.uniform_grid(4, 3)
    pts = c["pts"][:65536]
    ctx.set_points(pts)
    gl = ctx.loss_grad_s(pkg.MODEL_LRNR, s, mu)
    u_l_X = ctx.values(pkg.MODEL_LRNR, s, X)
    u_l_P = ctx.values(pkg.MODEL_LRNR, s, pts)
    S = pkg.hyper_forward(pkg.c3_hyper(), pkg.api.C2_FAST_MU_GRID)
    rows = []
    for r_hat in (4, 8, 16, 24, 32):
        t0 = time.perf_counter()
        f = ctx.build_fast(m, S, nx=4, nt=3, n_perturb=8, sigma=0.05, seed=777, r_hat=r_hat)
        t_build = time.perf_counter() - t0
        ctx.set_fast(f, pkg.F32)
        gf = ctx.loss_grad_s(pkg.MODEL_FAST, s, mu)
        dX = np.abs(ctx.values(pkg.MODEL_FAST, s, X) - u_l_X)
        dP = np.abs(ctx.values(pkg.MODEL_FAST, s, pts) - u_l_P)
        rows.append({"r_hat": list(map(int, f.red_ranks)), "u_abs_err_X_max": float(dX.max()),
                     "u_abs_err_X_mean": float(dX.mean()), "u_abs_err_65536_mean": float(dP.mean()),
                     "u_lrnr_abs_mean": float(np.abs(u_l_P).mean()),
                     "grad_s_rel_l2": float(np.linalg.norm(gf["grad_s"] - gl["grad_s"]) / np.linalg.norm(gl["grad_s"])),
                     "cosine": float(np.dot(gf["grad_s"], gl["grad_s"]) /
                                     (np.linalg.norm(gf["grad_s"]) * np.linalg.norm(gl["grad_s"]))),
                     "loss_rel": float(abs(gf["value"] - gl["value"]) / abs(gl["value"])),
                     "build_ms": t_build * 1e3})
    ctx.close()
    return {"what": "FastLRNR vs LRNR per reduction budget (c2 model, sin, FP32): |u_fast - u_lrnr| at the 4x3 "
                    "sampling set X and on 65,536 collocation points; dL/ds rel. L2 / cosine on those points; "
                    "FastLRNR built on the device (harvest + greedy EIM over the mu grid)", "rows": rows}


def solve_loops(env, pkg, with_reference):
    """The solve loops the model is trained / deployed with (training.cpp:428-607), on BASELINE c2
    shapes with tanh (the reference's activation): fast_solve of the FastLRNR (12-point X grid, lambda
    1e-2, 400 epochs) and fine_tune of the LRNR (1024 + 256 + 256 points re-sampled per epoch, 100
    epochs), device ms/epoch; the reference's own loops on the host cores beside them."""
    c = pkg.config2(n_points=0, act=pkg.ACT_TANH)
    m, f = c["model"], c["fast"]
    X = pkg.uniform_grid(4, 3)
    ctx = env.context(comm=False)
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
                          "workload": f"c2 FastLRNR r_hat {list(map(int, f.red_ranks))} (tanh), 12-point X (4x3 grid), "
                                      "lambda_local 1e-2, lr 1e-2",
                          "path": "lrnr_gpu_fast_solve (persistent cluster solver, one launch)"},
           "fine_tune": {"ms_per_epoch": t_ft * 1e3, "epochs": 100, "best_loss": ft["best_loss"], "dtype": "f32",
                         "workload": "c2 LRNR (tanh), 1024 + 256 + 256 points re-sampled per epoch, lr 1e-2",
                         "path": "lrnr_gpu_fine_tune"},
           "gpu_launches": launches}
    if with_reference:
        try:
            W = RefWorkloads()
            R, c2r = W.R, W.c2()
            s = c2r["s"]
            t0 = time.perf_counter()
            R.fast_solve(C2_RANKS, c2r["f"]["red_ranks"], c2r["f"]["fparams"], s, C2_MU, X, 1e-2, 1e-2, 400,
                         threads=W.cores)
            out["fast_solve"]["reference_ms_per_epoch"] = (time.perf_counter() - t0) / 400 * 1e3
            t0 = time.perf_counter()
            R.fine_tune(C2_WIDTHS, C2_RANKS, c2r["P"], s, C2_MU, 1e-2, 5, 1024, 256, 256, 1234, threads=W.cores)
            out["fine_tune"]["reference_ms_per_epoch"] = (time.perf_counter() - t0) / 5 * 1e3
            out["reference_cores"] = W.cores
            out["reference_note"] = "unmodified reference training::fast_solve / fine_tune, FP64, all host threads"
        except Exception as e:
            out["reference_error"] = str(e)
    return out


def run_ours(args):
    env = Env(args)
    import paper_2410_04001_b200 as pkg

    ctx = env.context()
    h = headline(env, pkg, args, ctx)
    ctx.close()
    configs = {}
    wanted = [k.strip() for k in args.configs.split(",") if k.strip()]
    for key in wanted:
        try:
            if key in ("c0", "c1"):
                if env.rank == 0:
                    configs[key] = single_gpu_fp64(env, pkg, args, key)
                env.barrier()
            elif key == "c3":
                configs[key] = config_c3(env, pkg, args)
            elif key == "c4":
                configs[key] = config_c4(env, pkg, args)
        except Exception as e:  # reported, never fatal
            configs[key] = {"error": f"{type(e).__name__}: {e}"}
            env.barrier()
    extra = {}
    if env.rank == 0 and not args.no_solves:
        for name, fn in (("fastlrnr_budget_curve", lambda: budget_curve(env, pkg, h["c"])),
                         ("solve_loops", lambda: solve_loops(env, pkg, not args.no_cpu_baseline))):
            try:
                extra[name] = fn()
            except Exception as e:
                extra[name] = {"error": f"{type(e).__name__}: {e}"}
    env.barrier()

    if env.rank == 0:
        f = h["c"]["fast"]
        line = {"metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": env.world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": h["ms"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "activation": "sin",
                "config": {"workload": C2_WORKLOAD, "points_per_gpu": h["n"]},
                "r_hat": list(map(int, f.red_ranks)),
                "flop_per_point": sum(v["flop_per_point"] for v in h["kernels"].values()),
                "parallelism": (f"dp{env.world}: points per rank, [loss, dL/ds] summed by the contexts' NCCL "
                                "communicator (lrnr_gpu_comm_init)" if env.world > 1 else "single GPU"),
                "l2": "flushed between timed steps (256 MiB write outside the step events)",
                "roofline": h["roofline"], "kernels": h["kernels"], "cpu_baseline": h["cpu"], "e2e": h["e2e"],
                "gpu_launches": h["launches"], "clocks": h["clocks"], "c2_strong": h["strong"],
                "fast_vs_lrnr": h["approx"], "configs": configs}
        line.update(extra)
        print(json.dumps(line))
    if env.dist is not None:
        env.barrier()
        env.dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execvp(cmd[0], cmd)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
