"""CPU, world_size 2 over gloo: the multi-GPU decomposition of the path.

Each rank computes its shard's [loss, dL/ds] rows (points sharded for config 2,
whole instances for config 3) with the FP64 oracle standing in for the device
sweep, then the rows are summed with the same all-reduce helper bench.py uses
(NCCL on the GPU box).  The result must equal the single-process sweep over
all points / instances.  Config 4 (meta step): whole instances per rank, the
packed [U, V, b, theta] gradient summed."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def meta_grads(O, g, a, b):
    """Sum over instances a..b-1 of 4 (24 golden c4 points each) of the meta gradient."""
    nP = g["c4_params"].size
    out = np.zeros(nP + g["c4_hparams"].size)
    for i in range(a, b):
        mu = g["c4_mus"][24 * i]
        s_i = O.hyper_forward(g["c4_hw"], g["c4_hparams"], g["c3_lo"], g["c3_hi"], mu)
        r = O.lrnr_grad(g["c4_widths"], g["c4_ranks"], g["c4_params"], s_i, mu, g["c4_pts"][24 * i:24 * (i + 1)],
                        w=1.0 / 96, params_grad=True)
        out[:nP] += r["grad_params"]
        O.hyper_vjp(g["c4_hw"], g["c4_hparams"], g["c3_lo"], g["c3_hi"], mu, r["grad_s"], out=out[nP:])
    return out


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2410_04001_b200.dist import allreduce_sum_, shard_instances, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz")))
    # config-2 style: points sharded, weight 1/N_global
    pts = g["c2_pts"]
    n = len(pts)
    lo, hi = shard_range(n, world, rank)
    r = O.lrnr_grad(g["c2_widths"], g["c2_ranks"], g["c2_params"], g["c2_s"], g["c2_mu"], pts[lo:hi], w=1.0 / n)
    row = torch.tensor(np.concatenate([[r["value"]], r["grad_s"]]))
    allreduce_sum_(row)
    # config-3 style: instances sharded, hypernetwork gradient summed
    mus = g["c3_mu"]
    a, b = shard_instances(len(mus), world, rank)
    hw, H, lo3, hi3 = g["c3_hw"], g["c3_hparams"], g["c3_lo"], g["c3_hi"]
    sub = pts[:64]
    ght = np.zeros(H.size)
    for i in range(a, b):
        s_i = O.hyper_forward(hw, H, lo3, hi3, mus[i])
        ri = O.fast_grad(g["c2_ranks"], g["c2_red_ranks"], g["c2_fparams"], s_i, mus[i], sub,
                         w=1.0 / (len(mus) * len(sub)))
        O.hyper_vjp(hw, H, lo3, hi3, mus[i], ri["grad_s"], out=ght)
    th = torch.tensor(ght)
    allreduce_sum_(th)
    # config-4 style: meta gradient (U, V, b then theta, ParamPacker order), instances sharded
    mg = meta_grads(O, g, *shard_instances(4, world, rank))
    tm = torch.tensor(mg)
    allreduce_sum_(tm)
    if rank == 0:
        q.put((row.numpy(), th.numpy(), tm.numpy()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_sharding_equals_single_process(oracle, golden):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    row, th, tm = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = golden
    full = oracle.lrnr_grad(g["c2_widths"], g["c2_ranks"], g["c2_params"], g["c2_s"], g["c2_mu"], g["c2_pts"])
    assert abs(row[0] - full["value"]) <= 1e-13 * full["value"]
    np.testing.assert_allclose(row[1:], full["grad_s"], rtol=1e-11, atol=1e-14 * np.abs(full["grad_s"]).max())
    mus = g["c3_mu"]
    sub = g["c2_pts"][:64]
    ref = np.zeros(g["c3_hparams"].size)
    for i in range(len(mus)):
        s_i = oracle.hyper_forward(g["c3_hw"], g["c3_hparams"], g["c3_lo"], g["c3_hi"], mus[i])
        ri = oracle.fast_grad(g["c2_ranks"], g["c2_red_ranks"], g["c2_fparams"], s_i, mus[i], sub,
                              w=1.0 / (len(mus) * len(sub)))
        oracle.hyper_vjp(g["c3_hw"], g["c3_hparams"], g["c3_lo"], g["c3_hi"], mus[i], ri["grad_s"], out=ref)
    np.testing.assert_allclose(th, ref, rtol=1e-11, atol=1e-14 * np.abs(ref).max())
    ref4 = meta_grads(oracle, g, 0, 4)
    np.testing.assert_allclose(tm, ref4, rtol=1e-11, atol=1e-14 * np.abs(ref4).max())


# ---------------------------------------------------------------------------
# the product path: 2 ranks over gloo, each driving its own context on cuda:0
# ---------------------------------------------------------------------------
def _gpu_case():
    import paper_2410_04001_b200 as pkg

    c2 = pkg.config2(n_points=6000)
    c3 = pkg.config3(n_inst=6, pts_per_inst=300)
    c4 = pkg.config4(n_inst=4, pts_per_inst=96)
    return pkg, c2, c3, c4


def _gpu_rows(pkg, c2, c3, c4, rank, world):
    """One rank's share through the C ABI: c2 points, c3 / c4 whole instances; global weights."""
    from paper_2410_04001_b200.dist import shard_instances, shard_range

    ctx = pkg.GpuContext(0)
    try:
        n = len(c2["pts"])
        lo, hi = shard_range(n, world, rank)
        ctx.set_lrnr(c2["model"], pkg.F32)
        ctx.set_fast(c2["fast"], pkg.F32)
        ctx.set_points(c2["pts"][lo:hi])
        r = ctx.loss_grad_s(pkg.MODEL_LRNR, c2["s"], c2["mu"], w=1.0 / n)
        rf = ctx.loss_grad_s(pkg.MODEL_FAST, c2["s"], c2["mu"], w=1.0 / n)
        a, b = shard_instances(c3["n_inst"], world, rank)
        per = len(c3["pts"]) // c3["n_inst"]
        ctx.set_fast(c3["fast"], pkg.F32)
        ctx.set_hyper(c3["hyper"])
        ctx.set_points(c3["pts"][a * per:b * per], n_inst=b - a)
        h = ctx.hyper_loss_grad(pkg.MODEL_FAST, c3["mus"][a:b], w=1.0 / len(c3["pts"]))
        a4, b4 = shard_instances(c4["n_inst"], world, rank)
        per4 = len(c4["pts"]) // c4["n_inst"]
        ctx.set_option(pkg.OPT_META_PREC, 1)
        ctx.set_lrnr(c4["model"], pkg.F32)
        ctx.set_hyper(c4["hyper"])
        ctx.set_points(c4["pts"][a4 * per4:b4 * per4], n_inst=b4 - a4)
        g4 = ctx.meta_loss_grad(c4["mus"][a4:b4], c4["model"].params.size, w=1.0 / len(c4["pts"]))
        return (np.concatenate([[r["value"]], r["grad_s"]]), np.concatenate([[rf["value"]], rf["grad_s"]]),
                np.concatenate([[h["value"]], h["grad_theta"]]), np.concatenate([[g4["value"]], g4["grad"]]))
    finally:
        ctx.close()


def _gpu_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2410_04001_b200.dist import allreduce_sum_

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pkg, c2, c3, c4 = _gpu_case()
    out = [allreduce_sum_(torch.from_numpy(x.copy())).numpy() for x in _gpu_rows(pkg, c2, c3, c4, rank, world)]
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_rank_product_path_equals_single_context():
    """Two processes on one GPU (their kernels never wait on each other), each running its shard
    through the product C ABI; the rows summed over gloo equal one context over everything."""
    pytest.importorskip("torch")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=540)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pkg, c2, c3, c4 = _gpu_case()
    want = _gpu_rows(pkg, c2, c3, c4, 0, 1)
    for name, g, w, tol in zip(("c2 LRNR", "c2 FastLRNR", "c3 theta", "c4 meta"), got, want,
                               (1e-6, 1e-6, 1e-6, 1e-5)):
        err = np.linalg.norm(g - w) / np.linalg.norm(w)
        assert err <= tol, (name, err)


@pytest.mark.gpu
@pytest.mark.timeout(480)
def test_bench_two_ranks_orchestration_on_one_gpu(tmp_path):
    """bench.py --gpus 2 re-launches itself under torch.distributed.run with 2 ranks (here both on
    cuda:0, gloo process group, no NCCL communicator -- LRNR_BENCH_GLOO), shards c2 / c3, times with
    max over ranks and prints one line with n_gpus 2 from rank 0."""
    import json
    import subprocess

    env = dict(os.environ, LRNR_BENCH_GLOO="1")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--configs", "c0,c3", "--no-solves", "--no-cpu-baseline", "--no-e2e", "--points", "65536"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["c2_strong"]["n_gpus"] == 2
    assert d["configs"]["c3"]["n_gpus"] == 2 and d["configs"]["c3"]["instances_per_gpu"] == 512
    assert d["configs"]["c0"]["n_gpus"] == 1 and d["configs"]["c0"]["value"] > 0
