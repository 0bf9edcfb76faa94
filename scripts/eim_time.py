"""Dev aid: FastLRNR construction (harvest_snapshots + eim_greedy + build_fastparams)
on the device vs the host restatement (the reference's algorithm, one thread), c2
widths, r_hat = 32, n_mu coefficient vectors (the hyper_forward outputs of a mu grid).

    python scripts/eim_time.py [--host-max 256] [--out profiles/r01_eim_time.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_04001_b200 as pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--host-max", type=int, default=64)
    ap.add_argument("--out", default="")
    ap.add_argument("--only", type=int, default=0, help="run this n_mu only")
    a = ap.parse_args()
    from paper_2410_04001_b200.api import C2_RANKS, C2_WIDTHS

    m, s0 = pkg.make_baseline_model(C2_WIDTHS, C2_RANKS, 2411)
    gpu = pkg.GpuContext(0)
    rng = np.random.default_rng(0)
    rows = []
    for n_mu in ([a.only] if a.only else (1, 16, 64, 256, 1024, 4096)):
        s = s0[None, :] * rng.uniform(0.5, 1.5, (n_mu, m.r_total))
        fd = gpu.build_fast(m, s, r_hat=32)  # warm-up (module load, allocation at this size)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fd = gpu.build_fast(m, s, r_hat=32)
            ts.append(time.perf_counter() - t0)
        td = float(np.median(ts))
        row = dict(n_mu=n_mu, n_cols=n_mu * 108, device_s=td, red=fd.red_ranks.tolist())
        if n_mu <= a.host_max:
            t0 = time.perf_counter()
            fh = pkg.build_fast(m, s, r_hat=32)
            row["host_s"] = time.perf_counter() - t0
            row["indices_equal"] = bool(np.array_equal(fh.indices, fd.indices))
            row["fparams_maxnorm_rel"] = float(np.abs(fh.fparams - fd.fparams).max() / np.abs(fh.fparams).max())
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(dict(config="c2 widths (2,256x6,1) ranks (2,32x5,1), tanh, nx=4 nt=3 n_perturb=8 r_hat=32",
                           rows=rows), f, indent=1)


if __name__ == "__main__":
    main()
