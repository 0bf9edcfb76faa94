"""Round-2 golden fixtures from the UNMODIFIED reference (oracle/_ref, built by
``make -C oracle`` in the build container):

    python tests/golden/make_golden_r2.py   ->  tests/golden/reference_golden_r2.npz

* hyper_forward of the c3 hypernetwork (3-64-64-163, seed 4003) at the 8 corners of
  the c3 mu box, and the c2 FastLRNR built from them by the reference's own
  harvest_snapshots (mu grid) / eim_greedy / build_fastparams, budget 32 (tanh: the
  reference's activation);
* the plain losses loss_tune (with boundary terms), loss_fast (sampling sets 4x3
  and 7x5) and loss_meta (per-sample mu), and lrnr_forward / fast_forward values on
  BASELINE config 0 / 1.
Every array is produced by the reference's own code; nothing is restated.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
C2_WIDTHS, C2_RANKS = [2] + [256] * 6 + [1], [2, 32, 32, 32, 32, 32, 1]
C0_WIDTHS, C0_RANKS = [2, 100, 100, 100, 1], [2, 10, 10, 1]
LO, HI = (1.0, 0.0, 0.0), (40.0, 0.1, 10.0)
GRID = np.array([(a, b, c) for a in (LO[0], HI[0]) for b in (LO[1], HI[1]) for c in (LO[2], HI[2])])


def main():
    R = Reference()
    g = {"mu_grid": GRID}
    P2, s2 = R.make_baseline_model(C2_WIDTHS, C2_RANKS, 2411)
    hw, H = R.make_hyper_params(C2_RANKS, 2, 64, LO, HI, 4003)
    g["c3_hparams"] = H
    g["grid_s"] = np.array([R.hyper_forward(hw, H, C2_RANKS, LO, HI, mu) for mu in GRID])
    f = R.build_fast_hyper(C2_WIDTHS, C2_RANKS, P2, hw, H, LO, HI, GRID, r_hat=32)
    g.update(c2grid_red=f["red_ranks"], c2grid_idx=f["indices"], c2grid_fparams=f["fparams"],
             c2grid_exh=f["exhausted"])

    P0, s0 = R.make_baseline_model(C0_WIDTHS, C0_RANKS, 2410)
    mu0 = np.array([30.0, 0.0, 0.0])
    b = R.sample_collocation(4009, 600, 70, 50)
    g.update(c0_params=P0, c0_s=s0, lt_pts=b["interior"], lt_icx=b["initial_x"], lt_pert=b["periodic_t"])
    g["lt_out"] = R.loss_tune(C0_WIDTHS, C0_RANKS, P0, s0, mu0, b["interior"], b["initial_x"], b["periodic_t"])
    f0 = R.build_fast(C0_WIDTHS, C0_RANKS, P0, s0, mu0, r_hat=10)
    g.update(c1_red=f0["red_ranks"], c1_fparams=f0["fparams"])
    for nx, nt in ((4, 3), (7, 5)):
        X = np.array([(2 * np.pi * i / (nx - 1) if nx > 1 else 0.0, j / (nt - 1) if nt > 1 else 0.0)
                      for j in range(nt) for i in range(nx)])
        X[:, 0] = np.where(np.arange(len(X)) % nx == nx - 1, 6.283185307179586476925286766559, X[:, 0])
        g[f"lf_{nx}x{nt}_X"] = X
        g[f"lf_{nx}x{nt}_out"] = R.loss_fast(C0_RANKS, f0["red_ranks"], f0["fparams"], s0, mu0, X)
    vp = R.sample_collocation(4010, 257)["interior"]
    g["val_pts"] = vp
    g["val_lrnr"] = R.values(0, C0_WIDTHS, C0_RANKS, P0, None, None, s0, vp)
    g["val_fast"] = R.values(1, None, C0_RANKS, None, f0["red_ranks"], f0["fparams"], s0, vp)

    # loss_meta: per-sample mu (sample_collocation with mu), hypernetwork 3-16-16-23 on c0
    hwm, Hm = R.make_hyper_params(C0_RANKS, 2, 16, LO, HI, 4012)
    mb = R.sample_collocation(4011, 300, 40, 30, LO, HI, with_mu=True)
    g.update(lm_hparams=Hm, lm_pts=mb["interior"], lm_mu=mb["interior_mu"], lm_icx=mb["initial_x"],
             lm_icmu=mb["initial_mu"], lm_pert=mb["periodic_t"], lm_permu=mb["periodic_mu"])
    g["lm_out"] = R.loss_meta(C0_WIDTHS, C0_RANKS, P0, hwm, Hm, LO, HI, mb["interior"], mb["interior_mu"],
                              mb["initial_x"], mb["initial_mu"], mb["periodic_t"], mb["periodic_mu"])
    path = os.path.join(OUT, "reference_golden_r2.npz")
    np.savez_compressed(path, **g)
    print("wrote", path, os.path.getsize(path), "bytes;", len(g), "arrays")


if __name__ == "__main__":
    main()
