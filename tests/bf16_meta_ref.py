"""TEST INFRASTRUCTURE: numpy reference of the meta gradient with the meta
tensor-core kernel's numerics (pinn_meta_tc.cuh): every tensor-core operand
rounded to bf16 (RNE; or tf32 RNA for comparison), FP32 values elsewhere, the
reference's jet / VJP algebra (autodiff.cpp:473-563, 644-666, 720-730) in
float64 arithmetic.  Two uses: the GPU parity test compares the BF16 kernel
with it (same roundings, so only accumulation order differs), and running it
as a script reports the precision of each operand format against FP64 (the
design study that chose BF16 for config 4: python tests/bf16_meta_ref.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_04001_b200 as pkg  # noqa: E402


def rnd(x, fmt, kind="a"):
    if fmt == "f64" or (fmt == "bf16w" and kind == "a") or (fmt == "bf16a" and kind == "w"):
        return x
    if fmt in ("bf16w", "bf16a"):
        fmt = "bf16"
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    if fmt == "bf16":
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    elif fmt == "tf32":
        u = (u + 0x1000) & 0xFFFFE000
    elif fmt == "f32":
        pass
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def f32(x, fmt):
    return x if fmt == "f64" else np.asarray(x, np.float32).astype(np.float64)


def act3(a, act):
    """sigma and its first three derivatives (tanh: model.hpp:28-33; sin extension)."""
    if act == pkg.ACT_SIN:
        sg, c = np.sin(a), np.cos(a)
        return sg, c, -sg, -c
    sg = np.tanh(a)
    e = 1 - sg * sg
    return sg, e, -2 * sg * e, -2 * e * e + 4 * sg * sg * e


def meta_grad(m, s, mu, pts, fmt, act=pkg.ACT_SIN):
    W, R = [int(v) for v in m.widths], [int(v) for v in m.ranks]
    L = len(R)
    offs, _ = m.offsets()
    U = [m.params[o[0]:o[0] + W[l + 1] * R[l]].reshape(W[l + 1], R[l]) for l, o in enumerate(offs)]
    V = [m.params[o[1]:o[1] + W[l] * R[l]].reshape(W[l], R[l]) for l, o in enumerate(offs)]
    b = [m.params[o[2]:o[2] + W[l + 1]] for l, o in enumerate(offs)]
    so = np.cumsum([0] + R)
    sl = [s[so[l]:so[l + 1]] for l in range(L)]
    P = len(pts)
    z = np.zeros((P, 4, 2))
    z[:, 0, :] = pts
    z[:, 1, 0] = 1
    z[:, 2, 1] = 1
    ys, As, zs = [], [], [z]
    y = f32(z @ V[0], fmt)  # input layer on CUDA cores
    for l in range(L):
        ys.append(y)
        sy = f32(sl[l] * y, fmt)
        if l == L - 1:
            a = sy @ U[l].T
            a[:, 0] += b[l]
            u = f32(a[:, :, 0], fmt)
            break
        a = f32(rnd(sy, fmt) @ rnd(U[l], fmt, "w").T, fmt)
        a[:, 0] += b[l]
        a = f32(a, fmt)
        As.append(a)
        sg, d1, d2, _ = act3(a[:, 0], act)
        zn = np.empty_like(a)
        zn[:, 0] = sg
        zn[:, 1] = d1 * a[:, 1]
        zn[:, 2] = d1 * a[:, 2]
        zn[:, 3] = d2 * a[:, 1] ** 2 + d1 * a[:, 3]
        zn = f32(zn, fmt)
        zs.append(zn)
        y = f32(rnd(zn, fmt) @ rnd(V[l + 1], fmt, "w"), fmt)
    mu0, mu1, mu2 = mu
    N = u[:, 2] + mu0 * u[:, 1] - mu1 * u[:, 3] - mu2 * u[:, 0] * (1 - u[:, 0])
    w = 1.0 / P
    loss = w * np.sum(N * N)
    gN = 2 * N * w
    gu = np.stack([gN * (-mu2 * (1 - 2 * u[:, 0])), gN * mu0, gN, -gN * mu1], 1)  # (P,4)
    dU = [None] * L
    dV = [None] * L
    db = [None] * L
    ds = [None] * L
    # output layer
    g = gu[:, :, None]  # (P,4,1) = dL/da_L
    t = g @ U[L - 1]  # (P,4,r)
    dU[L - 1] = np.einsum("pci,pcj->ij", g, sl[L - 1] * ys[L - 1])
    db[L - 1] = g[:, 0].sum(0)
    ds[L - 1] = np.einsum("pcj,pcj->j", t, ys[L - 1])
    st = f32(sl[L - 1] * t, fmt)
    for l in range(L - 2, -1, -1):
        # transition l: neurons of hidden layer l+1
        dz = f32(rnd(st, fmt) @ rnd(V[l + 1], fmt, "w").T, fmt)  # (P,4,M)
        dV[l + 1] = np.einsum("pci,pcj->ij", rnd(zs[l + 1], fmt), rnd(st, fmt))
        a = As[l]
        sg, d1, d2, d3 = act3(a[:, 0], act)
        ax, at, aw = a[:, 1], a[:, 2], a[:, 3]
        g0, g1, g2, g3 = dz[:, 0], dz[:, 1], dz[:, 2], dz[:, 3]
        gg = np.stack([g0 * d1 + g1 * d2 * ax + g2 * d2 * at + g3 * (d3 * ax * ax + d2 * aw),
                       g1 * d1 + g3 * 2 * d2 * ax, g2 * d1, g3 * d1], 1)
        gg = f32(gg, fmt)
        t = f32(rnd(gg, fmt) @ rnd(U[l], fmt, "w"), fmt)
        sy = f32(sl[l] * ys[l], fmt)
        dU[l] = np.einsum("pci,pcj->ij", rnd(gg, fmt), rnd(sy, fmt))
        db[l] = gg[:, 0].sum(0)
        ds[l] = np.einsum("pcj,pcj->j", t, ys[l])
        st = f32(sl[l] * t, fmt)
    # input layer dV_0 = z0^T st
    dV[0] = np.einsum("pci,pcj->ij", zs[0], st)
    grad = np.concatenate([np.concatenate([dU[l].ravel(), dV[l].ravel(), db[l].ravel()]) for l in range(L)])
    return loss, np.concatenate(ds), grad


if __name__ == "__main__":
    per = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    c = pkg.config4(n_inst=2, pts_per_inst=per)
    m = c["model"]
    rng = np.random.default_rng(0)
    s = np.sort(rng.uniform(0, 1, int(np.sum(m.ranks))))[::-1].copy()
    for i in range(2):
        mu = c["mus"][i]
        pts = c["pts"][i * per:(i + 1) * per]
        ref = meta_grad(m, s, mu, pts, "f64")
        for fmt in ("f32", "tf32", "bf16"):
            got = meta_grad(m, s, mu, pts, fmt)
            nrm = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
            cos = lambda a, b: a @ b / np.linalg.norm(a) / np.linalg.norm(b)
            print(f"inst {i} mu={np.round(mu, 3)} {fmt:5s} loss rel {abs(got[0] - ref[0]) / ref[0]:.2e} "
                  f"ds norm {nrm(got[1], ref[1]):.2e} grad norm {nrm(got[2], ref[2]):.2e} cos {cos(got[2], ref[2]):.7f}")
