// Persistent fast-phase solver: the whole fast_solve loop (training.cpp:498-607)
// in ONE CTA and ONE launch, for FastLRNR networks whose widths and ranks fit a
// warp (r_hat_l <= 32, r_l <= 32 -- the EIM budget of BASELINE configs 1 and 2).
//
// The fast phase evaluates 12 sampling points per epoch for hundreds of epochs.
// Batch kernels are pure latency there: launches, grid-wide reductions, and ~30
// block barriers per point and pass. Here:
//   * one warp per loss term: an interior point, an initial point, or one side
//     of a periodic pair (the two sides exchange u through shared memory under
//     a 64-thread named barrier);
//   * inside a warp, lane = neuron k (affine + activation jet / VJP) or lane =
//     rank j (the V^T / U^T contractions); operands move by __shfl_sync, so a
//     transition needs no block barrier;
//   * every transition's factor block sits in shared memory for all epochs;
//   * per epoch the CTA reduces the per-warp [term, dL/ds] rows in warp order
//     (deterministic), adds lambda ||s - s_init||_1, applies the stop rules, the
//     best iterate, adam_step (autodiff.cpp:1062-1075) and the projection
//     (autodiff.cpp:967-977), and starts the next epoch -- no host involvement.
// The math per term is the streaming / small kernels' (TermSpec kinds 1 and 3,
// the Abs VJP sgn(.), 0 at 0).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include "pinn_kernels.cuh"
#include "pinn_small.cuh"

namespace lrnr_b200 {
namespace solve {

struct Problem {
    int n_int, n_ic, n_bc;  // interior points, initial points, periodic pairs
    int n_warps;            // n_int + n_ic + 2 n_bc
    // cluster layout: global warp gw = cluster rank * wpc + warp; terms at gw < n_int + n_ic,
    // periodic pairs at pair_base + 2 j (pair_base even, wpc even: a pair never straddles CTAs)
    int wpc, pair_base, n_gw;
    int yoff[kMaxL + 1];    // per-warp state: y_l at 4 * yoff[l], A_l at 4 * (ylen + aoff[l])
    int aoff[kMaxL];
    int ylen, alen;
    int wlen;               // factor blocks (elements), copied once
    int woff[kMaxL];        // transition l's block in shared memory
    int wrow[kMaxL];        // its row stride there: trow_l rounded up to odd (lane k reads row k:
                            // an odd stride spreads the 32 rows over all 32 banks)
    double lr, lambda_local;
    int64_t epochs;
};

struct State {
    double best_loss;
    double initial;
    int64_t epoch, best_epoch, t;
    int stopped, flags;
};

// smem (bytes): T weights + T per-warp state + double s, s0, m, v, best, per-warp ds rows, terms
__host__ inline size_t smem_bytes(const Problem& p, int rtotal, size_t elem) {
    return elem * (static_cast<size_t>(p.wlen) + 8 + static_cast<size_t>(p.wpc) * (4 * (p.ylen + p.alen) + 128)) +
           8 * (5 * static_cast<size_t>(rtotal) + static_cast<size_t>(p.wpc) * (rtotal + 1) + 64 + 33);
}

template <typename T>
__device__ __forceinline__ T wshfl(T v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}

template <typename T, int ACT>
__global__ void __launch_bounds__(512, 1)
fast_solve_kernel(const DevNet<T> net, const Problem pb, const double* __restrict__ terms,
                  const double* __restrict__ mu, const double* __restrict__ s_init, const double* __restrict__ bt,
                  double* __restrict__ best_out, double* __restrict__ losses, State* __restrict__ st_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int L = net.L, G = net.rtotal;
    // ---- shared-memory carve-up ----
    double* s = reinterpret_cast<double*>(smem_raw);
    double* s0 = s + G;
    double* am = s0 + G;
    double* av = am + G;
    double* best = av + G;
    double* rows = best + G;                         // [warp][term, ds (G)]
    double* misc = rows + pb.wpc * (G + 1);          // u exchange (32) + reduction scratch
    double* pair_u = misc;                           // [warp] value of u
    double* terms_s = misc + 32;                     // 32 (x / t / target per warp)
    // factor blocks, V0, per-warp state: 16-B aligned (vector loads)
    T* wsm = reinterpret_cast<T*>(terms_s + 32 + ((5 * G + pb.wpc * (G + 1)) & 1));
    T* v0s = wsm + pb.wlen;
    T* states = v0s + 8;                              // [warp][4 (ylen + alen) + 128]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nthr = blockDim.x;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = static_cast<int>(cluster.block_rank()), csize = static_cast<int>(cluster.num_blocks());
    const int gw = crank * pb.wpc + warp;  // global warp: this warp's term
    // ---- one-time staging: factor blocks, V_0, u_last; s, s0 ----
    for (int l = 0; l + 1 < L; ++l) {
        const int trow = net.trow[l], wr = pb.wrow[l];
        const int n = net.M[l + 1] * trow;
        for (int i = tid; i < n; i += nthr) wsm[pb.woff[l] + (i / trow) * wr + (i % trow)] = net.trans[l][i];
    }
    for (int i = tid; i < 2 * net.r[0] && i < 8; i += nthr) v0s[i] = net.V0[i];
    for (int i = tid; i < G; i += nthr) {
        s[i] = s_init[i];
        s0[i] = s_init[i];
        best[i] = s_init[i];
        am[i] = 0.0;
        av[i] = 0.0;
    }
    for (int i = tid; i < pb.wpc * (G + 1); i += nthr) rows[i] = 0.0;  // idle warps keep zero rows
    __shared__ State st;
    __shared__ int go, copy;
    if (tid == 0) {
        st.best_loss = __longlong_as_double(0x7ff0000000000000LL);  // +inf
        st.initial = 0.0;
        st.epoch = st.best_epoch = st.t = 0;
        st.stopped = st.flags = 0;
    }
    __syncthreads();
    const T mu0 = T(mu[0]), mu1 = T(mu[1]), mu2 = T(mu[2]);

    // ---- this warp's term ----
    const bool is_pair = gw >= pb.pair_base && gw < pb.pair_base + 2 * pb.n_bc;
    const bool active = gw < pb.n_int + pb.n_ic || is_pair;
    int kind = 0;       // 0 interior |N|, 1 initial |u - sin x|, 2 periodic side 0, 3 periodic side 1
    T px = T(0), pt = T(0);
    double tgt = 0.0;
    if (active) {
        if (gw < pb.n_int) {
            px = T(terms[2 * gw]);
            pt = T(terms[2 * gw + 1]);
        } else if (gw < pb.n_int + pb.n_ic) {
            kind = 1;
            const int i = gw - pb.n_int;
            px = T(terms[2 * pb.n_int + i]);
            tgt = sin(terms[2 * pb.n_int + i]);
        } else {
            const int j = gw - pb.pair_base;
            kind = 2 + (j & 1);
            px = (j & 1) ? T(6.283185307179586476925286766559) : T(0);
            pt = T(terms[2 * pb.n_int + pb.n_ic + (j >> 1)]);
        }
    }
    T* ys = states + static_cast<int64_t>(warp) * (4 * (pb.ylen + pb.alen) + 128);
    T* as = ys + 4 * pb.ylen;
    T* vb = as + 4 * pb.alen;  // 32 x 4: the operand a lane loop broadcasts (LDS.128, no shuffles)
    const T* ulast = net.ulast;

    for (int64_t ep = 0; ep < pb.epochs; ++ep) {
        if (st.stopped) break;  // uniform: written by thread 0 before the last barrier
        T term = T(0);
        if (active) {
            // ---------------- forward: lane j = rank, lane k = neuron ----------------
            {
                const int r0 = net.r[0];
                if (lane < r0) {
                    const T v0 = v0s[lane], v1 = v0s[r0 + lane];
                    ys[(pb.yoff[0] + lane) * 4 + 0] = v0 * px + v1 * pt;
                    ys[(pb.yoff[0] + lane) * 4 + 1] = v0;
                    ys[(pb.yoff[0] + lane) * 4 + 2] = v1;
                    ys[(pb.yoff[0] + lane) * 4 + 3] = T(0);
                }
            }
            __syncwarp();
            for (int l = 0; l + 1 < L; ++l) {
                const int rl = net.r[l], rn = net.r[l + 1], M = net.M[l + 1], trow = pb.wrow[l];
                const T* tr = wsm + pb.woff[l];
                // sy (lane j): s_l o y_l
                T sy0 = T(0), sy1 = T(0), sy2 = T(0), sy3 = T(0);
                if (lane < rl) {
                    const T sj = T(s[net.soff[l] + lane]);
                    const T* y = ys + (pb.yoff[l] + lane) * 4;
                    sy0 = sj * y[0];
                    sy1 = sj * y[1];
                    sy2 = sj * y[2];
                    sy3 = sj * y[3];
                }
                if (lane < rl) v2::st4(vb + lane * 4, sy0, sy1, sy2, sy3);
                __syncwarp();
                // A (lane k)
                T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
                const T* row = tr + (lane < M ? lane : 0) * trow;
#pragma unroll 8
                for (int j = 0; j < rl; ++j) {
                    const T u = row[j];
                    T b4[4];
                    v2::ld4(vb + j * 4, b4);
                    a0 = fma(u, b4[0], a0);
                    a1 = fma(u, b4[1], a1);
                    a2 = fma(u, b4[2], a2);
                    a3 = fma(u, b4[3], a3);
                }
                __syncwarp();
                T z0 = T(0), z1 = T(0), z2 = T(0), z3 = T(0);
                if (lane < M) {
                    a0 += row[rl + rn];
                    T* ak = as + (pb.aoff[l] + lane) * 4;
                    ak[0] = a0;
                    ak[1] = a1;
                    ak[2] = a2;
                    ak[3] = a3;
                    T sg, d1, d2, d3;
                    small::act_jet<T, ACT>(a0, sg, d1, d2, d3);
                    z0 = sg;
                    z1 = d1 * a1;
                    z2 = d1 * a2;
                    z3 = d2 * a1 * a1 + d1 * a3;
                }
                if (lane < M) v2::st4(vb + lane * 4, z0, z1, z2, z3);
                __syncwarp();
                // y_{l+1} (lane j) = sum_k V[k][j] z_k
                T y0 = T(0), y1 = T(0), y2 = T(0), y3 = T(0);
                const int jj = lane < rn ? lane : 0;
#pragma unroll 8
                for (int k = 0; k < M; ++k) {
                    const T v = tr[k * trow + rl + jj];
                    T b4[4];
                    v2::ld4(vb + k * 4, b4);
                    y0 = fma(v, b4[0], y0);
                    y1 = fma(v, b4[1], y1);
                    y2 = fma(v, b4[2], y2);
                    y3 = fma(v, b4[3], y3);
                }
                __syncwarp();
                if (lane < rn) {
                    T* y = ys + (pb.yoff[l + 1] + lane) * 4;
                    y[0] = y0;
                    y[1] = y1;
                    y[2] = y2;
                    y[3] = y3;
                }
                __syncwarp();
            }
            // output jet u = u_last . (s o y_{L-1}) (+ b), warp reduction over ranks
            const int rL = net.r[L - 1];
            T u0 = T(0), u1 = T(0), u2 = T(0), u3 = T(0);
            if (lane < rL) {
                const T c = ulast[lane] * T(s[net.soff[L - 1] + lane]);
                const T* y = ys + (pb.yoff[L - 1] + lane) * 4;
                u0 = c * y[0];
                u1 = c * y[1];
                u2 = c * y[2];
                u3 = c * y[3];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                u0 += __shfl_xor_sync(0xffffffffu, u0, o);
                u1 += __shfl_xor_sync(0xffffffffu, u1, o);
                u2 += __shfl_xor_sync(0xffffffffu, u2, o);
                u3 += __shfl_xor_sync(0xffffffffu, u3, o);
            }
            u0 += ulast[rL];
            // ---------------- term and seed ----------------
            T g0 = T(0), g1 = T(0), g2 = T(0), g3 = T(0);
            if (kind == 0) {
                const T N = u2 + mu0 * u1 - mu1 * u3 - mu2 * u0 * (T(1) - u0);
                term = fabs(N);
                const T gN = sgn0(N);
                g0 = gN * (-mu2 * (T(1) - T(2) * u0));
                g1 = gN * mu0;
                g2 = gN;
                g3 = -gN * mu1;
            } else if (kind == 1) {
                const T d = u0 - T(tgt);
                term = fabs(d);
                g0 = sgn0(d);
            } else {
                if (lane == 0) pair_u[warp] = double(u0);
                // the two sides of a pair: local warps (w, w + 1), w even
                asm volatile("bar.sync %0, 64;" ::"r"(1 + ((gw - pb.pair_base) >> 1) % 15) : "memory");
                const double other = pair_u[kind == 2 ? warp + 1 : warp - 1];
                const T d = kind == 2 ? u0 - T(other) : T(other) - u0;  // u(0,t) - u(2pi,t)
                if (kind == 2) term = fabs(d);
                g0 = kind == 2 ? sgn0(d) : -sgn0(d);
            }
            // ---------------- reverse ----------------
            double* drow = rows + warp * (G + 1);
            T st0 = T(0), st1 = T(0), st2 = T(0), st3 = T(0);  // lane j: s o T for the next transition
            if (lane < rL) {
                const T uj = ulast[lane], sj = T(s[net.soff[L - 1] + lane]);
                const T* y = ys + (pb.yoff[L - 1] + lane) * 4;
                const T t0 = uj * g0, t1 = uj * g1, t2 = uj * g2, t3 = uj * g3;
                drow[1 + net.soff[L - 1] + lane] = double(t0 * y[0] + t1 * y[1] + t2 * y[2] + t3 * y[3]);
                st0 = sj * t0;
                st1 = sj * t1;
                st2 = sj * t2;
                st3 = sj * t3;
            }
            for (int l = L - 2; l >= 0; --l) {
                const int rl = net.r[l], rn = net.r[l + 1], M = net.M[l + 1], trow = pb.wrow[l];
                const T* tr = wsm + pb.woff[l];
                const T* row = tr + (lane < M ? lane : 0) * trow;
                if (lane < rn) v2::st4(vb + lane * 4, st0, st1, st2, st3);
                __syncwarp();
                T d0 = T(0), d1v = T(0), d2v = T(0), d3v = T(0);
#pragma unroll 8
                for (int j = 0; j < rn; ++j) {
                    const T v = row[rl + j];
                    T b4[4];
                    v2::ld4(vb + j * 4, b4);
                    d0 = fma(v, b4[0], d0);
                    d1v = fma(v, b4[1], d1v);
                    d2v = fma(v, b4[2], d2v);
                    d3v = fma(v, b4[3], d3v);
                }
                __syncwarp();
                T ga0 = T(0), ga1 = T(0), ga2 = T(0), ga3 = T(0);
                if (lane < M) {
                    const T* ak = as + (pb.aoff[l] + lane) * 4;
                    const T a0 = ak[0], ax = ak[1], at = ak[2], aw = ak[3];
                    T sg, e1, e2, e3;
                    small::act_jet<T, ACT>(a0, sg, e1, e2, e3);
                    ga0 = d0 * e1 + d1v * e2 * ax + d2v * e2 * at + d3v * (e3 * ax * ax + e2 * aw);
                    ga1 = d1v * e1 + d3v * T(2) * e2 * ax;
                    ga2 = d2v * e1;
                    ga3 = d3v * e1;
                }
                if (lane < M) v2::st4(vb + lane * 4, ga0, ga1, ga2, ga3);
                __syncwarp();
                // T_l (lane j) = sum_k U[k][j] ga_k
                T t0 = T(0), t1 = T(0), t2 = T(0), t3 = T(0);
                const int jl = lane < rl ? lane : 0;
#pragma unroll 8
                for (int k = 0; k < M; ++k) {
                    const T uu = tr[k * trow + jl];
                    T b4[4];
                    v2::ld4(vb + k * 4, b4);
                    t0 = fma(uu, b4[0], t0);
                    t1 = fma(uu, b4[1], t1);
                    t2 = fma(uu, b4[2], t2);
                    t3 = fma(uu, b4[3], t3);
                }
                __syncwarp();
                st0 = st1 = st2 = st3 = T(0);
                if (lane < rl) {
                    const T* y = ys + (pb.yoff[l] + lane) * 4;
                    drow[1 + net.soff[l] + lane] = double(t0 * y[0] + t1 * y[1] + t2 * y[2] + t3 * y[3]);
                    const T sj = T(s[net.soff[l] + lane]);
                    st0 = sj * t0;
                    st1 = sj * t1;
                    st2 = sj * t2;
                    st3 = sj * t3;
                }
            }
            if (lane == 0) drow[0] = double(term);
        }
        cluster.sync();  // every CTA's rows are complete
        // ---------------- step: rank 0 reduces all CTAs' rows (DSMEM) in global warp order ----------------
        if (crank == 0) {
            if (warp == 0) {
                // loss = sum of the warp terms + lambda ||s - s0||_1: lane-strided partials, then a
                // fixed xor tree (deterministic)
                double value = 0.0;
                for (int g2 = lane; g2 < csize * pb.wpc; g2 += 32) {
                    const double* rr = cluster.map_shared_rank(rows, g2 / pb.wpc);
                    value += rr[(g2 % pb.wpc) * (G + 1)];
                }
                double local = 0.0;
                if (pb.lambda_local > 0.0)
                    for (int i = lane; i < G; i += 32) local += fabs(s[i] - s0[i]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    value += __shfl_xor_sync(0xffffffffu, value, o);
                    local += __shfl_xor_sync(0xffffffffu, local, o);
                }
                if (lane == 0) misc[63] = value + pb.lambda_local * local;
                __syncwarp();
            }
            __syncthreads();
            if (tid == 0) {
                go = 0;
                copy = 0;
                const int64_t e = ++st.epoch;
                const double value = misc[63];
                if (!isfinite(value)) {
                    st.flags |= 3;
                    st.stopped = 1;
                } else {
                    losses[e - 1] = value;
                    if (e == 1) st.initial = value;
                    if (value > 1e3 * st.initial) {
                        st.flags |= 2;
                        st.stopped = 1;
                    } else {
                        if (value < st.best_loss) {
                            st.best_loss = value;
                            st.best_epoch = e;
                            copy = 1;
                        }
                        ++st.t;
                        go = 1;
                    }
                }
            }
            __syncthreads();
            if (go) {
                const double b1t = bt[2 * (st.t - 1)], b2t = bt[2 * (st.t - 1) + 1];
                for (int i = tid; i < G; i += nthr) {
                    const double si = s[i];
                    if (copy) best[i] = si;
                    double g = 0.0;
                    for (int r = 0; r < csize; ++r) {
                        const double* rr = cluster.map_shared_rank(rows, r);
                        for (int w = 0; w < pb.wpc; ++w) g += rr[w * (G + 1) + 1 + i];
                    }
                    if (pb.lambda_local > 0.0) {
                        const double d = si - s0[i];
                        g += pb.lambda_local * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0));
                    }
                    const double mi = 0.9 * am[i] + (1.0 - 0.9) * g;
                    const double vi = 0.999 * av[i] + (1.0 - 0.999) * g * g;
                    am[i] = mi;
                    av[i] = vi;
                    const double x = si - pb.lr * (mi / b1t) / (sqrt(vi / b2t) + 1e-8);
                    s[i] = x < 0.0 ? 0.0 : x;
                }
            }
        }
        cluster.sync();  // rank 0's step is complete
        if (crank != 0) {  // pull the new s and the stop flag
            const double* s_r0 = cluster.map_shared_rank(s, 0);
            for (int i = tid; i < G; i += nthr) s[i] = s_r0[i];
            if (tid == 0) st.stopped = cluster.map_shared_rank(&st, 0)->stopped;
        }
        __syncthreads();
    }
    cluster.sync();  // no CTA exits while others may still read its shared memory
    if (crank != 0) return;
    for (int i = tid; i < G; i += nthr) best_out[i] = best[i];
    if (tid == 0) *st_out = st;
}

}  // namespace solve
}  // namespace lrnr_b200
