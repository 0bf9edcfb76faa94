// Latency kernel for small point batches (solve loops: the fast phase's
// 12-point X, fine_tune's 1024 + 256 + 256 batches, boundary passes).
//
// The throughput kernels give each CTA a tile of 64-128 points. A batch of a
// few hundred points leaves most of the 148 SMs idle, and every tile still
// walks the whole network serially (~0.3-0.6 ms). Here one CTA of 256 threads owns ONE point and
// spreads each layer over its threads:
//   forward transition l (widths M = M_{l+1}, ranks rl -> rn):
//     (a) thread per neuron k:   A_k = U_k . (s_l o y_l) (+ b_k)   4 slots, K = rl
//                                Z_k = sigma-jet(A_k); A kept in shared memory
//     (b) thread per (slot, j):  y_{l+1,j} = sum_k V_kj Z_k        4 partial sums over k
//   reverse transition l:
//     (a') thread per neuron k:  DZ_k = V_k . (s_{l+1} o T_{l+1});  G_k = VJP(A_k, DZ_k)
//     (b') thread per (slot, j): T_{l,j} = sum_k U_kj G_k;  dL/ds_lj = sum_c T y
// The math (and the per-point term kinds, TermSpec) is the streaming kernel's
// (pinn_kernels.cuh), i.e. the reference's jet ops (model.cpp:85-181) and their
// VJPs (autodiff.cpp:473-666). Output: one [term, dL/ds] row per point,
// reduced per instance in fixed order (reduce_units_kernel): deterministic.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pinn_kernels.cuh"
#include "pinn_v2.cuh"

namespace lrnr_b200 {
namespace small {

constexpr int NT = 256;

struct Geom {
    int64_t n_total;  // points over all instances
    int64_t n_per;    // points per instance
    int aoff[kMaxL];  // A of transition l at 4 * aoff[l] in shared memory
    int a_len;        // sum of hidden widths
    int mmax, rmax;
    int stage;        // 1: each transition's factor block is staged in shared memory (cp.async.bulk,
                      //    two buffers: the next block's copy overlaps the current layer)
    int blk;          // elements of the largest block (multiple of 4)
};

// shared-memory carve-up (elements of T)
__host__ __device__ inline int smem_elems(int rtotal, int a_len, int mmax, int rmax) {
    const int e = 4 * rtotal        // y of every layer: [(soff_l + j) * 4 + c]
                  + 4 * a_len       // pre-activation jets A: [(aoff_l + k) * 4 + c]
                  + 4 * mmax        // Z / G of the current transition: [c * M + k]
                  + 8 * rmax        // S o Y / S o T (sb) and T (tb): [c * r + j]
                  + rtotal + 1 + 8; // [term, dL/ds] of the point (+ u, gu)
    return (e + 7) & ~7;            // staged blocks follow, 32-B aligned
}

template <typename T, int ACT>
__device__ __forceinline__ void act_jet(T a, T& sg, T& d1, T& d2, T& d3) {
    if constexpr (sizeof(T) == 4) {
        v2::act3<ACT, false>(a, sg, d1, d2, d3);
    } else if constexpr (ACT == 0) {
        const T s = tanh(a), e = T(1) - s * s;
        sg = s;
        d1 = e;
        d2 = T(-2) * s * e;
        d3 = T(-2) * e * e + T(4) * s * s * e;
    } else {
        T sn, cs;
        sincos(a, &sn, &cs);
        sg = sn;
        d1 = cs;
        d2 = -sn;
        d3 = -cs;
    }
}

// MODE 0: term + dL/ds rows;  MODE 1: term + output jets (no reverse sweep)
template <typename T, int ACT, int MODE>
__global__ void __launch_bounds__(NT) pinn_small_kernel(const DevNet<T> net, const Geom g,
                                                        const double* __restrict__ pts,
                                                        const double* __restrict__ svec,
                                                        const double* __restrict__ mus, const T w,
                                                        T* __restrict__ part, double* __restrict__ jets_out,
                                                        unsigned long long* __restrict__ bad,
                                                        const TermSpec* __restrict__ spec, const int objective) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* ys = reinterpret_cast<T*>(smem_raw);
    T* as = ys + 4 * net.rtotal;
    T* zb = as + 4 * g.a_len;
    T* sb = zb + 4 * g.mmax;
    T* tb = sb + 4 * g.rmax;
    T* acc = tb + 4 * g.rmax;   // [0] term, [1 + i] dL/ds_i
    T* uu = acc + net.rtotal + 1;  // u[4], gu[4]
    T* wb = reinterpret_cast<T*>(smem_raw) + smem_elems(net.rtotal, g.a_len, g.mmax, g.rmax);  // 2 x blk
    __shared__ __align__(8) uint64_t wbar[2];
    const int tid = threadIdx.x;
    const int L = net.L;
    const int R1 = 1 + net.rtotal;
    if (tid == 0) {
        v2::mbar_init(&wbar[0], 1);
        v2::mbar_init(&wbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // factor-block stages of one point: forward transitions 0..L-2, then (MODE 0)
    // the reverse L-2..0; gq counts stages over the CTA's points (buffer gq & 1)
    const int nst = MODE == 0 ? 2 * (L - 1) : (L - 1);
    auto layer_of = [&](int q) { return q < L - 1 ? q : 2 * (L - 1) - 1 - q; };
    int64_t gq = 0;
    uint32_t wph0 = 0, wph1 = 0;
    auto issue = [&](int q, int64_t qq) {
        if (g.stage && tid == 0 && q < nst) {
            const int l = layer_of(q), b = static_cast<int>(qq & 1);
            const uint32_t bytes = static_cast<uint32_t>(net.M[l + 1]) * net.trow[l] * sizeof(T);
            v2::fence_proxy_async();
            v2::mbar_expect_tx(&wbar[b], bytes);
            v2::bulk_g2s(wb + b * g.blk, net.trans[l], bytes, &wbar[b]);
        }
    };
    // the block of transition l for the current stage (staged copy or global)
    auto acquire = [&](int q) -> const T* {
        const int l = layer_of(q);
        if (!g.stage) return net.trans[l];
        const int b = static_cast<int>(gq & 1);
        if (b == 0) {
            v2::mbar_wait(&wbar[0], wph0);
            wph0 ^= 1u;
        } else {
            v2::mbar_wait(&wbar[1], wph1);
            wph1 ^= 1u;
        }
        issue(q + 1, gq + 1);  // the other buffer: its last readers passed the previous stage's barrier
        ++gq;
        return wb + b * g.blk;
    };

    for (int64_t gp = blockIdx.x; gp < g.n_total; gp += gridDim.x) {
        issue(0, gq);
        const int64_t inst = gp / g.n_per;
        const double* sv = svec + inst * net.rtotal;
        const T x = T(pts[2 * gp]), t = T(pts[2 * gp + 1]);
        // ---- y_0 = V_0^T z_0, z_0 = (x,t),(1,0),(0,1),(0,0) ----
        {
            const int r0 = net.r[0];
            for (int idx = tid; idx < 4 * r0; idx += NT) {
                const int c = idx / r0, j = idx % r0;
                const T z0 = c == 0 ? x : (c == 1 ? T(1) : T(0));
                const T z1 = c == 0 ? t : (c == 2 ? T(1) : T(0));
                ys[(net.soff[0] + j) * 4 + c] = net.V0[j] * z0 + net.V0[r0 + j] * z1;
            }
        }
        __syncthreads();
        // ---- forward transitions ----
        for (int l = 0; l + 1 < L; ++l) {
            const int rl = net.r[l], rn = net.r[l + 1], M = net.M[l + 1], trow = net.trow[l];
            const T* tr = acquire(l);
            for (int idx = tid; idx < 4 * rl; idx += NT) {
                const int c = idx / rl, j = idx % rl;
                sb[idx] = T(sv[net.soff[l] + j]) * ys[(net.soff[l] + j) * 4 + c];
            }
            __syncthreads();
            for (int k = tid; k < M; k += NT) {
                const T* row = tr + static_cast<int64_t>(k) * trow;
                T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
                for (int j = 0; j < rl; ++j) {
                    const T u = row[j];
                    a0 = fma(u, sb[j], a0);
                    a1 = fma(u, sb[rl + j], a1);
                    a2 = fma(u, sb[2 * rl + j], a2);
                    a3 = fma(u, sb[3 * rl + j], a3);
                }
                a0 += row[rl + rn];
                T* ak = as + (g.aoff[l] + k) * 4;
                ak[0] = a0;
                ak[1] = a1;
                ak[2] = a2;
                ak[3] = a3;
                T sg, d1, d2, d3;
                act_jet<T, ACT>(a0, sg, d1, d2, d3);
                zb[k] = sg;
                zb[M + k] = d1 * a1;
                zb[2 * M + k] = d1 * a2;
                zb[3 * M + k] = d2 * a1 * a1 + d1 * a3;
            }
            __syncthreads();
            for (int idx = tid; idx < 4 * rn; idx += NT) {
                const int c = idx / rn, j = idx % rn;
                const T* v = tr + rl + j;
                const T* z = zb + c * M;
                T p0 = T(0), p1 = T(0), p2 = T(0), p3 = T(0);
                int k = 0;
                for (; k + 3 < M; k += 4) {
                    p0 = fma(v[static_cast<int64_t>(k) * trow], z[k], p0);
                    p1 = fma(v[static_cast<int64_t>(k + 1) * trow], z[k + 1], p1);
                    p2 = fma(v[static_cast<int64_t>(k + 2) * trow], z[k + 2], p2);
                    p3 = fma(v[static_cast<int64_t>(k + 3) * trow], z[k + 3], p3);
                }
                for (; k < M; ++k) p0 = fma(v[static_cast<int64_t>(k) * trow], z[k], p0);
                ys[(net.soff[l + 1] + j) * 4 + c] = (p0 + p1) + (p2 + p3);
            }
            __syncthreads();
        }
        // ---- output layer (M_L = 1) + per-point term ----
        const int rL = net.r[L - 1];
        const double* sL = sv + net.soff[L - 1];
        if (tid < 4) {
            T u = T(0);
            for (int j = 0; j < rL; ++j) u = fma(net.ulast[j] * T(sL[j]), ys[(net.soff[L - 1] + j) * 4 + tid], u);
            if (tid == 0) u += net.ulast[rL];
            uu[tid] = u;
        }
        __syncthreads();
        if (tid == 0) {
            const T mu0 = T(mus[3 * inst]), mu1 = T(mus[3 * inst + 1]), mu2 = T(mus[3 * inst + 2]);
            const T u0 = uu[0];
            const T N = uu[2] + mu0 * uu[1] - mu1 * uu[3] - mu2 * u0 * (T(1) - u0);
            int kind = objective;
            T tw = w, sw = w, tgt = T(0);
            if (spec != nullptr) {
                const TermSpec sp = spec[gp];
                kind = sp.kind;
                tgt = T(sp.target);
                tw = T(sp.w_term);
                sw = T(sp.w_seed);
            }
            const T d = u0 - tgt;
            const T term = kind == 0 ? tw * (N * N) : (kind == 1 ? tw * fabs(N) : (kind == 2 ? tw * (d * d) : tw * fabs(d)));
            if (!isfinite(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
            acc[0] = term;
            if (kind <= 1) {
                const T gN = kind == 0 ? T(2) * N * sw : sgn0(N) * sw;
                uu[4] = gN * (-mu2 * (T(1) - T(2) * u0));
                uu[5] = gN * mu0;
                uu[6] = gN;
                uu[7] = -gN * mu1;
            } else {
                uu[4] = kind == 2 ? T(2) * d * sw : sgn0(d) * sw;
                uu[5] = uu[6] = uu[7] = T(0);
            }
        }
        if constexpr (MODE == 1) {
            if (tid < 4 && jets_out != nullptr) jets_out[gp * 4 + tid] = double(uu[tid]);
            __syncthreads();
            for (int k = tid; k < R1; k += NT) part[gp * R1 + k] = k == 0 ? acc[0] : T(0);
            __syncthreads();
            continue;
        } else {
            __syncthreads();
            // output layer reverse: t_j = u_j gu, dL/ds_{L-1} = sum_c t y, S o T
            for (int j = tid; j < rL; j += NT) {
                const T uj = net.ulast[j], sj = T(sL[j]);
                T cd = T(0);
                for (int c = 0; c < 4; ++c) {
                    const T tj = uj * uu[4 + c];
                    cd = fma(tj, ys[(net.soff[L - 1] + j) * 4 + c], cd);
                    sb[c * rL + j] = sj * tj;
                }
                acc[1 + net.soff[L - 1] + j] = cd;
            }
            __syncthreads();
            for (int l = L - 2; l >= 0; --l) {
                const int rl = net.r[l], rn = net.r[l + 1], M = net.M[l + 1], trow = net.trow[l];
                const T* tr = acquire(2 * (L - 1) - 1 - l);
                for (int k = tid; k < M; k += NT) {
                    const T* row = tr + static_cast<int64_t>(k) * trow;
                    T g0 = T(0), g1 = T(0), g2 = T(0), g3 = T(0);
                    for (int j = 0; j < rn; ++j) {
                        const T v = row[rl + j];
                        g0 = fma(v, sb[j], g0);
                        g1 = fma(v, sb[rn + j], g1);
                        g2 = fma(v, sb[2 * rn + j], g2);
                        g3 = fma(v, sb[3 * rn + j], g3);
                    }
                    const T* ak = as + (g.aoff[l] + k) * 4;
                    const T av = ak[0], ax = ak[1], at = ak[2], aw = ak[3];
                    T sg, d1, d2, d3;
                    act_jet<T, ACT>(av, sg, d1, d2, d3);
                    zb[k] = g0 * d1 + g1 * d2 * ax + g2 * d2 * at + g3 * (d3 * ax * ax + d2 * aw);
                    zb[M + k] = g1 * d1 + g3 * T(2) * d2 * ax;
                    zb[2 * M + k] = g2 * d1;
                    zb[3 * M + k] = g3 * d1;
                }
                __syncthreads();
                for (int idx = tid; idx < 4 * rl; idx += NT) {
                    const int c = idx / rl, j = idx % rl;
                    const T* uc = tr + j;
                    const T* gz = zb + c * M;
                    T p0 = T(0), p1 = T(0), p2 = T(0), p3 = T(0);
                    int k = 0;
                    for (; k + 3 < M; k += 4) {
                        p0 = fma(uc[static_cast<int64_t>(k) * trow], gz[k], p0);
                        p1 = fma(uc[static_cast<int64_t>(k + 1) * trow], gz[k + 1], p1);
                        p2 = fma(uc[static_cast<int64_t>(k + 2) * trow], gz[k + 2], p2);
                        p3 = fma(uc[static_cast<int64_t>(k + 3) * trow], gz[k + 3], p3);
                    }
                    for (; k < M; ++k) p0 = fma(uc[static_cast<int64_t>(k) * trow], gz[k], p0);
                    tb[idx] = (p0 + p1) + (p2 + p3);
                }
                __syncthreads();
                for (int j = tid; j < rl; j += NT) {
                    const T sj = T(sv[net.soff[l] + j]);
                    T cd = T(0);
                    for (int c = 0; c < 4; ++c) {
                        const T tn = tb[c * rl + j];
                        cd = fma(tn, ys[(net.soff[l] + j) * 4 + c], cd);
                        sb[c * rl + j] = sj * tn;
                    }
                    acc[1 + net.soff[l] + j] = cd;
                }
                __syncthreads();
            }
            for (int k = tid; k < R1; k += NT) part[gp * R1 + k] = acc[k];
            __syncthreads();
        }
    }
}

}  // namespace small
}  // namespace lrnr_b200
