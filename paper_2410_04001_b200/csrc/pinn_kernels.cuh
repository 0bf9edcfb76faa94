// Fused LRNR / FastLRNR residual + reverse-to-s kernels for sm_100a.
//
// One thread group of TPP lanes owns one collocation point; lane q of the
// group owns jet slots [q*SPT, (q+1)*SPT) of (u, u_x, u_t, u_xx) (SPT = 4/TPP).
// The network is swept neuron by neuron ("streaming"): for a transition
// through the M_{l+1} hidden neurons of layer l,
//     a_k   = U_l[k,:] . (s_l (.) y_l) + b_l[k]          (jet_affine_factored, model.cpp:85-122)
//     z_k   = sigma-jet(a_k)                             (jet_activation,      model.cpp:170-181)
//     y_{l+1} += V_{l+1}[k,:] z_k
// so the M-wide activations never exist anywhere: only the rank-r vectors y_l
// (4 r_l values per point per layer) are kept, in an L2-resident per-CTA
// scratch, for the reverse sweep.  The reverse sweep recomputes a_k from y_l
// (one extra rank-r dot product per neuron, +25% FMAs, not counted as
// algorithmic work) and streams the same rows again:
//     dz_k  = V_{l+1}[k,:] . (s_{l+1} (.) t_{l+1})       (AffineFactoredJet VJP, autodiff.cpp:540-552)
//     g_k   = sigma-jet VJP(a_k, dz_k)                   (ActivationJet VJP,     autodiff.cpp:644-666)
//     t_l  += U_l[k,:]^T g_k                             (autodiff.cpp:491-500)
//     dL/ds_l[j] = sum_slots t_l[j] y_l[j]               (autodiff.cpp:506-513)
// Matrix rows are read with warp-uniform addresses (one L1 transaction feeds
// every lane), the 4 jet slots share each matrix element.
//
// FastLRNR is the same network with hidden widths rhat_l and (U_l, V_{l+1},
// b_l) -> (u_hat_l, v_hat_l, b_hat_l), V_0 -> v_in, U_{L-1} -> u_out
// (emit_fast_jet, autodiff.cpp:905-922): the ScaleJet VJP (autodiff.cpp:624-643)
// equals the factored-affine coefficient gradient, so one kernel serves both.
//
// Per-point loss terms, dL/ds partials and the loss are reduced
// deterministically: warp shuffle tree -> per-warp smem rows -> per-unit (a
// fixed contiguous range of tiles of one PDE instance) smem accumulator ->
// global unit partial -> fixed-order double reduction per instance.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lrnr_b200 {

constexpr int kMaxL = 32;
constexpr int kThreads = 128;  // threads per CTA (4 warps)

template <typename T>
struct DevNet {
    int L;
    int M[kMaxL + 1];     // widths (M[0] = 2, M[L] = 1)
    int r[kMaxL];         // ranks
    int soff[kMaxL + 1];  // offsets of s_l in the coefficient vector; soff[L] = r_total
    int trow[kMaxL];      // row stride of transition l: [U_l row | V_{l+1} row | b_l[k] | pad]
    const T* V0;          // 2 x r[0]
    const T* trans[kMaxL];
    const T* ulast;       // U_{L-1} row 0 (r[L-1]) then b_{L-1}[0]
    int rtotal;
};

// One loss term per point: kind 0 = w N^2, 1 = w |N| (interior, N = CDR
// residual), 2 = w (u - target)^2, 3 = w |u - target| (value terms: initial
// u(x,0) - sin x, periodic u(0,t) - u(2pi,t) with the partner's u as target).
// w_term scales the term's value, w_seed its gradient; a periodic pair puts the
// term on its first point and a seed-only (w_term = 0) copy on the second.
struct TermSpec {
    double target;
    double w_term;
    double w_seed;
    int kind;
    int pad;
};

// per-layer offsets of s_l inside the coefficient vector (meta regularizers)
struct BandLayout {
    int L;
    int off[kMaxL + 1];
};

struct RunGeom {
    int64_t n_per_inst;     // points per instance
    int tiles_per_inst;
    int tiles_per_unit;
    int units_per_inst;
    int64_t n_units;
    int P;                  // points per tile
};

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}
template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
    return __shfl_xor_sync(0xffffffffu, v, m);
}

template <int ACT, typename T>
__device__ __forceinline__ void act_fwd(T a, T& sg, T& d1, T& d2) {
    if constexpr (ACT == 0) {
        T s;
        if constexpr (sizeof(T) == 8) s = tanh(a);
        else s = tanhf(a);
        sg = s;
        d1 = T(1) - s * s;
        d2 = T(-2) * s * d1;
    } else {
        T sn, cs;
        if constexpr (sizeof(T) == 8) sincos(a, &sn, &cs);
        else sincosf(a, &sn, &cs);
        sg = sn;
        d1 = cs;
        d2 = -sn;
    }
}

// sigma', sigma'', sigma''' at a (tanh: from the value, model.hpp:28-33)
template <int ACT, typename T>
__device__ __forceinline__ void act_bwd(T a, T& d1, T& d2, T& d3) {
    if constexpr (ACT == 0) {
        T s;
        if constexpr (sizeof(T) == 8) s = tanh(a);
        else s = tanhf(a);
        const T e = T(1) - s * s;
        d1 = e;
        d2 = T(-2) * s * e;
        d3 = T(-2) * e * e + T(4) * s * s * e;
    } else {
        T sn, cs;
        if constexpr (sizeof(T) == 8) sincos(a, &sn, &cs);
        else sincosf(a, &sn, &cs);
        d1 = cs;
        d2 = -sn;
        d3 = -cs;
    }
}

template <typename T>
__device__ __forceinline__ bool finite_val(T v) {
    return isfinite(v);
}

// Gather all 4 slots of a per-point jet quantity held SPT-per-lane in a TPP group.
template <int TPP, typename T>
__device__ __forceinline__ void gather4(const T* own, T (&all)[4], int base) {
    constexpr int SPT = 4 / TPP;
    if constexpr (TPP == 1) {
        all[0] = own[0];
        all[1] = own[1];
        all[2] = own[2];
        all[3] = own[3];
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) all[c] = shfl(own[c % SPT], base + c / SPT);
    }
}

template <typename T, int RMAX>
__device__ __forceinline__ void warp_sum_store(T (&v)[RMAX], int r, T* dst, int lane) {
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
        if (j < r) {
            T x = v[j];
            x += shfl_xor(x, 16);
            x += shfl_xor(x, 8);
            x += shfl_xor(x, 4);
            x += shfl_xor(x, 2);
            x += shfl_xor(x, 1);
            if (lane == 0) dst[j] = x;
        }
    }
}

template <typename T>
__device__ __forceinline__ T sgn0(T v) {
    return v > T(0) ? T(1) : (v < T(0) ? T(-1) : T(0));
}

// MODE 0: residual + dL/ds;  MODE 1: forward only (loss terms + output jets).
// Per-point term (TermSpec, internal.h): spec == nullptr -> every point is an
// interior term of `objective` (0: w N^2, 1: w |N|); otherwise spec[point]
// gives the kind (adds 2: w (u - c)^2, 3: w |u - c|), the target c and the
// term / seed weights (training.cpp:286-327, 521-549).
template <typename T, int TPP, int RMAX, int ACT, int MODE>
__global__ void __launch_bounds__(kThreads)
pinn_kernel(const DevNet<T> net, const RunGeom g, const double* __restrict__ pts,
            const double* __restrict__ svec, const double* __restrict__ mus, const T w,
            T* __restrict__ scratch, T* __restrict__ part, double* __restrict__ jets_out,
            unsigned long long* __restrict__ bad, const TermSpec* __restrict__ spec, const int objective) {
    constexpr int SPT = 4 / TPP;
    constexpr int NW = kThreads / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int R1 = 1 + net.rtotal;
    T* wpart = reinterpret_cast<T*>(smem_raw);  // NW x R1
    T* acc = wpart + NW * R1;                    // R1

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int q = tid % TPP;
    const int pl = tid / TPP;
    const int base = lane & ~(TPP - 1);
    const int P = g.P;
    T* scr = scratch + static_cast<int64_t>(blockIdx.x) * P * 4 * net.rtotal;
    const int L = net.L;

    for (int k = tid; k < (NW + 1) * R1; k += kThreads) wpart[k] = T(0);  // wpart + acc
    __syncthreads();

    for (int64_t unit = blockIdx.x; unit < g.n_units; unit += gridDim.x) {
        const int64_t inst = unit / g.units_per_inst;
        const int seg = static_cast<int>(unit % g.units_per_inst);
        const int t_lo = seg * g.tiles_per_unit;
        const int t_hi = min(g.tiles_per_inst, t_lo + g.tiles_per_unit);
        const double* sv = svec + inst * net.rtotal;
        const T mu0 = T(mus[3 * inst]), mu1 = T(mus[3 * inst + 1]), mu2 = T(mus[3 * inst + 2]);

        for (int tile = t_lo; tile < t_hi; ++tile) {
            const int64_t pi = static_cast<int64_t>(tile) * P + pl;
            const bool valid = pi < g.n_per_inst;
            const int64_t gp = inst * g.n_per_inst + pi;
            const T x = valid ? T(pts[2 * gp]) : T(0);
            const T t = valid ? T(pts[2 * gp + 1]) : T(0);

            T y[SPT][RMAX];
            T sy[SPT][RMAX];
            // ---- layer 0 input: y_0 = V_0^T z_0, z_0 = (x,t),(1,0),(0,1),(0,0) ----
            {
                const int r0 = net.r[0];
#pragma unroll
                for (int j = 0; j < RMAX; ++j) {
                    if (j < r0) {
                        const T v0 = net.V0[j], v1 = net.V0[r0 + j];
#pragma unroll
                        for (int i = 0; i < SPT; ++i) {
                            const int c = q * SPT + i;
                            const T z0 = c == 0 ? x : (c == 1 ? T(1) : T(0));
                            const T z1 = c == 0 ? t : (c == 2 ? T(1) : T(0));
                            y[i][j] = v0 * z0 + v1 * z1;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < SPT; ++i) y[i][j] = T(0);
                    }
                }
                if constexpr (MODE == 0) {
#pragma unroll
                    for (int j = 0; j < RMAX; ++j)
                        if (j < r0)
#pragma unroll
                            for (int i = 0; i < SPT; ++i)
                                scr[((net.soff[0] + j) * P + pl) * 4 + q * SPT + i] = y[i][j];
                }
            }
            // ---- forward transitions ----
            for (int l = 0; l + 1 < L; ++l) {
                const int rl = net.r[l], rn = net.r[l + 1], Mn = net.M[l + 1], stride = net.trow[l];
                const double* sl = sv + net.soff[l];
#pragma unroll
                for (int j = 0; j < RMAX; ++j) {
                    const T sj = j < rl ? T(sl[j]) : T(0);
#pragma unroll
                    for (int i = 0; i < SPT; ++i) sy[i][j] = sj * y[i][j];
                }
#pragma unroll
                for (int j = 0; j < RMAX; ++j)
#pragma unroll
                    for (int i = 0; i < SPT; ++i) y[i][j] = T(0);
                const T* row = net.trans[l];
                for (int k = 0; k < Mn; ++k, row += stride) {
                    T a[SPT];
#pragma unroll
                    for (int i = 0; i < SPT; ++i) a[i] = T(0);
#pragma unroll
                    for (int j = 0; j < RMAX; ++j) {
                        if (j < rl) {
                            const T u = row[j];
#pragma unroll
                            for (int i = 0; i < SPT; ++i) a[i] = fma(u, sy[i][j], a[i]);
                        }
                    }
                    if (q == 0) a[0] += row[rl + rn];
                    T av, ax;
                    if constexpr (TPP == 1) {
                        av = a[0];
                        ax = a[1];
                    } else {
                        av = shfl(a[0], base);
                        ax = shfl(a[1 % SPT], base + 1 / SPT);
                    }
                    T sg, d1, d2;
                    act_fwd<ACT>(av, sg, d1, d2);
                    T z[SPT];
#pragma unroll
                    for (int i = 0; i < SPT; ++i) {
                        const int c = q * SPT + i;
                        z[i] = c == 0 ? sg : (c == 3 ? d2 * ax * ax + d1 * a[i] : d1 * a[i]);
                    }
#pragma unroll
                    for (int j = 0; j < RMAX; ++j) {
                        if (j < rn) {
                            const T v = row[rl + j];
#pragma unroll
                            for (int i = 0; i < SPT; ++i) y[i][j] = fma(v, z[i], y[i][j]);
                        }
                    }
                }
                if constexpr (MODE == 0) {
#pragma unroll
                    for (int j = 0; j < RMAX; ++j)
                        if (j < rn)
#pragma unroll
                            for (int i = 0; i < SPT; ++i)
                                scr[((net.soff[l + 1] + j) * P + pl) * 4 + q * SPT + i] = y[i][j];
                }
            }
            // ---- output layer (M_L = 1) + residual ----
            const int rL = net.r[L - 1];
            const double* sL = sv + net.soff[L - 1];
            T u[SPT];
#pragma unroll
            for (int i = 0; i < SPT; ++i) u[i] = T(0);
#pragma unroll
            for (int j = 0; j < RMAX; ++j) {
                if (j < rL) {
                    const T us = net.ulast[j] * T(sL[j]);
#pragma unroll
                    for (int i = 0; i < SPT; ++i) u[i] = fma(us, y[i][j], u[i]);
                }
            }
            if (q == 0) u[0] += net.ulast[rL];
            T u4[4];
            gather4<TPP>(u, u4, base);
            const T N = u4[2] + mu0 * u4[1] - mu1 * u4[3] - mu2 * u4[0] * (T(1) - u4[0]);
            int kind = objective;
            T tw = w, sw = w, tgt = T(0);
            if (spec != nullptr && valid) {
                const TermSpec sp = spec[gp];
                kind = sp.kind;
                tgt = T(sp.target);
                tw = T(sp.w_term);
                sw = T(sp.w_seed);
            }
            const T d = u4[0] - tgt;  // value kinds: u - c
            T term = kind == 0 ? tw * (N * N) : (kind == 1 ? tw * fabs(N) : (kind == 2 ? tw * (d * d) : tw * fabs(d)));
            term = valid ? term : T(0);
            if (valid && q == 0 && !finite_val(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
            {
                T tv = q == 0 ? term : T(0);
                tv += shfl_xor(tv, 16);
                tv += shfl_xor(tv, 8);
                tv += shfl_xor(tv, 4);
                tv += shfl_xor(tv, 2);
                tv += shfl_xor(tv, 1);
                if (lane == 0) wpart[warp * R1] = tv;
            }
            if constexpr (MODE == 1) {
                if (valid && jets_out != nullptr) {
#pragma unroll
                    for (int i = 0; i < SPT; ++i) jets_out[gp * 4 + q * SPT + i] = double(u[i]);
                }
            } else {
                // ---- reverse sweep ----
                T gu[SPT];
                if (kind <= 1) {
                    const T gN = valid ? (kind == 0 ? T(2) * N * sw : sgn0(N) * sw) : T(0);
#pragma unroll
                    for (int i = 0; i < SPT; ++i) {
                        const int c = q * SPT + i;
                        gu[i] = c == 0 ? gN * (-mu2 * (T(1) - T(2) * u4[0]))
                                       : (c == 1 ? gN * mu0 : (c == 2 ? gN : -gN * mu1));
                    }
                } else {
                    // value terms seed the value slot only (PickValue VJP, autodiff.cpp:715-760)
                    const T gd = valid ? (kind == 2 ? T(2) * d * sw : sgn0(d) * sw) : T(0);
#pragma unroll
                    for (int i = 0; i < SPT; ++i) gu[i] = (q * SPT + i) == 0 ? gd : T(0);
                }
                T st[SPT][RMAX];
                {
                    T cds[RMAX];
#pragma unroll
                    for (int j = 0; j < RMAX; ++j) {
                        const T uj = j < rL ? net.ulast[j] : T(0);
                        const T sj = j < rL ? T(sL[j]) : T(0);
                        T cd = T(0);
#pragma unroll
                        for (int i = 0; i < SPT; ++i) {
                            const T tj = uj * gu[i];
                            cd = fma(tj, y[i][j], cd);
                            st[i][j] = sj * tj;
                        }
                        cds[j] = cd;
                    }
                    warp_sum_store<T, RMAX>(cds, rL, wpart + warp * R1 + 1 + net.soff[L - 1], lane);
                }
                for (int l = L - 2; l >= 0; --l) {
                    const int rl = net.r[l], rn = net.r[l + 1], Mn = net.M[l + 1], stride = net.trow[l];
                    const double* sl = sv + net.soff[l];
#pragma unroll
                    for (int j = 0; j < RMAX; ++j) {
                        const T sj = j < rl ? T(sl[j]) : T(0);
#pragma unroll
                        for (int i = 0; i < SPT; ++i)
                            sy[i][j] = j < rl ? sj * scr[((net.soff[l] + j) * P + pl) * 4 + q * SPT + i] : T(0);
                    }
                    T tn[SPT][RMAX];
#pragma unroll
                    for (int j = 0; j < RMAX; ++j)
#pragma unroll
                        for (int i = 0; i < SPT; ++i) tn[i][j] = T(0);
                    const T* row = net.trans[l];
                    for (int k = 0; k < Mn; ++k, row += stride) {
                        T a[SPT], dz[SPT];
#pragma unroll
                        for (int i = 0; i < SPT; ++i) {
                            a[i] = T(0);
                            dz[i] = T(0);
                        }
#pragma unroll
                        for (int j = 0; j < RMAX; ++j) {
                            if (j < rn) {
                                const T v = row[rl + j];
#pragma unroll
                                for (int i = 0; i < SPT; ++i) dz[i] = fma(v, st[i][j], dz[i]);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < RMAX; ++j) {
                            if (j < rl) {
                                const T uu = row[j];
#pragma unroll
                                for (int i = 0; i < SPT; ++i) a[i] = fma(uu, sy[i][j], a[i]);
                            }
                        }
                        if (q == 0) a[0] += row[rl + rn];
                        T a4[4], g4[4];
                        gather4<TPP>(a, a4, base);
                        gather4<TPP>(dz, g4, base);
                        T d1, d2, d3;
                        act_bwd<ACT>(a4[0], d1, d2, d3);
                        const T gav = g4[0] * d1 + g4[1] * d2 * a4[1] + g4[2] * d2 * a4[2] +
                                      g4[3] * (d3 * a4[1] * a4[1] + d2 * a4[3]);
                        const T gax = g4[1] * d1 + g4[3] * T(2) * d2 * a4[1];
                        const T gat = g4[2] * d1;
                        const T gaw = g4[3] * d1;
                        T ga[SPT];
#pragma unroll
                        for (int i = 0; i < SPT; ++i) {
                            const int c = q * SPT + i;
                            ga[i] = c == 0 ? gav : (c == 1 ? gax : (c == 2 ? gat : gaw));
                        }
#pragma unroll
                        for (int j = 0; j < RMAX; ++j) {
                            if (j < rl) {
                                const T uu = row[j];
#pragma unroll
                                for (int i = 0; i < SPT; ++i) tn[i][j] = fma(uu, ga[i], tn[i][j]);
                            }
                        }
                    }
                    T cds[RMAX];
#pragma unroll
                    for (int j = 0; j < RMAX; ++j) {
                        T cd = T(0);
                        const T sj = j < rl ? T(sl[j]) : T(0);
#pragma unroll
                        for (int i = 0; i < SPT; ++i) {
                            const T yv = j < rl ? scr[((net.soff[l] + j) * P + pl) * 4 + q * SPT + i] : T(0);
                            cd = fma(tn[i][j], yv, cd);
                            st[i][j] = sj * tn[i][j];
                        }
                        cds[j] = cd;
                    }
                    warp_sum_store<T, RMAX>(cds, rl, wpart + warp * R1 + 1 + net.soff[l], lane);
                }
            }
            __syncthreads();
            for (int k = tid; k < R1; k += kThreads) {
                T sacc = acc[k];
#pragma unroll
                for (int ww = 0; ww < NW; ++ww) sacc += wpart[ww * R1 + k];
                acc[k] = sacc;
            }
            __syncthreads();
        }
        for (int k = tid; k < R1; k += kThreads) {
            part[unit * R1 + k] = acc[k];
            acc[k] = T(0);
        }
        __syncthreads();
    }
}

// Fixed-order per-instance reduction of unit partials, in double.
template <typename T>
__global__ void reduce_units_kernel(const T* __restrict__ part, int units_per_inst, int R1,
                                    int64_t n_inst, double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t inst = blockIdx.y;
    if (k >= R1 || inst >= n_inst) return;
    const T* p = part + inst * units_per_inst * static_cast<int64_t>(R1) + k;
    double s = 0.0;
    for (int u = 0; u < units_per_inst; ++u) s += double(p[static_cast<int64_t>(u) * R1]);
    out[inst * R1 + k] = s;
}

// First level of a two-level fixed-order unit reduction (many units, e.g. the
// dynamically claimed single-tile units of the tensor-core sweep): group g of
// instance inst sums units [g G, (g + 1) G) into out2[inst][g][k] in double.
template <typename T>
__global__ void reduce_unit_groups_kernel(const T* __restrict__ part, int units_per_inst, int R1, int G,
                                          double* __restrict__ out2) {
    const int g = blockIdx.x, ngroups = gridDim.x;
    const int64_t inst = blockIdx.y;
    const int u0 = g * G, u1 = min(units_per_inst, u0 + G);
    const T* p = part + (inst * units_per_inst + u0) * static_cast<int64_t>(R1);
    for (int k = threadIdx.x; k < R1; k += blockDim.x) {
        double s = 0.0;
        for (int u = 0; u < u1 - u0; ++u) s += double(p[static_cast<int64_t>(u) * R1 + k]);
        out2[(inst * ngroups + g) * R1 + k] = s;
    }
}

// out[i] = sum_r rows[r][i] in double, rows in fixed order (per-CTA partials).
template <typename T>
__global__ void reduce_rows_kernel(const T* __restrict__ rows, int n_rows, int64_t stride, int64_t n,
                                   double* __restrict__ out, int accumulate = 0) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int r = 0; r < n_rows; ++r) s += double(rows[r * stride + i]);
    out[i] = accumulate ? out[i] + s : s;
}

}  // namespace lrnr_b200
