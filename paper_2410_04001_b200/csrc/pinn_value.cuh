// Value-only (1-slot) forward: u(x, t) of the LRNR or the FastLRNR at a batch of
// points, the reference's lrnr_forward / fast_forward (model.cpp:260-292) with
// value_affine_factored / value_affine_dense / value_activation (model.cpp:183-223).
//
// The boundary terms of loss_tune / loss_meta / loss_fast (training.cpp:76-189)
// and the L1 evaluation grid (pde.cpp:166-178) need u only; the 4-slot jet sweep
// costs 4x the FMAs for them.  One thread owns one point and streams the network
// neuron by neuron over the same DevNet rows as the jet kernels
// (pinn_kernels.cuh): a_k = U_l[k,:] . (s_l (.) y_l) + b_l[k], z_k = sigma(a_k),
// y_{l+1} += V_{l+1}[k,:] z_k.  Row reads are warp-uniform (one L1 transaction
// feeds all 32 lanes); only the rank-r vectors live in registers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pinn_kernels.cuh"

namespace lrnr_b200 {
namespace value {

constexpr int NT = 128;

template <int ACT, typename T>
__device__ __forceinline__ T act_value(T a) {
    if constexpr (ACT == 0) {
        if constexpr (sizeof(T) == 8) return tanh(a);
        else return tanhf(a);
    } else {
        if constexpr (sizeof(T) == 8) return sin(a);
        else return sinf(a);
    }
}

// pts: n_inst groups of n_per (x, t) pairs; svec: n_inst x r_total; out_u: n_inst * n_per
// values (double). bad: first non-finite point index (atomicMin), ULLONG_MAX when clean.
template <typename T, int RMAX, int ACT>
__global__ void __launch_bounds__(NT)
value_kernel(const DevNet<T> net, const double* __restrict__ pts, int64_t n_per, int64_t n_total,
             const double* __restrict__ svec, double* __restrict__ out_u, unsigned long long* __restrict__ bad) {
    const int64_t gp = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
    if (gp >= n_total) return;
    const int64_t inst = gp / n_per;
    const double* sv = svec + inst * net.rtotal;
    const T x = T(pts[2 * gp]), t = T(pts[2 * gp + 1]);
    const int L = net.L;
    T y[RMAX], sy[RMAX];
    const int r0 = net.r[0];
#pragma unroll
    for (int j = 0; j < RMAX; ++j) y[j] = j < r0 ? net.V0[j] * x + net.V0[r0 + j] * t : T(0);
    for (int l = 0; l + 1 < L; ++l) {
        const int rl = net.r[l], rn = net.r[l + 1], Mn = net.M[l + 1], stride = net.trow[l];
        const double* sl = sv + net.soff[l];
#pragma unroll
        for (int j = 0; j < RMAX; ++j) {
            sy[j] = j < rl ? T(sl[j]) * y[j] : T(0);
            y[j] = T(0);
        }
        const T* row = net.trans[l];
        for (int k = 0; k < Mn; ++k, row += stride) {
            T a = row[rl + rn];
#pragma unroll
            for (int j = 0; j < RMAX; ++j)
                if (j < rl) a = fma(row[j], sy[j], a);
            const T z = act_value<ACT>(a);
#pragma unroll
            for (int j = 0; j < RMAX; ++j)
                if (j < rn) y[j] = fma(row[rl + j], z, y[j]);
        }
    }
    const int rL = net.r[L - 1];
    const double* sL = sv + net.soff[L - 1];
    T u = net.ulast[rL];
#pragma unroll
    for (int j = 0; j < RMAX; ++j)
        if (j < rL) u = fma(net.ulast[j] * T(sL[j]), y[j], u);
    const double ud = static_cast<double>(u);
    out_u[gp] = ud;
    if (!isfinite(ud)) atomicMin(bad, static_cast<unsigned long long>(gp));
}

}  // namespace value
}  // namespace lrnr_b200
