// Hypernetwork mu -> s, batched over PDE-parameter instances, and its VJP
// (BASELINE config 3/4).  Restates hyper_forward (model.cpp:294-318),
// normalize_mu (model.cpp:74-81), emit_hyper + the AffineDenseVec / TanhVec /
// ReluVec / SliceVec VJPs (autodiff.cpp:155-209,667-714,883-903).
// The network is tiny (3-64-64-r_total: 15K-34K parameters) next to the
// point sweep it feeds (16K-1M points per instance), so it runs once per
// instance (the reference re-runs it per point in meta mode,
// training.cpp:283-288) and in FP64.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lrnr_b200 {

constexpr int kHyperMaxLayers = 8;

struct HyperDev {
    int K;                       // affine layers
    int hw[kHyperMaxLayers + 1]; // widths, hw[0] = 3
    int oW[kHyperMaxLayers], ob[kHyperMaxLayers];
    int max_w;
    int n_params;
    const double* P;             // flat W_k, b_k
    double lo[3], hi[3];
};

// acts[inst][k][max_w]: input of layer k (k = 0..K; acts[K] = ReLU output = s)
__global__ void hyper_forward_kernel(const HyperDev h, const double* __restrict__ mus,
                                     int64_t n_inst, double* __restrict__ acts,
                                     double* __restrict__ s_out) {
    const int64_t inst = blockIdx.x;
    if (inst >= n_inst) return;
    const int MW = h.max_w;
    double* A = acts + inst * (h.K + 1) * MW;
    if (threadIdx.x < 3) {
        const int i = threadIdx.x;
        const double extent = h.hi[i] - h.lo[i];
        A[i] = extent > 0.0 ? (mus[3 * inst + i] - h.lo[i]) / extent : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < h.K; ++k) {
        const int rows = h.hw[k + 1], cols = h.hw[k];
        const double* W = h.P + h.oW[k];
        const double* b = h.P + h.ob[k];
        const double* in = A + k * MW;
        double* out = A + (k + 1) * MW;
        for (int i = threadIdx.x; i < rows; i += blockDim.x) {
            double acc = 0.0;
            for (int j = 0; j < cols; ++j) acc += W[i * cols + j] * in[j];
            const double a = acc + b[i];
            out[i] = (k + 1 < h.K) ? tanh(a) : (a > 0.0 ? a : 0.0);
        }
        __syncthreads();
    }
    const int od = h.hw[h.K];
    for (int i = threadIdx.x; i < od; i += blockDim.x) s_out[inst * od + i] = A[h.K * MW + i];
}

// Per-instance backward: G[inst][k][i] = dL/d(pre-activation of layer k)_i.
// gs: rows of the per-instance result buffer [value, dL/ds (r_total)] (stride R1).
__global__ void hyper_backward_kernel(const HyperDev h, const double* __restrict__ acts,
                                      const double* __restrict__ gs, int R1, int64_t n_inst,
                                      double* __restrict__ G) {
    const int64_t inst = blockIdx.x;
    if (inst >= n_inst) return;
    const int MW = h.max_w, K = h.K;
    const double* A = acts + inst * (K + 1) * MW;
    double* Gi = G + inst * K * MW;
    const int od = h.hw[K];
    // ReLU VJP (autodiff.cpp:698-707): pass where out > 0
    for (int i = threadIdx.x; i < od; i += blockDim.x)
        Gi[(K - 1) * MW + i] = A[K * MW + i] > 0.0 ? gs[inst * R1 + 1 + i] : 0.0;
    __syncthreads();
    for (int k = K - 1; k >= 1; --k) {
        const int rows = h.hw[k + 1], cols = h.hw[k];
        const double* W = h.P + h.oW[k];
        const double* g = Gi + k * MW;
        const double* sig = A + k * MW;  // tanh output feeding layer k
        for (int j = threadIdx.x; j < cols; j += blockDim.x) {
            double acc = 0.0;
            for (int i = 0; i < rows; ++i) acc += W[i * cols + j] * g[i];
            Gi[(k - 1) * MW + j] = acc * (1.0 - sig[j] * sig[j]);  // TanhVec VJP
        }
        __syncthreads();
    }
}

// dW_k[i][j] = sum_inst G[inst][k][i] * acts[inst][k][j]; db_k[i] = sum_inst G[inst][k][i]
// (fixed instance order -> deterministic).
__global__ void hyper_param_grad_kernel(const HyperDev h, const double* __restrict__ acts,
                                        const double* __restrict__ G, int64_t n_inst,
                                        double* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= h.n_params) return;
    int k = 0;
    while (k + 1 < h.K && p >= h.oW[k + 1]) ++k;
    const int MW = h.max_w, K = h.K;
    const int cols = h.hw[k];
    double s = 0.0;
    if (p < h.ob[k]) {
        const int e = p - h.oW[k];
        const int i = e / cols, j = e % cols;
        for (int64_t n = 0; n < n_inst; ++n)
            s += G[(n * K + k) * MW + i] * acts[(n * (K + 1) + k) * MW + j];
    } else {
        const int i = p - h.ob[k];
        for (int64_t n = 0; n < n_inst; ++n) s += G[(n * K + k) * MW + i];
    }
    out[p] = s;
}

}  // namespace lrnr_b200
