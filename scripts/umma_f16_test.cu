// Self-test (dev aid, run on a B200) of the FP16 two-term split GEMM the tensor-core
// LRNR kernel uses: x = hi + lo with hi = fp16(x S), lo = fp16(x S - hi), S a power
// of two (per row for A, per matrix for B); the product is hi*hi + hi*lo + lo*hi
// (kind::f16, FP32 accumulate), unscaled per row.  Checks
//   * the K-major SWIZZLE_NONE canonical layout of 16-bit operands in shared memory (SS),
//   * A in tensor memory, two 16-bit K elements per 32-bit column (TS),
//   * accuracy against a double reference, with rows spanning 2^-30 .. 2^10 in magnitude.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/umma_f16_test.cu -o scripts/umma_f16_test
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200::umma;

constexpr int M = 128, N = 32, K = 32;

__host__ __device__ inline int kmaj16(int row, int k, int rows) {
    return (((k >> 3) * (rows >> 3) + (row >> 3)) << 6) + ((row & 7) << 3) + (k & 7);
}
__device__ inline uint32_t idesc_f16(int m, int n) {
    return (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ inline void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ inline void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ inline float pow2_scale(float amax) {  // 2^(14 - e), amax <= 2^e
    int e;
    frexpf(amax, &e);
    e = max(-100, min(100, e));
    return ldexpf(1.f, 14 - e);
}

__global__ void k_test(const float* A, const float* B, float* D_ss, float* D_ts) {
    __shared__ __align__(128) __half sAh[M * K], sAl[M * K], sBh[N * K], sBl[N * K];
    __shared__ float rowinv[M];
    __shared__ float bscale;
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (tid == 0) {
        float bm = 0.f;
        for (int i = 0; i < N * K; ++i) bm = fmaxf(bm, fabsf(B[i]));
        bscale = pow2_scale(bm);
    }
    __syncthreads();
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int n = i / K, k = i % K;
        const float x = B[i] * bscale;
        const __half h = __float2half_rn(x);
        sBh[kmaj16(n, k, N)] = h;
        sBl[kmaj16(n, k, N)] = __float2half_rn(x - __half2float(h));
    }
    if (warp == 0) tmem_alloc<256>(&tbase);
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    const uint32_t t0 = tbase;
    const uint32_t dss = t0, dts = t0 + 32, ah_t = t0 + 64, al_t = t0 + 96;  // A hi / lo in TMEM: K/2 columns each
    if (warp < 4) {
        const int m = warp * 32 + lane;
        float am = 0.f;
        for (int k = 0; k < K; ++k) am = fmaxf(am, fabsf(A[m * K + k]));
        const float s = pow2_scale(am);
        rowinv[m] = 1.f / (s * bscale);
        uint32_t hw[K / 2], lw[K / 2];
        for (int k = 0; k < K; ++k) {
            const float x = A[m * K + k] * s;
            const __half h = __float2half_rn(x), l = __float2half_rn(x - __half2float(h));
            sAh[kmaj16(m, k, M)] = h;
            sAl[kmaj16(m, k, M)] = l;
            const uint32_t hb = __half_as_ushort(h), lb = __half_as_ushort(l);
            if (k & 1) { hw[k / 2] |= hb << 16; lw[k / 2] |= lb << 16; } else { hw[k / 2] = hb; lw[k / 2] = lb; }
        }
        float v[16];
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(hw[i]);
        tmem_st16(ah_t + ((warp * 32) << 16), v);
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(lw[i]);
        tmem_st16(al_t + ((warp * 32) << 16), v);
        tmem_st_wait();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
        const uint32_t id = idesc_f16(M, N);
        for (int s = 0; s < K / 16; ++s) {
            // K step of 16 = two 8-element core-matrix columns: start at 2 s LBO
            const uint64_t dah = smem_desc(sAh + s * 2 * (M / 8) * 64, (M / 8) * 128, 128);
            const uint64_t dal = smem_desc(sAl + s * 2 * (M / 8) * 64, (M / 8) * 128, 128);
            const uint64_t dbh = smem_desc(sBh + s * 2 * (N / 8) * 64, (N / 8) * 128, 128);
            const uint64_t dbl = smem_desc(sBl + s * 2 * (N / 8) * 64, (N / 8) * 128, 128);
            mma_ss(dss, dah, dbh, id, s > 0);
            mma_ss(dss, dah, dbl, id, 1);
            mma_ss(dss, dal, dbh, id, 1);
            mma_ts(dts, ah_t + s * 8, dbh, id, s > 0);
            mma_ts(dts, ah_t + s * 8, dbl, id, 1);
            mma_ts(dts, al_t + s * 8, dbh, id, 1);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    if (warp < 4) {
        const int m = warp * 32 + lane;
        float v[16];
        for (int h = 0; h < 2; ++h) {
            tmem_ld16(dss + ((warp * 32) << 16) + h * 16, v);
            tmem_ld_wait();
            for (int i = 0; i < 16; ++i) D_ss[m * N + h * 16 + i] = v[i] * rowinv[m];
            tmem_ld16(dts + ((warp * 32) << 16) + h * 16, v);
            tmem_ld_wait();
            for (int i = 0; i < 16; ++i) D_ts[m * N + h * 16 + i] = v[i] * rowinv[m];
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(t0);
}

int main() {
    std::vector<float> A(M * K), B(N * K), dss(M * N), dts(M * N);
    std::vector<double> ref(M * N, 0.0);
    srand(1);
    auto urand = [] { return (rand() + 0.5) / (RAND_MAX + 1.0); };
    for (int m = 0; m < M; ++m) {
        const double rs = std::ldexp(1.0, -30 + (m * 40) / M);  // rows from 2^-30 to 2^10
        for (int k = 0; k < K; ++k) {
            double x = (2 * urand() - 1) * rs;
            if ((m + k) % 7 == 0) x *= 1e-4;  // small entries inside a row
            A[m * K + k] = float(x);
        }
    }
    for (auto& b : B) b = float((2 * urand() - 1) * 0.2);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * B[n * K + k];
            ref[m * N + n] = s;
        }
    float *dA, *dB, *d1, *d2;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&d1, dss.size() * 4); cudaMalloc(&d2, dts.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    k_test<<<1, 256>>>(dA, dB, d1, d2);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 2;
    cudaMemcpy(dss.data(), d1, dss.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(dts.data(), d2, dts.size() * 4, cudaMemcpyDeviceToHost);
    // per-row normwise relative error, worst row; plus plain fp32-rounding of the reference for scale
    double w1 = 0, w2 = 0;
    for (int m = 0; m < M; ++m) {
        double n0 = 0, e1 = 0, e2 = 0;
        for (int n = 0; n < N; ++n) {
            const double r = ref[m * N + n];
            n0 += r * r;
            e1 += (dss[m * N + n] - r) * (dss[m * N + n] - r);
            e2 += (dts[m * N + n] - r) * (dts[m * N + n] - r);
        }
        w1 = fmax(w1, sqrt(e1 / n0));
        w2 = fmax(w2, sqrt(e2 / n0));
        if (m % 32 == 0) printf("row %3d |ref| %.3e  SS rel %.2e  TS rel %.2e\n", m, sqrt(n0 / N), sqrt(e1 / n0), sqrt(e2 / n0));
    }
    printf("worst row normwise rel err: SS %.3e  TS %.3e\n", w1, w2);
    return (w1 < 2e-6 && w2 < 2e-6) ? 0 : 1;
}
