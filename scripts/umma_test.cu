// Self-test of the tcgen05 primitives in csrc/umma.cuh (dev aid; run on a B200).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200::umma;

constexpr int M = 128, N = 32, K = 32;

__global__ void k_test(const float* A, const float* B, float* D_ss, float* D_ts) {
    __shared__ __align__(128) float sA[M * K];
    __shared__ __align__(128) float sB[N * K];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < M * K; i += blockDim.x) { int m = i / K, k = i % K; sA[kmaj_off(m, k, M)] = A[i]; }
    for (int i = tid; i < N * K; i += blockDim.x) { int n = i / K, k = i % K; sB[kmaj_off(n, k, N)] = B[i]; }
    if (warp == 0) tmem_alloc<128>(&tbase);
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t t0 = tbase;
    const uint32_t dss = t0, dts = t0 + 32, atm = t0 + 64;   // columns
    // A into TMEM for the TS variant: lane = row m, column = k
    if (warp < 4) {
        const int m = warp * 32 + lane;
        float v[16];
        for (int h = 0; h < 2; ++h) {
            for (int i = 0; i < 16; ++i) v[i] = A[m * K + h * 16 + i];
            tmem_st16(atm + ((warp * 32) << 16) + h * 16, v);
        }
        tmem_st_wait();
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(M, N);
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t da = smem_desc(sA + s * 2 * (M / 8) * 32, (M / 8) * 128, 128);
            const uint64_t db = smem_desc(sB + s * 2 * (N / 8) * 32, (N / 8) * 128, 128);
            mma_tf32_ss(dss, da, db, idesc, s > 0);
            mma_tf32_ts(dts, atm + s * 8, db, idesc, s > 0);
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
            for (int i = 0; i < 16; ++i) D_ss[m * N + h * 16 + i] = v[i];
            tmem_ld16(dts + ((warp * 32) << 16) + h * 16, v);
            tmem_ld_wait();
            for (int i = 0; i < 16; ++i) D_ts[m * N + h * 16 + i] = v[i];
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(t0);
}

int main() {
    std::vector<float> A(M * K), B(N * K), ref(M * N, 0.f), dss(M * N), dts(M * N);
    srand(1);
    for (auto& a : A) a = float(rand() % 17 - 8) / 8.f;
    for (auto& b : B) b = float(rand() % 17 - 8) / 4.f;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < K; ++k) s += double(A[m*K+k]) * B[n*K+k]; ref[m*N+n] = float(s); }
    float *dA, *dB, *d1, *d2;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&d1, dss.size() * 4); cudaMalloc(&d2, dts.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    k_test<<<1, 256>>>(dA, dB, d1, d2);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 2;
    cudaMemcpy(dss.data(), d1, dss.size() * 4, cudaMemcpyDeviceToHost); cudaMemcpy(dts.data(), d2, dts.size() * 4, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0;
    for (int i = 0; i < M * N; ++i) { e1 = fmax(e1, fabs(dss[i] - ref[i])); e2 = fmax(e2, fabs(dts[i] - ref[i])); }
    printf("SS max abs err %g (ref[0]=%g got %g)\nTS max abs err %g (got %g)\n", e1, ref[0], dss[0], e2, dts[0]);
    if (e1 > 1e-3) { for (int i = 0; i < 8; ++i) printf("  ref %g ss %g\n", ref[i], dss[i]); }
    return (e1 < 1e-3 && e2 < 1e-3) ? 0 : 1;
}
