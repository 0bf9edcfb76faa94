// K-dependence of 3xTF32 accumulation error on tcgen05 (dev aid).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200::umma;
constexpr int M = 128, N = 32, K = 128, KC = 32;
// mode 0: single acc (hh, hl, lh per k-step); 1: hh acc + cross acc; 2: per-KC fresh acc, fp32 sum in registers
__global__ void k(const float* A, const float* B, float* D, int mode) {
    extern __shared__ __align__(128) float sm[];
    float *sAh = sm, *sAl = sAh + M * K, *sBh = sAl + M * K, *sBl = sBh + N * K;
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < M * K; i += blockDim.x) { int m = i / K, kk = i % K; float h, l; split_tf32(A[i], h, l); sAh[kmaj_off(m, kk, M)] = h; sAl[kmaj_off(m, kk, M)] = l; }
    for (int i = tid; i < N * K; i += blockDim.x) { int n = i / K, kk = i % K; float h, l; split_tf32(B[i], h, l); sBh[kmaj_off(n, kk, N)] = h; sBl[kmaj_off(n, kk, N)] = l; }
    if (warp == 0) tmem_alloc<128>(&tbase);
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    fence_async_smem(); fence_before(); __syncthreads(); fence_after();
    const uint32_t d0 = tbase, d1 = tbase + 32;
    const uint32_t id = idesc_tf32(M, N);
    float accr[32];
    for (int i = 0; i < 32; ++i) accr[i] = 0.f;
    const int nchunk = mode == 2 ? K / KC : 1;
    for (int ch = 0; ch < nchunk; ++ch) {
        if (tid == 0) {
            const int s0 = mode == 2 ? ch * KC / 8 : 0, s1 = mode == 2 ? (ch + 1) * KC / 8 : K / 8;
            for (int s = s0; s < s1; ++s) {
                uint64_t ah = smem_desc(sAh + s * 2 * (M / 8) * 32, (M / 8) * 128, 128), al = smem_desc(sAl + s * 2 * (M / 8) * 32, (M / 8) * 128, 128);
                uint64_t bh = smem_desc(sBh + s * 2 * (N / 8) * 32, (N / 8) * 128, 128), bl = smem_desc(sBl + s * 2 * (N / 8) * 32, (N / 8) * 128, 128);
                const uint32_t first = s > s0;
                if (mode == 1) { mma_tf32_ss(d0, ah, bh, id, first); mma_tf32_ss(d1, ah, bl, id, first); mma_tf32_ss(d1, al, bh, id, 1); }
                else { mma_tf32_ss(d0, ah, bh, id, first); mma_tf32_ss(d0, ah, bl, id, 1); mma_tf32_ss(d0, al, bh, id, 1); }
            }
            mma_commit(&bar);
        }
        mbar_wait(&bar, ch & 1); fence_after();
        if (warp < 4) {
            float v[16], v1[16];
            for (int h = 0; h < 2; ++h) {
                tmem_ld16(d0 + ((warp * 32) << 16) + h * 16, v); tmem_ld16(d1 + ((warp * 32) << 16) + h * 16, v1); tmem_ld_wait();
                for (int i = 0; i < 16; ++i) accr[h * 16 + i] += (mode == 1 ? v[i] + v1[i] : v[i]);
            }
        }
        fence_before(); __syncthreads(); fence_after();
    }
    if (warp < 4) { const int m = warp * 32 + lane; for (int i = 0; i < 32; ++i) D[m * N + i] = accr[i]; }
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tbase);
}
int main() {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    std::vector<double> ref(M * N);
    srand(7);
    for (int trial = 0; trial < 2; ++trial) {
        // trial 0: zero-mean data; trial 1: positive (coherent) data
        for (auto& a : A) a = trial ? rand() / (float)RAND_MAX : (rand() / (float)RAND_MAX - 0.5f) * 3.f;
        for (auto& b : B) b = trial ? rand() / (float)RAND_MAX : (rand() / (float)RAND_MAX - 0.5f) * 2.f;
        double nr = 0, ef = 0;
        for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { double s = 0; float f = 0; for (int kk = 0; kk < K; ++kk) { s += double(A[m*K+kk]) * B[n*K+kk]; f = fmaf(A[m*K+kk], B[n*K+kk], f); } ref[m*N+n] = s; nr += s*s; ef += (f - s) * (f - s); }
        printf("trial %d (K=%d): fp32 FMA normwise err %.3e\n", trial, K, sqrt(ef / nr));
        float *dA, *dB, *dD;
        cudaMalloc(&dA, A.size()*4); cudaMalloc(&dB, B.size()*4); cudaMalloc(&dD, D.size()*4);
        cudaMemcpy(dA, A.data(), A.size()*4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size()*4, cudaMemcpyHostToDevice);
        const int smem = (2 * M * K + 2 * N * K) * 4;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const char* names[3] = {"3xTF32 single acc", "3xTF32 hh + cross acc", "3xTF32 fresh per 32, fp32 sum"};
        for (int mode = 0; mode < 3; ++mode) {
            k<<<1, 256, smem>>>(dA, dB, dD, mode); if (cudaGetLastError() != cudaSuccess) { printf("launch fail\n"); return 1; }
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("fail\n"); return 1; }
            cudaMemcpy(D.data(), dD, D.size()*4, cudaMemcpyDeviceToHost);
            double e = 0, bias = 0;
            for (int i = 0; i < M * N; ++i) { e += (D[i] - ref[i]) * (D[i] - ref[i]); bias += (D[i] - ref[i]); }
            printf("  %-32s normwise err %.3e  mean err/|ref| %.3e\n", names[mode], sqrt(e / nr), bias / (M * N) / sqrt(nr / (M * N)));
        }
    }
    return 0;
}
