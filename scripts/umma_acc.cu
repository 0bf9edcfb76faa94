// 3xTF32 accuracy probe of tcgen05.mma kind::tf32 (dev aid).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200::umma;
constexpr int M = 128, N = 32, K = 32;
// mode 0: 1xTF32, 1: hi*hi, hi*lo, lo*hi (big first), 2: small first, 3: separate accumulators summed in fp32
__global__ void k(const float* A, const float* B, float* D, int mode) {
    __shared__ __align__(128) float sAh[M * K], sAl[M * K];
    __shared__ __align__(128) float sBh[N * K], sBl[N * K];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < M * K; i += blockDim.x) { int m = i / K, kk = i % K; float h, l; split_tf32(A[i], h, l); sAh[kmaj_off(m, kk, M)] = h; sAl[kmaj_off(m, kk, M)] = l; }
    for (int i = tid; i < N * K; i += blockDim.x) { int n = i / K, kk = i % K; float h, l; split_tf32(B[i], h, l); sBh[kmaj_off(n, kk, N)] = h; sBl[kmaj_off(n, kk, N)] = l; }
    if (warp == 0) tmem_alloc<128>(&tbase);
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    fence_async_smem(); fence_before(); __syncthreads(); fence_after();
    const uint32_t d0 = tbase, d1 = tbase + 32, d2 = tbase + 32, aH = tbase + 64, aL = tbase + 96;
    if (mode >= 4 && warp < 4) {
        const int m = warp * 32 + lane;
        float vh[16], vl[16];
        for (int h = 0; h < 2; ++h) {
            for (int i = 0; i < 16; ++i) split_tf32(A[m * K + h * 16 + i], vh[i], vl[i]);
            tmem_st16(aH + ((warp * 32) << 16) + h * 16, vh);
            tmem_st16(aL + ((warp * 32) << 16) + h * 16, vl);
        }
        tmem_st_wait();
    }
    fence_before(); __syncthreads(); fence_after();
    if (tid == 0) {
        const uint32_t id = idesc_tf32(M, N);
        for (int s = 0; s < K / 8; ++s) {
            uint64_t ah = smem_desc(sAh + s * 2 * (M / 8) * 32, (M / 8) * 128, 128), al = smem_desc(sAl + s * 2 * (M / 8) * 32, (M / 8) * 128, 128);
            uint64_t bh = smem_desc(sBh + s * 2 * (N / 8) * 32, (N / 8) * 128, 128), bl = smem_desc(sBl + s * 2 * (N / 8) * 32, (N / 8) * 128, 128);
            if (mode == 0) { mma_tf32_ss(d0, ah, bh, id, s > 0); }
            else if (mode == 1) { mma_tf32_ss(d0, ah, bh, id, s > 0); mma_tf32_ss(d0, ah, bl, id, 1); mma_tf32_ss(d0, al, bh, id, 1); }
            else if (mode == 2) { mma_tf32_ss(d0, al, bh, id, s > 0); mma_tf32_ss(d0, ah, bl, id, 1); mma_tf32_ss(d0, ah, bh, id, 1); }
            else if (mode == 3) { mma_tf32_ss(d0, ah, bh, id, s > 0); mma_tf32_ss(d1, ah, bl, id, s > 0); mma_tf32_ss(d2, al, bh, id, s > 0); }
            else if (mode == 4) { mma_tf32_ts(d0, aH + s * 8, bh, id, s > 0); }
            else { mma_tf32_ts(d0, aH + s * 8, bh, id, s > 0); mma_tf32_ts(d0, aH + s * 8, bl, id, 1); mma_tf32_ts(d0, aL + s * 8, bh, id, 1); }
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0); fence_after();
    if (warp < 4) {
        const int m = warp * 32 + lane;
        float v[16], v1[16], v2[16];
        for (int h = 0; h < 2; ++h) {
            tmem_ld16(d0 + ((warp * 32) << 16) + h * 16, v); tmem_ld16(d1 + ((warp * 32) << 16) + h * 16, v1); tmem_ld16(d2 + ((warp * 32) << 16) + h * 16, v2);
            tmem_ld_wait();
            for (int i = 0; i < 16; ++i) D[m * N + h * 16 + i] = mode == 3 ? v[i] + (v1[i] + v2[i]) : v[i];
        }
    }
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tbase);
}
int main() {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    std::vector<double> ref(M * N);
    srand(7);
    for (auto& a : A) a = (rand() / (float)RAND_MAX - 0.5f) * 3.f;
    for (auto& b : B) b = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int kk = 0; kk < K; ++kk) s += double(A[m*K+kk]) * B[n*K+kk]; ref[m*N+n] = s; }
    // fp32 FMA reference error
    double ef = 0, nr = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { float s = 0; for (int kk = 0; kk < K; ++kk) s = fmaf(A[m*K+kk], B[n*K+kk], s); ef += (s - ref[m*N+n]) * (s - ref[m*N+n]); nr += ref[m*N+n]*ref[m*N+n]; }
    printf("fp32 FMA   normwise err %.3e\n", sqrt(ef / nr));
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size()*4); cudaMalloc(&dB, B.size()*4); cudaMalloc(&dD, D.size()*4);
    cudaMemcpy(dA, A.data(), A.size()*4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size()*4, cudaMemcpyHostToDevice);
    const char* names[6] = {"1xTF32", "3xTF32 big-first", "3xTF32 small-first", "3xTF32 separate acc", "TS 1xTF32", "TS 3xTF32"};
    for (int mode = 0; mode < 6; ++mode) {
        k<<<1, 256>>>(dA, dB, dD, mode);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("fail\n"); return 1; }
        cudaMemcpy(D.data(), dD, D.size()*4, cudaMemcpyDeviceToHost);
        double e = 0;
        for (int i = 0; i < M * N; ++i) e += (D[i] - ref[i]) * (D[i] - ref[i]);
        printf("%-22s normwise err %.3e\n", names[mode], sqrt(e / nr));
    }
    return 0;
}
