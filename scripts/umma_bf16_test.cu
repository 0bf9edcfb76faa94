// Self-test of the bf16 tcgen05 layouts used by the meta tensor-core kernel
// (dev aid; run on a B200):
//   (1) K-major A (points x ranks tile) x K-major B, M = 128, N = 16
//   (2) MN-major A (the same tile read as ranks x points) x MN-major B (points x
//       neurons tile), M = 64, N = 16, K = 128 points; D in the M = 64 TMEM layout
//       (row m -> lane (m % 16) + 32 (m / 16)); also at TMEM lane offset 16
//   (3) K-major A (points x neurons tile, K = 16) x K-major B, M = 128, N = 64
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200::umma;

constexpr int P = 128, R = 64, NK = 16, N3 = 64;

// tile element (row p, col j) of a [colgroup][rowgroup (P/8)][8 rows][8 cols] bf16 tile
__host__ __device__ inline int toff(int p, int j, int rows) { return ((j >> 3) * (rows >> 3) + (p >> 3)) * 64 + (p & 7) * 8 + (j & 7); }

__device__ inline uint32_t idesc_bf16(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(amaj) << 15) | (uint32_t(bmaj) << 16) |
           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ inline uint64_t desc(const void* base, uint32_t lbo, uint32_t sbo) { return smem_desc(base, lbo, sbo); }
__device__ inline void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}

__global__ void k_test(const float* A, const float* B1, const float* G, const float* W3, float* D1, float* D2,
                       float* D2b, float* D3) {
    extern __shared__ __align__(128) unsigned char sm[];
    __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(sm);   // P x R tile: 16 KB
    __nv_bfloat16* sB1 = sA + P * R;                             // NK x R (K-major B): 2 KB
    __nv_bfloat16* sG = sB1 + NK * R;                            // P x NK tile: 4 KB
    __nv_bfloat16* sW3 = sG + P * NK;                            // N3 x NK (K-major B): 2 KB
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < P * R; i += blockDim.x) sA[toff(i / R, i % R, P)] = __float2bfloat16(A[i]);
    for (int i = tid; i < NK * R; i += blockDim.x) sB1[toff(i / R, i % R, NK)] = __float2bfloat16(B1[i]);
    for (int i = tid; i < P * NK; i += blockDim.x) sG[toff(i / NK, i % NK, P)] = __float2bfloat16(G[i]);
    for (int i = tid; i < N3 * NK; i += blockDim.x) sW3[toff(i / NK, i % NK, N3)] = __float2bfloat16(W3[i]);
    if (warp == 0) tmem_alloc<256>(&tbase);
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t t0 = tbase;
    if (tid == 0) {
        // (1) D1[p][n] = sum_j A[p][j] B1[n][j]: K-major, LBO = col-group stride, SBO = 128
        for (int s = 0; s < R / 16; ++s)
            mma_bf16(t0 + 0, desc(sA + s * 2 * (P / 8) * 64, (P / 8) * 128, 128),
                     desc(sB1 + s * 2 * (NK / 8) * 64, (NK / 8) * 128, 128), idesc_bf16(128, NK, 0, 0), s > 0);
        // (2) D2[j][n] = sum_p A[p][j] G[p][n]: MN-major, LBO = K-group (8 points) stride 128 B,
        //     SBO = MN-group stride
        for (int s = 0; s < P / 16; ++s) {
            const uint64_t a = desc(sA + s * 2 * 64, 128, (P / 8) * 128);
            const uint64_t b = desc(sG + s * 2 * 64, 128, (P / 8) * 128);
            mma_bf16(t0 + 32, a, b, idesc_bf16(64, NK, 1, 1), s > 0);
            mma_bf16(t0 + 48 + (16u << 16), a, b, idesc_bf16(64, NK, 1, 1), s > 0);
        }
        // (3) D3[p][n] = sum_k G[p][k] W3[n][k]: K = 16 (one step)
        mma_bf16(t0 + 64, desc(sG, (P / 8) * 128, 128), desc(sW3, (N3 / 8) * 128, 128), idesc_bf16(128, N3, 0, 0), 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    if (warp < 4) {
        const uint32_t tl = t0 + ((warp * 32) << 16);
        float v[16];
        tmem_ld16(tl + 0, v);
        tmem_ld_wait();
        for (int i = 0; i < 16; ++i) D1[(warp * 32 + lane) * NK + i] = v[i];
        tmem_ld16(tl + 32, v);
        tmem_ld_wait();
        if (lane < 16)
            for (int i = 0; i < 16; ++i) D2[(warp * 16 + lane) * NK + i] = v[i];
        tmem_ld16(tl + 48, v);
        tmem_ld_wait();
        if (lane >= 16)
            for (int i = 0; i < 16; ++i) D2b[(warp * 16 + lane - 16) * NK + i] = v[i];
        for (int h = 0; h < 4; ++h) {
            tmem_ld16(tl + 64 + h * 16, v);
            tmem_ld_wait();
            for (int i = 0; i < 16; ++i) D3[(warp * 32 + lane) * N3 + h * 16 + i] = v[i];
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(t0);
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
    std::vector<float> A(P * R), B1(NK * R), G(P * NK), W3(N3 * NK);
    srand(3);
    auto rnd = [] { return float(rand() % 2001 - 1000) / 700.f; };
    for (auto& a : A) a = rnd();
    for (auto& a : B1) a = rnd();
    for (auto& a : G) a = rnd();
    for (auto& a : W3) a = rnd();
    std::vector<float> r1(P * NK), r2(R * NK), r3(P * N3);
    for (int p = 0; p < P; ++p)
        for (int n = 0; n < NK; ++n) {
            double s = 0;
            for (int j = 0; j < R; ++j) s += double(bf(A[p * R + j])) * bf(B1[n * R + j]);
            r1[p * NK + n] = float(s);
        }
    for (int j = 0; j < R; ++j)
        for (int n = 0; n < NK; ++n) {
            double s = 0;
            for (int p = 0; p < P; ++p) s += double(bf(A[p * R + j])) * bf(G[p * NK + n]);
            r2[j * NK + n] = float(s);
        }
    for (int p = 0; p < P; ++p)
        for (int n = 0; n < N3; ++n) {
            double s = 0;
            for (int k = 0; k < NK; ++k) s += double(bf(G[p * NK + k])) * bf(W3[n * NK + k]);
            r3[p * N3 + n] = float(s);
        }
    float *dA, *dB1, *dG, *dW3, *d1, *d2, *d2b, *d3;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB1, B1.size() * 4);
    cudaMalloc(&dG, G.size() * 4);
    cudaMalloc(&dW3, W3.size() * 4);
    cudaMalloc(&d1, r1.size() * 4);
    cudaMalloc(&d2, r2.size() * 4);
    cudaMalloc(&d2b, r2.size() * 4);
    cudaMalloc(&d3, r3.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB1, B1.data(), B1.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dW3, W3.data(), W3.size() * 4, cudaMemcpyHostToDevice);
    const int smem = (P * R + NK * R + P * NK + N3 * NK) * 2;
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_test<<<1, 128, smem>>>(dA, dB1, dG, dW3, d1, d2, d2b, d3);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 2;
    std::vector<float> g1(r1.size()), g2(r2.size()), g2b(r2.size()), g3(r3.size());
    cudaMemcpy(g1.data(), d1, g1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(g2.data(), d2, g2.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(g2b.data(), d2b, g2b.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(g3.data(), d3, g3.size() * 4, cudaMemcpyDeviceToHost);
    auto err = [](const std::vector<float>& a, const std::vector<float>& b) {
        double e = 0;
        for (size_t i = 0; i < a.size(); ++i) e = fmax(e, fabs(a[i] - b[i]) / (1.0 + fabs(b[i])));
        return e;
    };
    const double e1 = err(g1, r1), e2 = err(g2, r2), e2b = err(g2b, r2), e3 = err(g3, r3);
    printf("(1) K-major M128 N16 K64: %g\n(2) MN-major M64 N16 K128: %g (lane-16 copy: %g)\n(3) K-major M128 N64 K16: %g\n",
           e1, e2, e2b, e3);
    if (e2 > 1e-4)
        for (int i = 0; i < 4; ++i) printf("  r2 %g got %g\n", r2[i * NK], g2[i * NK]);
    return (e1 < 1e-4 && e2 < 1e-4 && e3 < 1e-4) ? 0 : 1;
}
