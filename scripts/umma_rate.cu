// Microbenchmark (dev aid): cycles per tcgen05.mma (bf16, SS, no swizzle) issued
// back to back from one warp, for the shapes the meta kernel uses.
#include <cstdio>
#include <cstdint>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200::umma;

__device__ __forceinline__ uint32_t idesc_bf16(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(amaj) << 15) | (uint32_t(bmaj) << 16) |
           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma64(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
template <int M, int N, int AMAJ, int NMMA, int NACC>
__global__ void k_rate(unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int warp = __shfl_sync(0xffffffff, threadIdx.x >> 5, 0);
    for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    fence_async_smem(); fence_before(); __syncthreads(); fence_after();
    if (warp == 0) {
        const uint32_t sb = __shfl_sync(0xffffffff, smem_addr(sm) >> 4, 0);
        const uint64_t hk = uint64_t(desc_hi(AMAJ ? 2048 : 128)) << 32;
        const uint64_t a = hk | (sb + ((AMAJ ? 128u : 2048u) >> 4 << 16));
        const uint64_t b = (uint64_t(desc_hi(128)) << 32) | (sb + (0x20000 >> 4) + ((256u >> 4) << 16));
        const uint32_t id = idesc_bf16(M, N, AMAJ, AMAJ);
        // warm-up
        for (int i = 0; i < 8; ++i) mma64(0, a, b, id, 0);
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_addr(&bar)) : "memory");
        mbar_wait(&bar, 0);
        const long long t0 = clock64();
#pragma unroll 16
        for (int i = 0; i < NMMA; ++i) mma64((i % NACC) * (NACC == 16 ? 16 : 64) + ((NACC == 2 && M == 64) ? 0 : 0), a + ((i & 7) * 256 >> 4), b + ((i & 3) * 512 >> 4), id, i >= NACC);
        const long long t1 = clock64();
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_addr(&bar)) : "memory");
        mbar_wait(&bar, 1);
        const long long t2 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tb);
}
template <int M, int N, int AMAJ, int NACC>
void run(const char* name) {
    unsigned long long* d; cudaMalloc(&d, 16);
    const int NM = 1024;
    cudaFuncSetAttribute(k_rate<M, N, AMAJ, NM, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_rate<M, N, AMAJ, NM, NACC><<<1, 128, 200 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double macs = double(M) * N * 16;
    printf("%-22s acc x%-2d %s issue %.1f cyc/mma, complete %.1f cyc/mma (math floor %.1f)\n", name, NACC, cudaGetErrorString(e),
           double(h[0]) / NM, double(h[1]) / NM, macs / 4096.0);
    cudaFree(d);
}
int main() {
    run<128, 16, 0, 1>("M128 N16 K-major");
    run<128, 16, 0, 2>("M128 N16 K-major");
    run<128, 16, 0, 4>("M128 N16 K-major");
    run<128, 16, 0, 16>("M128 N16 K-major");
    run<128, 64, 0, 1>("M128 N64 K-major");
    run<128, 64, 0, 4>("M128 N64 K-major");
    run<128, 128, 0, 1>("M128 N128 K-major");
    run<128, 128, 0, 4>("M128 N128 K-major");
    run<64, 16, 1, 1>("M64 N16 MN-major");
    run<64, 16, 1, 2>("M64 N16 MN-major");
    run<64, 16, 1, 4>("M64 N16 MN-major");
    run<64, 16, 1, 16>("M64 N16 MN-major");
    run<64, 32, 1, 1>("M64 N32 MN-major");
    run<64, 32, 1, 4>("M64 N32 MN-major");
    return 0;
}
