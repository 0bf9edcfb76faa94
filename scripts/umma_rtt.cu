// Microbenchmark (dev aid): round-trip latency MMA -> tcgen05.commit -> mbarrier ->
// waiting warp -> mbarrier arrive -> issuing thread, as in the meta kernel's
// issuer / epilogue handshake.
#include <cstdio>
#include <cstdint>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200::umma;
__global__ void k_rtt(unsigned long long* out, int iters, int nmma) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t full, back;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) { mbar_init(&full, 1); mbar_init(&back, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    fence_async_smem(); fence_before(); __syncthreads(); fence_after();
    const uint32_t sb = smem_addr(sm) >> 4;
    const uint64_t a = (uint64_t(desc_hi(128)) << 32) | (sb + (2048u >> 4 << 16));
    const uint64_t b = (uint64_t(desc_hi(128)) << 32) | (sb + (0x8000 >> 4) + (256u >> 4 << 16));
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (2u << 17) | (8u << 24);
    if (warp == 1 && lane == 0) {
        long long tot = 0;
        for (int it = 0; it < iters; ++it) {
            const long long t0 = clock64();
            for (int m = 0; m < nmma; ++m)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(0u), "l"(a), "l"(b), "r"(id), "r"(m) : "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(&full)) : "memory");
            mbar_wait(&back, it & 1);
            tot += clock64() - t0;
        }
        out[0] = tot / iters;
    } else if (warp == 2) {
        for (int it = 0; it < iters; ++it) {
            mbar_wait(&full, it & 1);
            fence_after();
            __syncwarp();
            if (lane == 0) mbar_arrive(&back);
        }
    }
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tb);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_rtt, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int nm : {1, 4, 16, 64}) {
        k_rtt<<<1, 128, 64 * 1024>>>(d, 200, nm);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%2d MMAs (M128 N16) + commit -> wait -> arrive -> wait: %llu cycles per round trip (%s)\n", nm, h, cudaGetErrorString(e));
    }
    return 0;
}
