// Microbenchmark (dev aid): MMA issue cost from a single-lane region when the
// descriptor / TMEM operands live in regular registers (R2UR.BROADCAST waterfall
// per MMA, as in the meta kernels' issuer) vs uniform-register operands.
#include <cstdio>
#include <cstdint>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
#include "../paper_2410_04001_b200/csrc/pinn_meta_tc.cuh"
using namespace lrnr_b200;
__global__ void k_issue(unsigned long long* out, const uint32_t* __restrict__ vals, int mode) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) umma::tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) { umma::mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    umma::fence_async_smem(); umma::fence_before(); __syncthreads(); umma::fence_after();
    if (warp == 1 && lane == 0) {
        const uint32_t sb = umma::smem_addr(sm) >> 4;
        // "non-uniform" operands: loaded from global memory by the single thread
        const uint32_t boff = vals[0], d = vals[1], id = mtc::idesc_bf16(128, 64, 1, 1);
        constexpr uint32_t H = (2048u >> 4) | (1u << 14);
        const long long t0 = clock64();
        for (int it = 0; it < 64; ++it) {
            const uint32_t a = sb + (128u << 16) + (it & 1) * 256, b = sb + boff + (128u << 16) + (it & 1) * 512;
            if (mode == 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k) mtc::mma_lo<H, H>(d, a + k * 16, b + k * 16, id, k > 0);
            } else {
                mtc::mma_x8<H, H, 16, 16>(d, a, b, id, 0);
            }
        }
        mtc::commit1(&bar);
        umma::mbar_wait(&bar, 0);
        out[0] = (clock64() - t0) / (64 * 8);
    }
    umma::fence_before(); __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tb);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    uint32_t* v; cudaMalloc(&v, 8);
    uint32_t hv[2] = {0x4000u >> 4, 256u};
    cudaMemcpy(v, hv, 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    for (int mode = 0; mode < 2; ++mode) {
        k_issue<<<1, 128, 96 * 1024>>>(d, v, mode);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %llu cycles per MMA (M128 N64 K16, floor 32-48) (%s)\n", mode, mode ? "mma_x8" : "mma_lo", h, cudaGetErrorString(e));
    }
    return 0;
}
