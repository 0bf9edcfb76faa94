// Microbenchmark (dev aid): tcgen05.ld throughput per SM (16 warps, 32x32b.x16 / x32 loads).
#include <cstdio>
#include <cstdint>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200;
template <int NW>
__global__ void k_bw(unsigned long long* out, float* sink, int iters) {
    __shared__ uint32_t tb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) umma::tmem_alloc<512>(&tb);
    umma::fence_before(); __syncthreads(); umma::fence_after();
    const uint32_t tl = tb + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        float v[16], w[16];
        umma::tmem_ld16(tl + (it & 1) * 16, v);
        umma::tmem_ld16(tl + 32 + (it & 1) * 16, w);
        umma::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += v[i] + w[i];
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    umma::fence_before(); __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tb);
}
template <int NW>
void run() {
    unsigned long long* d; cudaMalloc(&d, 8);
    float* s; cudaMalloc(&s, 148 * 1024 * 4);
    const int iters = 4096;
    k_bw<NW><<<148, NW * 32>>>(d, s, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = double(NW) * 32 * 32 * 4 * iters;
    printf("%2d warps: %.1f B/clk per SM (%s)\n", NW, bytes / h, cudaGetErrorString(e));
}
int main() { run<4>(); run<8>(); run<16>(); run<32>(); return 0; }
