// Dev aid: per-SM throughput of f32 reductions into global memory (the meta kernel's dU / dV flush):
//   (a) red.global.add.v4.f32, 16 B per lane, lanes 256 B apart (one request per lane);
//   (b) the same with 8 consecutive lanes covering one 128-byte line;
//   (c) cp.reduce.async.bulk.global.shared::cta.add.f32 of a 16 KB shared-memory block.
// One CTA per SM, each into its own 64 KB partial (L2 resident).  Prints bytes / clk / SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/red_bw scripts/red_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* part, int iters, long long* cyc) {
    extern __shared__ __align__(128) unsigned char sm[];
    float* mine = part + (size_t)blockIdx.x * 16384;  // 64 KB
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 4096; i += 512) reinterpret_cast<float4*>(sm)[i % 1024] = make_float4(1.f, 1.f, 1.f, 1.f);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            // thread = row (tid & 127), 16 floats of the row's quarter (tid >> 7): 4 red4 per pass, 2 passes (dU, dV)
            for (int m = 0; m < 2; ++m) {
                float* b = mine + m * 8192 + (tid & 127) * 64 + (tid >> 7) * 16;
#pragma unroll
                for (int i = 0; i < 4; ++i) red4(b + 4 * i, 1.f, 1.f, 1.f, 1.f);
            }
        } else if (MODE == 1) {
            // 8 lanes cover one 128-byte line; a warp instruction covers 4 lines; 8 instructions per thread
            float* b = mine + warp * 1024 + (lane >> 3) * 64 + (lane & 7) * 4;
#pragma unroll
            for (int i = 0; i < 8; ++i) red4(b + (i >> 2) * 32 + (i & 3) * 256, 1.f, 1.f, 1.f, 1.f);
        } else {
            if (tid == 0) {
                for (int q = 0; q < 4; ++q)
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(mine + q * 4096),
                                 "r"((uint32_t)__cvta_generic_to_shared(sm)), "r"(16384)
                                 : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncthreads();
        }
    }
    if (MODE == 2 && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    int sms = 148;
    float* part; long long* cyc;
    cudaMalloc(&part, (size_t)sms * 65536);
    cudaMemset(part, 0, (size_t)sms * 65536);
    cudaMalloc(&cyc, sms * sizeof(long long));
    const int iters = 2000;
    long long h[148];
    const char* names[3] = {"red.v4, lanes 256 B apart", "red.v4, 8 lanes per 128-B line", "cp.reduce.async.bulk 16 KB"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<sms, 512, 16384>>>(part, iters, cyc);
            if (mode == 1) k<1><<<sms, 512, 16384>>>(part, iters, cyc);
            if (mode == 2) k<2><<<sms, 512, 16384>>>(part, iters, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        }
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += h[i];
        avg /= sms;
        printf("%-34s %8.0f cycles per 64 KB flush, %6.1f B/clk/SM (148 SMs at once)\n", names[mode], avg / iters, 65536.0 * iters / avg);
    }
    // one SM alone
    for (int mode = 0; mode < 3; ++mode) {
        if (mode == 0) k<0><<<1, 512, 16384>>>(part, iters, cyc);
        if (mode == 1) k<1><<<1, 512, 16384>>>(part, iters, cyc);
        if (mode == 2) k<2><<<1, 512, 16384>>>(part, iters, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
        printf("%-34s %8.0f cycles per 64 KB flush, %6.1f B/clk/SM (one SM alone)\n", names[mode], (double)h[0] / iters, 65536.0 * iters / h[0]);
    }
    float v; cudaMemcpy(&v, part, 4, cudaMemcpyDeviceToHost);
    printf("check: part[0] = %g\n", v);
    return 0;
}
