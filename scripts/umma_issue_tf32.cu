// Microbenchmark (dev aid): issue cost of the tensor-core LRNR kernel's phase-1
// MMA group (4 jet slots x 4 K-steps x 3 products = 48 tcgen05.mma kind::tf32,
// M128 N32 K8, both operands in shared memory) in different issue forms:
//   0: warp-collective, elect.sync inside every MMA, runtime K loop (the kernel's form)
//   1: one elected lane, 12 MMAs per asm block (descriptor adds in PTX), 4 blocks
//   2: one elected lane, all 48 MMAs in one asm block
//   3: form 1 with kind::f16 (M128 N32 K16, 2 K-steps: 24 MMAs), for the rate
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/umma_issue_tf32.cu -o scripts/umma_issue_tf32
#include <cstdio>
#include <cstdint>
#include "../paper_2410_04001_b200/csrc/umma.cuh"
using namespace lrnr_b200;

// 12 MMAs of one jet slot: k-steps s = 0..3, products hi*hi, hi*lo, lo*hi.
// a / al: A hi / lo low words; b / bl: B hi / lo low words; per k-step the A low word
// advances by SA and the B low word by SB (16-byte units).
template <int SA, int SB>
__device__ __forceinline__ void mma12(uint32_t d, uint32_t a, uint32_t al, uint32_t b, uint32_t bl, uint32_t hi,
                                      uint32_t id) {
    asm volatile(
        "{\n\t.reg .b32 x, y, z, w;\n\t.reg .b64 da, db;\n\t.reg .pred pf, pt;\n\t"
        "setp.ne.b32 pf, 0, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
        "mov.b64 da, {%1, %5};\n\tmov.b64 db, {%3, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pf;\n\t"
        "mov.b64 db, {%4, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "mov.b64 da, {%2, %5};\n\tmov.b64 db, {%3, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "add.u32 x, %1, %7;\n\tadd.u32 y, %2, %7;\n\tadd.u32 z, %3, %8;\n\tadd.u32 w, %4, %8;\n\t"
        "mov.b64 da, {x, %5};\n\tmov.b64 db, {z, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "mov.b64 db, {w, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "mov.b64 da, {y, %5};\n\tmov.b64 db, {z, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "add.u32 x, x, %7;\n\tadd.u32 y, y, %7;\n\tadd.u32 z, z, %8;\n\tadd.u32 w, w, %8;\n\t"
        "mov.b64 da, {x, %5};\n\tmov.b64 db, {z, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "mov.b64 db, {w, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "mov.b64 da, {y, %5};\n\tmov.b64 db, {z, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "add.u32 x, x, %7;\n\tadd.u32 y, y, %7;\n\tadd.u32 z, z, %8;\n\tadd.u32 w, w, %8;\n\t"
        "mov.b64 da, {x, %5};\n\tmov.b64 db, {z, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "mov.b64 db, {w, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t"
        "mov.b64 da, {y, %5};\n\tmov.b64 db, {z, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %6, pt;\n\t}" ::"r"(d),
        "r"(a), "r"(al), "r"(b), "r"(bl), "r"(hi), "r"(id), "n"(SA), "n"(SB)
        : "memory");
}
__device__ __forceinline__ uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__global__ void k_issue(unsigned long long* out, int mode, int rk) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) umma::tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) {
        umma::mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tb;
    constexpr int P = 128, KC = 32, SY_TILE = P * 32;
    const uint32_t dhi = umma::desc_hi(128);
    const uint32_t lsy = umma::desc_lo(sm, (P / 8) * 128);
    const uint32_t lb32 = umma::desc_lo(sm + 8 * SY_TILE, (KC / 8) * 128);
    const uint32_t id = umma::idesc_tf32(P, KC);
    constexpr int SA_ = (2 * (P / 8) * 32) / 4, SB_ = (2 * (KC / 8) * 32) / 4;
    unsigned long long tiss = 0, ttot = 0;
    uint32_t ph = 0;
    if (warp == 1) {
        for (int it = 0; it < 65; ++it) {
            const long long t0 = clock64();
            if (mode == 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t dd = tbase + c * KC;
                    const uint32_t ah0 = lsy + ((2 * c) * SY_TILE >> 2), al0 = lsy + ((2 * c + 1) * SY_TILE >> 2);
                    const uint32_t bh0 = lb32, bl0 = lb32 + ((KC * rk) >> 2);
                    for (int s = 0; s < rk / 8; ++s) {
                        const uint32_t sa = s * (2 * (P / 8) * 32 >> 2), sb = s * (2 * (KC / 8) * 32 >> 2);
                        umma::mma_ss_w(dd, ah0 + sa, bh0 + sb, dhi, id, s > 0);
                        umma::mma_ss_w(dd, ah0 + sa, bl0 + sb, dhi, id, 1);
                        umma::mma_ss_w(dd, al0 + sa, bh0 + sb, dhi, id, 1);
                    }
                }
                umma::mma_commit_w(&bar);
            } else if (mode == 1 || mode == 2) {
                uint32_t e;
                asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
                if (e) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        mma12<SA_, SB_>(
                            tbase + c * KC, lsy + ((2 * c) * SY_TILE >> 2), lsy + ((2 * c + 1) * SY_TILE >> 2), lb32,
                            lb32 + ((KC * 32) >> 2), dhi, id);
                    umma::mma_commit_1(&bar);
                }
                __syncwarp();
            } else {
                uint32_t e;
                asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
                if (e) {
                    const uint32_t idf = idesc_f16(128, 32);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const uint32_t dd = tbase + c * KC;
                        const uint32_t a = lsy + ((2 * c) * SY_TILE >> 2), al = lsy + ((2 * c + 1) * SY_TILE >> 2);
#pragma unroll
                        for (int s = 0; s < 2; ++s) {
                            const uint32_t sa = s * (2 * (P / 8) * 32 >> 2), sb = s * (2 * (KC / 8) * 32 >> 2);
                            asm volatile(
                                "{\n\t.reg .b64 da, db;\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
                                "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(dd),
                                "r"(a + sa), "r"(lb32 + sb), "r"(dhi), "r"(s), "r"(idf)
                                : "memory");
                            asm volatile(
                                "{\n\t.reg .b64 da, db;\n\tmov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
                                "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t}" ::"r"(dd),
                                "r"(a + sa), "r"(lb32 + 1024 + sb), "r"(dhi), "r"(idf)
                                : "memory");
                            asm volatile(
                                "{\n\t.reg .b64 da, db;\n\tmov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
                                "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t}" ::"r"(dd),
                                "r"(al + sa), "r"(lb32 + sb), "r"(dhi), "r"(idf)
                                : "memory");
                        }
                    }
                    umma::mma_commit_1(&bar);
                }
                __syncwarp();
            }
            const long long t1 = clock64();
            umma::mbar_wait(&bar, ph & 1);
            ++ph;
            umma::fence_after();
            const long long t2 = clock64();
            if (it > 0) {
                tiss += t1 - t0;
                ttot += t2 - t0;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            out[0] = tiss / 64;
            out[1] = ttot / 64;
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tbase);
}


// generic: NW issuing warps, each NM single-lane MMAs (M128, N, K8 tf32 or K16 f16) into its own accumulator
template <int N, int NW, bool F16>
__global__ void k_rate(unsigned long long* out) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar[4];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) umma::tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) umma::mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tb;
    const uint32_t dhi = umma::desc_hi(128);
    const uint32_t la = umma::desc_lo(sm, 16 * 128);
    const uint32_t lb = umma::desc_lo(sm + 16384, (N / 8) * 128);
    const uint32_t id = F16 ? idesc_f16(128, N) : umma::idesc_tf32(128, N);
    constexpr int NM = 96;
    if (warp < NW) {
        const uint32_t d = tbase + warp * (512 / NW);
        __syncwarp();
        const long long t0 = clock64();
        uint32_t e;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
        if (e) {
#pragma unroll 8
            for (int i = 0; i < NM; ++i) {
                if (F16)
                    asm volatile(
                        "{\n\t.reg .b64 da, db;\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(d),
                        "r"(la + (i & 3) * 256), "r"(lb + (i & 3) * 64), "r"(dhi), "r"(i), "r"(id)
                        : "memory");
                else
                    asm volatile(
                        "{\n\t.reg .b64 da, db;\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t}" ::"r"(d),
                        "r"(la + (i & 3) * 256), "r"(lb + (i & 3) * 64), "r"(dhi), "r"(i), "r"(id)
                        : "memory");
            }
            umma::mma_commit_1(&bar[warp]);
        }
        __syncwarp();
        const long long t1 = clock64();
        umma::mbar_wait(&bar[warp], 0);
        const long long t2 = clock64();
        if ((threadIdx.x & 31) == 0) {
            out[2 * warp] = t1 - t0;
            out[2 * warp + 1] = t2 - t0;
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tbase);
}
template <int N, int NW, bool F16>
void rate() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    cudaFuncSetAttribute(k_rate<N, NW, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    k_rate<N, NW, F16><<<1, 128, 160 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[8];
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int w = 0; w < NW; ++w) mx = h[2 * w + 1] > mx ? h[2 * w + 1] : mx;
    const double floor_cyc = 128.0 * N / 256.0;
    printf("%s M128 N%-3d x %d warps: %s  %.1f cyc/MMA overall (floor %.0f) -> %.0f%% of peak\n", F16 ? "f16 " : "tf32", N,
           NW, cudaGetErrorString(e), double(mx) / (96 * NW), floor_cyc, 100.0 * floor_cyc / (double(mx) / (96 * NW)));
    cudaFree(d);
}

// TS form: A from TMEM (columns 256..), D at column 0; B from shared memory
template <int N, bool F16>
__global__ void k_rate_ts(unsigned long long* out) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) umma::tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) {
        umma::mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tb;
    const uint32_t dhi = umma::desc_hi(128);
    const uint32_t lb = umma::desc_lo(sm + 16384, (N / 8) * 128);
    const uint32_t id = F16 ? idesc_f16(128, N) : umma::idesc_tf32(128, N);
    constexpr int NM = 96;
    if (warp == 0) {
        const long long t0 = clock64();
        uint32_t e;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
        if (e) {
#pragma unroll 8
            for (int i = 0; i < NM; ++i) {
                const uint32_t a = tbase + 256 + (i & 15) * 8;
                if (F16)
                    asm volatile(
                        "{\n\t.reg .b64 db;\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "mov.b64 db, {%2, %3};\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %5, p;\n\t}" ::"r"(tbase),
                        "r"(a), "r"(lb + (i & 3) * 64), "r"(dhi), "r"(i), "r"(id)
                        : "memory");
                else
                    asm volatile(
                        "{\n\t.reg .b64 db;\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "mov.b64 db, {%2, %3};\n\t"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], db, %5, p;\n\t}" ::"r"(tbase),
                        "r"(a), "r"(lb + (i & 3) * 64), "r"(dhi), "r"(i), "r"(id)
                        : "memory");
            }
            umma::mma_commit_1(&bar);
        }
        __syncwarp();
        umma::mbar_wait(&bar, 0);
        const long long t2 = clock64();
        if ((threadIdx.x & 31) == 0) out[0] = t2 - t0;
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tbase);
}
template <int N, bool F16>
void rate_ts() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k_rate_ts<N, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    k_rate_ts<N, F16><<<1, 128, 160 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[1];
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    const double floor_cyc = 128.0 * N / 256.0;
    printf("TS %s M128 N%-3d: %s  %.1f cyc/MMA (floor %.0f)\n", F16 ? "f16 " : "tf32", N, cudaGetErrorString(e),
           double(h[0]) / 96, floor_cyc);
    cudaFree(d);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const char* names[] = {"warp-collective, elect per MMA (kernel form)", "elected lane, 12-MMA asm blocks",
                           "elected lane, 12-MMA asm blocks (repeat)", "elected lane, kind::f16 K16 (24 MMAs)"};
    for (int mode = 0; mode < 4; ++mode) {
        k_issue<<<1, 128, 160 * 1024>>>(d, mode, 32);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[2] = {0, 0};
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const int n = mode == 3 ? 24 : 48;
        printf("mode %d %-46s %s: issue %llu cyc (%.1f/MMA), issue+complete %llu cyc (%.1f/MMA)\n", mode, names[mode],
               cudaGetErrorString(e), h[0], double(h[0]) / n, h[1], double(h[1]) / n);
    }
    cudaFree(d);
    rate<32, 1, false>(); rate<32, 2, false>(); rate<32, 4, false>();
    rate<64, 1, false>(); rate<64, 2, false>();
    rate<128, 1, false>(); rate<128, 2, false>();
    rate<256, 1, false>(); rate<256, 2, false>();
    rate<32, 1, true>(); rate<64, 1, true>(); rate<128, 1, true>(); rate<256, 1, true>(); rate<256, 2, true>();
    rate_ts<16, false>(); rate_ts<32, false>(); rate_ts<64, false>(); rate_ts<128, false>(); rate_ts<32, true>(); rate_ts<64, true>();
    return 0;
}
