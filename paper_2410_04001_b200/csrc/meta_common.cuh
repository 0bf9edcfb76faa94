// Shared pieces of the tcgen05 meta kernel (pinn_meta_tc2.cuh): BF16 operand
// packing, the MMA issue helpers (32-bit descriptor words, 8-MMA batches),
// commit, reduction helpers and the activation jet with the SFU sin/cos.
// The first meta kernel (points on TMEM lanes, 16-neuron chunks; 118 TFLOP/s on
// c4) was retired in round 2: its N = 16 MMAs ran at 20 % tensor
// efficiency and the neurons-on-lanes kernel replaced it.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pinn_kernels.cuh"
#include "pinn_v2.cuh"
#include "umma.cuh"

namespace lrnr_b200 {
namespace mtc {

constexpr int P = 128;           // points per tile (MMA M, TMEM lanes)
constexpr int KC = 16;           // neurons per chunk
constexpr int RP = 64;           // max padded rank
constexpr int NWE = 16;          // epilogue warps
constexpr int ISSUER = NWE;      // MMA warp
constexpr int PRODUCER = NWE + 1;  // TMA warp
constexpr int NT = 32 * (NWE + 2);
constexpr int NBUF = 3;          // factor ring slots
constexpr int SLOT = (RP / 8) * (P / 8) * 128;  // bytes of one slot tile of SY / ST (16 KB)
constexpr int ZSLOT = (KC / 8) * (P / 8) * 128;  // bytes of one slot tile of a Z / G chunk (4 KB)
constexpr int BLK = 32 * (3 * RP) + 64;          // max factor block (reverse): 6208 B
constexpr int BLKS = (BLK + 127) / 128 * 128;
constexpr int OFF_SY = 0;
constexpr int OFF_ST = OFF_SY + 4 * SLOT;
constexpr int OFF_ZG = OFF_ST + 4 * SLOT;        // 2 buffers x [Z 4 slots | G 4 slots]
constexpr int ZGBUF = 8 * ZSLOT;
constexpr int OFF_RING = OFF_ZG + 2 * ZGBUF;
constexpr int OFF_ACC = OFF_RING + NBUF * BLKS;  // float acc4[4][R1]
constexpr int MAX_R1 = 512;
constexpr int SMEM_BYTES = OFF_ACC + 4 * MAX_R1 * 4;
// TMEM columns
constexpr uint32_t TM_P1 = 0, TM_DZ = 64, TM_D = 128, TM_Y = 256;



__device__ __forceinline__ int toff(int row, int col, int rows) {
    return ((col >> 3) * (rows >> 3) + (row >> 3)) * 64 + (row & 7) * 8 + (col & 7);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(amaj) << 15) |
           (static_cast<uint32_t>(bmaj) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
// One MMA, issued by the single MMA thread.
__device__ __forceinline__ void mma1(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// single-thread MMA from 32-bit descriptor low words (start >> 4 | LBO >> 4 << 16)
// with compile-time high words (SBO, version): keeps only 32-bit values live
template <uint32_t HA, uint32_t HB>
__device__ __forceinline__ void mma_lo(uint32_t d, uint32_t alo, uint32_t blo, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %5};\n\t"
        "mov.b64 db, {%2, %6};\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, p;\n\t}" ::"r"(d),
        "r"(alo), "r"(blo), "r"(idesc), "r"(acc), "n"(HA), "n"(HB)
        : "memory");
}
// 8 MMAs into one accumulator in a single asm block (one warp-uniformity region
// for ptxas instead of one per MMA): descriptor low words advance by AST / BST
// (16-byte units) per MMA; the first MMA accumulates iff acc0 != 0.
template <uint32_t HA, uint32_t HB, uint32_t AST, uint32_t BST>
__device__ __forceinline__ void mma_x8(uint32_t d, uint32_t alo, uint32_t blo, uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p0, pt;\n\t.reg .b32 al, bl;\n\t.reg .b64 da, db;\n\t"
        "setp.ne.b32 p0, %4, 0;\n\t"
        "setp.eq.b32 pt, 0, 0;\n\t"
        "mov.b64 da, {%1, %5};\n\t"
        "mov.b64 db, {%2, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, p0;\n\t"
        "add.u32 al, %1, %7;\n\tadd.u32 bl, %2, %8;\n\tmov.b64 da, {al, %5};\n\tmov.b64 db, {bl, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, pt;\n\t"
        "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 da, {al, %5};\n\tmov.b64 db, {bl, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, pt;\n\t"
        "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 da, {al, %5};\n\tmov.b64 db, {bl, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, pt;\n\t"
        "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 da, {al, %5};\n\tmov.b64 db, {bl, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, pt;\n\t"
        "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 da, {al, %5};\n\tmov.b64 db, {bl, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, pt;\n\t"
        "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 da, {al, %5};\n\tmov.b64 db, {bl, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, pt;\n\t"
        "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 da, {al, %5};\n\tmov.b64 db, {bl, %6};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, pt;\n\t}" ::"r"(d),
        "r"(alo), "r"(blo), "r"(idesc), "r"(acc0), "n"(HA), "n"(HB), "n"(AST), "n"(BST)
        : "memory");
}
__device__ __forceinline__ void commit1(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(umma::smem_addr(bar))
                 : "memory");
}
// timing knobs (dev aid; results are wrong when set): bit 0 skips the dU / dV
// MMAs, bit 1 the partial-gradient reductions, bit 2 the activation math
#ifndef MTC_SKIP
#define MTC_SKIP 0
#endif
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void sts64(unsigned char* p, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(umma::smem_addr(p)), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void sts128(unsigned char* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(umma::smem_addr(p)), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void red1(float* p, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}
// named barrier over the 16 epilogue warps
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NWE * 32) : "memory"); }

// Transpose-reduce over the warp: v[N] per lane (N = 4 or 16); returns the
// warp sum of v[idx], idx = the lane's bits (16, 8[, 4, 2]) read as a number;
// the lanes with the remaining low bits zero hold distinct indices.
template <int N>
__device__ __forceinline__ float treduce(float (&v)[N], int lane, int& idx) {
    int cnt = N, off = 16;
    idx = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (cnt > 1) {
            const int half = cnt / 2;
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int i = 0; i < N / 2; ++i)
                if (i < half) {
                    const float snd = up ? v[i] : v[i + half];
                    const float kp = up ? v[i + half] : v[i];
                    v[i] = kp + __shfl_xor_sync(0xffffffffu, snd, off);
                }
            if (up) idx += half;
            cnt = half;
            off >>= 1;
        }
    }
    float s = v[0];
    for (int o = off; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-phase cycle counters of CTA 0 (dev aid, -DMTC_TIMING): epilogue warp 0 and
// the MMA warp accumulate clock64 deltas per site; read g_mtc_timing[32].
#ifdef MTC_TIMING
__device__ unsigned long long g_mtc_timing[32];
#define MT(slot, ...)                                                                     \
    do {                                                                                  \
        const long long _t0 = clock64();                                                  \
        __VA_ARGS__;                                                                      \
        if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == ISSUER * 32))          \
            atomicAdd(&::lrnr_b200::mtc::g_mtc_timing[slot], static_cast<unsigned long long>(clock64() - _t0)); \
    } while (0)
#else
#define MT(slot, ...) __VA_ARGS__
#endif

template <int ACT>
__device__ __forceinline__ void act3(float a, float& sg, float& d1, float& d2, float& d3) {
    v2::act3<ACT, true, float>(a, sg, d1, d2, d3);  // sin: SFU after a Cody-Waite reduction (~1e-6)
}

}  // namespace mtc
}  // namespace lrnr_b200
