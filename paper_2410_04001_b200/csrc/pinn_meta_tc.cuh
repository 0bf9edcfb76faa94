// Tensor-core (tcgen05, BF16 operands, FP32 accumulate) kernel for the meta
// step: the fused LRNR jet forward + residual + reverse sweep to s, U, V and b
// (training.cpp:335-426 with the PinnTermEmitter interior terms; the factor
// VJPs are AffineFactoredJet's U/V/b branches, autodiff.cpp:501-505,524-534,
// 553-560).  BASELINE config 4 names BF16/TF32 inputs with FP32 accumulation.
//
// A CTA owns a tile of P = 128 collocation points (TMEM lane = point = MMA M)
// and walks every transition l (rank space y_l -> the M_{l+1} neurons of hidden
// layer l+1 -> y_{l+1}) in chunks of KC = 16 neurons.  The 4 jet slots are 4
// independent MMAs, so the epilogue thread that owns a point sees all 4 slots
// of a neuron.  Per chunk:
//   forward   P1  A_c  = SY_l U_c^T            (M 128, N 16, K rp_l)  -> TMEM
//             epi Z_c  = sigma-jet(A_c + b_c)  -> bf16 smem
//             P2  Y   += Z_c V_c               (M 128, N rp_{l+1}, K 16) -> TMEM
//   reverse   P1  A_c  = SY_l U_c^T  (recompute: the forward A is not stored --
//                                     at c4 it would be 57 KB/point of HBM traffic)
//                 DZ_c = ST_{l+1} V_c^T
//             epi G_c  = sigma-jet VJP(A_c + b_c, DZ_c), Z_c again -> bf16 smem
//                 db_l[c] += sum_p G_c[p][u-slot]
//             P2  T   += G_c U_c               (M 128, N rp_l, K 16)
//             P3  dU_l^T[:, c]     = SY_l^T G_c      (M 64 ranks, N 16, K = 4 slots x 128 points,
//                 dV_{l+1}^T[:, c] = ST_{l+1}^T Z_c   MN-major operands, TMEM lanes 0-15 / 16-31)
//             flush: dU / dV chunk -> this CTA's partial (red.global.add, one writer per address)
// Shared memory (bf16 canonical no-swizzle tiles, [col group][row group][8][8]):
//   SY, ST: 4 slots x 128 points x 64 ranks (64 KB each)
//   Z/G chunk buffers (double buffered, 64 KB), factor-chunk ring (TMA bulk copies)
// TMEM (512 columns): P1 [0,128) | dU/dV D [128,160) | Y / T [256,512).
// Warp roles: 16 epilogue warps (lane quarter = warp % 4, neuron / rank group =
// warp / 4), warp 16 issues the MMAs, warp 17 feeds the factor ring.
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

struct MetaNet {
    int L;
    int M[kMaxL + 1];
    int r[kMaxL];
    int rp[kMaxL];          // ranks padded to a multiple of 16
    int nc[kMaxL];          // chunks of transition l (M_{l+1} / 16, rounded up)
    int soff[kMaxL + 1];
    int yoff[kMaxL];        // y_l in the per-CTA scratch: [p][rp_l][4] floats, l <= L-2
    int64_t ystride;
    int rtotal;
    const unsigned char* blocks;  // bf16 factor blocks (bias fp32 inside)
    const int64_t* sched_off;     // byte offset per schedule entry
    const int* sched_bytes;
    int sched_len;                // entries per tile (forward then reverse chunks)
    const float* V0;              // 2 x r[0]
    const float* ulast;           // r[L-1] then b_{L-1}[0]
    // per-CTA partial gradient (floats): transition l, chunk c at gbase[l] + c * 2048:
    // dU_l^T [64][16] then dV_{l+1}^T [64][16]; then 4 quarter copies (stride QS) of
    // db_l (qdb[l] + k), dU_{L-1} (qdUL + j), db_{L-1} (qdbL), dV_0 (qdV0 + i * r0 + j)
    int64_t gbase[kMaxL];
    int64_t qbase;
    int QS;
    int qdb[kMaxL];
    int qdUL, qdbL, qdV0;
    int64_t wg_stride;
};

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

template <int ACT>
__global__ void __launch_bounds__(NT, 1)
meta_tc_kernel(const MetaNet net, const RunGeom g, const double* __restrict__ pts, const double* __restrict__ svec,
               const double* __restrict__ mus, const float w, float* __restrict__ scratch, float* __restrict__ part,
               float* __restrict__ wgrad, unsigned long long* __restrict__ bad, const TermSpec* __restrict__ spec,
               const int objective) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[NBUF], slotfree[NBUF], p1full[2], p1empty[2], zgfull[2], zgfree[2],
        dready[2], dfree[2], tdone, sready;
    __shared__ uint32_t tmem_base;
    float* acc4 = reinterpret_cast<float*>(sm + OFF_ACC);

    const int tid = threadIdx.x, lane = tid & 31;
    // warp index through a shuffle: provably warp-uniform, so the MMA warp's
    // descriptor arithmetic stays on the uniform datapath (no R2UR per MMA)
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int quarter = warp & 3, grp = warp >> 2;
    const int p = quarter * 32 + lane;  // epilogue: the point (TMEM lane) of this thread
    const int L = net.L;
    const int R1 = 1 + net.rtotal;
    float* scr = scratch + static_cast<int64_t>(blockIdx.x) * net.ystride;
    float* wg = wgrad + static_cast<int64_t>(blockIdx.x) * net.wg_stride;
    float* wq = wg + net.qbase + quarter * net.QS;  // this quarter's copy of the small gradients

    for (int k = tid; k < 4 * MAX_R1; k += NT) acc4[k] = 0.f;
    for (int k = tid; k < (OFF_RING - OFF_SY) / 16; k += NT)
        reinterpret_cast<uint4*>(sm + OFF_SY)[k] = make_uint4(0, 0, 0, 0);
    if (warp == 0) umma::tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < NBUF; ++i) {
            umma::mbar_init(&full[i], 1);
            umma::mbar_init(&slotfree[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&p1full[i], 1);
            umma::mbar_init(&p1empty[i], NWE);
            umma::mbar_init(&zgfull[i], NWE);
            umma::mbar_init(&zgfree[i], 1);
            umma::mbar_init(&dready[i], 1);
            umma::mbar_init(&dfree[i], NWE);
        }
        umma::mbar_init(&tdone, 1);
        umma::mbar_init(&sready, NWE);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    // all 512 columns are allocated, so the TMEM base address is 0 (lane 0, column 0)
    const uint32_t tbase = 0;
    if (tid == 0 && tmem_base != 0) __trap();

    int64_t total_tiles = 0;
    for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
        const int seg = static_cast<int>(u % g.units_per_inst);
        const int t_lo = seg * g.tiles_per_unit;
        total_tiles += min(g.tiles_per_inst, t_lo + g.tiles_per_unit) - t_lo;
    }
    const int64_t total_chunks = total_tiles * net.sched_len;

    auto wait = [](uint64_t* bar, uint32_t parity) {
        umma::mbar_wait(bar, parity);
        umma::fence_after();
    };

#ifdef MTC_TIMING
    const long long t_start = clock64();
#endif
    // =========================== TMA producer ===========================
    if (warp == PRODUCER) {
        if (lane == 0) {
            for (int64_t q = 0; q < total_chunks; ++q) {
                const int s = static_cast<int>(q % NBUF);
                if (q >= NBUF) umma::mbar_wait(&slotfree[s], static_cast<uint32_t>(((q / NBUF) - 1) & 1));
                const int e = static_cast<int>(q % net.sched_len);
                v2::mbar_expect_tx(&full[s], static_cast<uint32_t>(net.sched_bytes[e]));
                v2::bulk_g2s(sm + OFF_RING + s * BLKS, net.blocks + net.sched_off[e],
                             static_cast<uint32_t>(net.sched_bytes[e]), &full[s]);
            }
        }
        __syncwarp();
    }
    // =========================== MMA issuer ===========================
    // One thread (lane 0) issues every MMA: in a single-thread region ptxas keeps
    // the descriptors on the uniform datapath (UIADD3 + UTCHMMA per MMA); the
    // warp-collective elected form cost ~165 cycles per MMA (R2UR.BROADCAST chains).
    else if (warp == ISSUER) {
      if (lane == 0) {
        const uint32_t sbase = umma::smem_addr(sm) >> 4;
        constexpr uint32_t HK = (128u >> 4) | (1u << 14);   // SBO 128 B (K-major tiles, ring tiles)
        constexpr uint32_t HM = (2048u >> 4) | (1u << 14);  // SBO 2048 B (MN-major SY / ST / G / Z)
        // descriptor low word: start address >> 4 | LBO >> 4 << 16
        auto lo = [&](uint32_t off, uint32_t lbo) -> uint32_t { return sbase + (off >> 4) + ((lbo >> 4) << 16); };
        uint32_t qc = 0, rc = 0, pe = 0;  // chunk counter, reverse-chunk counter, p1empty completions consumed
        uint32_t tcount = 0;
        auto drain_p1empty = [&](uint32_t end) {  // consume p1empty completions of chunks < end, in order
            for (; pe < end; ++pe) MT(18, wait(&p1empty[pe & 1], static_cast<uint32_t>((pe >> 1) & 1)));
        };
        auto ring = [&](uint32_t q) { return static_cast<uint32_t>(OFF_RING + static_cast<int>(q % NBUF) * BLKS); };
        auto wait_full = [&](uint32_t q) { MT(17, wait(&full[q % NBUF], static_cast<uint32_t>((q / NBUF) & 1))); };
        for (int64_t t = 0; t < total_tiles; ++t) {
            // ---------------- forward ----------------
            for (int l = 0; l + 1 < L; ++l) {
                MT(16, wait(&sready, tcount & 1));  // SY_l in shared memory
                const int RL = net.rp[l], RN = net.rp[l + 1], n = net.nc[l];
                const uint32_t id1 = idesc_bf16(P, KC, 0, 0), id2 = idesc_bf16(P, RN, 0, 0);
                auto p1 = [&](uint32_t q) {
                    wait_full(q);
                    const uint32_t a0 = lo(OFF_SY, 2048), b0 = lo(ring(q), 256);
                    const uint32_t d0 = tbase + TM_P1 + static_cast<uint32_t>(q & 1) * 64;
                    const int nk = RL / 16;
#pragma unroll
                    for (int k = 0; k < RP / 16; ++k)
                        if (k < nk)
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                mma_lo<HK, HK>(d0 + c * 16, a0 + ((c * SLOT + k * 4096) >> 4), b0 + ((k * 512) >> 4), id1, k > 0);
                    commit1(&p1full[q & 1]);
                };
                const uint32_t q0 = qc;
                MT(21, p1(q0));
                for (int ch = 0; ch < n; ++ch) {
                    const uint32_t q = q0 + ch;
                    if (ch + 1 < n) {
                        drain_p1empty(q);
                        MT(21, p1(q + 1));
                    }
                    MT(19, wait(&zgfull[q & 1], static_cast<uint32_t>((q >> 1) & 1)));
                    const uint32_t a0 = lo(OFF_ZG + static_cast<uint32_t>(q & 1) * ZGBUF, 2048);
                    const uint32_t b0 = lo(ring(q) + RL * 32 + 64, (RN / 8) * 128);
#pragma unroll
                    for (int c = 0; c < 4; ++c) mma_lo<HK, HK>(tbase + TM_Y + c * 64, a0 + ((c * ZSLOT) >> 4), b0, id2, ch > 0);
                    commit1(&zgfree[q & 1]);
                    commit1(&slotfree[q % NBUF]);
                }
                commit1(&tdone);
                drain_p1empty(q0 + n);
                qc += n;
                ++tcount;
            }
            // ---------------- reverse ----------------
            for (int l = L - 2; l >= 0; --l) {
                MT(16, wait(&sready, tcount & 1));  // ST_{l+1} and SY_l in shared memory
                const int RL = net.rp[l], RN = net.rp[l + 1], n = net.nc[l];
                const uint32_t id1 = idesc_bf16(P, KC, 0, 0), id2 = idesc_bf16(P, RL, 0, 0);
                const uint32_t id3 = idesc_bf16(64, KC, 1, 1);
                auto p1 = [&](uint32_t q) {
                    wait_full(q);
                    const uint32_t ay = lo(OFF_SY, 2048), at = lo(OFF_ST, 2048), bu = lo(ring(q), 256),
                                   bv = lo(ring(q) + RL * 32 + 64, 256);
                    const int nkl = RL / 16, nkn = RN / 16;
#pragma unroll
                    for (int k = 0; k < RP / 16; ++k)
                        if (k < nkl)
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                mma_lo<HK, HK>(tbase + TM_P1 + c * 16, ay + ((c * SLOT + k * 4096) >> 4), bu + ((k * 512) >> 4),
                                               id1, k > 0);
#pragma unroll
                    for (int k = 0; k < RP / 16; ++k)
                        if (k < nkn)
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                mma_lo<HK, HK>(tbase + TM_DZ + c * 16, at + ((c * SLOT + k * 4096) >> 4), bv + ((k * 512) >> 4),
                                               id1, k > 0);
                    commit1(&p1full[q & 1]);
                };
                const uint32_t q0 = qc;
                MT(22, p1(q0));
                for (int ch = 0; ch < n; ++ch) {
                    const uint32_t q = q0 + ch;
                    if (ch + 1 < n) {
                        drain_p1empty(q + 1);
                        MT(22, p1(q + 1));
                    }
                    MT(19, wait(&zgfull[q & 1], static_cast<uint32_t>((q >> 1) & 1)));
                    if (rc >= 2) MT(20, wait(&dfree[rc & 1], static_cast<uint32_t>(((rc - 2) >> 1) & 1)));
                    const uint32_t zo = OFF_ZG + static_cast<uint32_t>(q & 1) * ZGBUF, go = zo + 4 * ZSLOT;
                    // T += G U
                    const uint32_t ag = lo(go, 2048), but = lo(ring(q) + RL * 32 + 64 + RN * 32, (RL / 8) * 128);
#pragma unroll
                    for (int c = 0; c < 4; ++c) mma_lo<HK, HK>(tbase + TM_Y + c * 64, ag + ((c * ZSLOT) >> 4), but, id2, ch > 0);
                    // dU_l^T = SY^T G (lanes 0-15), dV_{l+1}^T = ST^T Z (lanes 16-31), interleaved
                    const uint32_t dd = tbase + TM_D + static_cast<uint32_t>(rc & 1) * 16;
                    const uint32_t my = lo(OFF_SY, 128), mg = lo(go, 128), mt = lo(OFF_ST, 128), mz = lo(zo, 128);
                    if (!(MTC_SKIP & 1)) {
#pragma unroll
                        for (int c = 0; c < 4; ++c)
#pragma unroll
                            for (int k = 0; k < P / 16; ++k) {
                                mma_lo<HM, HM>(dd, my + ((c * SLOT + k * 256) >> 4), mg + ((c * ZSLOT + k * 256) >> 4), id3,
                                               (c | k) != 0);
                                mma_lo<HM, HM>(dd + (16u << 16), mt + ((c * SLOT + k * 256) >> 4),
                                               mz + ((c * ZSLOT + k * 256) >> 4), id3, (c | k) != 0);
                            }
                    }
                    commit1(&zgfree[q & 1]);
                    commit1(&dready[rc & 1]);
                    commit1(&slotfree[q % NBUF]);
                    ++rc;
                }
                commit1(&tdone);
                drain_p1empty(q0 + n);
                qc += n;
                ++tcount;
            }
        }
      }
      __syncwarp();  // converge the MMA warp before the CTA barrier at the end
    }
    // =========================== epilogue warps ===========================
    else {
        int64_t qc = 0, rc = 0;
        uint32_t tcount = 0;
        const uint32_t tl = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
        auto signal = [&](uint64_t* bar) {
            umma::fence_before();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(bar);
        };
        // SY_l (bf16) for this thread's point from the y_l scratch, ranks of group grp
        auto build_sy = [&](int l, const double* sv) {
            const int RL = net.rp[l];
            if (16 * grp >= RL) return;
            const float* yp = scr + net.yoff[l] + (p * RL + 16 * grp) * 4;
            const double* sl = sv + net.soff[l];
            const int rt = net.r[l];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float v[4][8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int j = 16 * grp + 8 * h + i;
                    const float4 y4 = *reinterpret_cast<const float4*>(yp + (8 * h + i) * 4);
                    const float sj = j < rt ? static_cast<float>(sl[j]) : 0.f;
                    v[0][i] = sj * y4.x;
                    v[1][i] = sj * y4.y;
                    v[2][i] = sj * y4.z;
                    v[3][i] = sj * y4.w;
                }
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    sts128(sm + OFF_SY + c * SLOT + toff(p, 16 * grp + 8 * h, P) * 2, pack_bf16(v[c][0], v[c][1]),
                           pack_bf16(v[c][2], v[c][3]), pack_bf16(v[c][4], v[c][5]), pack_bf16(v[c][6], v[c][7]));
            }
        };
        // flush reverse chunk rr (transition l, chunk ch): dU_l^T / dV_{l+1}^T columns 4 grp .. 4 grp + 3
        auto flush = [&](int64_t rr, int l, int ch) {
            MT(8, wait(&dready[rr & 1], static_cast<uint32_t>((rr >> 1) & 1)));
            float v[4];
            umma::tmem_ld4(tl + TM_D + static_cast<uint32_t>(rr & 1) * 16 + 4 * grp, v);
            umma::tmem_ld_wait();
            signal(&dfree[rr & 1]);
            const int row = 16 * quarter + (lane & 15);
            const bool isV = lane >= 16;
            if (!(MTC_SKIP & 2) && row < (isV ? net.r[l + 1] : net.r[l]))
                red4(wg + net.gbase[l] + static_cast<int64_t>(ch) * 2048 + (isV ? 1024 : 0) + row * 16 + 4 * grp, v[0],
                     v[1], v[2], v[3]);
        };

        for (int64_t unit = blockIdx.x; unit < g.n_units; unit += gridDim.x) {
            const int64_t inst = unit / g.units_per_inst;
            const int seg = static_cast<int>(unit % g.units_per_inst);
            const int t_lo = seg * g.tiles_per_unit;
            const int t_hi = min(g.tiles_per_inst, t_lo + g.tiles_per_unit);
            const double* sv = svec + inst * net.rtotal;
            const float mu0 = float(mus[3 * inst]), mu1 = float(mus[3 * inst + 1]), mu2 = float(mus[3 * inst + 2]);

            for (int tile = t_lo; tile < t_hi; ++tile) {
                const int64_t pi = static_cast<int64_t>(tile) * P + p;
                const bool valid = pi < g.n_per_inst;
                const int64_t gp = inst * g.n_per_inst + pi;
                const float x = valid ? float(pts[2 * gp]) : 0.f;
                const float tt = valid ? float(pts[2 * gp + 1]) : 0.f;
                // ---------------- input layer: y_0 = V_0^T z_0 ----------------
                if (grp == 0) {
                    const int r0 = net.r[0], RL = net.rp[0];
                    float* yp = scr + net.yoff[0] + p * RL * 4;
                    for (int h = 0; h < RL / 8; ++h) {
                        float v[4][8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int j = 8 * h + i;
                            float y0 = 0.f, y1 = 0.f, y2 = 0.f, sj = 0.f;
                            if (j < r0) {
                                const float a = net.V0[j], b = net.V0[r0 + j];
                                y0 = a * x + b * tt;
                                y1 = a;
                                y2 = b;
                                sj = static_cast<float>(sv[j]);
                            }
                            *reinterpret_cast<float4*>(yp + j * 4) = make_float4(y0, y1, y2, 0.f);
                            v[0][i] = sj * y0;
                            v[1][i] = sj * y1;
                            v[2][i] = sj * y2;
                            v[3][i] = 0.f;
                        }
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            sts128(sm + OFF_SY + c * SLOT + toff(p, 8 * h, P) * 2, pack_bf16(v[c][0], v[c][1]),
                                   pack_bf16(v[c][2], v[c][3]), pack_bf16(v[c][4], v[c][5]),
                                   pack_bf16(v[c][6], v[c][7]));
                    }
                }
                umma::fence_async_smem();
                signal(&sready);

                // ---------------- forward transitions ----------------
                for (int l = 0; l + 1 < L; ++l) {
                    const int RL = net.rp[l], n = net.nc[l];
                    for (int ch = 0; ch < n; ++ch, ++qc) {
                        MT(0, wait(&p1full[qc & 1], static_cast<uint32_t>((qc >> 1) & 1)));
                        float a[4][4] = {};
                        if (!(MTC_SKIP & 8)) {
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                umma::tmem_ld4(tl + TM_P1 + static_cast<uint32_t>(qc & 1) * 64 + c * 16 + 4 * grp, a[c]);
                            umma::tmem_ld_wait();
                        }
                        signal(&p1empty[qc & 1]);
                        wait(&full[qc % NBUF], static_cast<uint32_t>((qc / NBUF) & 1));
                        const float4 bias = *reinterpret_cast<const float4*>(
                            sm + OFF_RING + static_cast<int>(qc % NBUF) * BLKS + RL * 32 + 16 * grp);
                        const float bb[4] = {bias.x, bias.y, bias.z, bias.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float av = a[0][k] + bb[k], ax = a[1][k], at = a[2][k], aw = a[3][k];
                            float sg, d1, d2, d3;
                            act3<ACT>(av, sg, d1, d2, d3);
                            a[0][k] = sg;
                            a[1][k] = d1 * ax;
                            a[2][k] = d1 * at;
                            a[3][k] = d2 * ax * ax + d1 * aw;
                        }
                        if (qc >= 2) MT(1, wait(&zgfree[qc & 1], static_cast<uint32_t>(((qc - 2) >> 1) & 1)));
                        unsigned char* zb = sm + OFF_ZG + static_cast<int>(qc & 1) * ZGBUF + toff(p, 4 * grp, P) * 2;
                        if (!(MTC_SKIP & 16))
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            sts64(zb + c * ZSLOT, pack_bf16(a[c][0], a[c][1]), pack_bf16(a[c][2], a[c][3]));
                        umma::fence_async_smem();
                        signal(&zgfull[qc & 1]);
                    }
                    MT(2, wait(&tdone, tcount & 1));
                    ++tcount;
                    // transition end: Y -> y_{l+1} scratch + SY_{l+1}, or the output layer
                    const int RN = net.rp[l + 1];
                    if (l + 2 < L) {
                        if (16 * grp < RN) {
                            float y[4][16];
#pragma unroll
                            for (int c = 0; c < 4; ++c) umma::tmem_ld16(tl + TM_Y + c * 64 + 16 * grp, y[c]);
                            umma::tmem_ld_wait();
                            float* yp = scr + net.yoff[l + 1] + (p * RN + 16 * grp) * 4;
                            const double* sl = sv + net.soff[l + 1];
                            const int rt = net.r[l + 1];
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                *reinterpret_cast<float4*>(yp + i * 4) = make_float4(y[0][i], y[1][i], y[2][i], y[3][i]);
                                const int j = 16 * grp + i;
                                const float sj = j < rt ? static_cast<float>(sl[j]) : 0.f;
#pragma unroll
                                for (int c = 0; c < 4; ++c) y[c][i] *= sj;
                            }
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int c = 0; c < 4; ++c)
                                    sts128(sm + OFF_SY + c * SLOT + toff(p, 16 * grp + 8 * h, P) * 2,
                                           pack_bf16(y[c][8 * h], y[c][8 * h + 1]), pack_bf16(y[c][8 * h + 2], y[c][8 * h + 3]),
                                           pack_bf16(y[c][8 * h + 4], y[c][8 * h + 5]),
                                           pack_bf16(y[c][8 * h + 6], y[c][8 * h + 7]));
                        }
                    } else {
                        // ---------------- output layer (M_L = 1) + residual ----------------
                        if (grp == 0) {
                            float y[4][16];
#pragma unroll
                            for (int c = 0; c < 4; ++c) umma::tmem_ld16(tl + TM_Y + c * 64, y[c]);
                            umma::tmem_ld_wait();
                            const int rL = net.r[L - 1];
                            const double* sL = sv + net.soff[L - 1];
                            float u[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (j < rL) {
                                    const float us = net.ulast[j] * float(sL[j]);
#pragma unroll
                                    for (int c = 0; c < 4; ++c) u[c] = fmaf(us, y[c][j], u[c]);
                                }
                            u[0] += net.ulast[rL];
                            const float N = u[2] + mu0 * u[1] - mu1 * u[3] - mu2 * u[0] * (1.f - u[0]);
                            int kind = objective;
                            float tw = w, sw = w, tgt = 0.f;
                            if (spec != nullptr && valid) {
                                const TermSpec sp = spec[gp];
                                kind = sp.kind;
                                tgt = float(sp.target);
                                tw = float(sp.w_term);
                                sw = float(sp.w_seed);
                            }
                            const float dv = u[0] - tgt;
                            float term = kind == 0 ? tw * (N * N)
                                                   : (kind == 1 ? tw * fabsf(N) : (kind == 2 ? tw * (dv * dv) : tw * fabsf(dv)));
                            term = valid ? term : 0.f;
                            if (valid && !isfinite(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
                            float gu[4];
                            if (kind <= 1) {
                                const float gN = valid ? (kind == 0 ? 2.f * N * sw : sgn0(N) * sw) : 0.f;
                                gu[0] = gN * (-mu2 * (1.f - 2.f * u[0]));
                                gu[1] = gN * mu0;
                                gu[2] = gN;
                                gu[3] = -gN * mu1;
                            } else {
                                gu[0] = valid ? (kind == 2 ? 2.f * dv * sw : sgn0(dv) * sw) : 0.f;
                                gu[1] = gu[2] = gu[3] = 0.f;
                            }
                            const float ts = wsum(term);
                            const float gb = wsum(gu[0]);
                            if (lane == 0) {
                                acc4[quarter * MAX_R1] += ts;
                                red1(wq + net.qdbL, gb);
                            }
                            // dL/ds_{L-1}, dU_{L-1} (ranks < r_{L-1}), then ST_{L-1} = s (.) u_last (.) gu
                            float co[16];
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                co[j] = 0.f;
                                if (j < rL) {
                                    const float uj = net.ulast[j], sj = float(sL[j]);
                                    co[j] = sj * uj;
                                    float cd = 0.f, du = 0.f;
#pragma unroll
                                    for (int c = 0; c < 4; ++c) {
                                        cd = fmaf(uj * gu[c], y[c][j], cd);
                                        du = fmaf(gu[c], sj * y[c][j], du);
                                    }
                                    cd = wsum(cd);
                                    du = wsum(du);
                                    if (lane == 0) {
                                        acc4[quarter * MAX_R1 + 1 + net.soff[L - 1] + j] += cd;
                                        red1(wq + net.qdUL + j, du);
                                    }
                                }
                            }
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int c = 0; c < 4; ++c) {
                                    const float* q8 = co + 8 * h;
                                    const float gc = gu[c];
                                    sts128(sm + OFF_ST + c * SLOT + toff(p, 8 * h, P) * 2, pack_bf16(q8[0] * gc, q8[1] * gc),
                                           pack_bf16(q8[2] * gc, q8[3] * gc), pack_bf16(q8[4] * gc, q8[5] * gc),
                                           pack_bf16(q8[6] * gc, q8[7] * gc));
                                }
                        }
                        build_sy(L - 2, sv);
                    }
                    umma::fence_async_smem();
                    signal(&sready);
                }

                // ---------------- reverse transitions ----------------
                for (int l = L - 2; l >= 0; --l) {
                    const int RL = net.rp[l], n = net.nc[l];
                    const int Mn = net.M[l + 1];
                    for (int ch = 0; ch < n; ++ch, ++qc, ++rc) {
                        MT(4, wait(&p1full[qc & 1], static_cast<uint32_t>((qc >> 1) & 1)));
                        float a[4][4] = {}, dz[4][4] = {};
                        if (!(MTC_SKIP & 8)) {
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                umma::tmem_ld4(tl + TM_P1 + c * 16 + 4 * grp, a[c]);
                                umma::tmem_ld4(tl + TM_DZ + c * 16 + 4 * grp, dz[c]);
                            }
                            umma::tmem_ld_wait();
                        }
                        signal(&p1empty[qc & 1]);
                        wait(&full[qc % NBUF], static_cast<uint32_t>((qc / NBUF) & 1));
                        const float4 bias = *reinterpret_cast<const float4*>(
                            sm + OFF_RING + static_cast<int>(qc % NBUF) * BLKS + RL * 32 + 16 * grp);
                        const float bb[4] = {bias.x, bias.y, bias.z, bias.w};
                        float gv[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float av = a[0][k] + bb[k], ax = a[1][k], at = a[2][k], aw = a[3][k];
                            const float g0 = dz[0][k], g1 = dz[1][k], g2 = dz[2][k], g3 = dz[3][k];
                            float sg, d1, d2, d3;
                            if (MTC_SKIP & 4) {
                                sg = av; d1 = ax; d2 = at; d3 = aw;
                            } else {
                                act3<ACT>(av, sg, d1, d2, d3);
                            }
                            dz[0][k] = g0 * d1 + g1 * d2 * ax + g2 * d2 * at + g3 * (d3 * ax * ax + d2 * aw);
                            dz[1][k] = g1 * d1 + g3 * 2.f * d2 * ax;
                            dz[2][k] = g2 * d1;
                            dz[3][k] = g3 * d1;
                            gv[k] = dz[0][k];
                            a[0][k] = sg;
                            a[1][k] = d1 * ax;
                            a[2][k] = d1 * at;
                            a[3][k] = d2 * ax * ax + d1 * aw;
                        }
                        if (qc >= 2) MT(5, wait(&zgfree[qc & 1], static_cast<uint32_t>(((qc - 2) >> 1) & 1)));
                        unsigned char* zb = sm + OFF_ZG + static_cast<int>(qc & 1) * ZGBUF + toff(p, 4 * grp, P) * 2;
                        if (!(MTC_SKIP & 16))
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            sts64(zb + c * ZSLOT, pack_bf16(a[c][0], a[c][1]), pack_bf16(a[c][2], a[c][3]));
                            sts64(zb + (4 + c) * ZSLOT, pack_bf16(dz[c][0], dz[c][1]), pack_bf16(dz[c][2], dz[c][3]));
                        }
                        umma::fence_async_smem();
                        signal(&zgfull[qc & 1]);
                        // db_l over this warp's 32 points (one writer per (quarter, neuron))
                        int idx;
                        const float dbs = treduce<4>(gv, lane, idx);
                        const int k = ch * KC + 4 * grp + idx;
                        if ((lane & 7) == 0 && k < Mn) red1(wq + net.qdb[l] + k, dbs);
                        if (ch > 0) MT(6, flush(rc - 1, l, ch - 1));
                    }
                    MT(6, flush(rc - 1, l, n - 1));
                    MT(7, wait(&tdone, tcount & 1));
                    ++tcount;
                    // transition end: T -> dL/ds_l, ST_l (or dV_0), SY_{l-1}
                    if (16 * grp < RL) {
                        float tv[4][16];
#pragma unroll
                        for (int c = 0; c < 4; ++c) umma::tmem_ld16(tl + TM_Y + c * 64 + 16 * grp, tv[c]);
                        umma::tmem_ld_wait();
                        const float* yp = scr + net.yoff[l] + (p * RL + 16 * grp) * 4;
                        const double* sl = sv + net.soff[l];
                        const int rt = net.r[l];
                        float cd[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float4 y4 = *reinterpret_cast<const float4*>(yp + i * 4);
                            cd[i] = tv[0][i] * y4.x + tv[1][i] * y4.y + tv[2][i] * y4.z + tv[3][i] * y4.w;
                            const int j = 16 * grp + i;
                            const float sj = j < rt ? static_cast<float>(sl[j]) : 0.f;
#pragma unroll
                            for (int c = 0; c < 4; ++c) tv[c][i] *= sj;
                        }
                        int idx;
                        const float cs = treduce<16>(cd, lane, idx);
                        const int j = 16 * grp + idx;
                        if ((lane & 1) == 0 && j < rt) acc4[quarter * MAX_R1 + 1 + net.soff[l] + j] += cs;
                        if (l > 0) {
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int c = 0; c < 4; ++c)
                                    sts128(sm + OFF_ST + c * SLOT + toff(p, 16 * grp + 8 * h, P) * 2,
                                           pack_bf16(tv[c][8 * h], tv[c][8 * h + 1]), pack_bf16(tv[c][8 * h + 2], tv[c][8 * h + 3]),
                                           pack_bf16(tv[c][8 * h + 4], tv[c][8 * h + 5]),
                                           pack_bf16(tv[c][8 * h + 6], tv[c][8 * h + 7]));
                        } else if (grp == 0) {
                            // dV_0[i][j] = sum_{p,c} z0_c[i] st_0[c][j], z0 = (x,t),(1,0),(0,1),(0,0)
                            for (int jj = 0; jj < rt; ++jj) {
                                const float v0 = wsum(x * tv[0][jj] + tv[1][jj]);
                                const float v1 = wsum(tt * tv[0][jj] + tv[2][jj]);
                                if (lane == 0) {
                                    red1(wq + net.qdV0 + jj, v0);
                                    red1(wq + net.qdV0 + rt + jj, v1);
                                }
                            }
                        }
                    }
                    if (l > 0) {
                        build_sy(l - 1, sv);
                        umma::fence_async_smem();
                        signal(&sready);
                    }
                }
            }
            // unit end: [loss, dL/ds] row = sum of the 4 quarter copies (fixed order)
            epi_sync();
            for (int k = tid; k < R1; k += NWE * 32) {
                part[unit * R1 + k] = ((acc4[k] + acc4[MAX_R1 + k]) + acc4[2 * MAX_R1 + k]) + acc4[3 * MAX_R1 + k];
                acc4[k] = acc4[MAX_R1 + k] = acc4[2 * MAX_R1 + k] = acc4[3 * MAX_R1 + k] = 0.f;
            }
            epi_sync();
        }
    }
#ifdef MTC_TIMING
    if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == ISSUER * 32))
        atomicAdd(&g_mtc_timing[threadIdx.x == 0 ? 15 : 31], static_cast<unsigned long long>(clock64() - t_start));
#endif
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tbase);
}

}  // namespace mtc
}  // namespace lrnr_b200
