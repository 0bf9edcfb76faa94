// Tensor-core (tcgen05 / TMEM) tile kernel for the fused LRNR / FastLRNR
// residual + reverse-to-s sweep, FP32-grade accuracy via 3xTF32.
//
// Same math as the FMA tile kernel (pinn_v2.cuh); the two tile GEMMs of every
// chunk run on the 5th-generation tensor cores:
//   * a CTA owns P = 128 collocation points = the MMA M dimension (TMEM lane =
//     point); the 4 jet slots (u, u_x, u_t, u_xx) are 4 independent MMAs, so
//     the epilogue thread that owns a point sees all 4 slots of every neuron
//     (the activation jet and its VJP mix slots) without shuffles;
//   * phase 1 (K = rank):   P1_c = SY_c U^T  (forward)  |  P1_c = ST_c V^T (reverse)
//     A operand SY_c / ST_c from shared memory, B operand = factor chunk (TMA bulk);
//   * epilogue (CUDA cores): tcgen05.ld P1 -> (+b) activation jet / its VJP with
//     the pre-activation A reloaded from the forward's store -> 3xTF32 split ->
//     tcgen05.st into TMEM (Z_c hi / lo);
//   * phase 2 (K = KC neurons): Y_c += Z_c V (forward) | T_c += G_c U (reverse),
//     A operand from TMEM, accumulated in TMEM over the chunks of the transition.
// 3xTF32: x = hi + lo with hi = tf32(x); a*b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi
// (fp32 accumulate), giving ~fp32 accuracy (the dropped lo*lo term is 2^-22).
// TMEM (512 columns): P1_c 4x32 | Z hi 4x32 | Z lo 4x32 | Y/T 4x32.
// Shared memory: SY/ST hi/lo for 4 slots (128 KB) + a 3-slot factor-chunk ring.
// One CTA per SM owns the whole TMEM; two issuer warps issue the phase-1 and
// phase-2 MMAs warp-collectively, completion via tcgen05.commit -> mbarrier.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pinn_kernels.cuh"
#include "pinn_v2.cuh"
#include "umma.cuh"

namespace lrnr_b200 {
namespace tc {

constexpr int P = 128;    // points per tile (MMA M)
constexpr int KC = 32;    // neurons per chunk (phase-1 N, phase-2 K)
constexpr int RP = 32;    // max padded rank
#ifndef TC_NWE
#define TC_NWE 16
#endif
constexpr int NWE = TC_NWE;  // epilogue warps: lane quarter = warp % 4, neuron / rank group of NG = warp / 4
// Two dedicated MMA issuer warps after the epilogue warps: MMA issue is
// latency-bound (~57 cycles per MMA from one warp), so the phase-1 and phase-2
// MMAs are issued concurrently by warps ISSUER and ISSUER2 (one issuer: 24.40 ms
// on c2; two: 23.51 ms; four, with each phase's jet slots split: 27.1 ms).
constexpr int ISSUER = NWE;       // phase-1 issuer
constexpr int ISSUER2 = NWE + 1;  // phase-2 issuer
constexpr int NT = 32 * (NWE + 2);
constexpr int NG = KC / (NWE / 4);  // neurons (epilogue) / ranks (sums) per thread
// Units (single tiles) after each CTA's first are claimed from a global counter:
// SMs run at slightly different speeds (a static split spread by up to 5 %).
#define TC_MMA_SS umma::mma_ss_w
#define TC_MMA_TS umma::mma_ts_w
#define TC_COMMIT umma::mma_commit_w
constexpr int TM_P1 = 0, TM_ZH = 128, TM_ZL = 256, TM_Y = 384;
// Phase-2 products of YACC consecutive chunks accumulate in TMEM before the
// epilogue reads them into the FP32 running sum (the tensor-core accumulator
// truncates: 1 chunk = 12 MMAs keeps it at ~3e-6 on c2, 2 chunks ~6e-6, the
// full K = 256 reached 1.2e-4). Halves the TMEM load round trips of Y.
#ifndef TC_YACC
#define TC_YACC 2
#endif
constexpr int YACC = TC_YACC;

template <typename T = float>
struct NetTC {
    int L;
    int M[kMaxL + 1];
    int r[kMaxL];
    int rk[kMaxL];         // padded rank as MMA K (multiple of 8, <= 32)
    int rn[kMaxL];         // padded rank as MMA N (16 or 32)
    int nc[kMaxL];
    int soff[kMaxL + 1];
    int yoff[kMaxL];       // y_l in per-CTA scratch: [p][j (r_l)][4]
    int ystride;
    int64_t aoff[kMaxL];   // A in per-CTA scratch: [chunk][KC][p][4]
    int64_t astride;
    int rtotal;
    const float* blocks;
    const int64_t* sched_off;
    const int* sched_bytes;
    int sched_len;
    const float* V0;       // 2 x r[0]
    const float* ulast;    // r[L-1] then b_{L-1}[0]
};

// smem layout (floats)
constexpr int SY_TILE = P * RP;               // one canonical K-major tile (rows = 128, K = 32)
constexpr int OFF_SY = 0;                     // [c][hi/lo] tiles: 8 x 4096 floats = 128 KB
constexpr int BUF = 4 * KC * RP + KC + 32;    // factor chunk (max): 4 canonical 32x32 tiles + bias
#ifndef TC_NBUF
#define TC_NBUF 3
#endif
constexpr int NBUF = TC_NBUF;                 // factor-chunk ring (NBUF - 1 chunks in flight)
constexpr int OFF_B0 = OFF_SY + 8 * SY_TILE;
constexpr int OFF_RED = OFF_B0 + NBUF * BUF;  // [P][RP] + P (loss) + [16][RP] partials
constexpr int RPS = RP + 1;                   // red[] point stride (odd: conflict-free column writes)
constexpr int OFF_ACC = OFF_RED + P * RPS + P + 16 * RP;  // partials: up to 16 groups
constexpr int SMEM_FLOATS = OFF_ACC + 1024;

__device__ __forceinline__ float* sy_tile(float* sm, int c, int lo) { return sm + OFF_SY + (2 * c + lo) * SY_TILE; }

// write an fp32 value split into the hi / lo canonical tiles of slot c at (row p, k j)
// four consecutive k (j0 % 4 == 0) of row p as one 16-byte store per tile: a
// quarter-warp's 8 rows then fill one 128-byte core matrix (no bank conflicts; the
// scalar form hits each bank 4 times per warp)
__device__ __forceinline__ void put_split4(float* sm, int c, int p, int j0, float v0, float v1, float v2, float v3) {
    float h[4], l[4];
    umma::split_tf32(v0, h[0], l[0]);
    umma::split_tf32(v1, h[1], l[1]);
    umma::split_tf32(v2, h[2], l[2]);
    umma::split_tf32(v3, h[3], l[3]);
    const int o = umma::kmaj_off(p, j0, P);
    *reinterpret_cast<float4*>(sy_tile(sm, c, 0) + o) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(sy_tile(sm, c, 1) + o) = make_float4(l[0], l[1], l[2], l[3]);
}
__device__ __forceinline__ void put_split(float* sm, int c, int p, int j, float v) {
    float h, l;
    umma::split_tf32(v, h, l);
    const int o = umma::kmaj_off(p, j, P);
    sy_tile(sm, c, 0)[o] = h;
    sy_tile(sm, c, 1)[o] = l;
}

// Optional phase timing (dev aid): -DLRNR_TC_TIMING records clock64 deltas of
// CTA 0 / thread 32 into a global array (see scripts/tc_timing.py).
#ifdef LRNR_TC_TIMING
__device__ unsigned long long g_tc_timing[16];
// accumulated in shared memory (a few cycles per mark) and flushed once at the end
#define TC_T0()                                                \
    __shared__ unsigned long long _tc_acc[16];                 \
    if (threadIdx.x < 16) _tc_acc[threadIdx.x] = 0;            \
    __syncthreads();                                           \
    long long _tt = clock64();
#define TC_ISSUE_BEGIN() const long long _ti = clock64();
#define TC_ISSUE_END()                                                                    \
    do {                                                                                  \
        if (blockIdx.x == 0) _tc_acc[15] += static_cast<unsigned long long>(clock64() - _ti); \
    } while (0)
#define TC_MARK(i)                                                         \
    do {                                                                   \
        if (blockIdx.x == 0 && threadIdx.x == 32) {                        \
            const long long _n = clock64();                                \
            _tc_acc[i] += static_cast<unsigned long long>(_n - _tt);       \
            _tt = _n;                                                      \
        }                                                                  \
    } while (0)
#define TC_FLUSH()                                                          \
    do {                                                                    \
        __syncthreads();                                                    \
        if (blockIdx.x == 0 && threadIdx.x < 16) g_tc_timing[threadIdx.x] += _tc_acc[threadIdx.x]; \
    } while (0)
#else
#define TC_T0()
#define TC_ISSUE_BEGIN()
#define TC_ISSUE_END()
#define TC_MARK(i)
#define TC_FLUSH()
#endif

// acc[1 + off + j] += sum_p red[p][j] for j < r, fixed order: NRG groups of
// P / NRG points in parallel (one thread per (group, rank)), then the partials.
constexpr int NRG = NWE;
__device__ __forceinline__ void reduce_points(float* red, float* acc, int off, int r, int tid) {
    float* part = red + P * RPS + P;
    if (tid < NRG * RP) {
        const int j = tid % RP, g = tid / RP;
        float s = 0.f;
        if (j < r)
#pragma unroll
            for (int i = 0; i < P / NRG; ++i) s += red[((P / NRG) * g + i) * RPS + j];
        part[g * RP + j] = s;
    }
    __syncthreads();
    if (tid < r) {
        float s = 0.f;
#pragma unroll
        for (int g = 0; g < NRG; ++g) s += part[g * RP + tid];
        acc[1 + off + tid] += s;
    }
}

__device__ __forceinline__ void tld(uint32_t taddr, float (&v)[8]) { umma::tmem_ld8(taddr, v); }
__device__ __forceinline__ void tld(uint32_t taddr, float (&v)[16]) { umma::tmem_ld16(taddr, v); }
__device__ __forceinline__ void tst(uint32_t taddr, const float (&v)[8]) { umma::tmem_st8(taddr, v); }
__device__ __forceinline__ void tst(uint32_t taddr, const float (&v)[16]) { umma::tmem_st16(taddr, v); }

// acc[c][n] += TMEM[taddr + c * 32 + n] (the previous chunk's phase-2 product),
// one load batch, one wait
__device__ __forceinline__ void add_y(uint32_t taddr, float (&acc)[4][NG]) {
    float v[4][NG];
#pragma unroll
    for (int c = 0; c < 4; ++c) tld(taddr + c * 32, v[c]);
    umma::tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int n = 0; n < NG; ++n) acc[c][n] += v[c][n];
}

// P1 columns of this thread (4 slots x NG neurons) in two column halves: the first
// half is waited for here, the second is in flight while the first half's math runs
// (the caller waits before touching column NG / 2)
__device__ __forceinline__ void ld_p1_halves(uint32_t taddr, float (&v)[4][NG]) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int h = 0; h < NG / 2; h += 4) umma::tmem_ld4(taddr + c * KC + h, v[c] + h);
    umma::tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int h = NG / 2; h < NG; h += 4) umma::tmem_ld4(taddr + c * KC + h, v[c] + h);
}

// stored pre-activation A of (neuron k, point p) inside its chunk: [k][p][4]
// (a warp's 32 points are one contiguous 512-B segment)
__device__ __forceinline__ int aidx(int k, int p) { return (k * P + p) * 4; }

template <int ACT, bool FAST>
__device__ __forceinline__ void act3f(float a, float& sg, float& d1, float& d2, float& d3) {
    v2::act3<ACT, FAST>(a, sg, d1, d2, d3);
}

template <int ACT, bool FAST>
__global__ void __launch_bounds__(NT, 1)
pinn_tc_kernel(const NetTC<> net, const RunGeom g, const double* __restrict__ pts, const double* __restrict__ svec,
               const double* __restrict__ mus, const float w, float* __restrict__ scratch,
               float* __restrict__ ascratch, float* __restrict__ part, unsigned long long* __restrict__ bad,
               unsigned long long* __restrict__ unit_ctr) {
    extern __shared__ __align__(128) float sm[];
    float* red = sm + OFF_RED;
    float* acc = sm + OFF_ACC;
    __shared__ __align__(8) uint64_t wbar[NBUF];
    __shared__ __align__(8) uint64_t mbar1, mbar2;
    __shared__ __align__(8) uint64_t p1free, zready;  // epilogue -> issuer (one arrive per epilogue warp)
    __shared__ uint32_t tmem_base;
    __shared__ int64_t next_unit;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int quarter = warp & 3, half = warp >> 2;  // half: neuron / rank group of NG
    const int p = quarter * 32 + lane;  // the point (TMEM lane) this thread serves in epilogues
    const int R1 = 1 + net.rtotal;
    const int L = net.L;
    float* scr = scratch + static_cast<int64_t>(blockIdx.x) * net.ystride;
    float* ascr = ascratch + static_cast<int64_t>(blockIdx.x) * net.astride;

#ifdef TC_CTA_TIMES
    unsigned long long _t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t_start));
#endif
    for (int k = tid; k < R1; k += NT) acc[k] = 0.f;
    if (warp == 0) umma::tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < NBUF; ++i) umma::mbar_init(&wbar[i], 1);
        umma::mbar_init(&mbar1, 1);
        umma::mbar_init(&mbar2, 1);
        umma::mbar_init(&p1free, NWE);
        umma::mbar_init(&zready, NWE);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tmem_base;
    const uint32_t tlane = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
    uint32_t ph1 = 0, ph2 = 0;  // mbarrier phase counters (epilogue warps)
    uint32_t phf = 0, phz = 0;  // p1free / zready phase counters (issuer warp)
    // epilogue warp -> issuer handshakes (after warp-collective tcgen05 ld / st waits)
    auto signal = [&](uint64_t* bar) {
        umma::fence_before();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(bar);
    };
    auto await = [&](uint64_t* bar, uint32_t& ph) {
        umma::mbar_wait(bar, ph & 1);
        ++ph;
        umma::fence_after();
    };

    // ---- factor-chunk pipeline (TMA bulk copies) ----
    // every tile runs the same chunk schedule, so the ring is refilled without knowing the
    // CTA's tile count; the NBUF - 1 copies in flight past the last chunk are drained at exit
    const int64_t total_chunks = INT64_MAX;
#ifdef TC_CTA_TIMES
    int64_t total_tiles = 0;
#endif
    int64_t q = 0;
    auto issue = [&](int64_t qq) {
        if (qq < total_chunks) {
            const int e = static_cast<int>(qq % net.sched_len);
            const int b = static_cast<int>(qq % NBUF);
            v2::fence_proxy_async();
            v2::mbar_expect_tx(&wbar[b], static_cast<uint32_t>(net.sched_bytes[e]));
            v2::bulk_g2s(sm + OFF_B0 + b * BUF, net.blocks + net.sched_off[e], static_cast<uint32_t>(net.sched_bytes[e]),
                         &wbar[b]);
        }
    };
    if (tid == 0) {
        for (int i = 0; i + 1 < NBUF; ++i) issue(i);
    }
    TC_T0();
    auto wait_mma1 = [&]() {
        umma::mbar_wait(&mbar1, ph1 & 1);
        ++ph1;
        umma::fence_after();
    };
    auto wait_mma2 = [&]() {
        umma::mbar_wait(&mbar2, ph2 & 1);
        ++ph2;
        umma::fence_after();
    };
    const uint32_t id_p1 = umma::idesc_tf32(P, KC);
    // descriptor low words (start >> 4 | LBO >> 4 << 16); advancing the start by
    // a float offset f adds f >> 2.  Common high word: SBO = 128 B, version 1.
    const uint32_t dhi = umma::desc_hi(128);
    const uint32_t lsy = umma::desc_lo(sm + OFF_SY, (P / 8) * 128);     // SY / ST tiles (rows = P)
    const uint32_t lb32 = umma::desc_lo(sm + OFF_B0, (KC / 8) * 128);   // factor tiles with 32 rows
    const uint32_t lb16 = umma::desc_lo(sm + OFF_B0, (16 / 8) * 128);   // factor tiles with 16 rows
    // phase 1 (issuer warp, converged): P1_c = S_c B (3xTF32), S = SY / ST from smem,
    // B = factor tiles at float offset bo (hi) / bo + KC * rk (lo) of the ring slot
    auto mma_p1 = [&](int bo, int rk) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t d = tbase + TM_P1 + c * KC;
            const uint32_t ah0 = lsy + ((2 * c) * SY_TILE >> 2), al0 = lsy + ((2 * c + 1) * SY_TILE >> 2);
            const uint32_t bh0 = lb32 + (bo >> 2), bl0 = lb32 + ((bo + KC * rk) >> 2);
            for (int s = 0; s < rk / 8; ++s) {
                const uint32_t sa = s * (2 * (P / 8) * 32 >> 2), sb = s * (2 * (KC / 8) * 32 >> 2);
                TC_MMA_SS(d, ah0 + sa, bh0 + sb, dhi, id_p1, s > 0);
                TC_MMA_SS(d, ah0 + sa, bl0 + sb, dhi, id_p1, 1);
                TC_MMA_SS(d, al0 + sa, bh0 + sb, dhi, id_p1, 1);
            }
        }
        TC_COMMIT(&mbar1);
    };
    // phase 2 (issuer warp 2, converged): Y_c = Z_c B (fresh accumulator, A from TMEM),
    // B = factor tiles (rows rn) at float offset bo (hi) / bo + rn * KC (lo)
    auto mma_p2 = [&](int bo, int rn, bool acc0) {
        const uint32_t id_p2 = umma::idesc_tf32(P, rn);
        const uint32_t lb = rn == 16 ? lb16 : lb32;
        const uint32_t bh0 = lb + (bo >> 2), bl0 = lb + ((bo + rn * KC) >> 2);
        const uint32_t sb = 2 * (rn / 8) * 32 >> 2;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t d = tbase + TM_Y + c * 32;
#pragma unroll
            for (int s = 0; s < KC / 8; ++s) {
                const uint32_t azh = tbase + TM_ZH + c * KC + s * 8, azl = tbase + TM_ZL + c * KC + s * 8;
                TC_MMA_TS(d, azh, bh0 + s * sb, dhi, id_p2, (s > 0 || acc0) ? 1u : 0u);
                TC_MMA_TS(d, azh, bl0 + s * sb, dhi, id_p2, 1);
                TC_MMA_TS(d, azl, bh0 + s * sb, dhi, id_p2, 1);
            }
        }
        TC_COMMIT(&mbar2);
    };
    auto wait_slot = [&](int64_t qq) {
        umma::mbar_wait(&wbar[qq % NBUF], static_cast<uint32_t>((qq / NBUF) & 1));
        umma::fence_after();
    };

    // claims: the counter starts at all-ones (memset 0xff), so the first claim returns unit gridDim.x
    unsigned long long claim = 0;
    if (tid == 0) claim = atomicAdd(unit_ctr, 1ull) + 1ull + gridDim.x;
    for (int64_t unit = blockIdx.x; unit < g.n_units;) {
#ifdef TC_CTA_TIMES
        ++total_tiles;
#endif
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
            // ---------------- input layer: y_0 = V_0^T z_0 ----------------
            if (half == 0) {
                const float x = valid ? float(pts[2 * gp]) : 0.f;
                const float t = valid ? float(pts[2 * gp + 1]) : 0.f;
                const int r0 = net.r[0];
                for (int j = 0; j < net.rk[0]; ++j) {
                    float y4[4] = {0.f, 0.f, 0.f, 0.f};
                    float sj = 0.f;
                    if (j < r0) {
                        const float v0 = net.V0[j], v1 = net.V0[r0 + j];
                        y4[0] = v0 * x + v1 * t;
                        y4[1] = v0;
                        y4[2] = v1;
                        sj = float(sv[j]);
                        v2::st4(scr + net.yoff[0] + (p * r0 + j) * 4, y4[0], y4[1], y4[2], y4[3]);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) put_split(sm, c, p, j, sj * y4[c]);
                }
            }
            umma::fence_async_smem();
            __syncthreads();

            // ---------------- forward transitions ----------------
            for (int l = 0; l + 1 < L; ++l) {
                const int rk = net.rk[l], rnn = net.rn[l + 1];
                // Y = sum over chunks of fresh per-chunk tensor-core products, summed
                // here in FP32 (the tensor-core accumulator truncates; one K = 32
                // chunk per accumulator keeps that bias at the FP32 level)
                float ysum[4][NG];
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int n = 0; n < NG; ++n) ysum[c][n] = 0.f;
                // factor block of chunk qq: UT_H | UT_L (KC x rk, rows KC) | bias (KC, padded 32) | VT_H | VT_L (rnn x KC)
                auto fwd_p1 = [&](int64_t qq) {
                    wait_slot(qq);
                    mma_p1(static_cast<int>(qq % NBUF) * BUF, rk);
                };
                auto fwd_p2 = [&](int64_t qq, int ch) {
                    mma_p2(static_cast<int>(qq % NBUF) * BUF + 2 * KC * rk + 32, rnn, ch % YACC != 0);
                };
                if (warp == ISSUER) fwd_p1(q);
                // pipeline per chunk ch: [P1(ch) | P2(ch-1)] on the tensor core while the
                // epilogue of ch computes the activation jet; Z / Y are touched only after
                // P2(ch-1) completes.  P1(ch+1) is issued ahead of P2(ch).
                for (int ch = 0; ch < net.nc[l]; ++ch, ++q) {
                    const float* bias = sm + OFF_B0 + static_cast<int>(q % NBUF) * BUF + 2 * KC * rk;
                    if (warp < NWE) {
                        TC_MARK(1);
                        wait_mma1();
                        TC_MARK(2);
                        // ring slot of chunk q-1 is free once P2(q-1) is complete
                        if (ch == 0 && tid == 0) issue(q + NBUF - 1);
                        {
                            float a[4][NG];
                            float* Ast = ascr + net.aoff[l] + static_cast<int64_t>(ch) * (P * KC * 4);
                            // two column halves: the second half's TMEM read overlaps the first half's math
                            ld_p1_halves(tlane + TM_P1 + half * NG, a);
    #pragma unroll
                            for (int n = 0; n < NG; ++n) {
                                if (n == NG / 2) {
                                    umma::tmem_ld_wait();
                                    signal(&p1free);  // P1 may be overwritten by P1(ch+1)
                                }
                                const int k = half * NG + n;
                                const float av = a[0][n] + bias[k], ax = a[1][n], at = a[2][n], aw = a[3][n];
                                v2::st4(Ast + aidx(k, p), av, ax, at, aw);
                                float sg, d1, d2, d3;
                                act3f<ACT, FAST>(av, sg, d1, d2, d3);
                                a[0][n] = sg;
                                a[1][n] = d1 * ax;
                                a[2][n] = d1 * at;
                                a[3][n] = d2 * ax * ax + d1 * aw;
                            }
                            TC_MARK(3);
                            if (ch > 0) {
                                wait_mma2();  // P2(ch-1): Z free, its Y product ready
                                if (tid == 0) issue(q + NBUF - 1);
                                if (ch % YACC == 0) add_y(tlane + TM_Y + half * NG, ysum);  // a group of YACC chunks is complete
                            }
                            TC_MARK(0);
    #pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                float hi[NG], lo[NG];
    #pragma unroll
                                for (int n = 0; n < NG; ++n) umma::split_tf32(a[c][n], hi[n], lo[n]);
                                tst(tlane + TM_ZH + c * KC + half * NG, hi);
                                tst(tlane + TM_ZL + c * KC + half * NG, lo);
                            }
                            umma::tmem_st_wait();
                            signal(&zready);
                        }
                    }
                    TC_MARK(4);
                    if (warp == ISSUER) {
                        TC_ISSUE_BEGIN();
                        await(&p1free, phf);  // every chunk (keeps the phase count)
                        if (ch + 1 < net.nc[l]) fwd_p1(q + 1);
                        if (lane == 0) TC_ISSUE_END();
                    }
                    if (warp == ISSUER2) {
                        await(&zready, phz);
                        fwd_p2(q, ch);
                    }
                    TC_MARK(5);
                }
                // transition end: Y -> y_{l+1} (scratch), SY = s (.) y (smem hi / lo)
                TC_MARK(0);
                if (warp < NWE) {
                    wait_mma2();
                    TC_MARK(5);
                    const double* sl = sv + net.soff[l + 1];
                    const int rtrue = net.r[l + 1];
                    float (&y)[4][NG] = ysum;
                    add_y(tlane + TM_Y + half * NG, y);
#pragma unroll
                    for (int n4 = 0; n4 < NG / 4; ++n4) {
                        const int j0 = half * NG + 4 * n4;
                        if (j0 < net.rk[l + 1]) {  // rk is a multiple of 8: a group of 4 is all in or all out
                            float sj[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int j = j0 + i, n = 4 * n4 + i;
                                sj[i] = j < rtrue ? float(sl[j]) : 0.f;
                                if (j < rtrue)
                                    v2::st4(scr + net.yoff[l + 1] + (p * rtrue + j) * 4, y[0][n], y[1][n], y[2][n],
                                            y[3][n]);
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                put_split4(sm, c, p, j0, sj[0] * y[c][4 * n4], sj[1] * y[c][4 * n4 + 1],
                                           sj[2] * y[c][4 * n4 + 2], sj[3] * y[c][4 * n4 + 3]);
                        }
                    }
                }
                umma::fence_async_smem();
                umma::fence_before();
                __syncthreads();
            }

            TC_MARK(6);
            // ---------------- output layer (M_L = 1) + residual ----------------
            {
                const int rL = net.r[L - 1];
                const double* sL = sv + net.soff[L - 1];
                if (half == 0) {
                    float u[4] = {0.f, 0.f, 0.f, 0.f};
                    for (int j = 0; j < rL; ++j) {
                        float y4[4];
                        v2::ld4(scr + net.yoff[L - 1] + (p * rL + j) * 4, y4);
                        const float us = net.ulast[j] * float(sL[j]);
#pragma unroll
                        for (int c = 0; c < 4; ++c) u[c] = fmaf(us, y4[c], u[c]);
                    }
                    u[0] += net.ulast[rL];
                    const float N = u[2] + mu0 * u[1] - mu1 * u[3] - mu2 * u[0] * (1.f - u[0]);
                    const float term = valid ? w * (N * N) : 0.f;
                    if (valid && !isfinite(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
                    const float gN = valid ? 2.f * N * w : 0.f;
                    const float gu[4] = {gN * (-mu2 * (1.f - 2.f * u[0])), gN * mu0, gN, -gN * mu1};
                    red[P * RPS + p] = term;
                    for (int j = 0; j < net.rk[L - 1]; ++j) {
                        const float uj = j < rL ? net.ulast[j] : 0.f;
                        const float sj = j < rL ? float(sL[j]) : 0.f;
                        float cd = 0.f;
                        if (j < rL) {
                            float y4[4];
                            v2::ld4(scr + net.yoff[L - 1] + (p * rL + j) * 4, y4);
#pragma unroll
                            for (int c = 0; c < 4; ++c) cd = fmaf(uj * gu[c], y4[c], cd);
                        }
                        red[p * RPS + j] = cd;
#pragma unroll
                        for (int c = 0; c < 4; ++c) put_split(sm, c, p, j, sj * uj * gu[c]);
                    }
                }
                umma::fence_async_smem();
                __syncthreads();
                reduce_points(red, acc, net.soff[L - 1], rL, tid);
                if (tid == NT - 1) {
                    float sacc = 0.f;
                    for (int pp = 0; pp < P; ++pp) sacc += red[P * RPS + pp];
                    acc[0] += sacc;
                }
                __syncthreads();
            }

            TC_MARK(7);
            // ---------------- reverse transitions ----------------
            for (int l = L - 2; l >= 0; --l) {
                const int rkn = net.rk[l + 1], rnl = net.rn[l];
                float tsum[4][NG];
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int n = 0; n < NG; ++n) tsum[c][n] = 0.f;
                // factor block of chunk qq: V_H | V_L (KC x rkn, rows KC) | UT_H | UT_L (rnl x KC)
                auto bwd_p1 = [&](int64_t qq) {
                    wait_slot(qq);
                    mma_p1(static_cast<int>(qq % NBUF) * BUF, rkn);
                };
                auto bwd_p2 = [&](int64_t qq, int ch) {
                    mma_p2(static_cast<int>(qq % NBUF) * BUF + 2 * KC * rkn, rnl, ch % YACC != 0);
                };
                if (warp == ISSUER) bwd_p1(q);
                for (int ch = 0; ch < net.nc[l]; ++ch, ++q) {
                    if (warp < NWE) {
                        // stored pre-activations of this chunk (in flight during the MMAs)
                        const float* Ast = ascr + net.aoff[l] + static_cast<int64_t>(ch) * (P * KC * 4);
                        float a[4][NG];
    #pragma unroll
                        for (int n = 0; n < NG; ++n) {
                            float a4[4];
                            v2::ld4(Ast + aidx(half * NG + n, p), a4);
    #pragma unroll
                            for (int c = 0; c < 4; ++c) a[c][n] = a4[c];
                        }
                        TC_MARK(9);
                        wait_mma1();
                        TC_MARK(10);
                        if (ch == 0 && tid == 0) issue(q + NBUF - 1);
                        {
                            float dz[4][NG];
                            ld_p1_halves(tlane + TM_P1 + half * NG, dz);
    #pragma unroll
                            for (int n = 0; n < NG; ++n) {
                                if (n == NG / 2) {
                                    umma::tmem_ld_wait();
                                    signal(&p1free);
                                }
                                const float av = a[0][n], ax = a[1][n], at = a[2][n], aw = a[3][n];
                                const float g0 = dz[0][n], g1 = dz[1][n], g2 = dz[2][n], g3 = dz[3][n];
                                float sg, d1, d2, d3;
                                act3f<ACT, FAST>(av, sg, d1, d2, d3);
                                dz[0][n] = g0 * d1 + g1 * d2 * ax + g2 * d2 * at + g3 * (d3 * ax * ax + d2 * aw);
                                dz[1][n] = g1 * d1 + g3 * 2.f * d2 * ax;
                                dz[2][n] = g2 * d1;
                                dz[3][n] = g3 * d1;
                            }
                            TC_MARK(11);
                            if (ch > 0) {
                                wait_mma2();  // P2(ch-1): G free, its T product ready
                                if (tid == 0) issue(q + NBUF - 1);
                                if (ch % YACC == 0) add_y(tlane + TM_Y + half * NG, tsum);
                            }
                            TC_MARK(8);
    #pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                float hi[NG], lo[NG];
    #pragma unroll
                                for (int n = 0; n < NG; ++n) umma::split_tf32(dz[c][n], hi[n], lo[n]);
                                tst(tlane + TM_ZH + c * KC + half * NG, hi);
                                tst(tlane + TM_ZL + c * KC + half * NG, lo);
                            }
                            umma::tmem_st_wait();
                            signal(&zready);
                        }
                    }
                    TC_MARK(12);
                    if (warp == ISSUER) {
                        await(&p1free, phf);  // every chunk (keeps the phase count)
                        if (ch + 1 < net.nc[l]) bwd_p1(q + 1);
                    }
                    if (warp == ISSUER2) {
                        await(&zready, phz);
                        bwd_p2(q, ch);
                    }
                }
                // transition end: T -> dL/ds_l partials, ST = s_l (.) T (smem hi / lo)
                TC_MARK(8);
                if (warp < NWE) {
                    const double* sl = sv + net.soff[l];
                    const int rtrue = net.r[l];
                    // this thread's y_l (scratch, usually an L2 / HBM round trip): all loads issued
                    // together and before the wait for the last phase-2 product
                    float4 yv[NG];
#pragma unroll
                    for (int n = 0; n < NG; ++n) {
                        const int j = half * NG + n;
                        yv[n] = j < rtrue ? *reinterpret_cast<const float4*>(scr + net.yoff[l] + (p * rtrue + j) * 4)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    wait_mma2();
                    TC_MARK(13);
                    float (&tt)[4][NG] = tsum;
                    add_y(tlane + TM_Y + half * NG, tt);
#pragma unroll
                    for (int n4 = 0; n4 < NG / 4; ++n4) {
                        const int j0 = half * NG + 4 * n4;
                        if (j0 < net.rk[l]) {  // rk is a multiple of 8
                            float sj[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int j = j0 + i, n = 4 * n4 + i;
                                float cd = 0.f;
                                sj[i] = 0.f;
                                if (j < rtrue) {
                                    sj[i] = float(sl[j]);
                                    const float y4[4] = {yv[n].x, yv[n].y, yv[n].z, yv[n].w};
#pragma unroll
                                    for (int c = 0; c < 4; ++c) cd = fmaf(tt[c][n], y4[c], cd);
                                }
                                red[p * RPS + j] = cd;
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                put_split4(sm, c, p, j0, sj[0] * tt[c][4 * n4], sj[1] * tt[c][4 * n4 + 1],
                                           sj[2] * tt[c][4 * n4 + 2], sj[3] * tt[c][4 * n4 + 3]);
                        }
                    }
                }
                umma::fence_async_smem();
                umma::fence_before();
                __syncthreads();
                reduce_points(red, acc, net.soff[l], net.r[l], tid);
                __syncthreads();
                TC_MARK(14);
            }
        }
        for (int k = tid; k < R1; k += NT) {
            part[unit * R1 + k] = acc[k];
            acc[k] = 0.f;
        }
        if (tid == 0) {
            next_unit = static_cast<int64_t>(claim);
            if (claim < static_cast<unsigned long long>(g.n_units)) claim = atomicAdd(unit_ctr, 1ull) + 1ull + gridDim.x;
        }
        __syncthreads();
        unit = next_unit;
    }
    if (tid == 0)
        for (int64_t qq = q; qq < q + NBUF - 1; ++qq) wait_slot(qq);  // prefetches past the last chunk
    TC_FLUSH();
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tbase);
#ifdef TC_CTA_TIMES
    if (tid == 0) {
        unsigned long long _t_end;
        unsigned _smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(_smid));
        printf("CTA %d %u %llu %llu %lld\n", blockIdx.x, _smid, _t_start, _t_end, (long long)total_tiles);
    }
#endif
}

}  // namespace tc
}  // namespace lrnr_b200
