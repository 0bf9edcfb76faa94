// Tensor-core (tcgen05 / TMEM) tile kernel for the fused LRNR / FastLRNR
// residual + reverse-to-s sweep, FP32-grade accuracy from an FP16 two-term split.
//
// Same math as the FMA tile kernel (pinn_v2.cuh; reference: jet_affine_factored /
// jet_activation, proj/src/model.cpp:85-223, and their VJPs, proj/src/autodiff.cpp:473-563).
// A CTA owns P = 128 collocation points = the MMA M dimension (TMEM lane = point); the
// 4 jet slots (u, u_x, u_t, u_xx) are 4 independent MMAs, so the epilogue thread that
// owns a point sees all 4 slots of each of its neurons without shuffles.  Per chunk of
// KC = 32 neurons of transition l:
//   forward   P1  A_c  = SY_c U^T          TS: A = SY (TMEM), B = U^T chunk (ring)  -> TMEM
//             epilogue: A -> (+b) sigma-jet Z_c -> TMEM (fp16 hi | lo)
//             P2  Y_c += Z_c V             TS: A = Z (TMEM),  B = V chunk           -> TMEM
//   reverse   P1r A_c  = SY_c U^T (recomputed from SY_l in smem, no stash in HBM)
//             P1d DZ_c = ST_c V^T          SS: A = ST (smem)
//             epilogue: G_c = VJP(A, DZ) -> TMEM (fp16 hi | lo)
//             P2r T_c += G_c U             TS: A = G (TMEM)
// FP16 two-term split: every operand x is scaled by a power of two S (per point and jet
// slot for SY / ST / Z / G, per matrix for the factors), hi = fp16(x S), lo =
// fp16(x S - hi), and a*b ~ hi*hi + hi*lo + lo*hi with FP32 accumulation; the products
// are unscaled exactly in the epilogue (2^-22 relative, scripts/umma_f16_test.cu).  SY /
// ST rows are scaled by their exact 2-norm; Z / G rows by a Cauchy-Schwarz bound from
// the SY / ST row norms and the factors' row norms (|sigma^(k)| <= 1 for sin, <= 2 for
// tanh), so no per-chunk reduction is needed.  FP16 operands halve the shared-memory
// bytes of the SS MMAs (which are shared-memory bound at N = 32: 42 cycles for
// tf32 K8 vs 42 for f16 K16, scripts/umma_issue_tf32.cu) and let SY_l stay resident
// for the reverse recompute.
// TMEM (512 columns): forward P1 | SY | Z | Y;  reverse A | DZ | G | T.
// Warp roles: 16 epilogue warps; warp 16 issues P1-type MMAs; warp 17 issues P2-type
// MMAs and the factor-chunk TMA bulk copies (4-slot ring).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pinn_kernels.cuh"
#include "pinn_v2.cuh"
#include "umma.cuh"

namespace lrnr_b200 {
namespace tc {

constexpr int P = 128;    // points per tile (MMA M)
constexpr int KC = 32;    // neurons per chunk (N of the P1-type MMAs, K of the P2-type)
constexpr int RP = 32;    // max padded rank
constexpr int NWE = 16;   // epilogue warps: lane quarter = warp % 4, neuron / rank group h = warp / 4
constexpr int ISSUER = NWE;       // P1-type MMAs
constexpr int ISSUER2 = NWE + 1;  // P2-type MMAs + TMA producer
constexpr int NT = 32 * (NWE + 2);
constexpr int NG = 8;             // neurons / ranks per epilogue thread
// TMEM columns
constexpr int TM_R = 0;     // forward: P1; reverse: A at 0, DZ at 128
constexpr int TM_SY = 128;  // forward: SY (fp16 hi | lo per slot, like Z): the A operand of P1 (TS)
constexpr int TM_Z = 256;   // Z / G: per slot 32 columns = fp16 hi (16 columns) | lo (16 columns)
constexpr int TM_Y = 384;   // Y / T: per slot 32 fp32 columns
// Phase-2 products of YACC consecutive chunks accumulate in TMEM before the epilogue
// adds them to its FP32 running sum (a long tensor-core accumulation loses precision:
// K = 256 in one accumulator reached 1.2e-4 with 3xTF32).
constexpr int YACC = 2;
// reverse: T products of YACC_R chunks per accumulator.  Measured on c2 (scripts/c2_err.py):
// the reverse tolerates a whole transition (8 chunks) in one accumulator with no change in
// the error (dL/ds 7.8e-6), the forward does not (8 chunks: dL/ds 3.3e-5, loss 6.4e-5), so
// YACC = 2, YACC_R = 8 (c2 LRNR 13.18 -> 12.87 ms: no running T sum live in the chunk loop)
constexpr int YACC_R = 8;

// shared memory (bytes)
constexpr int OPD_HALF = P * RP * 2;           // one fp16 tile of a jet slot (128 rows x 32 K)
constexpr int OPD_SLOT = 2 * OPD_HALF;         // hi | lo
constexpr int OFF_X = 0;                       // SY (forward) / ST (reverse): P1-type A operand
constexpr int OFF_W = OFF_X + 4 * OPD_SLOT;    // reverse: SY_l for the recomputed pre-activations
constexpr int BUF = 3 * (4 * KC * RP) + 4 * KC;  // largest chunk block: three fp16 hi / lo 32 x 32 tiles + bias
constexpr int NBUF = 4;
constexpr int OFF_B0 = OFF_W + 4 * OPD_SLOT;
constexpr int OFF_RED = OFF_B0 + NBUF * BUF;   // floats: per-warp-quarter partials [layer][4][RP], loss [4]
constexpr int OFF_XCH = OFF_RED + (kMaxL * 4 * RP + 4) * 4;  // floats [4 groups][P][8]
constexpr int OFF_ACC = OFF_XCH + 4 * P * 8 * 4;
constexpr int OFF_S = OFF_ACC + 1024 * 4;      // the unit's s vector (FP32)
constexpr int SMEM_BYTES = OFF_S + 1024 * 4;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
static_assert(BUF % 16 == 0 && OFF_B0 % 1024 == 0, "alignment");

struct NetTC {
    int L;
    int M[kMaxL + 1];
    int r[kMaxL];
    int rk[kMaxL];         // padded rank as MMA K (multiple of 16, <= 32)
    int rn[kMaxL];         // padded rank as MMA N (16 or 32)
    int nc[kMaxL];
    int soff[kMaxL + 1];
    int yoff[kMaxL];       // y_l in per-CTA scratch: [j (r_l)][p][4] (a layer is one contiguous block)
    int ystride;
    int kU[kMaxL];         // factor scales 2^kU (U_l) and 2^kV (V_l)
    int kV[kMaxL];
    float muU[kMaxL];      // max row 2-norm of U_l / V_l (bounds of the pre-activation jets)
    float muV[kMaxL];
    float c3;              // max |sigma'''| (1 sin, 2 tanh)
    int rtotal;
    const unsigned char* blocks;
    const int64_t* sched_off;  // bytes
    const int* sched_bytes;
    int sched_len;
    const float* V0;       // 2 x r[0]
    const float* ulast;    // r[L-1] then b_{L-1}[0]
};

// Optional phase timing (dev aid): -DLRNR_TC_TIMING records clock64 deltas of
// CTA 0 / thread 32 into a global array (see scripts/tc_timing.py).
#ifdef LRNR_TC_TIMING
__device__ unsigned long long g_tc_timing[16];
#define TC_T0()                                                \
    __shared__ unsigned long long _tc_acc[16];                 \
    if (threadIdx.x < 16) _tc_acc[threadIdx.x] = 0;            \
    __syncthreads();                                           \
    long long _tt = clock64();
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
#define TC_MARK(i)
#define TC_FLUSH()
#endif

// Sum of v[0..7] over the warp's 32 lanes (points), fixed butterfly order: lanes with
// (lane & 3) == 0 return the sum of value ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1).
__device__ __forceinline__ float warp_sum8(const float (&v)[8], int lane) {
    float a[4], b[2];
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = (u16 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, u16 ? v[i] : v[i + 4], 16);
#pragma unroll
    for (int i = 0; i < 2; ++i) b[i] = (u8 ? a[i + 2] : a[i]) + __shfl_xor_sync(0xffffffffu, u8 ? a[i] : a[i + 2], 8);
    float c = (u4 ? b[1] : b[0]) + __shfl_xor_sync(0xffffffffu, u4 ? b[0] : b[1], 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    return c;
}
__device__ __forceinline__ int warp_sum8_index(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }

// acc[c][n] += iv[c] * TMEM[taddr + c * 32 + n] (YACC chunks of phase-2 products, unscaled)
__device__ __forceinline__ void add_acc(uint32_t taddr, const float (&iv)[4], float (&acc)[4][NG]) {
    float v[4][NG];
#pragma unroll
    for (int c = 0; c < 4; ++c) umma::tmem_ld8(taddr + c * 32, v[c]);
    umma::tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int n = 0; n < NG; ++n) acc[c][n] = fmaf(v[c][n], iv[c], acc[c][n]);
}

// Write this thread's 8 values (K block h = ranks 8h..8h+7) of point p of the four jet
// slots into an operand buffer (fp16 hi / lo tiles) after scaling slot c by 2^e[c]:
// a quarter-warp's 8 points fill one 128-byte core matrix (conflict-free 16-B stores).
__device__ __forceinline__ void put_rows(unsigned char* buf, int p, int h, const float (&v)[4][NG], const int (&e)[4]) {
    const int o = umma::kmaj16_off(p, 8 * h, P);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float s = umma::exp2i(e[c]);
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) umma::split16x2_fh(v[c][2 * i] * s, v[c][2 * i + 1] * s, hw[i], lw[i]);
        *reinterpret_cast<uint4*>(buf + c * OPD_SLOT + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(buf + c * OPD_SLOT + OPD_HALF + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// named barrier over the 4 epilogue warps that share a TMEM lane quarter (the same 32 points):
// enough for the per-point norm exchanges through xch
__device__ __forceinline__ void quarter_bar(int quarter) { asm volatile("bar.sync %0, 128;" ::"r"(8 + quarter) : "memory"); }

// The same 8 values into the forward SY operand in TMEM (this thread's lane = point p,
// K block h): per slot, 4 packed hi columns at c * 32 + 4h and 4 lo columns 16 further.
__device__ __forceinline__ void put_rows_tmem(uint32_t tsy, int h, const float (&v)[4][NG], const int (&e)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float s = umma::exp2i(e[c]);
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) umma::split16x2_fh(v[c][2 * i] * s, v[c][2 * i + 1] * s, hw[i], lw[i]);
        umma::tmem_st4u(tsy + c * 32 + 4 * h, hw[0], hw[1], hw[2], hw[3]);
        umma::tmem_st4u(tsy + c * 32 + 16 + 4 * h, lw[0], lw[1], lw[2], lw[3]);
    }
}

template <int ACT, bool FAST>
__device__ __forceinline__ void act3f(float a, float& sg, float& d1, float& d2, float& d3) {
    v2::act3<ACT, FAST>(a, sg, d1, d2, d3);
}

// Row norms only select power-of-two scales and bounds (one bit of FP16 headroom is kept), so the
// SFU square root (2 ulp) replaces the correctly rounded sequence at the transition ends.
__device__ __forceinline__ float sqrt_fast(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^k for an integer exponent, clamped to the normal range
__device__ __forceinline__ float exp2c(int k) { return umma::exp2i(max(-126, min(127, k))); }

// Per-point constants of one transition with the power-of-two unscale (P1 / P2 products)
// and scale (Z / G operands) factors folded in.  Exponents, each in [-40, 40]: Ea / Ed = the
// combined scale of a raw P1-type product (row scale of SY / ST + factor scale), ez / eg =
// Z / G row scales, kV / kU = the P2-type factor scales.  Every constant combines at most
// three of them, so it is a normal FP32 power of two.
struct FwdScales {
    float ia0;          // A_v = P1_v 2^-Ea0 + b
    float f1, f2, f3;   // Z_c 2^ez_c = d1 P1_c 2^(ez_c - Ea_c), c = 1, 2; u_w term d1 P1_3 f3
    float g3;           // Z_3 2^ez3 = d2 P1_1^2 2^(ez3 - 2 Ea1) + d1 P1_3 f3
    float s0;           // Z_0 2^ez0 = sigma s0
    float iy[4];        // Y unscale 2^-(ez_c + kV)
};
struct RevScales {
    float ia0, ia1;                  // A_v = P1r_v 2^-Ea0 + b;  A_x = P1r_x 2^-Ea1
    float k0, k01, k02, k03, k04;    // G0 2^eg0 = d1 e0 k0 + d2 (e1 r1 k01 + e2 r2 k02 + e3 r3 k03) + d3 e3 r1 A_x k04
    float k1, k13, k2, k3;           // G1 2^eg1 = d1 e1 k1 + d2 r1 e3 k13; G2 = d1 e2 k2; G3 = d1 e3 k3
    float it[4];                     // T unscale 2^-(eg_c + kU)
};
// (r = recomputed P1r columns, scaled by 2^Ea; e = DZ columns, scaled by 2^Ed)

// Combined exponents of the raw P1-type products: E_c = clamp(e_c + k) for the natural row
// exponents e_c; the row is then written with scale 2^(E_c - k) (e_c updated to it)
__device__ __forceinline__ void combine_exp(int (&e)[4], int k, int (&E)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        E[c] = max(-40, min(40, e[c] + k));
        e[c] = E[c] - k;
    }
}

// Forward constants from the exact SY row norms (combined exponents Ea[c]) of transition l.
__device__ __forceinline__ void fwd_scales(FwdScales& f, const NetTC& net, int l, const float (&nr)[4], const int (&Ea)[4]) {
    const int kV = net.kV[l];
    const float mu = net.muU[l];
    const float bx = nr[1] * mu, bt = nr[2] * mu, bw = nr[3] * mu;
    const int ez[4] = {umma::pow2_exp(1.f), umma::pow2_exp(bx), umma::pow2_exp(bt), umma::pow2_exp(fmaf(bx, bx, bw))};
    f.ia0 = exp2c(-Ea[0]);
    f.f1 = exp2c(ez[1] - Ea[1]);
    f.f2 = exp2c(ez[2] - Ea[2]);
    f.f3 = exp2c(ez[3] - Ea[3]);
    f.g3 = exp2c(ez[3] - 2 * Ea[1]);
    f.s0 = exp2c(ez[0]);
#pragma unroll
    for (int c = 0; c < 4; ++c) f.iy[c] = exp2c(-ez[c] - kV);
}

// NARROW: every transition is a single chunk (the FastLRNR).  The chunk-loop operand splits then
// use the mixed-precision FMA form as well: those sweeps are latency-bound (c2 FastLRNR 4.55 ->
// 4.49 ms), while the issue-bound wide sweeps keep cvt + sub (c2 LRNR 12.66 vs 12.80 ms).
template <int ACT, bool FAST, bool NARROW>
__global__ void __launch_bounds__(NT, 1)
pinn_tc_kernel(const NetTC net, const RunGeom g, const double* __restrict__ pts, const double* __restrict__ svec,
               const double* __restrict__ mus, const float w, float* __restrict__ scratch, float* __restrict__ part,
               unsigned long long* __restrict__ bad, unsigned long long* __restrict__ unit_ctr) {
    extern __shared__ __align__(1024) unsigned char smb[];
    float* tpart = reinterpret_cast<float*>(smb + OFF_RED);  // [layer][quarter][rank], then loss [quarter]
    float* xch = reinterpret_cast<float*>(smb + OFF_XCH);
    float* acc = reinterpret_cast<float*>(smb + OFF_ACC);
    float* ssm = reinterpret_cast<float*>(smb + OFF_S);
    unsigned char* X = smb + OFF_X;
    unsigned char* W = smb + OFF_W;
    __shared__ __align__(8) uint64_t wbar[NBUF];           // ring slot filled (TMA)
    __shared__ __align__(8) uint64_t p1full;     // forward P1 written (tcgen05.commit)
    __shared__ __align__(8) uint64_t rfull;      // reverse A / DZ written
    __shared__ __align__(8) uint64_t afull;      // reverse A written (the DZ MMAs still run)
    __shared__ __align__(8) uint64_t zfree;      // P2 done: Z / G free, Y / T product ready
    __shared__ __align__(8) uint64_t ybar;       // y_l block copied into W (TMA)
    __shared__ uint32_t tmem_base;
    __shared__ int64_t next_unit;

    const int tid = threadIdx.x;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const int quarter = warp & 3, h = warp >> 2;  // h: neuron / rank group (epilogue warps)
    const int p = quarter * 32 + lane;            // the point (TMEM lane) this thread serves
    const int R1 = 1 + net.rtotal;
    const int L = net.L;
    float* scr = scratch + static_cast<int64_t>(blockIdx.x) * net.ystride;

    for (int k = tid; k < R1; k += NT) acc[k] = 0.f;
    if (warp == 0) umma::tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < NBUF; ++i) umma::mbar_init(&wbar[i], 1);
        umma::mbar_init(&p1full, 1);
        umma::mbar_init(&rfull, 1);
        umma::mbar_init(&afull, 1);
        umma::mbar_init(&zfree, 1);
        umma::mbar_init(&ybar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tmem_base;
    const uint32_t tlane = tbase + (static_cast<uint32_t>(quarter * 32) << 16);

    auto wait = [&](uint64_t* bar, uint32_t parity) {
        umma::mbar_wait(bar, parity);
        umma::fence_after();
    };
    // epilogue -> issuer hand-offs are hardware named barriers (the 16 epilogue warps
    // arrive, the issuer warp syncs: it blocks without spinning; at most one generation
    // of each is outstanding): Z / G written, forward P1 buffer 0 / 1 read, reverse A / DZ read
    // (barrier 1 is the epilogue-only barrier)
    constexpr int BAR_ZFULL = 2, BAR_P1FREE = 3, BAR_RFREE = 5, BAR_N = NWE * 32 + 32;
    auto signal = [&](int id) {
        umma::fence_before();
        __syncwarp();
        asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(BAR_N) : "memory");
    };
    auto await = [&](int id) {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(BAR_N) : "memory");
        umma::fence_after();
    };

    // ---- factor-chunk ring (TMA bulk copies, issued by ISSUER2's elected lane) ----
    // every tile runs the same chunk schedule; the copies in flight past the last chunk
    // are drained at exit
    auto tma = [&](int64_t qq) {
        const int e = static_cast<int>(qq % net.sched_len);
        const int b = static_cast<int>(qq % NBUF);
        v2::fence_proxy_async();
        v2::mbar_expect_tx(&wbar[b], static_cast<uint32_t>(net.sched_bytes[e]));
        v2::bulk_g2s(smb + OFF_B0 + b * BUF, net.blocks + net.sched_off[e], static_cast<uint32_t>(net.sched_bytes[e]),
                     &wbar[b]);
    };
    const bool producer = warp == ISSUER2 && lane == 0;
    if (producer)
        for (int i = 0; i < NBUF; ++i) tma(i);
    auto wait_slot = [&](int64_t qq) { wait(&wbar[qq % NBUF], static_cast<uint32_t>((qq / NBUF) & 1)); };
    auto slot = [&](int64_t qq) { return smb + OFF_B0 + static_cast<int>(qq % NBUF) * BUF; };

    // descriptor words: high word SBO = 128 B, version 1; low words start >> 4 | LBO >> 4 << 16
    const uint32_t dhi = umma::desc_hi(128);
    auto dlo = [&](const unsigned char* ptr, int rows) { return umma::desc_lo(ptr, (rows / 8) * 128); };
    const uint32_t idP1 = umma::idesc_f16(P, KC);
    // P1-type MMAs (SS) into d: A = operand buffer (4 slots), B = fp16 hi / lo tile of
    // 32 neuron rows at bsrc; K = rk (multiple of 16).  One elected lane issues.
    auto mma_p1 = [&](uint32_t d, const unsigned char* abuf, const unsigned char* bsrc, int rk) {
        const uint32_t bh = dlo(bsrc, KC), bl = dlo(bsrc + 2 * KC * rk, KC);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t ah = dlo(abuf + c * OPD_SLOT, P), al = dlo(abuf + c * OPD_SLOT + OPD_HALF, P);
            for (int s = 0; s < rk / 16; ++s) {
                const uint32_t sa = s * 2 * P, sb = s * 2 * KC;  // 16-B units per K step of 16
                umma::mma16_ss(d + c * 32, ah + sa, bh + sb, dhi, idP1, s > 0);
                umma::mma16_ss(d + c * 32, ah + sa, bl + sb, dhi, idP1, 1);
                umma::mma16_ss(d + c * 32, al + sa, bh + sb, dhi, idP1, 1);
            }
        }
    };
    // forward P1 (TS): A = SY in TMEM (fp16 hi / lo columns per slot), B = U^T chunk; K = rk
    auto mma_p1_ts = [&](const unsigned char* bsrc, int rk) {
        const uint32_t bh = dlo(bsrc, KC), bl = dlo(bsrc + 2 * KC * rk, KC);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t d = tbase + TM_R + c * 32, ay = tbase + TM_SY + c * 32;
            for (int s = 0; s < rk / 16; ++s) {
                const uint32_t sb = s * 2 * KC;
                umma::mma16_ts(d, ay + 8 * s, bh + sb, dhi, idP1, s > 0);
                umma::mma16_ts(d, ay + 8 * s, bl + sb, dhi, idP1, 1);
                umma::mma16_ts(d, ay + 16 + 8 * s, bh + sb, dhi, idP1, 1);
            }
        }
    };
    // P2-type MMAs (TS): D = TM_Y, A = Z / G in TMEM, B = fp16 hi / lo tile of rn rows x KC at bsrc
    auto mma_p2 = [&](const unsigned char* bsrc, int rn, bool acc0) {
        const uint32_t id2 = umma::idesc_f16(P, rn);
        const uint32_t bh = dlo(bsrc, rn), bl = dlo(bsrc + 2 * rn * KC, rn);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t d = tbase + TM_Y + c * 32, az = tbase + TM_Z + c * 32;
#pragma unroll
            for (int s = 0; s < KC / 16; ++s) {
                const uint32_t sb = s * 2 * rn;
                umma::mma16_ts(d, az + 8 * s, bh + sb, dhi, id2, (s > 0 || acc0) ? 1u : 0u);
                umma::mma16_ts(d, az + 8 * s, bl + sb, dhi, id2, 1);
                umma::mma16_ts(d, az + 16 + 8 * s, bh + sb, dhi, id2, 1);
            }
        }
    };

    int64_t q = 0;      // global chunk counter (ring schedule)
    uint32_t fq = 0;    // forward chunks (P1 buffer uses)
    uint32_t rq = 0;    // reverse chunks
    uint32_t zw = 0;    // epilogue: zfree completions consumed

    // ISSUER2 per chunk: wait for Z / G, refill the previous chunk's ring slot (Z / G of
    // chunk qq are written only after P2(qq - 1), the slot's last reader, completed),
    // then issue the phase-2 MMAs
    auto issue_p2 = [&](int64_t qq, const unsigned char* bsrc, int rn, bool acc0) {
        await(BAR_ZFULL);
        if (umma::elect_one()) {
            mma_p2(bsrc, rn, acc0);
            umma::mma_commit_1(&zfree);
        }
        __syncwarp();
        if (lane == 0 && qq >= 1) tma(qq - 1 + NBUF);  // after the MMAs: the epilogue may be waiting for them
        __syncwarp();
    };
    // ISSUER: forward P1 of chunk qq into buffer fq & 1
    auto issue_fwd_p1 = [&](int64_t qq, uint32_t fqq, int rk) {
        wait_slot(qq);
        if (fqq >= 1) await(BAR_P1FREE);  // the epilogue has read P1(qq - 1)
        if (umma::elect_one()) {
            mma_p1_ts(slot(qq), rk);
            umma::mma_commit_1(&p1full);
        }
        __syncwarp();
    };
    // ISSUER: reverse A (recomputed) and DZ of chunk qq
    auto issue_rev_p1 = [&](int64_t qq, uint32_t rqq, int rkl, int rkn) {
        wait_slot(qq);
        if (rqq >= 1) await(BAR_RFREE);
        if (umma::elect_one()) {
            const unsigned char* b = slot(qq);
            mma_p1(tbase + TM_R, W, b, rkl);                               // A = SY_l U^T
            umma::mma_commit_1(&afull);  // the epilogue starts the activation jets of its first neurons on A
            mma_p1(tbase + TM_R + 128, X, b + 4 * KC * rkl + 4 * KC, rkn);  // DZ = ST_{l+1} V^T
            umma::mma_commit_1(&rfull);
        }
        __syncwarp();
    };

    // ISSUER lane 0: copy the y_l block of this CTA's scratch into W (the epilogue builds
    // SY_l there); the writers fenced their stores for the async proxy
    uint32_t yq = 0;  // ybar uses (issuer and epilogue count alike)
    auto prefetch_y = [&](int l) {
        if (lane == 0) {
            const uint32_t bytes = static_cast<uint32_t>(P * net.r[l] * 16);
            v2::mbar_expect_tx(&ybar, bytes);
            v2::bulk_g2s(W, scr + net.yoff[l], bytes, &ybar);
        }
        __syncwarp();
    };

    // Reverse scales of transition lr from the exchanged squared row norms of ST_{lr+1}
    // (nst) and SY_lr (nsy); writes this thread's K block of ST_{lr+1} into X and of
    // SY_lr into W.  G bound (|sigma'|, |sigma''| <= 1, |sigma'''| <= c3, |DZ_c| <= |ST_c| muV,
    // |A_c| <= |SY_c| muU): |G0| <= B0 + B1 bx + B2 bt + B3 (c3 bx^2 + bw), |G1| <= B1 + 2 B3 bx.
    auto rev_scales = [&](RevScales& r, float (&nst)[4], float (&nsy)[4], int lr, const float (&st)[4][NG],
                          const float (&sy)[4][NG]) {
        int est[4], esy[4], Ed[4], Ea[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            nst[c] = sqrt_fast(nst[c]);
            nsy[c] = sqrt_fast(nsy[c]);
            est[c] = umma::pow2_exp(nst[c]);
            esy[c] = umma::pow2_exp(nsy[c]);
        }
        const int kU = net.kU[lr], kV = net.kV[lr];
        combine_exp(est, kV, Ed);  // DZ = ST V^T
        combine_exp(esy, kU, Ea);  // A = SY U^T
        if (NG * h < net.rk[lr + 1]) put_rows(X, p, h, st, est);
        if (NG * h < net.rk[lr]) put_rows(W, p, h, sy, esy);
        const float mu = net.muU[lr], mv = net.muV[lr];
        const float bx = nsy[1] * mu, bt = nsy[2] * mu, bw = nsy[3] * mu;
        const float B0 = nst[0] * mv, B1 = nst[1] * mv, B2 = nst[2] * mv, B3 = nst[3] * mv;
        const int eg0 = umma::pow2_exp(B0 + B1 * bx + B2 * bt + B3 * fmaf(net.c3 * bx, bx, bw));
        const int eg1 = umma::pow2_exp(fmaf(2.f * B3, bx, B1));
        const int eg2 = umma::pow2_exp(B2), eg3 = umma::pow2_exp(B3);
        r.ia0 = exp2c(-Ea[0]);
        r.ia1 = exp2c(-Ea[1]);
        r.k0 = exp2c(eg0 - Ed[0]);
        r.k01 = exp2c(eg0 - Ed[1] - Ea[1]);
        r.k02 = exp2c(eg0 - Ed[2] - Ea[2]);
        r.k03 = exp2c(eg0 - Ed[3] - Ea[3]);
        r.k04 = exp2c(eg0 - Ed[3] - Ea[1]);  // times A_x (unscaled) in the A_x^2 term
        r.k1 = exp2c(eg1 - Ed[1]);
        r.k13 = 2.f * exp2c(eg1 - Ed[3] - Ea[1]);
        r.k2 = exp2c(eg2 - Ed[2]);
        r.k3 = exp2c(eg3 - Ed[3]);
        r.it[0] = exp2c(-eg0 - kU);
        r.it[1] = exp2c(-eg1 - kU);
        r.it[2] = exp2c(-eg2 - kU);
        r.it[3] = exp2c(-eg3 - kU);
    };

    TC_T0();
    // claims: the counter starts at all-ones (memset 0xff), so the first claim returns unit gridDim.x
    unsigned long long claim = 0;
    if (tid == 0) claim = atomicAdd(unit_ctr, 1ull) + 1ull + gridDim.x;
    int64_t s_inst = -1;  // the instance whose s vector is staged
    for (int64_t unit = blockIdx.x; unit < g.n_units;) {
        const int64_t inst = unit / g.units_per_inst;
        const int seg = static_cast<int>(unit % g.units_per_inst);
        const int t_lo = seg * g.tiles_per_unit;
        const int t_hi = min(g.tiles_per_inst, t_lo + g.tiles_per_unit);
        // the instance's s coefficients in shared memory (read at every transition end)
        if (inst != s_inst) {
            for (int k = tid; k < net.rtotal; k += NT) ssm[k] = static_cast<float>(svec[inst * net.rtotal + k]);
            s_inst = inst;
            __syncthreads();
        }
        const float* sv = ssm;
        const float mu0 = float(mus[3 * inst]), mu1 = float(mus[3 * inst + 1]), mu2 = float(mus[3 * inst + 2]);

        for (int tile = t_lo; tile < t_hi; ++tile) {
            const int64_t pi = static_cast<int64_t>(tile) * P + p;
            const bool valid = pi < g.n_per_inst;
            const int64_t gp = inst * g.n_per_inst + pi;
            FwdScales fs;
            // ---------------- input layer: y_0 = V_0^T z_0, SY_0 = s_0 (.) y_0 ----------------
            {
                float sy[4][NG];
                if (warp < NWE) {
                    const float x = valid ? float(pts[2 * gp]) : 0.f;
                    const float t = valid ? float(pts[2 * gp + 1]) : 0.f;
                    const int r0 = net.r[0];
                    float ss[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int n = 0; n < NG; ++n) {
                        const int j = NG * h + n;
                        float y4[4] = {0.f, 0.f, 0.f, 0.f};
                        float sj = 0.f;
                        if (j < r0) {
                            const float v0 = net.V0[j], v1 = net.V0[r0 + j];
                            y4[0] = v0 * x + v1 * t;
                            y4[1] = v0;
                            y4[2] = v1;
                            sj = float(sv[j]);
                            v2::st4(scr + net.yoff[0] + (j * P + p) * 4, y4[0], y4[1], y4[2], y4[3]);
                        }
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            sy[c][n] = sj * y4[c];
                            ss[c] = fmaf(sy[c][n], sy[c][n], ss[c]);
                        }
                    }
                    *reinterpret_cast<float4*>(xch + (h * P + p) * 8) = make_float4(ss[0], ss[1], ss[2], ss[3]);
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // y_0 may be read by a bulk copy
                    quarter_bar(quarter);
                }
                if (warp < NWE) {
                    float nr[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int hh = 0; hh < 4; ++hh) {
                        const float4 v = *reinterpret_cast<const float4*>(xch + (hh * P + p) * 8);
                        nr[0] += v.x;
                        nr[1] += v.y;
                        nr[2] += v.z;
                        nr[3] += v.w;
                    }
                    int e[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        nr[c] = sqrt_fast(nr[c]);
                        e[c] = umma::pow2_exp(nr[c]);
                    }
                    int Ea[4];
                    combine_exp(e, net.kU[0], Ea);
                    if (NG * h < net.rk[0]) put_rows_tmem(tlane + TM_SY, h, sy, e);
                    umma::tmem_st_wait();
                    fwd_scales(fs, net, 0, nr, Ea);
                }
                umma::fence_before();  // SY in TMEM -> the first P1
                __syncthreads();
            }

            // ---------------- forward transitions ----------------
            RevScales rs;
            for (int l = 0; l + 1 < L; ++l) {
                const int rk = net.rk[l], rnn = net.rn[l + 1], nc = net.nc[l];
                const int fbias = 4 * KC * rk, fv = fbias + 4 * KC;  // byte offsets in the forward block
                float ysum[4][NG];
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int n = 0; n < NG; ++n) ysum[c][n] = 0.f;
                if (warp == ISSUER) {
                    issue_fwd_p1(q, fq, rk);
                    if (l + 2 == L) prefetch_y(L - 2);  // W is free in the forward sweep (after the MMAs: the epilogue waits for them)
                }
                for (int ch = 0; ch < nc; ++ch, ++q, ++fq) {
                    if (warp == ISSUER) {
                        if (ch + 1 < nc) issue_fwd_p1(q + 1, fq + 1, rk);
                    } else if (warp == ISSUER2) {
                        issue_p2(q, slot(q) + fv, rnn, ch % YACC != 0);
                    } else {
                        TC_MARK(1);
                        wait(&p1full, fq & 1);
                        TC_MARK(2);
                        const float* bias = reinterpret_cast<const float*>(slot(q) + fbias);
                        float a[4][NG];
#pragma unroll
                        for (int c = 0; c < 4; ++c) umma::tmem_ld8(tlane + TM_R + c * 32 + NG * h, a[c]);
                        umma::tmem_ld_wait();
                        signal(BAR_P1FREE);  // P1 may take chunk q + 1
                        uint32_t zh[4][NG / 2], zl[4][NG / 2];
#pragma unroll
                        for (int n = 0; n < NG; n += 2) {
                            float z[2][4];
#pragma unroll
                            for (int i = 0; i < 2; ++i) {
                                const float r1 = a[1][n + i], r2 = a[2][n + i], r3 = a[3][n + i];
                                const float av = fmaf(a[0][n + i], fs.ia0, bias[NG * h + n + i]);
                                float sg, d1, d2, d3;
                                act3f<ACT, FAST>(av, sg, d1, d2, d3);
                                z[i][0] = sg * fs.s0;
                                z[i][1] = d1 * (r1 * fs.f1);
                                z[i][2] = d1 * (r2 * fs.f2);
                                z[i][3] = fmaf(d2 * r1, r1 * fs.g3, d1 * (r3 * fs.f3));
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                if constexpr (NARROW) umma::split16x2_fh(z[0][c], z[1][c], zh[c][n / 2], zl[c][n / 2]);
                                else umma::split16x2(z[0][c], z[1][c], zh[c][n / 2], zl[c][n / 2]);
                            }
                        }
                        TC_MARK(3);
                        if (ch > 0) {
                            wait(&zfree, zw & 1);  // P2(q - 1): Z free, its Y product ready
                            ++zw;
                            if (ch % YACC == 0) add_acc(tlane + TM_Y + NG * h, fs.iy, ysum);
                        }
                        TC_MARK(0);
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint32_t zc = tlane + TM_Z + c * 32 + (NG / 2) * h;
                            umma::tmem_st4u(zc, zh[c][0], zh[c][1], zh[c][2], zh[c][3]);
                            umma::tmem_st4u(zc + 16, zl[c][0], zl[c][1], zl[c][2], zl[c][3]);
                        }
                        umma::tmem_st_wait();
                        signal(BAR_ZFULL);
                        TC_MARK(4);
                    }
                }
                // transition end: Y -> y_{l+1} (scratch), then SY_{l+1} or the output layer
                const bool last = l + 2 == L;
                const float* sl = sv + net.soff[l + 1];
                const int rtrue = net.r[l + 1];
                if (warp < NWE) {
                    wait(&zfree, zw & 1);
                    ++zw;
                    add_acc(tlane + TM_Y + NG * h, fs.iy, ysum);
                    TC_MARK(13);
                    float pr[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int n = 0; n < NG; ++n) {
                        const int j = NG * h + n;
                        float sj = 0.f;
                        if (j < rtrue) {
                            v2::st4(scr + net.yoff[l + 1] + (j * P + p) * 4, ysum[0][n], ysum[1][n], ysum[2][n],
                                    ysum[3][n]);
                            sj = float(sl[j]);
                            if (last) sj *= net.ulast[j];
                        }
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float v = sj * ysum[c][n];
                            pr[c] = last ? pr[c] + v : fmaf(v, v, pr[c]);
                            if (!last) ysum[c][n] = v;  // SY_{l+1}
                        }
                    }
                    *reinterpret_cast<float4*>(xch + (h * P + p) * 8) = make_float4(pr[0], pr[1], pr[2], pr[3]);
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // y_{l+1} may be read by a bulk copy
                    quarter_bar(quarter);
                }
                TC_MARK(5);
                if (warp < NWE) {
                    float nr[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int hh = 0; hh < 4; ++hh) {
                        const float4 v = *reinterpret_cast<const float4*>(xch + (hh * P + p) * 8);
                        nr[0] += v.x;
                        nr[1] += v.y;
                        nr[2] += v.z;
                        nr[3] += v.w;
                    }
                    if (!last) {
                        int e[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            nr[c] = sqrt_fast(nr[c]);
                            e[c] = umma::pow2_exp(nr[c]);
                        }
                        int Ea[4];
                        combine_exp(e, net.kU[l + 1], Ea);
                        if (NG * h < net.rk[l + 1]) put_rows_tmem(tlane + TM_SY, h, ysum, e);
                        umma::tmem_st_wait();
                        fwd_scales(fs, net, l + 1, nr, Ea);
                    } else {
                        // ---------------- output layer (M_L = 1) + residual ----------------
                        float u[4] = {nr[0] + net.ulast[rtrue], nr[1], nr[2], nr[3]};
                        const float N = u[2] + mu0 * u[1] - mu1 * u[3] - mu2 * u[0] * (1.f - u[0]);
                        const float term = valid ? w * (N * N) : 0.f;
                        if (h == 0) {
                            if (valid && !isfinite(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
                            float tsm = term;
#pragma unroll
                            for (int o = 16; o >= 1; o >>= 1) tsm += __shfl_xor_sync(0xffffffffu, tsm, o);
                            if (lane == 0) tpart[kMaxL * 4 * RP + quarter] = tsm;
                        }
                        const float gN = valid ? 2.f * N * w : 0.f;
                        const float gu[4] = {gN * (-mu2 * (1.f - 2.f * u[0])), gN * mu0, gN, -gN * mu1};
                        // ST_{L-1} (own ranks) and the dL/ds_{L-1} partials; y_{L-1} is ysum
                        float st[4][NG], cd[NG];
                        float ss[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int n = 0; n < NG; ++n) {
                            const int j = NG * h + n;
                            const float uj = j < rtrue ? net.ulast[j] : 0.f;
                            const float sj = j < rtrue ? float(sl[j]) : 0.f;
                            cd[n] = 0.f;
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                cd[n] = fmaf(uj * gu[c], ysum[c][n], cd[n]);
                                st[c][n] = sj * uj * gu[c];
                                ss[c] = fmaf(st[c][n], st[c][n], ss[c]);
                            }
                        }
                        {
                            const float v = warp_sum8(cd, lane);
                            if ((lane & 3) == 0) tpart[((L - 1) * 4 + quarter) * RP + NG * h + warp_sum8_index(lane)] = v;
                        }
                        // SY_{L-2} from y_{L-2} (copied into W during the last forward transition);
                        // the first reverse transition recomputes A_{L-2} from it
                        const int lr = L - 2, rr = net.r[lr];
                        const float* sr = sv + net.soff[lr];
                        float sy[4][NG];
                        float ssy[4] = {0.f, 0.f, 0.f, 0.f};
                        wait(&ybar, yq & 1);
                        ++yq;
#pragma unroll
                        for (int n = 0; n < NG; ++n) {
                            const int j = NG * h + n;
                            float y4[4] = {0.f, 0.f, 0.f, 0.f};
                            float sj = 0.f;
                            if (j < rr) {
                                v2::ld4(reinterpret_cast<const float*>(W) + (j * P + p) * 4, y4);
                                sj = float(sr[j]);
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                sy[c][n] = sj * y4[c];
                                ssy[c] = fmaf(sy[c][n], sy[c][n], ssy[c]);
                            }
                        }
                        // the 4 warps of this lane quarter have read the u partials and their y_{L-2}
                        // (the y block and the SY operand tiles both keep a point's bytes at p * 16 of
                        // every 2 KB row block, so a quarter only ever touches its own 512-byte columns of W)
                        quarter_bar(quarter);
                        *reinterpret_cast<float4*>(xch + (h * P + p) * 8) = make_float4(ss[0], ss[1], ss[2], ss[3]);
                        *reinterpret_cast<float4*>(xch + (h * P + p) * 8 + 4) = make_float4(ssy[0], ssy[1], ssy[2], ssy[3]);
                        quarter_bar(quarter);
                        float nst[4] = {0.f, 0.f, 0.f, 0.f}, nsy[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int hh = 0; hh < 4; ++hh) {
                            const float4 v = *reinterpret_cast<const float4*>(xch + (hh * P + p) * 8);
                            const float4 v2 = *reinterpret_cast<const float4*>(xch + (hh * P + p) * 8 + 4);
                            nst[0] += v.x;
                            nst[1] += v.y;
                            nst[2] += v.z;
                            nst[3] += v.w;
                            nsy[0] += v2.x;
                            nsy[1] += v2.y;
                            nsy[2] += v2.z;
                            nsy[3] += v2.w;
                        }
                        rev_scales(rs, nst, nsy, lr, st, sy);
                    }
                }
                umma::fence_async_smem();
                umma::fence_before();
                __syncthreads();
                TC_MARK(6);
            }

            // ---------------- reverse transitions ----------------
            for (int l = L - 2; l >= 0; --l) {
                const int rkl = net.rk[l], rkn = net.rk[l + 1], rnl = net.rn[l], nc = net.nc[l];
                const int bbias = 4 * KC * rkl, bu = bbias + 4 * KC + 4 * KC * rkn;  // byte offsets in the reverse block
                float tsum[4][NG];
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int n = 0; n < NG; ++n) tsum[c][n] = 0.f;
                if (warp == ISSUER) issue_rev_p1(q, rq, rkl, rkn);
                for (int ch = 0; ch < nc; ++ch, ++q, ++rq) {
                    if (warp == ISSUER) {
                        if (ch + 1 < nc) issue_rev_p1(q + 1, rq + 1, rkl, rkn);
                    } else if (warp == ISSUER2) {
                        issue_p2(q, slot(q) + bu, rnl, ch % YACC_R != 0);
                    } else {
                        TC_MARK(7);
                        const float* bias = reinterpret_cast<const float*>(slot(q) + bbias);
                        uint32_t gh[4][NG / 2], gl[4][NG / 2];
                        // A lands first: the activation jets of the first 4 neurons overlap the DZ MMAs
                        float a0[4][NG / 2], j0[NG / 2][4];
                        wait(&afull, rq & 1);
#pragma unroll
                        for (int c = 0; c < 4; ++c) umma::tmem_ld4(tlane + TM_R + c * 32 + NG * h, a0[c]);
                        umma::tmem_ld_wait();
#pragma unroll
                        for (int n = 0; n < NG / 2; ++n)
                            act3f<ACT, FAST>(fmaf(a0[0][n], rs.ia0, bias[NG * h + n]), j0[n][0], j0[n][1], j0[n][2], j0[n][3]);
                        wait(&rfull, rq & 1);
                        TC_MARK(8);
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf) {
                            float a[4][NG / 2], dz[4][NG / 2];
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                if (hf == 1) umma::tmem_ld4(tlane + TM_R + c * 32 + NG * h + 4 * hf, a[c]);
                                umma::tmem_ld4(tlane + TM_R + 128 + c * 32 + NG * h + 4 * hf, dz[c]);
                            }
                            umma::tmem_ld_wait();
                            if (hf == 0) {
#pragma unroll
                                for (int c = 0; c < 4; ++c)
#pragma unroll
                                    for (int n = 0; n < NG / 2; ++n) a[c][n] = a0[c][n];
                            }
                            if (hf == 1) signal(BAR_RFREE);  // A / DZ consumed: the next chunk's MMAs may start
#pragma unroll
                            for (int n = 0; n < NG / 2; n += 2) {
                                float gg[2][4];
#pragma unroll
                                for (int i = 0; i < 2; ++i) {
                                    const float r1 = a[1][n + i], r2 = a[2][n + i], r3 = a[3][n + i];
                                    const float e0 = dz[0][n + i], e1 = dz[1][n + i], e2 = dz[2][n + i], e3 = dz[3][n + i];
                                    float sg, d1, d2, d3;
                                    if (hf == 0) {
                                        sg = j0[n + i][0];
                                        d1 = j0[n + i][1];
                                        d2 = j0[n + i][2];
                                        d3 = j0[n + i][3];
                                    } else {
                                        const float av = fmaf(a[0][n + i], rs.ia0, bias[NG * h + 4 * hf + n + i]);
                                        act3f<ACT, FAST>(av, sg, d1, d2, d3);
                                    }
                                    float wv = (e3 * rs.k03) * r3;
                                    wv = fmaf(e2 * rs.k02, r2, wv);
                                    wv = fmaf(e1 * rs.k01, r1, wv);
                                    const float xv = ((e3 * rs.k04) * r1) * (r1 * rs.ia1);
                                    gg[i][0] = fmaf(d1, e0 * rs.k0, fmaf(d2, wv, d3 * xv));
                                    gg[i][1] = fmaf(d1, e1 * rs.k1, (d2 * r1) * (e3 * rs.k13));
                                    gg[i][2] = d1 * (e2 * rs.k2);
                                    gg[i][3] = d1 * (e3 * rs.k3);
                                }
#pragma unroll
                                for (int c = 0; c < 4; ++c) {
                                    if constexpr (NARROW)
                                        umma::split16x2_fh(gg[0][c], gg[1][c], gh[c][2 * hf + n / 2], gl[c][2 * hf + n / 2]);
                                    else
                                        umma::split16x2(gg[0][c], gg[1][c], gh[c][2 * hf + n / 2], gl[c][2 * hf + n / 2]);
                                }
                            }
                        }
                        TC_MARK(9);
                        if (ch > 0) {
                            wait(&zfree, zw & 1);  // P2r(q - 1): G free, its T product ready
                            ++zw;
                            if (ch % YACC_R == 0) add_acc(tlane + TM_Y + NG * h, rs.it, tsum);
                        }
                        TC_MARK(10);
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint32_t zc = tlane + TM_Z + c * 32 + (NG / 2) * h;
                            umma::tmem_st4u(zc, gh[c][0], gh[c][1], gh[c][2], gh[c][3]);
                            umma::tmem_st4u(zc + 16, gl[c][0], gl[c][1], gl[c][2], gl[c][3]);
                        }
                        umma::tmem_st_wait();
                        signal(BAR_ZFULL);
                        TC_MARK(11);
                    }
                }
                // transition end: T -> dL/ds_l partials; ST_l and SY_{l-1} for the next reverse transition
                const int rl = net.r[l];
                const float* sl = sv + net.soff[l];
                if (warp < NWE) {
                    float4 yv[NG];
#pragma unroll
                    for (int n = 0; n < NG; ++n) {
                        const int j = NG * h + n;
                        yv[n] = j < rl ? *reinterpret_cast<const float4*>(scr + net.yoff[l] + (j * P + p) * 4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    wait(&zfree, zw & 1);
                    ++zw;
                    add_acc(tlane + TM_Y + NG * h, rs.it, tsum);
                    TC_MARK(14);
                    float ss[4] = {0.f, 0.f, 0.f, 0.f};
                    {
                        float cd[NG];
#pragma unroll
                        for (int n = 0; n < NG; ++n) {
                            cd[n] = tsum[0][n] * yv[n].x;
                            cd[n] = fmaf(tsum[1][n], yv[n].y, cd[n]);
                            cd[n] = fmaf(tsum[2][n], yv[n].z, cd[n]);
                            cd[n] = fmaf(tsum[3][n], yv[n].w, cd[n]);
                        }
                        const float v = warp_sum8(cd, lane);
                        if ((lane & 3) == 0) tpart[(l * 4 + quarter) * RP + NG * h + warp_sum8_index(lane)] = v;
                    }
#pragma unroll
                    for (int n = 0; n < NG; ++n) {
                        const int j = NG * h + n;
                        const float sj = j < rl ? float(sl[j]) : 0.f;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            tsum[c][n] *= sj;  // ST_l
                            ss[c] = fmaf(tsum[c][n], tsum[c][n], ss[c]);
                        }
                    }
                    if (l >= 1) {
                        const int rr = net.r[l - 1];
                        const float* sr = sv + net.soff[l - 1];
                        float sy[4][NG];
                        float ssy[4] = {0.f, 0.f, 0.f, 0.f};
                        wait(&ybar, yq & 1);  // y_{l-1} copied into W
                        ++yq;
#pragma unroll
                        for (int n = 0; n < NG; ++n) {
                            const int j = NG * h + n;
                            float y4[4] = {0.f, 0.f, 0.f, 0.f};
                            float sj = 0.f;
                            if (j < rr) {
                                v2::ld4(reinterpret_cast<const float*>(W) + (j * P + p) * 4, y4);
                                sj = float(sr[j]);
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                sy[c][n] = sj * y4[c];
                                ssy[c] = fmaf(sy[c][n], sy[c][n], ssy[c]);
                            }
                        }
                        *reinterpret_cast<float4*>(xch + (h * P + p) * 8) = make_float4(ss[0], ss[1], ss[2], ss[3]);
                        *reinterpret_cast<float4*>(xch + (h * P + p) * 8 + 4) = make_float4(ssy[0], ssy[1], ssy[2], ssy[3]);
                        quarter_bar(quarter);  // also: this quarter's threads have read their y_{l-1} from W
                        float nst[4] = {0.f, 0.f, 0.f, 0.f}, nsy[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int hh = 0; hh < 4; ++hh) {
                            const float4 v = *reinterpret_cast<const float4*>(xch + (hh * P + p) * 8);
                            const float4 v2 = *reinterpret_cast<const float4*>(xch + (hh * P + p) * 8 + 4);
                            nst[0] += v.x;
                            nst[1] += v.y;
                            nst[2] += v.z;
                            nst[3] += v.w;
                            nsy[0] += v2.x;
                            nsy[1] += v2.y;
                            nsy[2] += v2.z;
                            nsy[3] += v2.w;
                        }
                        rev_scales(rs, nst, nsy, l - 1, tsum, sy);
                    }
                } else if (warp == ISSUER && l >= 1) {
                    wait(&rfull, (rq - 1) & 1);  // the last A MMAs of this transition have read W
                    prefetch_y(l - 1);
                }
                TC_MARK(15);
                umma::fence_async_smem();
                umma::fence_before();
                __syncthreads();
                TC_MARK(12);
            }
            // the tile's dL/ds partials (per warp quarter, fixed order) -> acc
            for (int l = 0; l < L; ++l)
                for (int j = tid; j < net.r[l]; j += NT) {
                    const float* t = tpart + l * 4 * RP + j;
                    acc[1 + net.soff[l] + j] += ((t[0] + t[RP]) + t[2 * RP]) + t[3 * RP];
                }
            if (tid == NT - 1) {
                const float* t = tpart + kMaxL * 4 * RP;
                acc[0] += ((t[0] + t[1]) + t[2]) + t[3];
            }
            __syncthreads();
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
    if (producer)
        for (int64_t qq = q; qq < q + NBUF - 1; ++qq) wait_slot(qq);  // copies past the last chunk
    TC_FLUSH();
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tbase);
}

}  // namespace tc
}  // namespace lrnr_b200
