// Kernel v3 ("tile"): tile-GEMM formulation of the fused LRNR / FastLRNR
// residual + reverse-to-s sweep (sm_100a).
//
// A CTA of NT = 8P threads owns a tile of P collocation points (P = 64 for
// FP32, 32 for FP64).  Rows of every GEMM are (point, jet slot) pairs with the
// 4 slots (u, u_x, u_t, u_xx) contiguous.  A transition through the M_{l+1}
// hidden neurons of layer l is swept in chunks of KC neurons; per chunk:
//   phase 1 (rows x KC tile, K = rank):
//     forward   A  = SY_l U_l^T (+ b)               (jet_affine_factored, model.cpp:85-122)
//               Z  = sigma-jet(A)  -> smem          (jet_activation,      model.cpp:170-181)
//     backward  A  = SY_l U_l^T (+ b)   [recompute]
//               DZ = ST_{l+1} V_{l+1}^T             (autodiff.cpp:540-552)
//               G  = sigma-jet VJP(A, DZ) -> smem   (autodiff.cpp:644-666)
//   phase 2 (rows x rank tile, K = KC):
//     forward   Y_{l+1} += Z V_{l+1}[chunk]
//     backward  T_l     += G U_l[chunk]             (autodiff.cpp:491-500)
// The M-wide activations exist only per chunk in shared memory.  The rank-side
// vectors y_l (4 r_l per point per layer) go to a per-CTA scratch (L2
// resident) for the reverse sweep; dL/ds_l[j] = sum_slots t_l[j] y_l[j]
// (autodiff.cpp:506-513) is reduced per tile in fixed order.
//
// Ranks are zero-padded to one of two compile-time classes, 4 or RPMAX, so
// every inner loop is fully unrolled with immediate smem offsets and no
// guards.  Register tiles: phase 1 = PT1 points x 4 slots x 4 neurons (one
// LDS.128 of U^T feeds 16*PT1 FMAs, one of SY feeds 16), phase 2 = 1 point x 4
// slots x 4 ranks per j-group.  Factor chunks are pre-laid-out on the host
// (lrnr_gpu.cu build_v2) into contiguous blocks and staged with cp.async.bulk
// (TMA bulk copy) into a double buffer; completion is tracked by mbarrier
// transaction counts and the next chunk is in flight while the current one is
// consumed.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pinn_kernels.cuh"

namespace lrnr_b200 {
namespace v2 {

constexpr int JG = 8;  // phase-2 j-groups per point row (NT / P)

template <typename T>
struct NetV2 {
    int L;
    int M[kMaxL + 1];      // widths
    int r[kMaxL];          // true ranks
    int rp[kMaxL];         // ranks padded to the class (4 or RPMAX)
    int nc[kMaxL];         // chunks of transition l
    int soff[kMaxL + 1];   // s / dL/ds offsets
    int yoff[kMaxL];       // y_l offsets in the per-CTA scratch (elements), layout [p][j][4]
    int ystride;           // scratch elements per CTA
    int rtotal;
    const T* blocks;       // chunk blocks (see lrnr_gpu.cu build_v2)
    const int64_t* sched_off;  // per schedule entry: element offset of the block
    const int* sched_bytes;    // per schedule entry: bytes
    int sched_len;         // entries per tile (forward chunks then backward chunks)
    const T* V0;           // 2 x r[0]
    const T* ulast;        // r[L-1] values then b_{L-1}[0]
    // META: flat ParamPacker offsets of U_l, V_l, b_l (autodiff.cpp:926-934)
    int64_t oU[kMaxL], oV[kMaxL], ob[kMaxL];
    int64_t wg_stride;     // per-CTA partial-gradient stride (elements)
    // pre-activation jets A stored by the forward sweep, reloaded by the reverse
    // sweep (no recompute): per CTA, transition l, chunk c at aoff[l] + c*P*KC*4
    int64_t aoff[kMaxL];
    int64_t astride;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ void ld4(const T* p, T (&v)[4]) {
    if constexpr (sizeof(T) == 4) {
        const float4 q = *reinterpret_cast<const float4*>(p);
        v[0] = q.x;
        v[1] = q.y;
        v[2] = q.z;
        v[3] = q.w;
    } else {
        const double2 a = *reinterpret_cast<const double2*>(p);
        const double2 b = *reinterpret_cast<const double2*>(p + 2);
        v[0] = a.x;
        v[1] = a.y;
        v[2] = b.x;
        v[3] = b.y;
    }
}
template <typename T>
__device__ __forceinline__ void st4(T* p, T a, T b, T c, T d) {
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
    } else {
        *reinterpret_cast<double2*>(p) = make_double2(a, b);
        *reinterpret_cast<double2*>(p + 2) = make_double2(c, d);
    }
}

// sin / cos with a 2-term Cody-Waite reduction to [-pi, pi] and the SFU
// approximations (|abs err| ~ 1e-6 on the reduced argument); FP32 only.
__device__ __forceinline__ void fast_sincos(float a, float& s, float& c) {
    const float k = rintf(a * 0.15915494309189535f);
    float x = fmaf(-k, 6.28318548202514648f, a);
    x = fmaf(-k, -1.7484556e-07f, x);
    s = __sinf(x);
    c = __cosf(x);
}

// FP32 sin/cos, branch-free: k = rint(a * 2/pi), 3-term Cody-Waite reduction to
// |r| <= pi/4, minimax polynomials (Cephes single-precision coefficients),
// quadrant select.  Max abs error 9.2e-8 (~1.5 ulp near 1) for |a| <= 1e3,
// measured against libm double; no local-memory slow path (unlike sincosf).
__device__ __forceinline__ void poly_sincos(float a, float& s, float& c) {
    const float k = rintf(a * 0.636619772367581343f);
    float r = fmaf(-k, 1.5703125f, a);
    r = fmaf(-k, 4.837512969970703125e-4f, r);
    r = fmaf(-k, 7.54978995489188216e-8f, r);
    const float r2 = r * r;
    float ps = fmaf(r2, -1.9515295891e-4f, 8.3321608736e-3f);
    ps = fmaf(r2, ps, -1.6666654611e-1f);
    ps = fmaf(r2 * r, ps, r);
    float pc = fmaf(r2, 2.443315711809948e-5f, -1.388731625493765e-3f);
    pc = fmaf(r2, pc, 4.166664568298827e-2f);
    pc = fmaf(r2 * r2, pc, fmaf(-0.5f, r2, 1.0f));
    const int q = static_cast<int>(k) & 3;
    const float sv = (q & 1) ? pc : ps, cv = (q & 1) ? ps : pc;
    s = (q & 2) ? -sv : sv;
    c = ((q + 1) & 2) ? -cv : cv;
}

// tanh jet from its value (the same expressions as act3<0>)
template <typename T>
__device__ __forceinline__ void act3_from_value(T s, T& sg, T& d1, T& d2, T& d3) {
    const T e = T(1) - s * s;
    sg = s;
    d1 = e;
    d2 = T(-2) * s * e;
    d3 = T(-2) * e * e + T(4) * s * s * e;
}

template <int ACT, bool FAST, typename T>
__device__ __forceinline__ void act3(T a, T& sg, T& d1, T& d2, T& d3) {
    if constexpr (ACT == 0) {
        T s;
        if constexpr (sizeof(T) == 8) s = tanh(a);
        else s = tanhf(a);
        const T e = T(1) - s * s;
        sg = s;
        d1 = e;
        d2 = T(-2) * s * e;
        d3 = T(-2) * e * e + T(4) * s * s * e;
    } else {
        T sn, cs;
        if constexpr (sizeof(T) == 8) {
            sincos(a, &sn, &cs);
        } else if constexpr (FAST) {
            fast_sincos(a, sn, cs);
        } else {
            poly_sincos(a, sn, cs);
        }
        sg = sn;
        d1 = cs;
        d2 = -sn;
        d3 = -cs;
    }
}

// Shared-memory carve-up (elements of T).
template <typename T, int P, int KC, int RPMAX, bool META = false>
struct Smem {
    static constexpr int ZS = KC * 4 + 4;      // Z/G point stride (padded: conflict-free phase-2 reads)
    static constexpr int SS = RPMAX * 4 + 4;   // SY/ST point stride
    static constexpr int BUF = 2 * RPMAX * KC + KC + 16;  // max block (fwd: U^T, b, V; bwd: V^T, U)
    static constexpr int OFF_Z = 0;
    static constexpr int OFF_SY = OFF_Z + P * ZS;
    static constexpr int OFF_ST = OFF_SY + P * SS;
    static constexpr int OFF_B0 = ((OFF_ST + P * SS + 31) / 32) * 32;
    static constexpr int OFF_B1 = OFF_B0 + ((BUF + 31) / 32) * 32;
    static constexpr int OFF_RED = OFF_B1 + ((BUF + 31) / 32) * 32;
    static constexpr int OFF_ACC = OFF_RED + P * RPMAX + 2 * P;
    static constexpr int OFF_ZZ = ((OFF_ACC + 1024 + 31) / 32) * 32;  // META: Z chunk (needs r_total < 1024)
    static constexpr int OFF_XT = OFF_ZZ + (META ? P * ZS : 0);        // META: (x, t) of the tile
    static constexpr int END = OFF_XT + (META ? 2 * P : 0);
};

template <typename T, int P, int PT1, int NG, int RPMAX, int ACT, bool FAST, bool META = false>
struct Tile {
    static constexpr int NT = JG * P;
    static constexpr int KC = 4 * NG;
    static constexpr int NJ = RPMAX / (4 * JG);
    using S = Smem<T, P, KC, RPMAX, META>;
    static_assert(NG * (P / PT1) == NT, "phase-1 mapping must cover the CTA");
    static_assert(RPMAX % (4 * JG) == 0, "RPMAX multiple of 32");

    // forward phase 1: Z = sigma-jet(SY U^T + b) for this thread's PT1 points x 4 neurons
    // KK: active neuron groups (k = ng + NG kk, kk < KK) of a narrow last chunk (warp-uniform)
    template <int RL, int KK = 4>
    static __device__ __forceinline__ void fwd_phase1(const T* __restrict__ UT, const T* __restrict__ bb,
                                                      const T* __restrict__ SY, T* __restrict__ Zg, int ng,
                                                      int pg, T* __restrict__ Ast) {
        T a1[PT1][4][4];
#pragma unroll
        for (int i = 0; i < PT1; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int kk = 0; kk < KK; ++kk) a1[i][c][kk] = T(0);
        const T* syb = SY + pg * PT1 * S::SS;
#pragma unroll
        for (int j = 0; j < RL; ++j) {
            T ut[4];
            ld4(UT + j * KC + ng * 4, ut);
#pragma unroll
            for (int i = 0; i < PT1; ++i) {
                T sy[4];
                ld4(syb + i * S::SS + j * 4, sy);
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int kk = 0; kk < KK; ++kk) a1[i][c][kk] = fma(sy[c], ut[kk], a1[i][c][kk]);
            }
        }
        T bias[4];
        ld4(bb + ng * 4, bias);
#pragma unroll
        for (int i = 0; i < PT1; ++i)
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) {
                const T av = a1[i][0][kk] + bias[kk], ax = a1[i][1][kk];
                const T at = a1[i][2][kk], aw = a1[i][3][kk];
                T sg, d1, d2, d3;
                act3<ACT, FAST>(av, sg, d1, d2, d3);
                // tanh: the reverse sweep needs only sigma (its derivatives are polynomials in it, the
                // reference's d*_from_value, autodiff.cpp:655-657), so sigma is stashed instead of a
                st4(Ast + ((pg * PT1 + i) * KC + ng + NG * kk) * 4, ACT == 0 ? sg : av, ax, at, aw);
                st4(Zg + (pg * PT1 + i) * S::ZS + (ng + NG * kk) * 4, sg, d1 * ax, d1 * at, d2 * ax * ax + d1 * aw);
            }
    }

    // backward phase 1: G = VJP(A, ST V^T), A reloaded from the forward sweep's store
    template <int RN, int KK = 4>
    static __device__ __forceinline__ void bwd_phase1(const T* __restrict__ Ast, const T* __restrict__ VT,
                                                      const T* __restrict__ ST, T* __restrict__ Zg, int ng,
                                                      int pg, T* __restrict__ Zz = nullptr) {
        T a1[PT1][4][4], dz[PT1][4][4];
        // issue the A loads first (L2 / HBM latency hidden behind the DZ GEMM)
#pragma unroll
        for (int i = 0; i < PT1; ++i)
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) {
                T a4[4];
                ld4(Ast + ((pg * PT1 + i) * KC + ng + NG * kk) * 4, a4);
#pragma unroll
                for (int c = 0; c < 4; ++c) a1[i][c][kk] = a4[c];
            }
#pragma unroll
        for (int i = 0; i < PT1; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int kk = 0; kk < KK; ++kk) dz[i][c][kk] = T(0);
        const T* stb = ST + pg * PT1 * S::SS;
#pragma unroll
        for (int j = 0; j < RN; ++j) {
            T vt[4];
            ld4(VT + j * KC + ng * 4, vt);
#pragma unroll
            for (int i = 0; i < PT1; ++i) {
                T st[4];
                ld4(stb + i * S::SS + j * 4, st);
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int kk = 0; kk < KK; ++kk) dz[i][c][kk] = fma(st[c], vt[kk], dz[i][c][kk]);
            }
        }
#pragma unroll
        for (int i = 0; i < PT1; ++i)
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) {
                const T av = a1[i][0][kk], ax = a1[i][1][kk];
                const T at = a1[i][2][kk], aw = a1[i][3][kk];
                const T g0 = dz[i][0][kk], g1 = dz[i][1][kk], g2 = dz[i][2][kk], g3 = dz[i][3][kk];
                T sg, d1, d2, d3;
                if constexpr (ACT == 0) act3_from_value(av, sg, d1, d2, d3);  // the stash holds sigma
                else act3<ACT, FAST>(av, sg, d1, d2, d3);
                const T gav = g0 * d1 + g1 * d2 * ax + g2 * d2 * at + g3 * (d3 * ax * ax + d2 * aw);
                const T gax = g1 * d1 + g3 * T(2) * d2 * ax;
                st4(Zg + (pg * PT1 + i) * S::ZS + (ng + NG * kk) * 4, gav, gax, g2 * d1, g3 * d1);
                if constexpr (META)
                    st4(Zz + (pg * PT1 + i) * S::ZS + (ng + NG * kk) * 4, sg, d1 * ax, d1 * at, d2 * ax * ax + d1 * aw);
            }
    }

    // META phase 3 (AffineFactoredJet VJP w.r.t. the factors, autodiff.cpp:501-505,524-534,553-560):
    //   dU_l[k][j]      += sum_{p,c} G[p][k][c] SY[p][j][c]
    //   dV_{l+1}[k][j'] += sum_{p,c} Z[p][k][c] ST[p][j'][c]
    //   db_l[k]         += sum_p G[p][k][0]
    // accumulated over the tile in registers, then added into this CTA's
    // partial-gradient rows (fixed order -> deterministic).
    template <int RL, int RN>
    static __device__ __forceinline__ void phase3(const T* __restrict__ Gs, const T* __restrict__ Zs,
                                                  const T* __restrict__ SY, const T* __restrict__ ST,
                                                  T* __restrict__ wg, int64_t oU, int64_t oV, int64_t ob, int k0,
                                                  int M, int rl_true, int rn_true, int tid) {
        // thread (kq, jq) owns neurons kq + KQ a and ranks jq + JQ b (a, b < 4): the 8 kq
        // lanes of a warp read 8 consecutive 16-B jets (all 32 banks, no conflicts)
        constexpr int KQ = KC / 4;
        constexpr int NU = KQ * (RL / 4), NV = KQ * (RN / 4);
        for (int idx = tid; idx < NU + NV; idx += NT) {
            const bool isU = idx < NU;
            const int e = isU ? idx : idx - NU;
            const int kq = e % KQ, jq = e / KQ;
            const int JQ = (isU ? RL : RN) / 4;
            const T* A = isU ? Gs : Zs;
            const T* B = isU ? SY : ST;
            T acc[4][4], db[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                db[a] = T(0);
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
            }
#pragma unroll 4
            for (int p = 0; p < P; ++p) {
                T g[4][4], y[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    ld4(A + p * S::ZS + (kq + KQ * a) * 4, g[a]);
                    ld4(B + p * S::SS + (jq + JQ * a) * 4, y[a]);
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    db[a] += g[a][0];
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[a][b] = fma(g[a][c], y[b][c], acc[a][b]);
                }
            }
            const int rtrue = isU ? rl_true : rn_true;
            const int64_t base = isU ? oU : oV;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int k = k0 + kq + KQ * a;
                if (k >= M) continue;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int j = jq + JQ * b;
                    if (j < rtrue) wg[base + static_cast<int64_t>(k) * rtrue + j] += acc[a][b];
                }
                if (isU && jq == 0) wg[ob + k] += db[a];
            }
        }
    }

    // phase 2: acc += Zg[p2] * Mat (Mat = KC x RN, row stride RN)
    // kc: neurons of this chunk (< KC in a narrow last chunk; padded rows are zero)
    template <int RN>
    static __device__ __forceinline__ void phase2(const T* __restrict__ Zg, const T* __restrict__ Mat,
                                                  T (&acc)[NJ][4][4], int p2, int jg, int kc) {
        constexpr int NJE = (RN + 4 * JG - 1) / (4 * JG);
        if (RN < 4 * JG && jg * 4 >= RN) return;
        const T* zb = Zg + p2 * S::ZS;
#pragma unroll 16
        for (int k = 0; k < kc; ++k) {
            T z[4];
            ld4(zb + k * 4, z);
#pragma unroll
            for (int a = 0; a < NJE; ++a) {
                T v[4];
                ld4(Mat + k * RN + (jg + JG * a) * 4, v);
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) acc[a][c][jj] = fma(z[c], v[jj], acc[a][c][jj]);
            }
        }
    }
};

// CTAs per SM: two 256-thread CTAs for FP32 P = 32 tiles (independent
// barriers overlap), one otherwise.
template <typename T, int P>
constexpr int tile_min_blocks() {
    return (sizeof(T) == 4 && P == 32) ? 2 : 1;
}

template <typename T, int P, int PT1, int NG, int RPMAX, int ACT, bool FAST, bool META = false>
__global__ void __launch_bounds__(JG * P, (META ? 1 : tile_min_blocks<T, P>()))
pinn_tile_kernel(const NetV2<T> net, const RunGeom g, const double* __restrict__ pts,
                 const double* __restrict__ svec, const double* __restrict__ mus, const T w,
                 T* __restrict__ scratch, T* __restrict__ part, unsigned long long* __restrict__ bad,
                 T* __restrict__ ascratch, T* __restrict__ wgrad = nullptr,
                 const TermSpec* __restrict__ spec = nullptr, const int objective = 0) {
    using K = Tile<T, P, PT1, NG, RPMAX, ACT, FAST, META>;
    using S = typename K::S;
    constexpr int NT = K::NT;
    constexpr int KC = K::KC;
    constexpr int NJ = K::NJ;
    constexpr bool R16 = sizeof(T) == 8 && !META;  // the host pads ranks 5..16 to 16 for these (build_v2)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    T* Zg = sm + S::OFF_Z;
    T* SY = sm + S::OFF_SY;
    T* ST = sm + S::OFF_ST;
    T* const buf0 = sm + S::OFF_B0;
    constexpr int BUFSTRIDE = S::OFF_B1 - S::OFF_B0;
    T* red = sm + S::OFF_RED;
    T* acc = sm + S::OFF_ACC;
    T* Zz = sm + S::OFF_ZZ;
    T* xts = sm + S::OFF_XT;
    __shared__ __align__(8) uint64_t mbar[2];
    T* wg = META ? wgrad + static_cast<int64_t>(blockIdx.x) * net.wg_stride : nullptr;

    const int tid = threadIdx.x;
    const int ng = tid % NG;
    const int pg = tid / NG;
    const int jg = tid % JG;
    const int p2 = tid / JG;
    const int R1 = 1 + net.rtotal;
    const int L = net.L;
    T* scr = scratch + static_cast<int64_t>(blockIdx.x) * net.ystride;
    T* ascr = ascratch + static_cast<int64_t>(blockIdx.x) * net.astride;

    for (int k = tid; k < R1; k += NT) acc[k] = T(0);
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    int64_t total_tiles = 0;
    for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
        const int seg = static_cast<int>(u % g.units_per_inst);
        const int t_lo = seg * g.tiles_per_unit;
        total_tiles += min(g.tiles_per_inst, t_lo + g.tiles_per_unit) - t_lo;
    }
    const int64_t total_chunks = total_tiles * net.sched_len;
    int64_t q = 0;
    auto issue = [&](int64_t qq) {
        if (qq < total_chunks && tid == 0) {
            const int e = static_cast<int>(qq % net.sched_len);
            const int b = static_cast<int>(qq & 1);
            fence_proxy_async();
            mbar_expect_tx(&mbar[b], static_cast<uint32_t>(net.sched_bytes[e]));
            bulk_g2s(buf0 + b * BUFSTRIDE, net.blocks + net.sched_off[e], static_cast<uint32_t>(net.sched_bytes[e]),
                     &mbar[b]);
        }
    };
    // wait for chunk q, prefetch q+1, return the chunk buffer
    auto acquire = [&]() -> const T* {
        const int b = static_cast<int>(q & 1);
        issue(q + 1);
        mbar_wait(&mbar[b], static_cast<uint32_t>((q >> 1) & 1));
        ++q;
        return buf0 + b * BUFSTRIDE;
    };
    issue(0);

    for (int64_t unit = blockIdx.x; unit < g.n_units; unit += gridDim.x) {
        const int64_t inst = unit / g.units_per_inst;
        const int seg = static_cast<int>(unit % g.units_per_inst);
        const int t_lo = seg * g.tiles_per_unit;
        const int t_hi = min(g.tiles_per_inst, t_lo + g.tiles_per_unit);
        const double* sv = svec + inst * net.rtotal;
        const T mu0 = T(mus[3 * inst]), mu1 = T(mus[3 * inst + 1]), mu2 = T(mus[3 * inst + 2]);

        for (int tile = t_lo; tile < t_hi; ++tile) {
            const int64_t pbase = static_cast<int64_t>(tile) * P;
            // ---------------- input layer: y_0 = V_0^T z_0 ----------------
            {
                const int64_t pi = pbase + p2;
                const bool valid = pi < g.n_per_inst;
                const int64_t gp = inst * g.n_per_inst + pi;
                const T x = valid ? T(pts[2 * gp]) : T(0);
                const T t = valid ? T(pts[2 * gp + 1]) : T(0);
                if (META && jg == 0) {
                    xts[2 * p2] = x;
                    xts[2 * p2 + 1] = t;
                }
                const int r0 = net.r[0], rp0 = net.rp[0];
                for (int jj = jg; jj < rp0; jj += JG) {
                    T y4[4] = {T(0), T(0), T(0), T(0)};
                    T sj = T(0);
                    if (jj < r0) {
                        const T v0 = net.V0[jj], v1 = net.V0[r0 + jj];
                        y4[0] = v0 * x + v1 * t;
                        y4[1] = v0;
                        y4[2] = v1;
                        sj = T(sv[jj]);
                    }
                    st4(scr + net.yoff[0] + (p2 * rp0 + jj) * 4, y4[0], y4[1], y4[2], y4[3]);
                    st4(SY + p2 * S::SS + jj * 4, sj * y4[0], sj * y4[1], sj * y4[2], sj * y4[3]);
                }
            }
            __syncthreads();

            // ---------------- forward transitions ----------------
            for (int l = 0; l + 1 < L; ++l) {
                const int rl = net.rp[l], rn = net.rp[l + 1];
                T yacc[NJ][4][4];
#pragma unroll
                for (int a = 0; a < NJ; ++a)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int b = 0; b < 4; ++b) yacc[a][c][b] = T(0);
                for (int ch = 0; ch < net.nc[l]; ++ch) {
                    const T* UT = acquire();
                    const T* bb = UT + rl * KC;
                    const T* Vm = bb + KC;
                    T* Ast = ascr + net.aoff[l] + static_cast<int64_t>(ch) * (P * KC * 4);
                    const int kc = META ? KC : min(KC, net.M[l + 1] - ch * KC);
                    const int kk = (kc + NG - 1) / NG;
#define V2_FWD1(RLV)                                                                         \
    switch (kk) {                                                                            \
        case 1: K::template fwd_phase1<RLV, 1>(UT, bb, SY, Zg, ng, pg, Ast); break;          \
        case 2: K::template fwd_phase1<RLV, 2>(UT, bb, SY, Zg, ng, pg, Ast); break;          \
        case 3: K::template fwd_phase1<RLV, 3>(UT, bb, SY, Zg, ng, pg, Ast); break;          \
        default: K::template fwd_phase1<RLV, 4>(UT, bb, SY, Zg, ng, pg, Ast); break;         \
    }
                    // rank classes 4 / RPMAX, and 16 for FP64 (R16: c0 / c1's rank 10 pads to 16, not 32)
                    if (rl == 4) {
                        V2_FWD1(4)
                    } else if (R16 && rl == 16) {
                        if constexpr (R16) { V2_FWD1(16) }
                    } else {
                        V2_FWD1(RPMAX)
                    }
#undef V2_FWD1
                    __syncthreads();
                    if (rn == 4) K::template phase2<4>(Zg, Vm, yacc, p2, jg, kc);
                    else if (R16 && rn == 16) K::template phase2<R16 ? 16 : RPMAX>(Zg, Vm, yacc, p2, jg, kc);
                    else K::template phase2<RPMAX>(Zg, Vm, yacc, p2, jg, kc);
                    __syncthreads();
                }
                // y_{l+1} -> scratch, SY = s_{l+1} (.) y_{l+1}
                const double* sl = sv + net.soff[l + 1];
                const int rtrue = net.r[l + 1];
#pragma unroll
                for (int a = 0; a < NJ; ++a) {
                    const int j0 = (jg + JG * a) * 4;
                    if (j0 < rn) {
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const int j = j0 + jj;
                            const T sj = j < rtrue ? T(sl[j]) : T(0);
                            st4(scr + net.yoff[l + 1] + (p2 * rn + j) * 4, yacc[a][0][jj], yacc[a][1][jj],
                                yacc[a][2][jj], yacc[a][3][jj]);
                            st4(SY + p2 * S::SS + j * 4, sj * yacc[a][0][jj], sj * yacc[a][1][jj],
                                sj * yacc[a][2][jj], sj * yacc[a][3][jj]);
                        }
                    }
                }
                __syncthreads();
            }

            // ---------------- output layer (M_L = 1) + residual ----------------
            {
                const int rL = net.r[L - 1], rpL = net.rp[L - 1];
                const double* sL = sv + net.soff[L - 1];
                if (tid < P) {
                    const int p = tid;
                    const int64_t pi = pbase + p;
                    const bool valid = pi < g.n_per_inst;
                    const int64_t gp = inst * g.n_per_inst + pi;
                    T u[4] = {T(0), T(0), T(0), T(0)};
                    for (int j = 0; j < rL; ++j) {
                        T sy[4];
                        ld4(SY + p * S::SS + j * 4, sy);
                        const T uj = net.ulast[j];
#pragma unroll
                        for (int c = 0; c < 4; ++c) u[c] = fma(uj, sy[c], u[c]);
                    }
                    u[0] += net.ulast[rL];
                    const T N = u[2] + mu0 * u[1] - mu1 * u[3] - mu2 * u[0] * (T(1) - u[0]);
                    // per-point term kind (TermSpec, pinn_kernels.cuh): interior w N^2 / w |N|,
                    // value terms w (u - c)^2 / w |u - c| (boundary terms)
                    int kind = objective;
                    T tw = w, sw = w, tgt = T(0);
                    if (spec != nullptr && valid) {
                        const TermSpec sp = spec[gp];
                        kind = sp.kind;
                        tgt = T(sp.target);
                        tw = T(sp.w_term);
                        sw = T(sp.w_seed);
                    }
                    const T dv = u[0] - tgt;
                    T term = kind == 0 ? tw * (N * N) : (kind == 1 ? tw * fabs(N) : (kind == 2 ? tw * (dv * dv) : tw * fabs(dv)));
                    term = valid ? term : T(0);
                    if (valid && !isfinite(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
                    T gu[4];
                    if (kind <= 1) {
                        const T gN = valid ? (kind == 0 ? T(2) * N * sw : sgn0(N) * sw) : T(0);
                        gu[0] = gN * (-mu2 * (T(1) - T(2) * u[0]));
                        gu[1] = gN * mu0;
                        gu[2] = gN;
                        gu[3] = -gN * mu1;
                    } else {
                        gu[0] = valid ? (kind == 2 ? T(2) * dv * sw : sgn0(dv) * sw) : T(0);
                        gu[1] = gu[2] = gu[3] = T(0);
                    }
                    red[P * RPMAX + p] = term;
                    if constexpr (META) red[P * RPMAX + P + p] = gu[0];
                    for (int j = 0; j < rpL; ++j) {
                        const T uj = j < rL ? net.ulast[j] : T(0);
                        const T sj = j < rL ? T(sL[j]) : T(0);
                        T y4[4];
                        ld4(scr + net.yoff[L - 1] + (p * rpL + j) * 4, y4);
                        T cd = T(0);
#pragma unroll
                        for (int c = 0; c < 4; ++c) cd = fma(uj * gu[c], y4[c], cd);
                        if constexpr (META) {
                            // dU_{L-1}[0][j] contribution sum_c gu[c] * sy[j][c]
                            T du = T(0);
#pragma unroll
                            for (int c = 0; c < 4; ++c) du = fma(gu[c], sj * y4[c], du);
                            Zz[p * S::ZS + j] = du;
                        }
                        red[p * RPMAX + j] = cd;
                        st4(ST + p * S::SS + j * 4, sj * uj * gu[0], sj * uj * gu[1], sj * uj * gu[2],
                            sj * uj * gu[3]);
                    }
                }
                __syncthreads();
                if (tid < rL) {
                    T sacc = T(0);
                    for (int p = 0; p < P; ++p) sacc += red[p * RPMAX + tid];
                    acc[1 + net.soff[L - 1] + tid] += sacc;
                }
                if (tid == NT - 1) {
                    T sacc = T(0);
                    for (int p = 0; p < P; ++p) sacc += red[P * RPMAX + p];
                    acc[0] += sacc;
                }
                if constexpr (META) {
                    if (tid >= 32 && tid < 32 + rL) {
                        const int j = tid - 32;
                        T du = T(0);
                        for (int p = 0; p < P; ++p) du += Zz[p * S::ZS + j];
                        wg[net.oU[L - 1] + j] += du;
                    }
                    if (tid == NT - 2) {
                        T dbl = T(0);
                        for (int p = 0; p < P; ++p) dbl += red[P * RPMAX + P + p];
                        wg[net.ob[L - 1]] += dbl;
                    }
                }
                __syncthreads();
            }

            // ---------------- backward transitions ----------------
            for (int l = L - 2; l >= 0; --l) {
                const int rl = net.rp[l], rn = net.rp[l + 1];
                const int rtrue = net.r[l];
                const double* sl = sv + net.soff[l];
                // SY = s_l (.) y_l (only the factor gradients of the meta path need it)
                if (META)
                for (int j = jg; j < rl; j += JG) {
                    const T sj = j < rtrue ? T(sl[j]) : T(0);
                    T y4[4];
                    ld4(scr + net.yoff[l] + (p2 * rl + j) * 4, y4);
                    st4(SY + p2 * S::SS + j * 4, sj * y4[0], sj * y4[1], sj * y4[2], sj * y4[3]);
                }
                __syncthreads();
                T tacc[NJ][4][4];
#pragma unroll
                for (int a = 0; a < NJ; ++a)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int b = 0; b < 4; ++b) tacc[a][c][b] = T(0);
                for (int ch = 0; ch < net.nc[l]; ++ch) {
                    const T* VT = acquire();
                    const T* Um = VT + rn * KC;
                    const T* Ast = ascr + net.aoff[l] + static_cast<int64_t>(ch) * (P * KC * 4);
                    const int kc = META ? KC : min(KC, net.M[l + 1] - ch * KC);
                    const int kk = (kc + NG - 1) / NG;
#define V2_BWD1(RNV)                                                                         \
    switch (kk) {                                                                            \
        case 1: K::template bwd_phase1<RNV, 1>(Ast, VT, ST, Zg, ng, pg, Zz); break;          \
        case 2: K::template bwd_phase1<RNV, 2>(Ast, VT, ST, Zg, ng, pg, Zz); break;          \
        case 3: K::template bwd_phase1<RNV, 3>(Ast, VT, ST, Zg, ng, pg, Zz); break;          \
        default: K::template bwd_phase1<RNV, 4>(Ast, VT, ST, Zg, ng, pg, Zz); break;         \
    }
                    if (rn == 4) {
                        V2_BWD1(4)
                    } else if (R16 && rn == 16) {
                        if constexpr (R16) { V2_BWD1(16) }
                    } else {
                        V2_BWD1(RPMAX)
                    }
#undef V2_BWD1
                    __syncthreads();
                    if (rl == 4) K::template phase2<4>(Zg, Um, tacc, p2, jg, kc);
                    else if (R16 && rl == 16) K::template phase2<R16 ? 16 : RPMAX>(Zg, Um, tacc, p2, jg, kc);
                    else K::template phase2<RPMAX>(Zg, Um, tacc, p2, jg, kc);
                    if constexpr (META) {
                        const int k0 = ch * KC;
                        const int M = net.M[l + 1];
                        if (rl == 4) {
                            if (rn == 4)
                                K::template phase3<4, 4>(Zg, Zz, SY, ST, wg, net.oU[l], net.oV[l + 1], net.ob[l], k0, M,
                                                         net.r[l], net.r[l + 1], tid);
                            else
                                K::template phase3<4, RPMAX>(Zg, Zz, SY, ST, wg, net.oU[l], net.oV[l + 1], net.ob[l],
                                                             k0, M, net.r[l], net.r[l + 1], tid);
                        } else {
                            if (rn == 4)
                                K::template phase3<RPMAX, 4>(Zg, Zz, SY, ST, wg, net.oU[l], net.oV[l + 1], net.ob[l],
                                                             k0, M, net.r[l], net.r[l + 1], tid);
                            else
                                K::template phase3<RPMAX, RPMAX>(Zg, Zz, SY, ST, wg, net.oU[l], net.oV[l + 1],
                                                                 net.ob[l], k0, M, net.r[l], net.r[l + 1], tid);
                        }
                    }
                    __syncthreads();
                }
                // dL/ds_l partials and ST = s_l (.) T
#pragma unroll
                for (int a = 0; a < NJ; ++a) {
                    const int j0 = (jg + JG * a) * 4;
                    if (j0 < rl) {
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const int j = j0 + jj;
                            const T sj = j < rtrue ? T(sl[j]) : T(0);
                            T y4[4];
                            ld4(scr + net.yoff[l] + (p2 * rl + j) * 4, y4);
                            T cd = T(0);
#pragma unroll
                            for (int c = 0; c < 4; ++c) cd = fma(tacc[a][c][jj], y4[c], cd);
                            red[p2 * RPMAX + j] = cd;
                            st4(ST + p2 * S::SS + j * 4, sj * tacc[a][0][jj], sj * tacc[a][1][jj],
                                sj * tacc[a][2][jj], sj * tacc[a][3][jj]);
                        }
                    }
                }
                __syncthreads();
                if (tid < rtrue) {
                    T sacc = T(0);
                    for (int p = 0; p < P; ++p) sacc += red[p * RPMAX + tid];
                    acc[1 + net.soff[l] + tid] += sacc;
                }
                __syncthreads();
            }
            if constexpr (META) {
                // dV_0[i][j] = sum_{p,c} z0[p][c][i] st_0[p][j][c], z0 = (x,t),(1,0),(0,1),(0,0)
                const int r0 = net.r[0];
                if (tid < 2 * r0) {
                    const int i = tid / r0, j = tid % r0;
                    T dv = T(0);
                    for (int p = 0; p < P; ++p) {
                        T st[4];
                        ld4(ST + p * S::SS + j * 4, st);
                        dv += xts[2 * p + i] * st[0] + st[1 + i];
                    }
                    wg[net.oV[0] + i * r0 + j] += dv;
                }
                __syncthreads();
            }
        }
        for (int k = tid; k < R1; k += NT) {
            part[unit * R1 + k] = acc[k];
            acc[k] = T(0);
        }
        __syncthreads();
    }
}

}  // namespace v2
}  // namespace lrnr_b200
