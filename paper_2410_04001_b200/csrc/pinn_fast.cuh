// Kernel "fast" (sm_100a, FP32): the fused residual + reverse-to-s sweep for
// networks whose every hidden width and rank is <= 32, i.e. the EIM-reduced
// FastLRNR of BASELINE configs 1-3 (emit_fast_jet, autodiff.cpp:905-922, and
// its VJPs, autodiff.cpp:491-666).
//
// Why a separate kernel: at width 32 the tile-GEMM kernel (pinn_v2.cuh) is
// shared-memory-bound (ncu: L1 73 % busy, 2.8 wavefronts per LDS, FMA pipe
// 33 %) because each factor value it loads feeds only a 4x4 register tile, and
// its CTA-wide phases pay a barrier per chunk. Here:
//   - the whole reduced network (V0, per transition U-hat, V-hat, b-hat, the
//     output row; <= 50 KB) sits in shared memory for the kernel's lifetime;
//   - a point is owned by a lane pair: the even lane carries jet slots
//     (u, u_x), the odd lane (u_t, u_xx), each as two 32-vectors in registers;
//   - every factor row is read as a warp-wide broadcast LDS.128 that feeds 8
//     FMAs per lane (2 slots x 2 neurons x ... per 4 values), both GEMMs of a
//     transition stream over neuron pairs with register accumulators, and the
//     activation jets couple the two lanes through shfl.xor;
//   - warps run their 16-point tiles independently (no CTA barrier inside a
//     tile); the pre-activations z (forward) and the unscaled rank vectors u
//     (for dL/ds) go to a per-warp stash (L2-resident at 8 warps per SM);
//   - dL/ds_l per tile: a 31-shuffle transpose reduction (lane k ends with
//     column k), added into the warp's shared row; rows are summed in fixed
//     warp order per unit, so results are bitwise reproducible.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pinn_v2.cuh"

namespace lrnr_b200 {
namespace fastk {

constexpr int R = 32;                 // padded rank and reduced width
constexpr int NW = 8;                 // warps per CTA
constexpr int NT = NW * 32;
constexpr int TP = 16;                // points per warp tile (two lanes per point)
constexpr int TRANS = 2 * R * R + R;  // floats per transition block: U[R][R] | V[R][R] | b[R]

struct NetF {
    int L;
    int np[kMaxL];          // neuron pairs of transition l: ceil(M_{l+1} / 2)
    int r[kMaxL];           // true ranks
    int soff[kMaxL + 1];
    int rtotal;
    const float* blk;       // V0[2][R] | per transition U[R][R] V[R][R] b[R] | ulast[R] b_last (zero padded)
    int blk_len;            // floats
    int64_t wstride;        // stash floats per warp
    int64_t zoff[kMaxL];    // per-warp stash offsets (floats): z of transition l ...
    int64_t uoff[kMaxL];    // ... and u_{l+1}
};

// Lane k ends with sum over the warp of v[k] (31 shuffles, fixed order).
__device__ __forceinline__ float transpose_reduce(float (&v)[R], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = up ? v[i] : v[i + o];
            const float keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// One forward transition: u_{l+1} (unscaled, yn) from y_l = s_l (.) u_l, the
// pre-activation jets z of every neuron pair to the stash. KJ / KK bound the
// rank loops of the two GEMMs (4 for the rank-2 input and rank-1 output
// layers of a FastLRNR; padded columns there are zero anyway).
// Activation jets (jet_activation, model.cpp:170-181): lane pair (even: slots
// u, u_x; odd: u_t, u_xx) trades z so the even lane evaluates neuron n and the
// odd lane neuron n+1 in full, then trades the results back.
template <int KJ>
__device__ __forceinline__ void gemm_pair(const float* __restrict__ ua, const float* __restrict__ ub,
                                          const float (&v)[2][R], float& c00, float& c01, float& c10, float& c11) {
#pragma unroll
    for (int j = 0; j < KJ; j += 4) {
        const float4 a = *reinterpret_cast<const float4*>(ua + j);
        const float4 b = *reinterpret_cast<const float4*>(ub + j);
        c00 = fmaf(a.x, v[0][j], c00);
        c01 = fmaf(a.x, v[1][j], c01);
        c10 = fmaf(b.x, v[0][j], c10);
        c11 = fmaf(b.x, v[1][j], c11);
        c00 = fmaf(a.y, v[0][j + 1], c00);
        c01 = fmaf(a.y, v[1][j + 1], c01);
        c10 = fmaf(b.y, v[0][j + 1], c10);
        c11 = fmaf(b.y, v[1][j + 1], c11);
        c00 = fmaf(a.z, v[0][j + 2], c00);
        c01 = fmaf(a.z, v[1][j + 2], c01);
        c10 = fmaf(b.z, v[0][j + 2], c10);
        c11 = fmaf(b.z, v[1][j + 2], c11);
        c00 = fmaf(a.w, v[0][j + 3], c00);
        c01 = fmaf(a.w, v[1][j + 3], c01);
        c10 = fmaf(b.w, v[0][j + 3], c10);
        c11 = fmaf(b.w, v[1][j + 3], c11);
    }
}

// acc[c][k] += va[k] * x0c + vb[k] * x1c for the lane's two slots c
template <int KK>
__device__ __forceinline__ void axpy_pair(const float* __restrict__ va, const float* __restrict__ vb, float x00,
                                          float x01, float x10, float x11, float (&acc)[2][R]) {
#pragma unroll
    for (int k = 0; k < KK; k += 4) {
        const float4 a = *reinterpret_cast<const float4*>(va + k);
        const float4 b = *reinterpret_cast<const float4*>(vb + k);
        acc[0][k] = fmaf(b.x, x10, fmaf(a.x, x00, acc[0][k]));
        acc[1][k] = fmaf(b.x, x11, fmaf(a.x, x01, acc[1][k]));
        acc[0][k + 1] = fmaf(b.y, x10, fmaf(a.y, x00, acc[0][k + 1]));
        acc[1][k + 1] = fmaf(b.y, x11, fmaf(a.y, x01, acc[1][k + 1]));
        acc[0][k + 2] = fmaf(b.z, x10, fmaf(a.z, x00, acc[0][k + 2]));
        acc[1][k + 2] = fmaf(b.z, x11, fmaf(a.z, x01, acc[1][k + 2]));
        acc[0][k + 3] = fmaf(b.w, x10, fmaf(a.w, x00, acc[0][k + 3]));
        acc[1][k + 3] = fmaf(b.w, x11, fmaf(a.w, x01, acc[1][k + 3]));
    }
}

// One forward transition: u_{l+1} (unscaled, yn) from y_l = s_l (.) u_l, the
// pre-activation jets z of every neuron pair to the stash. KJ / KK bound the
// rank loops of the two GEMMs (4 for the rank-2 input and rank-1 output
// layers of a FastLRNR; padded columns there are zero anyway).
// Activation jets (jet_activation, model.cpp:170-181): lane pair (even: slots
// u, u_x; odd: u_t, u_xx) trades z so the even lane evaluates neuron n and the
// odd lane neuron n+1 in full, then trades the results back. The next pair's
// z GEMM is issued before this pair's shuffle / sincos chain so the two overlap.
template <int ACT, bool FAST, int KJ, int KK>
__device__ __forceinline__ void fwd_transition(const float* __restrict__ Ub, const float* __restrict__ Vb,
                                               const float* __restrict__ bb, int np, float4* __restrict__ zst,
                                               int lane, int half, const float (&y)[2][R], float (&yn)[2][R]) {
#pragma unroll
    for (int k = 0; k < R; ++k) yn[0][k] = yn[1][k] = 0.f;
    float z00 = half ? 0.f : bb[0], z01 = 0.f, z10 = half ? 0.f : bb[1], z11 = 0.f;
    gemm_pair<KJ>(Ub, Ub + R, y, z00, z01, z10, z11);
    for (int q = 0; q < np; ++q) {
        const int n = 2 * q;
        zst[q * 32 + lane] = make_float4(z00, z01, z10, z11);
        // even lane: neuron n (z0, z1 own; z2, z3 from the odd lane); odd lane: neuron n+1
        const float e1 = __shfl_xor_sync(0xffffffffu, half ? z00 : z10, 1);
        const float e2 = __shfl_xor_sync(0xffffffffu, half ? z01 : z11, 1);
        const float z0 = half ? e1 : z00, z1 = half ? e2 : z01, z2 = half ? z10 : e1, z3 = half ? z11 : e2;
        if (q + 1 < np) {
            z00 = half ? 0.f : bb[n + 2];
            z01 = 0.f;
            z10 = half ? 0.f : bb[n + 3];
            z11 = 0.f;
            gemm_pair<KJ>(Ub + (n + 2) * R, Ub + (n + 3) * R, y, z00, z01, z10, z11);
        }
        float sg, d1, d2, d3;
        v2::act3<ACT, FAST>(z0, sg, d1, d2, d3);
        const float a0 = sg, a1 = d1 * z1, a2 = d1 * z2, a3 = fmaf(d2 * z1, z1, d1 * z3);
        const float e3 = __shfl_xor_sync(0xffffffffu, half ? a0 : a2, 1);
        const float e4 = __shfl_xor_sync(0xffffffffu, half ? a1 : a3, 1);
        axpy_pair<KK>(Vb + n * R, Vb + (n + 1) * R, half ? e3 : a0, half ? e4 : a1, half ? a2 : e3, half ? a3 : e4, yn);
    }
}

// One reverse transition: dL/dy_l (gp) from g = dL/du_{l+1} (already scaled by
// s_{l+1}). Activation-jet VJP (autodiff.cpp:644-666) split like the forward:
// each lane of the pair does one neuron's four slots.
template <int ACT, bool FAST, int KJ, int KK>
__device__ __forceinline__ void bwd_transition(const float* __restrict__ Ub, const float* __restrict__ Vb, int np,
                                               const float4* __restrict__ zst, int lane, int half,
                                               const float (&g)[2][R], float (&gp)[2][R]) {
#pragma unroll
    for (int j = 0; j < R; ++j) gp[0][j] = gp[1][j] = 0.f;
    float g00 = 0.f, g01 = 0.f, g10 = 0.f, g11 = 0.f;  // dL/da [neuron][slot]
    gemm_pair<KK>(Vb, Vb + R, g, g00, g01, g10, g11);
    float4 zz = zst[lane];
    for (int q = 0; q < np; ++q) {
        const int n = 2 * q;
        // gather neuron m = n + half's four slots of z and dL/da on each lane
        const float e1 = __shfl_xor_sync(0xffffffffu, half ? zz.x : zz.z, 1);
        const float e2 = __shfl_xor_sync(0xffffffffu, half ? zz.y : g10, 1);
        const float e3 = __shfl_xor_sync(0xffffffffu, half ? g00 : g11, 1);
        const float e4 = __shfl_xor_sync(0xffffffffu, half ? g01 : zz.w, 1);
        const float z0 = half ? e1 : zz.x, z1 = half ? e4 : zz.y, z2 = half ? zz.z : e1, z3 = half ? zz.w : e2;
        const float c0 = half ? e2 : g00, c1 = half ? e3 : g01, c2 = half ? g10 : e3, c3 = half ? g11 : e4;
        if (q + 1 < np) {  // the next pair's dL/da and z, overlapping this pair's VJP chain
            zz = zst[(q + 1) * 32 + lane];
            g00 = g01 = g10 = g11 = 0.f;
            gemm_pair<KK>(Vb + (n + 2) * R, Vb + (n + 3) * R, g, g00, g01, g10, g11);
        }
        float sg, s1, s2, s3;
        v2::act3<ACT, FAST>(z0, sg, s1, s2, s3);
        const float h0 = c0 * s1 + s2 * (c1 * z1 + c2 * z2) + c3 * (s3 * z1 * z1 + s2 * z3);
        const float h1 = c1 * s1 + 2.f * c3 * s2 * z1;
        const float h2 = c2 * s1, h3 = c3 * s1;
        const float e5 = __shfl_xor_sync(0xffffffffu, half ? h0 : h2, 1);
        const float e6 = __shfl_xor_sync(0xffffffffu, half ? h1 : h3, 1);
        axpy_pair<KJ>(Ub + n * R, Ub + (n + 1) * R, half ? e5 : h0, half ? e6 : h1, half ? h2 : e5, half ? h3 : e6, gp);
    }
}

template <int ACT, bool FAST>
__global__ void __launch_bounds__(NT, 1)
pinn_fast_kernel(const NetF net, const RunGeom g, const double* __restrict__ pts, const double* __restrict__ svec,
                 const double* __restrict__ mus, const float w, float* __restrict__ stash, float* __restrict__ part,
                 unsigned long long* __restrict__ bad, const TermSpec* __restrict__ spec, const int objective) {
    extern __shared__ __align__(16) float fsm[];
    const int RW = ((1 + net.rtotal) + 31) & ~31;
    float* Bk = fsm;
    float* S = fsm + ((net.blk_len + 3) & ~3);
    float* rows = S + RW;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int half = lane & 1;  // 0: slots (u, u_x); 1: slots (u_t, u_xx)
    const int pl = lane >> 1;
    const int R1 = 1 + net.rtotal;
    const int L = net.L;
    for (int i = tid; i < net.blk_len; i += NT) Bk[i] = net.blk[i];
    for (int i = tid; i < NW * RW; i += NT) rows[i] = 0.f;
    float* myrow = rows + warp * RW;
    float* wst = stash + (static_cast<int64_t>(blockIdx.x) * NW + warp) * net.wstride;
    const float* V0 = Bk;
    const float* UL = Bk + 2 * R + (L - 1) * TRANS;

    for (int64_t unit = blockIdx.x; unit < g.n_units; unit += gridDim.x) {
        const int64_t inst = unit / g.units_per_inst;
        const int seg = static_cast<int>(unit % g.units_per_inst);
        const int t_lo = seg * g.tiles_per_unit;
        const int t_hi = min(g.tiles_per_inst, t_lo + g.tiles_per_unit);
        __syncthreads();
        for (int k = tid; k < net.rtotal; k += NT) S[k] = static_cast<float>(svec[inst * net.rtotal + k]);
        const float mu0 = static_cast<float>(mus[3 * inst]), mu1 = static_cast<float>(mus[3 * inst + 1]),
                    mu2 = static_cast<float>(mus[3 * inst + 2]);
        __syncthreads();
        float loss = 0.f;

        for (int tile = t_lo + warp; tile < t_hi; tile += NW) {
            const int64_t pi = static_cast<int64_t>(tile) * TP + pl;
            const bool valid = pi < g.n_per_inst;
            const int64_t gp = inst * g.n_per_inst + pi;
            const float x = valid ? static_cast<float>(pts[2 * gp]) : 0.f;
            const float t = valid ? static_cast<float>(pts[2 * gp + 1]) : 0.f;
            float y[2][R], yn[2][R];
            // ---- input layer: y_0 = s_0 (.) V_0^T (x, t) jets ----
            {
                const int r0 = net.r[0];
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const float v0 = V0[j], v1 = V0[R + j];
                    const float sj = j < r0 ? S[j] : 0.f;
                    y[0][j] = sj * (half ? v1 : v0 * x + v1 * t);
                    y[1][j] = half ? 0.f : sj * v0;
                }
            }
            // ---- forward transitions ----
            const bool in4 = net.r[0] <= 4, out4 = net.r[L - 1] <= 4;
            for (int l = 0; l + 1 < L; ++l) {
                const float* Ub = Bk + 2 * R + l * TRANS;
                const float* Vb = Ub + R * R;
                const float* bb = Vb + R * R;
                float4* zst = reinterpret_cast<float4*>(wst + net.zoff[l]);
                const bool kj4 = l == 0 && in4, kk4 = l == L - 2 && out4;
                if (kj4 && kk4) fwd_transition<ACT, FAST, 4, 4>(Ub, Vb, bb, net.np[l], zst, lane, half, y, yn);
                else if (kj4) fwd_transition<ACT, FAST, 4, R>(Ub, Vb, bb, net.np[l], zst, lane, half, y, yn);
                else if (kk4) fwd_transition<ACT, FAST, R, 4>(Ub, Vb, bb, net.np[l], zst, lane, half, y, yn);
                else fwd_transition<ACT, FAST, R, R>(Ub, Vb, bb, net.np[l], zst, lane, half, y, yn);
                // u_{l+1} -> stash; y_{l+1} = s_{l+1} (.) u_{l+1}
                float4* ust = reinterpret_cast<float4*>(wst + net.uoff[l]);
                const int rn = net.r[l + 1], so = net.soff[l + 1];
#pragma unroll
                for (int k = 0; k < R; k += 4) {
                    ust[(k / 2) * 32 + lane] = make_float4(yn[0][k], yn[0][k + 1], yn[0][k + 2], yn[0][k + 3]);
                    ust[(k / 2 + 1) * 32 + lane] = make_float4(yn[1][k], yn[1][k + 1], yn[1][k + 2], yn[1][k + 3]);
                }
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const float sk = k < rn ? S[so + k] : 0.f;
                    y[0][k] = sk * yn[0][k];
                    y[1][k] = sk * yn[1][k];
                }
            }
            // ---- output layer (M_L = 1) + residual + term seed ----
            float gy[2][R];
            {
                float o0 = half ? 0.f : UL[R], o1 = 0.f;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    o0 = fmaf(UL[k], y[0][k], o0);
                    o1 = fmaf(UL[k], y[1][k], o1);
                }
                const float p0 = __shfl_xor_sync(0xffffffffu, o0, 1), p1 = __shfl_xor_sync(0xffffffffu, o1, 1);
                const float u0 = half ? p0 : o0, u1 = half ? p1 : o1, u2 = half ? o0 : p0, u3 = half ? o1 : p1;
                const float N = u2 + mu0 * u1 - mu1 * u3 - mu2 * u0 * (1.f - u0);
                int kind = objective;
                float tw = w, sw = w, tgt = 0.f;
                if (spec != nullptr && valid) {
                    const TermSpec sp = spec[gp];
                    kind = sp.kind;
                    tgt = static_cast<float>(sp.target);
                    tw = static_cast<float>(sp.w_term);
                    sw = static_cast<float>(sp.w_seed);
                }
                const float dv = u0 - tgt;
                float term = kind == 0 ? tw * (N * N)
                                       : (kind == 1 ? tw * fabsf(N) : (kind == 2 ? tw * (dv * dv) : tw * fabsf(dv)));
                term = valid ? term : 0.f;
                if (!half) {
                    loss += term;
                    if (valid && !isfinite(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
                }
                float g0, g1;
                if (kind <= 1) {
                    const float gN = valid ? (kind == 0 ? 2.f * N * sw : sgn0(N) * sw) : 0.f;
                    g0 = half ? gN : gN * (-mu2 * (1.f - 2.f * u0));
                    g1 = half ? -gN * mu1 : gN * mu0;
                } else {
                    g0 = (valid && !half) ? (kind == 2 ? 2.f * dv * sw : sgn0(dv) * sw) : 0.f;
                    g1 = 0.f;
                }
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    gy[0][k] = UL[k] * g0;
                    gy[1][k] = UL[k] * g1;
                }
            }
            // ---- reverse transitions ----
            for (int l = L - 2; l >= 0; --l) {
                // dL/ds_{l+1}[k] = sum_slots g_y[k] u[k] (autodiff.cpp:506-513)
                {
                    const float4* ust = reinterpret_cast<const float4*>(wst + net.uoff[l]);
                    float d[R];
#pragma unroll
                    for (int k = 0; k < R; k += 4) {
                        const float4 a = ust[(k / 2) * 32 + lane];
                        const float4 b = ust[(k / 2 + 1) * 32 + lane];
                        d[k] = fmaf(gy[1][k], b.x, gy[0][k] * a.x);
                        d[k + 1] = fmaf(gy[1][k + 1], b.y, gy[0][k + 1] * a.y);
                        d[k + 2] = fmaf(gy[1][k + 2], b.z, gy[0][k + 2] * a.z);
                        d[k + 3] = fmaf(gy[1][k + 3], b.w, gy[0][k + 3] * a.w);
                    }
                    const float ds = transpose_reduce(d, lane);
                    if (lane < net.r[l + 1]) myrow[1 + net.soff[l + 1] + lane] += ds;
                }
                const int rn = net.r[l + 1], so = net.soff[l + 1];
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const float sk = k < rn ? S[so + k] : 0.f;
                    gy[0][k] *= sk;
                    gy[1][k] *= sk;
                }
                const float* Ub = Bk + 2 * R + l * TRANS;
                const float* Vb = Ub + R * R;
                const float4* zst = reinterpret_cast<const float4*>(wst + net.zoff[l]);
                const bool kj4 = l == 0 && in4, kk4 = l == L - 2 && out4;
                if (kj4 && kk4) bwd_transition<ACT, FAST, 4, 4>(Ub, Vb, net.np[l], zst, lane, half, gy, yn);
                else if (kj4) bwd_transition<ACT, FAST, 4, R>(Ub, Vb, net.np[l], zst, lane, half, gy, yn);
                else if (kk4) bwd_transition<ACT, FAST, R, 4>(Ub, Vb, net.np[l], zst, lane, half, gy, yn);
                else bwd_transition<ACT, FAST, R, R>(Ub, Vb, net.np[l], zst, lane, half, gy, yn);
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    gy[0][j] = yn[0][j];
                    gy[1][j] = yn[1][j];
                }
            }
            // dL/ds_0[j] = sum_slots g_y0[j] u0[j], u0 = V_0^T (x, t) jets
            {
                float d[R];
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const float v0 = V0[j], v1 = V0[R + j];
                    d[j] = half ? gy[0][j] * v1 : fmaf(gy[1][j], v0, gy[0][j] * (v0 * x + v1 * t));
                }
                const float ds = transpose_reduce(d, lane);
                if (lane < net.r[0]) myrow[1 + lane] += ds;
            }
        }
        // the warp's loss, then the unit's row in fixed warp order
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, o);
        if (lane == 0) myrow[0] += loss;
        __syncthreads();
        for (int k = tid; k < R1; k += NT) {
            float a = 0.f;
            for (int ww = 0; ww < NW; ++ww) a += rows[ww * RW + k];
            part[unit * R1 + k] = a;
        }
        __syncthreads();
        for (int i = tid; i < NW * RW; i += NT) rows[i] = 0.f;
    }
}

}  // namespace fastk
}  // namespace lrnr_b200
