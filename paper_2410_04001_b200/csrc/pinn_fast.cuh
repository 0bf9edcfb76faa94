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
            for (int l = 0; l + 1 < L; ++l) {
                const float* Ub = Bk + 2 * R + l * TRANS;
                const float* Vb = Ub + R * R;
                const float* bb = Vb + R * R;
                float4* zst = reinterpret_cast<float4*>(wst + net.zoff[l]);
#pragma unroll
                for (int k = 0; k < R; ++k) yn[0][k] = yn[1][k] = 0.f;
                for (int q = 0; q < net.np[l]; ++q) {
                    const int n = 2 * q;
                    const float* ua = Ub + n * R;
                    const float* ub = ua + R;
                    float z00 = half ? 0.f : bb[n], z01 = 0.f, z10 = half ? 0.f : bb[n + 1], z11 = 0.f;
#pragma unroll
                    for (int j = 0; j < R; j += 4) {
                        const float4 a = *reinterpret_cast<const float4*>(ua + j);
                        const float4 b = *reinterpret_cast<const float4*>(ub + j);
                        z00 = fmaf(a.x, y[0][j], z00);
                        z01 = fmaf(a.x, y[1][j], z01);
                        z10 = fmaf(b.x, y[0][j], z10);
                        z11 = fmaf(b.x, y[1][j], z11);
                        z00 = fmaf(a.y, y[0][j + 1], z00);
                        z01 = fmaf(a.y, y[1][j + 1], z01);
                        z10 = fmaf(b.y, y[0][j + 1], z10);
                        z11 = fmaf(b.y, y[1][j + 1], z11);
                        z00 = fmaf(a.z, y[0][j + 2], z00);
                        z01 = fmaf(a.z, y[1][j + 2], z01);
                        z10 = fmaf(b.z, y[0][j + 2], z10);
                        z11 = fmaf(b.z, y[1][j + 2], z11);
                        z00 = fmaf(a.w, y[0][j + 3], z00);
                        z01 = fmaf(a.w, y[1][j + 3], z01);
                        z10 = fmaf(b.w, y[0][j + 3], z10);
                        z11 = fmaf(b.w, y[1][j + 3], z11);
                    }
                    zst[q * 32 + lane] = make_float4(z00, z01, z10, z11);
                    // activation jets (jet_activation, model.cpp:170-181): the even lane
                    // evaluates sigma at neuron n, the odd lane at n+1
                    const float zx = __shfl_xor_sync(0xffffffffu, z10, 1);
                    float sg, d1, d2, d3;
                    v2::act3<ACT, FAST>(half ? zx : z00, sg, d1, d2, d3);
                    const float e1 = __shfl_xor_sync(0xffffffffu, half ? sg : d1, 1);
                    const float e2 = __shfl_xor_sync(0xffffffffu, half ? d1 : d2, 1);
                    const float e3 = __shfl_xor_sync(0xffffffffu, z01, 1);
                    const float e4 = __shfl_xor_sync(0xffffffffu, z11, 1);
                    float a00, a01, a10, a11;
                    if (!half) {
                        a00 = sg;
                        a01 = d1 * z01;
                        a10 = e1;
                        a11 = e2 * z11;
                    } else {  // z00 = u_t slot, z01 = u_xx slot of neuron n; e1 = sigma'(n), e2 = sigma''(n)
                        a00 = e1 * z00;
                        a01 = fmaf(e2 * e3, e3, e1 * z01);
                        a10 = d1 * z10;
                        a11 = fmaf(d2 * e4, e4, d1 * z11);
                    }
                    const float* va = Vb + n * R;
                    const float* vb = va + R;
#pragma unroll
                    for (int k = 0; k < R; k += 4) {
                        const float4 a = *reinterpret_cast<const float4*>(va + k);
                        const float4 b = *reinterpret_cast<const float4*>(vb + k);
                        yn[0][k] = fmaf(b.x, a10, fmaf(a.x, a00, yn[0][k]));
                        yn[1][k] = fmaf(b.x, a11, fmaf(a.x, a01, yn[1][k]));
                        yn[0][k + 1] = fmaf(b.y, a10, fmaf(a.y, a00, yn[0][k + 1]));
                        yn[1][k + 1] = fmaf(b.y, a11, fmaf(a.y, a01, yn[1][k + 1]));
                        yn[0][k + 2] = fmaf(b.z, a10, fmaf(a.z, a00, yn[0][k + 2]));
                        yn[1][k + 2] = fmaf(b.z, a11, fmaf(a.z, a01, yn[1][k + 2]));
                        yn[0][k + 3] = fmaf(b.w, a10, fmaf(a.w, a00, yn[0][k + 3]));
                        yn[1][k + 3] = fmaf(b.w, a11, fmaf(a.w, a01, yn[1][k + 3]));
                    }
                }
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
#pragma unroll
                for (int j = 0; j < R; ++j) yn[0][j] = yn[1][j] = 0.f;
                for (int q = 0; q < net.np[l]; ++q) {
                    const int n = 2 * q;
                    const float* va = Vb + n * R;
                    const float* vb = va + R;
                    float g00 = 0.f, g01 = 0.f, g10 = 0.f, g11 = 0.f;  // dL/da [neuron][slot]
#pragma unroll
                    for (int k = 0; k < R; k += 4) {
                        const float4 a = *reinterpret_cast<const float4*>(va + k);
                        const float4 b = *reinterpret_cast<const float4*>(vb + k);
                        g00 = fmaf(a.x, gy[0][k], g00);
                        g01 = fmaf(a.x, gy[1][k], g01);
                        g10 = fmaf(b.x, gy[0][k], g10);
                        g11 = fmaf(b.x, gy[1][k], g11);
                        g00 = fmaf(a.y, gy[0][k + 1], g00);
                        g01 = fmaf(a.y, gy[1][k + 1], g01);
                        g10 = fmaf(b.y, gy[0][k + 1], g10);
                        g11 = fmaf(b.y, gy[1][k + 1], g11);
                        g00 = fmaf(a.z, gy[0][k + 2], g00);
                        g01 = fmaf(a.z, gy[1][k + 2], g01);
                        g10 = fmaf(b.z, gy[0][k + 2], g10);
                        g11 = fmaf(b.z, gy[1][k + 2], g11);
                        g00 = fmaf(a.w, gy[0][k + 3], g00);
                        g01 = fmaf(a.w, gy[1][k + 3], g01);
                        g10 = fmaf(b.w, gy[0][k + 3], g10);
                        g11 = fmaf(b.w, gy[1][k + 3], g11);
                    }
                    // activation-jet VJP (autodiff.cpp:644-666); the even lane does the
                    // coupled slots (u, u_x), the odd lane the diagonal ones (u_t, u_xx)
                    const float4 zz = zst[q * 32 + lane];
                    const float zx = __shfl_xor_sync(0xffffffffu, zz.z, 1);  // odd: z0(n+1); even: z2(n+1)
                    float sg, d1, d2, d3;
                    v2::act3<ACT, FAST>(half ? zx : zz.x, sg, d1, d2, d3);
                    const float x1 = __shfl_xor_sync(0xffffffffu, half ? g00 : d1, 1);  // even: g2(n); odd: s1(n)
                    const float x2 = __shfl_xor_sync(0xffffffffu, g01, 1);   // even: g3(n)
                    const float x3 = __shfl_xor_sync(0xffffffffu, zz.x, 1);  // even: z2(n)
                    const float x4 = __shfl_xor_sync(0xffffffffu, zz.y, 1);  // even: z3(n)
                    const float x5 = __shfl_xor_sync(0xffffffffu, g10, 1);   // even: g2(n+1)
                    const float x6 = __shfl_xor_sync(0xffffffffu, g11, 1);   // even: g3(n+1)
                    const float x8 = __shfl_xor_sync(0xffffffffu, zz.w, 1);  // even: z3(n+1)
                    const float x9 = __shfl_xor_sync(0xffffffffu, d1, 1);    // even: s1(n+1)
                    const float x10 = __shfl_xor_sync(0xffffffffu, d2, 1);   // even: s2(n+1)
                    const float x11 = __shfl_xor_sync(0xffffffffu, d3, 1);   // even: s3(n+1)
                    float h00, h01, h10, h11;  // dL/dz [neuron][slot]
                    if (!half) {
                        const float z1 = zz.y, z1b = zz.w;
                        h00 = g00 * d1 + d2 * (g01 * z1 + x1 * x3) + x2 * (d3 * z1 * z1 + d2 * x4);
                        h01 = g01 * d1 + 2.f * x2 * d2 * z1;
                        h10 = g10 * x9 + x10 * (g11 * z1b + x5 * zx) + x6 * (x11 * z1b * z1b + x10 * x8);
                        h11 = g11 * x9 + 2.f * x6 * x10 * z1b;
                    } else {
                        h00 = g00 * x1;
                        h01 = g01 * x1;
                        h10 = g10 * d1;
                        h11 = g11 * d1;
                    }
                    const float* ua = Ub + n * R;
                    const float* ub = ua + R;
#pragma unroll
                    for (int j = 0; j < R; j += 4) {
                        const float4 a = *reinterpret_cast<const float4*>(ua + j);
                        const float4 b = *reinterpret_cast<const float4*>(ub + j);
                        yn[0][j] = fmaf(b.x, h10, fmaf(a.x, h00, yn[0][j]));
                        yn[1][j] = fmaf(b.x, h11, fmaf(a.x, h01, yn[1][j]));
                        yn[0][j + 1] = fmaf(b.y, h10, fmaf(a.y, h00, yn[0][j + 1]));
                        yn[1][j + 1] = fmaf(b.y, h11, fmaf(a.y, h01, yn[1][j + 1]));
                        yn[0][j + 2] = fmaf(b.z, h10, fmaf(a.z, h00, yn[0][j + 2]));
                        yn[1][j + 2] = fmaf(b.z, h11, fmaf(a.z, h01, yn[1][j + 2]));
                        yn[0][j + 3] = fmaf(b.w, h10, fmaf(a.w, h00, yn[0][j + 3]));
                        yn[1][j + 3] = fmaf(b.w, h11, fmaf(a.w, h01, yn[1][j + 3]));
                    }
                }
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
