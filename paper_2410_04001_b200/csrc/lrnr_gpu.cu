// C-ABI core of include/lrnr_gpu.h: device-resident models and their kernel
// layouts, the launch planning and dispatch of the fused residual+gradient
// kernels, the boundary-term passes, the hypernetwork coupling
// (hyper_kernels.cuh), the L1 metric and the non-finite diagnosis
// (NonFiniteError semantics, autodiff.cpp:448-461). The solve loops live in
// solve.cu, the meta step in meta.cu, the FastLRNR construction in eim.cu and
// the narrow-network kernel's host side in fast_launch.cu.
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <climits>
#include <limits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "hyper_kernels.cuh"
#include "internal.h"
#include "instances.h"
#include "pinn_tc.cuh"

using namespace lrnr_b200;
using namespace lrnr_b200::detail;

namespace lrnr_b200 {
namespace detail {
void build_layout(Model& m) {
    const int L = m.L;
    m.soff.assign(L + 1, 0);
    for (int l = 0; l < L; ++l) m.soff[l + 1] = m.soff[l] + m.r[l];
    m.rtotal = m.soff[L];
    m.rmax = *std::max_element(m.r.begin(), m.r.end());
    m.trow.assign(L, 0);
    m.off_trans.assign(L, 0);
    size_t o = 0;
    m.off_V0 = o;
    o += static_cast<size_t>(2 * m.r[0]);
    o = (o + 3) & ~size_t(3);
    for (int l = 0; l + 1 < L; ++l) {
        const int stride = (m.r[l] + m.r[l + 1] + 1 + 3) & ~3;
        m.trow[l] = stride;
        m.off_trans[l] = o;
        o += static_cast<size_t>(m.M[l + 1]) * stride;
    }
    m.off_ulast = o;
    o += static_cast<size_t>(m.r[L - 1] + 1);
    m.packed.assign(o, 0.0);
}

small::Geom small_geom(const Model& m, int64_t n_inst, int64_t n_per) {
    small::Geom g{};
    g.n_total = n_inst * n_per;
    g.n_per = std::max<int64_t>(1, n_per);
    int a = 0, mm = 1;
    for (int l = 0; l + 1 < m.L; ++l) {
        g.aoff[l] = a;
        a += m.M[l + 1];
        mm = std::max(mm, m.M[l + 1]);
    }
    g.a_len = a;
    g.mmax = mm;
    g.rmax = m.rmax;
    int blk = 0;
    for (int l = 0; l + 1 < m.L; ++l) blk = std::max(blk, m.M[l + 1] * m.trow[l]);
    g.blk = (blk + 7) & ~7;
    const size_t elem = m.dtype == LRNR_F64 ? 8 : 4;
    const size_t base = static_cast<size_t>(small::smem_elems(m.rtotal, g.a_len, g.mmax, g.rmax)) * elem;
#ifndef SMALL_STAGE_MAX_KB
#define SMALL_STAGE_MAX_KB 100  // wide layers: several unstaged CTAs per SM beat one staged (fine_tune 1.29 -> 1.05 ms)
#endif
    g.stage = base + 2 * static_cast<size_t>(g.blk) * elem <= SMALL_STAGE_MAX_KB * 1024 ? 1 : 0;
    return g;
}

size_t small_smem_bytes(const Model& m, size_t elem) {
    const small::Geom g = small_geom(m, 1, 1);
    return static_cast<size_t>(small::smem_elems(m.rtotal, g.a_len, g.mmax, g.rmax)) * elem +
           (g.stage ? 2 * static_cast<size_t>(g.blk) * elem : 0);
}

void release_model(Model& m) {
    m.dev.release();
    m.v2.dblocks.release();
    m.v2.dsched_off.release();
    m.v2.dsched_bytes.release();
    m.v2meta.dblocks.release();
    m.v2meta.dsched_off.release();
    m.v2meta.dsched_bytes.release();
    m.tc.dblocks.release();
    m.fk.dblk.release();
    m.tc.dsched_off.release();
    m.tc.dsched_bytes.release();
    m.flat_dev.release();
    for (DevBuf* b : {&m.mtc2.dblocks, &m.mtc2.dblk_off, &m.mtc2.dblk_bytes, &m.mtc2.dmap, &m.mtc2.wg, &m.mtc2.sum})
        b->release();
}

void upload_model(Model& m) {
    const size_t n = m.packed.size();
    if (m.dtype == LRNR_F64) {
        m.dev.ensure(n * sizeof(double));
        CK(cudaMemcpy(m.dev.p, m.packed.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(n);
        for (size_t i = 0; i < n; ++i) f[i] = static_cast<float>(m.packed[i]);
        m.dev.ensure(n * sizeof(float));
        CK(cudaMemcpy(m.dev.p, f.data(), n * sizeof(float), cudaMemcpyHostToDevice));
    }
    m.set = true;
}

// Kernel-v2 layout (pinn_v2.cuh): per transition l and chunk c of KC neurons,
//   forward block  [U^T (rp_l x KC, permuted cols) | b (KC, permuted) | V (KC x rp_{l+1})]
//   backward block [U^T | b | V^T (rp_{l+1} x KC, permuted cols) | U (KC x rp_l)]
// with column q = ng*4 + kk holding local neuron ng + NG*kk (conflict-free Z/G
// stores in phase 1), zero padding for ranks (to multiples of 4) and neurons.
void build_v2(Model& m, bool meta) {
    auto& v = meta ? m.v2meta : m.v2;
    v = Model::V2{};
    const int L = m.L;
    int maxr = 0, maxM = 0;
    for (int l = 0; l < L; ++l) maxr = std::max(maxr, m.r[l]);
    for (int l = 1; l < L; ++l) maxM = std::max(maxM, m.M[l]);
    if (maxr > 64) return;  // the streaming kernel v1 handles larger ranks
    v.RPMAX = maxr <= 32 ? 32 : 64;
    // rank classes: 4 (first / last layers: r <= 4) or RPMAX
    v.rp.resize(L);
    // (FP64 gradient sweeps also have a class of 16: c0 / c1's rank 10 would otherwise pad to 32)
    const bool r16 = m.dtype == LRNR_F64 && !meta;
    for (int l = 0; l < L; ++l) v.rp[l] = m.r[l] <= 4 ? 4 : (r16 && m.r[l] <= 16 ? 16 : v.RPMAX);
    if (m.dtype == LRNR_F64 || meta) {
        v.P = 32;
        v.NG = 8;
        v.PT1 = 1;
    } else if (v.RPMAX == 64) {
        v.P = 32;
        v.NG = 16;
        v.PT1 = 2;
    } else if (maxM <= 32) {  // narrow (FastLRNR): one 32-neuron chunk per transition
        v.P = m.tile_p == 32 ? 32 : 64;
        v.NG = 8;
        v.PT1 = 1;
    } else {
        v.P = m.tile_p == 32 ? 32 : 64;
        v.NG = 16;
        v.PT1 = 2;
    }
    v.KC = 4 * v.NG;
    const int KC = v.KC, NG = v.NG;
    v.nc.assign(L, 0);
    v.yoff.assign(L, 0);
    int yo = 0;
    for (int l = 0; l < L; ++l) {
        v.yoff[l] = yo;
        yo += v.P * v.rp[l] * 4;
    }
    v.ystride = yo;
    int64_t ao = 0;
    v.aoff.assign(L, 0);
    for (int l = 0; l + 1 < L; ++l) {
        v.aoff[l] = ao;
        ao += static_cast<int64_t>((m.M[l + 1] + v.KC - 1) / v.KC) * v.P * v.KC * 4;
    }
    v.astride = ao;
    std::vector<int64_t> fwd_off(L), bwd_off(L);
    std::vector<int> fwd_cnt(L), bwd_cnt(L);
    std::vector<std::vector<int64_t>> foff(L), boff(L);
    auto pad8 = [](size_t n) { return (n + 7) & ~size_t(7); };
    for (int l = 0; l + 1 < L; ++l) {
        const int rl = m.r[l], rn = m.r[l + 1], rpl = v.rp[l], rpn = v.rp[l + 1], M = m.M[l + 1];
        v.nc[l] = (M + KC - 1) / KC;
        const double* rows = m.packed.data() + m.off_trans[l];
        auto U = [&](int k, int j) { return (k < M && j < rl) ? rows[static_cast<size_t>(k) * m.trow[l] + j] : 0.0; };
        auto V = [&](int k, int j) { return (k < M && j < rn) ? rows[static_cast<size_t>(k) * m.trow[l] + rl + j] : 0.0; };
        auto B = [&](int k) { return k < M ? rows[static_cast<size_t>(k) * m.trow[l] + rl + rn] : 0.0; };
        const size_t nf = pad8(static_cast<size_t>(rpl * KC + KC + KC * rpn));
        const size_t nb = pad8(static_cast<size_t>(rpn * KC + KC * rpl));
        for (int c = 0; c < v.nc[l]; ++c) {
            const int k0 = c * KC;
            auto kq = [&](int q) { return k0 + (q / 4) + NG * (q % 4); };
            // forward block
            foff[l].push_back(static_cast<int64_t>(v.blocks.size()));
            size_t o = v.blocks.size();
            v.blocks.resize(o + nf, 0.0);
            double* B0 = v.blocks.data() + o;
            for (int j = 0; j < rpl; ++j)
                for (int q = 0; q < KC; ++q) B0[j * KC + q] = U(kq(q), j);
            for (int q = 0; q < KC; ++q) B0[rpl * KC + q] = B(kq(q));
            for (int kl = 0; kl < KC; ++kl)
                for (int j = 0; j < rpn; ++j) B0[rpl * KC + KC + kl * rpn + j] = V(k0 + kl, j);
            // backward block: V^T (permuted cols) | U   (A is reloaded, not recomputed)
            boff[l].push_back(static_cast<int64_t>(v.blocks.size()));
            o = v.blocks.size();
            v.blocks.resize(o + nb, 0.0);
            double* B1 = v.blocks.data() + o;
            for (int j = 0; j < rpn; ++j)
                for (int q = 0; q < KC; ++q) B1[j * KC + q] = V(kq(q), j);
            for (int kl = 0; kl < KC; ++kl)
                for (int j = 0; j < rpl; ++j) B1[rpn * KC + kl * rpl + j] = U(k0 + kl, j);
        }
        fwd_cnt[l] = static_cast<int>(nf);
        bwd_cnt[l] = static_cast<int>(nb);
    }
    for (int l = 0; l + 1 < L; ++l)
        for (int c = 0; c < v.nc[l]; ++c) {
            v.sched_off.push_back(foff[l][c]);
            v.sched_cnt.push_back(fwd_cnt[l]);
        }
    for (int l = L - 2; l >= 0; --l)
        for (int c = 0; c < v.nc[l]; ++c) {
            v.sched_off.push_back(boff[l][c]);
            v.sched_cnt.push_back(bwd_cnt[l]);
        }
    const size_t esz = m.dtype == LRNR_F64 ? 8 : 4;
    const size_t nbl = std::max<size_t>(v.blocks.size(), 8);
    v.dblocks.ensure(nbl * esz);
    if (m.dtype == LRNR_F64) {
        if (!v.blocks.empty()) CK(cudaMemcpy(v.dblocks.p, v.blocks.data(), v.blocks.size() * 8, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(v.blocks.begin(), v.blocks.end());
        if (!f.empty()) CK(cudaMemcpy(v.dblocks.p, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
    }
    const size_t ns = std::max<size_t>(v.sched_off.size(), 1);
    std::vector<int> bytes(v.sched_cnt.size());
    for (size_t i = 0; i < bytes.size(); ++i) bytes[i] = static_cast<int>(v.sched_cnt[i] * esz);
    v.dsched_off.ensure(ns * sizeof(int64_t));
    v.dsched_bytes.ensure(ns * sizeof(int));
    if (!v.sched_off.empty()) {
        CK(cudaMemcpy(v.dsched_off.p, v.sched_off.data(), v.sched_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(v.dsched_bytes.p, bytes.data(), bytes.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    v.ok = true;
}

// Tensor-core layout (pinn_tc.cuh), FP16 two-term split of FP32 factors: x S = hi + lo,
// hi = fp16(x S), lo = fp16(x S - hi), S = 2^e per matrix (max |x| S < 2^15).  Per
// transition l and chunk of 32 neurons (16-bit K-major canonical tiles, hi then lo):
//   forward block [UT (N = 32 neurons x K = rk_l) | bias (32 floats) | V (N = rn_{l+1} x K = 32)]
//   reverse block [UT | bias | VT (N = 32 neurons x K = rk_{l+1}) | U (N = rn_l x K = 32)]
// plus, per layer, 1 / S and the max row 2-norm of U_l and V_l (the kernel's Z / G bounds).
void build_tc(Model& m) {
    auto& v = m.tc;
    v = Model::TC{};
    if (m.dtype != LRNR_F32 || m.L < 2) return;
    const int L = m.L;
    const int KC = tc::KC;
    for (int l = 0; l < L; ++l)
        if (m.r[l] > tc::RP) return;
    v.rk.resize(L);
    v.rn.resize(L);
    for (int l = 0; l < L; ++l) {
        v.rk[l] = (m.r[l] + 15) & ~15;
        v.rn[l] = m.r[l] <= 16 ? 16 : 32;
    }
    v.nc.assign(L, 0);
    v.yoff.assign(L, 0);
    v.kU.assign(L, 0);
    v.kV.assign(L, 0);
    v.muU.assign(L, 0.f);
    v.muV.assign(L, 0.f);
    int yo = 0;
    for (int l = 0; l < L; ++l) {
        v.yoff[l] = yo;
        yo += tc::P * m.r[l] * 4;
    }
    v.ystride = yo;
    for (int l = 0; l + 1 < L; ++l) v.nc[l] = (m.M[l + 1] + KC - 1) / KC;
    std::vector<std::vector<int64_t>> foff(L), boff(L);
    std::vector<int> fcnt(L), bcnt(L);
    // fp16 hi / lo of x * S at byte offset o of the hi tile (lo tile at hi + lo_off)
    auto put = [](unsigned char* hi, int lo_off, int o, double x, float S) {
        const float f = static_cast<float>(x) * S;
        const __half hh = __float2half_rn(f);
        const __half ll = __float2half_rn(f - __half2float(hh));
        std::memcpy(hi + o, &hh, 2);
        std::memcpy(hi + lo_off + o, &ll, 2);
    };
    auto pow2_for = [](double amax) {  // k with amax * 2^k < 2^15
        if (!(amax > 0.0) || !std::isfinite(amax)) return 0;
        int e;
        std::frexp(amax, &e);  // amax < 2^e
        return std::max(-40, std::min(40, 14 - e));  // the kernel's exponent range (umma::pow2_exp)
    };
    for (int l = 0; l + 1 < L; ++l) {
        const int rl = m.r[l], rn = m.r[l + 1], M = m.M[l + 1];
        const int rkl = v.rk[l], rkn = v.rk[l + 1], rnl = v.rn[l], rnn = v.rn[l + 1];
        const double* rows = m.packed.data() + m.off_trans[l];
        auto U = [&](int k, int j) {
            return (k < M && j < rl) ? static_cast<double>(static_cast<float>(rows[static_cast<size_t>(k) * m.trow[l] + j]))
                                     : 0.0;
        };
        auto V = [&](int k, int j) {
            return (k < M && j < rn)
                       ? static_cast<double>(static_cast<float>(rows[static_cast<size_t>(k) * m.trow[l] + rl + j]))
                       : 0.0;
        };
        auto B = [&](int k) { return k < M ? rows[static_cast<size_t>(k) * m.trow[l] + rl + rn] : 0.0; };
        double umax = 0.0, vmax = 0.0, un = 0.0, vn = 0.0;
        for (int k = 0; k < M; ++k) {
            double su = 0.0, svv = 0.0;
            for (int j = 0; j < rl; ++j) {
                umax = std::max(umax, std::fabs(U(k, j)));
                su += U(k, j) * U(k, j);
            }
            for (int j = 0; j < rn; ++j) {
                vmax = std::max(vmax, std::fabs(V(k, j)));
                svv += V(k, j) * V(k, j);
            }
            un = std::max(un, su);
            vn = std::max(vn, svv);
        }
        v.kU[l] = pow2_for(umax);
        v.kV[l] = pow2_for(vmax);
        const float SU = static_cast<float>(std::ldexp(1.0, v.kU[l])), SV = static_cast<float>(std::ldexp(1.0, v.kV[l]));
        // bounds are used as upper bounds: round the norms up a little
        v.muU[l] = static_cast<float>(std::sqrt(un) * (1.0 + 1e-6));
        v.muV[l] = static_cast<float>(std::sqrt(vn) * (1.0 + 1e-6));
        const int ut = 4 * KC * rkl;                 // UT hi + lo bytes
        const int nf = ut + 4 * KC + 4 * rnn * KC;   // forward block bytes
        const int nb = ut + 4 * KC + 4 * KC * rkn + 4 * rnl * KC;
        fcnt[l] = nf;
        bcnt[l] = nb;
        for (int c = 0; c < v.nc[l]; ++c) {
            const int k0 = c * KC;
            for (int dir = 0; dir < 2; ++dir) {
                size_t o = v.blocks.size();
                (dir == 0 ? foff : boff)[l].push_back(static_cast<int64_t>(o));
                v.blocks.resize(o + (dir == 0 ? nf : nb), 0);
                unsigned char* f = v.blocks.data() + o;
                for (int n = 0; n < KC; ++n)
                    for (int j = 0; j < rkl; ++j) put(f, 2 * KC * rkl, umma::kmaj16_off(n, j, KC), U(k0 + n, j), SU);
                float* bias = reinterpret_cast<float*>(f + ut);
                for (int n = 0; n < KC; ++n) bias[n] = static_cast<float>(B(k0 + n));
                unsigned char* g = f + ut + 4 * KC;
                if (dir == 0) {
                    for (int j = 0; j < rnn; ++j)
                        for (int n = 0; n < KC; ++n)
                            put(g, 2 * rnn * KC, umma::kmaj16_off(j, n, rnn), V(k0 + n, j), SV);
                } else {
                    for (int n = 0; n < KC; ++n)
                        for (int j = 0; j < rkn; ++j) put(g, 2 * KC * rkn, umma::kmaj16_off(n, j, KC), V(k0 + n, j), SV);
                    unsigned char* uu = g + 4 * KC * rkn;
                    for (int j = 0; j < rnl; ++j)
                        for (int n = 0; n < KC; ++n)
                            put(uu, 2 * rnl * KC, umma::kmaj16_off(j, n, rnl), U(k0 + n, j), SU);
                }
            }
        }
    }
    for (int l = 0; l + 1 < L; ++l)
        for (int c = 0; c < v.nc[l]; ++c) {
            v.sched_off.push_back(foff[l][c]);
            v.sched_cnt.push_back(fcnt[l]);
        }
    for (int l = L - 2; l >= 0; --l)
        for (int c = 0; c < v.nc[l]; ++c) {
            v.sched_off.push_back(boff[l][c]);
            v.sched_cnt.push_back(bcnt[l]);
        }
    v.dblocks.ensure(std::max<size_t>(v.blocks.size(), 16));
    if (!v.blocks.empty()) CK(cudaMemcpy(v.dblocks.p, v.blocks.data(), v.blocks.size(), cudaMemcpyHostToDevice));
    const size_t ns = std::max<size_t>(v.sched_off.size(), 1);
    v.dsched_off.ensure(ns * sizeof(int64_t));
    v.dsched_bytes.ensure(ns * sizeof(int));
    if (!v.sched_off.empty()) {
        CK(cudaMemcpy(v.dsched_off.p, v.sched_off.data(), v.sched_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(v.dsched_bytes.p, v.sched_cnt.data(), v.sched_cnt.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    v.ok = true;
}

}  // namespace detail
}  // namespace lrnr_b200

namespace lrnr_b200 {
namespace detail {


// ---------------------------------------------------------------------------
// launch planning
// ---------------------------------------------------------------------------
template <int ACT, bool FAST, bool NARROW>
void launch_tc(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
               double* dev_out) {
    const auto& v = m.tc;
    const int64_t n_inst = ctx->n_inst, n_per = ctx->n_per;
    const int R1 = 1 + m.rtotal;
    if (R1 > 1024) throw InvalidArg("tensor-core path supports r_total < 1024");
    const size_t smem = static_cast<size_t>(tc::SMEM_BYTES);
    auto kern = tc::pinn_tc_kernel<ACT, FAST, NARROW>;
    ctx->unit_ctr.ensure(sizeof(unsigned long long));
    CK(cudaMemsetAsync(ctx->unit_ctr.p, 0xff, sizeof(unsigned long long), ctx->stream));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    RunGeom g{};
    g.P = tc::P;
    g.n_per_inst = n_per;
    g.tiles_per_inst = static_cast<int>((n_per + tc::P - 1) / tc::P);
    const int64_t total_tiles = static_cast<int64_t>(g.tiles_per_inst) * n_inst;
    const int64_t max_grid = ctx->num_sms;  // one CTA per SM: it owns all 512 TMEM columns
    // units are claimed dynamically: one tile each up to 64 per CTA
    int64_t tpu = (total_tiles + max_grid * 64 - 1) / (max_grid * 64);
    tpu = std::max<int64_t>(1, std::min<int64_t>(tpu, g.tiles_per_inst));
    g.tiles_per_unit = static_cast<int>(tpu);
    g.units_per_inst = static_cast<int>((g.tiles_per_inst + tpu - 1) / tpu);
    g.n_units = static_cast<int64_t>(g.units_per_inst) * n_inst;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_grid, g.n_units)));
    ctx->scratch.ensure(static_cast<size_t>(grid) * v.ystride * sizeof(float) + 64);
    ensure_part<float>(ctx, n_inst, g.units_per_inst, R1);
    tc::NetTC net{};
    net.L = m.L;
    for (int l = 0; l <= m.L; ++l) {
        net.M[l] = m.M[l];
        net.soff[l] = m.soff[l];
    }
    for (int l = 0; l < m.L; ++l) {
        net.r[l] = m.r[l];
        net.rk[l] = v.rk[l];
        net.rn[l] = v.rn[l];
        net.nc[l] = v.nc[l];
        net.yoff[l] = v.yoff[l];
        net.kU[l] = v.kU[l];
        net.kV[l] = v.kV[l];
        net.muU[l] = v.muU[l];
        net.muV[l] = v.muV[l];
    }
    net.c3 = ACT == 1 ? 1.f : 2.f;
    net.ystride = v.ystride;
    net.rtotal = m.rtotal;
    net.blocks = v.dblocks.as<unsigned char>();
    net.sched_off = v.dsched_off.as<int64_t>();
    net.sched_bytes = v.dsched_bytes.as<int>();
    net.sched_len = static_cast<int>(v.sched_off.size());
    const float* base = m.dev.as<float>();
    net.V0 = base + m.off_V0;
    net.ulast = base + m.off_ulast;
    kern<<<grid, tc::NT, smem, ctx->stream>>>(net, g, ctx->pts, s_dev, mu_dev, static_cast<float>(w),
                                              ctx->scratch.as<float>(), ctx->part.as<float>(), bad_word(ctx, m),
                                              ctx->unit_ctr.as<unsigned long long>());
    CK(cudaGetLastError());
    reduce_units<float>(ctx, n_inst, g.units_per_inst, R1, dev_out);
    ctx->launches += 1;
}

bool dispatch_tc(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                 double* dev_out) {
    // auto (0): the tensor-core kernel for every eligible FP32 model (ranks <= 32): the
    // c2 LRNR, and the FastLRNR too (c2 r_hat 32: 5.1 vs 6.1 ms on the narrow FMA kernel;
    // c3: 80 vs 106 ms; scripts/fast_ab.py, scripts/c3_ab.py).  2 forces it.
    const bool want = ctx->opt_kernel == 2 || ctx->opt_kernel == 0;
    if (!m.tc.ok || !want) return false;
    const bool fast = ctx->opt_fast_sincos != 0;
    bool narrow = true;  // one chunk per transition (the FastLRNR)
    for (int l = 0; l + 1 < m.L; ++l) narrow = narrow && m.tc.nc[l] == 1;
#define TC_GO(A_, F_)                                                             \
    do {                                                                          \
        if (narrow) launch_tc<A_, F_, true>(ctx, m, s_dev, mu_dev, w, dev_out);    \
        else launch_tc<A_, F_, false>(ctx, m, s_dev, mu_dev, w, dev_out);          \
    } while (0)
    if (m.act == LRNR_ACT_SIN) {
        if (fast) TC_GO(1, true);
        else TC_GO(1, false);
    } else {
        TC_GO(0, false);
    }
#undef TC_GO
    return true;
}

bool dispatch_v2(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                 double* dev_out) {
    const auto& v = m.v2;
    if (!v.ok || ctx->opt_kernel == 1) return false;  // 0 / 2 (not tc-eligible) / 3 (force)
    const bool fast = ctx->opt_fast_sincos != 0;
#define V2CASE(T_, P_, PT1_, NG_, RP_, ACT_, FAST_)                                             \
    if (v.P == P_ && v.PT1 == PT1_ && v.NG == NG_ && v.RPMAX == RP_ && m.act == ACT_ && fast == FAST_) { \
        launch_v2<T_, P_, PT1_, NG_, RP_, ACT_, FAST_>(ctx, m, s_dev, mu_dev, w, dev_out);     \
        return true;                                                                           \
    }
    if (m.dtype == LRNR_F32) {
        V2CASE(float, 64, 2, 16, 32, 1, false)
        V2CASE(float, 64, 2, 16, 32, 1, true)
        V2CASE(float, 64, 2, 16, 32, 0, false)
        V2CASE(float, 64, 1, 8, 32, 1, false)
        V2CASE(float, 64, 1, 8, 32, 1, true)
        V2CASE(float, 64, 1, 8, 32, 0, false)
        V2CASE(float, 32, 1, 8, 32, 1, false)
        V2CASE(float, 32, 1, 8, 32, 1, true)
        V2CASE(float, 32, 1, 8, 32, 0, false)
        V2CASE(float, 32, 2, 16, 32, 1, false)
        V2CASE(float, 32, 2, 16, 32, 1, true)
        V2CASE(float, 32, 2, 16, 32, 0, false)
        V2CASE(float, 32, 2, 16, 64, 1, false)
        V2CASE(float, 32, 2, 16, 64, 1, true)
        V2CASE(float, 32, 2, 16, 64, 0, false)
    } else {
        V2CASE(double, 32, 1, 8, 32, 0, false)
        V2CASE(double, 32, 1, 8, 32, 1, false)
    }
#undef V2CASE
    return false;
}

// dispatch over (dtype, act, rmax, mode)
// The small-batch latency kernel: LRNR_OPT_KERNEL 4 forces it; auto (0) takes
// it for batches below one wave of the tile kernels.
bool use_small(const lrnr_gpu_ctx* ctx, const Model& m) {
    const size_t smem = small_smem_bytes(m, m.dtype == LRNR_F64 ? 8 : 4);
    if (smem > 220 * 1024 || m.rmax > 1024) return false;
    if (ctx->opt_kernel == 4) return true;
    return ctx->opt_kernel == 0 && ctx->n_inst * ctx->n_per <= static_cast<int64_t>(ctx->num_sms) * 16;
}

template <int MODE>
void dispatch_small(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                    double* dev_out, double* jets_dev) {
    if (m.dtype == LRNR_F64) {
        if (m.act == LRNR_ACT_TANH) launch_small<double, 0, MODE>(ctx, m, s_dev, mu_dev, w, dev_out, jets_dev);
        else launch_small<double, 1, MODE>(ctx, m, s_dev, mu_dev, w, dev_out, jets_dev);
    } else {
        if (m.act == LRNR_ACT_TANH) launch_small<float, 0, MODE>(ctx, m, s_dev, mu_dev, w, dev_out, jets_dev);
        else launch_small<float, 1, MODE>(ctx, m, s_dev, mu_dev, w, dev_out, jets_dev);
    }
}

template <int MODE>
void dispatch_pinn(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                   double* dev_out, double* jets_dev) {
    if (use_small(ctx, m)) {
        dispatch_small<MODE>(ctx, m, s_dev, mu_dev, w, dev_out, jets_dev);
        return;
    }
    const int rm = m.rmax;
#define LRNR_CASE(T, TPP, RM, ACT)                                                               \
    if (rm <= RM) {                                                                              \
        launch_pinn<T, TPP, RM, ACT, MODE>(ctx, m, s_dev, mu_dev, w, dev_out, jets_dev);        \
        return;                                                                                  \
    }
    if (m.dtype == LRNR_F64) {
        if (m.act == LRNR_ACT_TANH) {
            LRNR_CASE(double, 4, 16, 0)
            LRNR_CASE(double, 4, 32, 0)
            LRNR_CASE(double, 4, 64, 0)
        } else {
            LRNR_CASE(double, 4, 16, 1)
            LRNR_CASE(double, 4, 32, 1)
            LRNR_CASE(double, 4, 64, 1)
        }
    } else {
        if (m.act == LRNR_ACT_TANH) {
            LRNR_CASE(float, 4, 16, 0)
            LRNR_CASE(float, 4, 32, 0)
            LRNR_CASE(float, 4, 64, 0)
        } else {
            LRNR_CASE(float, 4, 16, 1)
            LRNR_CASE(float, 4, 32, 1)
            LRNR_CASE(float, 4, 64, 1)
        }
    }
#undef LRNR_CASE
    throw InvalidArg("rank above the compiled maximum (64)");
}

template void dispatch_small<0>(lrnr_gpu_ctx*, const Model&, const double*, const double*, double, double*, double*);
template void dispatch_small<1>(lrnr_gpu_ctx*, const Model&, const double*, const double*, double, double*, double*);
template void dispatch_pinn<0>(lrnr_gpu_ctx*, const Model&, const double*, const double*, double, double*, double*);
template void dispatch_pinn<1>(lrnr_gpu_ctx*, const Model&, const double*, const double*, double, double*, double*);

// ---------------------------------------------------------------------------
// boundary terms (PinnTermEmitter initial / periodic branches, training.cpp:307-327;
// fast-phase value terms, :533-549).  Points: [initial (x_i, 0)] then periodic
// pairs [(0, t_j), (2pi, t_j)]; the pair's term needs both u values, so a
// forward pass over the boundary points comes first and this kernel turns its
// output jets into per-point term specs for the seeded reverse pass.
// ---------------------------------------------------------------------------
__global__ void boundary_spec_kernel(const double* __restrict__ jets, const double* __restrict__ sin_x,
                                     int64_t n_ic, int64_t n_bc, double w_ic, double w_bc, int abs_obj,
                                     TermSpec* __restrict__ spec) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int kind = abs_obj ? 3 : 2;
    if (i < n_ic) {
        spec[i] = TermSpec{sin_x[i], w_ic, w_ic, kind, 0};
    } else if (i < n_ic + 2 * n_bc) {
        const int64_t j = i - n_ic, first = n_ic + (j & ~int64_t(1));
        if ((j & 1) == 0)  // u(0,t) - u(2pi,t): the term, target = the partner's u
            spec[i] = TermSpec{jets[4 * (first + 1)], w_bc, w_bc, kind, 0};
        else               // u(2pi,t) - u(0,t): seed only (its gradient is the negative)
            spec[i] = TermSpec{jets[4 * first], 0.0, w_bc, kind, 0};
    }
}

// The same for boundary points grouped by instance (meta mode: each instance's
// points use its own s = hyper(mu_i)): nb = n_ic + 2 n_bc points per instance.
__global__ void boundary_spec_multi_kernel(const double* __restrict__ jets, const double* __restrict__ sin_x,
                                           int64_t n_inst, int64_t n_ic, int64_t n_bc, double w_ic, double w_bc,
                                           TermSpec* __restrict__ spec) {
    const int64_t nb = n_ic + 2 * n_bc;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_inst * nb) return;
    const int64_t inst = i / nb, loc = i % nb, base = inst * nb;
    if (loc < n_ic) {
        spec[i] = TermSpec{sin_x[inst * n_ic + loc], w_ic, w_ic, 2, 0};
    } else {
        const int64_t j = loc - n_ic, first = base + n_ic + (j & ~int64_t(1));
        if ((j & 1) == 0) spec[i] = TermSpec{jets[4 * (first + 1)], w_bc, w_bc, 2, 0};
        else spec[i] = TermSpec{jets[4 * first], 0.0, w_bc, 2, 0};
    }
}

__global__ void add_rows_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                double* __restrict__ c) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) c[i] = a[i] + b[i];
}


// ---------------------------------------------------------------------------
// non-finite diagnosis: first non-finite node in tape order (autodiff.cpp:448-461)
// ---------------------------------------------------------------------------
int diagnose_tag(const Model& m, const double* s, double x, double t, const double* mu) {
    auto bad = [](double v) { return !std::isfinite(v); };
    // leaves: bias vectors (bind_lrnr / bind_fast) and s leaves, all tag -1;
    // the factor matrices are bound slots, not tape nodes (autodiff.cpp:47-59)
    for (int l = 0; l + 1 < m.L; ++l)
        for (int k = 0; k < m.M[l + 1]; ++k)
            if (bad(m.packed[m.off_trans[l] + static_cast<size_t>(k) * m.trow[l] + m.r[l] + m.r[l + 1]])) return -1;
    if (bad(m.packed[m.off_ulast + m.r[m.L - 1]])) return -1;
    for (int i = 0; i < m.rtotal; ++i)
        if (bad(s[i])) return -1;
    if (bad(x) || bad(t)) return -1;
    const bool fast = m.kind == LRNR_MODEL_FAST;
    const int L = m.L;
    const double* P = m.packed.data();
    std::vector<double> y(4 * m.rmax), yn(4 * m.rmax);
    const int r0 = m.r[0];
    const double z0[4][2] = {{x, t}, {1, 0}, {0, 1}, {0, 0}};
    for (int c = 0; c < 4; ++c)
        for (int j = 0; j < r0; ++j) y[c * m.rmax + j] = P[m.off_V0 + j] * z0[c][0] + P[m.off_V0 + r0 + j] * z0[c][1];
    if (fast)
        for (int c = 0; c < 4; ++c)
            for (int j = 0; j < r0; ++j)
                if (bad(y[c * m.rmax + j])) return 0;  // v_in dense node, tag 0 (autodiff.cpp:911)
    for (int l = 0; l + 1 < L; ++l) {
        const int rl = m.r[l], rn = m.r[l + 1];
        const double* sl = s + m.soff[l];
        bool nf = false;
        if (fast)
            for (int c = 0; c < 4; ++c)
                for (int j = 0; j < rl; ++j) nf |= bad(sl[j] * y[c * m.rmax + j]);  // scale node
        std::fill(yn.begin(), yn.end(), 0.0);
        for (int k = 0; k < m.M[l + 1]; ++k) {
            const double* row = P + m.off_trans[l] + static_cast<size_t>(k) * m.trow[l];
            double a[4] = {0, 0, 0, 0};
            for (int c = 0; c < 4; ++c)
                for (int j = 0; j < rl; ++j) a[c] += row[j] * sl[j] * y[c * m.rmax + j];
            a[0] += row[rl + rn];
            double sg, d1, d2;
            if (m.act == LRNR_ACT_TANH) {
                sg = std::tanh(a[0]);
                d1 = 1 - sg * sg;
                d2 = -2 * sg * d1;
            } else {
                sg = std::sin(a[0]);
                d1 = std::cos(a[0]);
                d2 = -sg;
            }
            const double z[4] = {sg, d1 * a[1], d1 * a[2], d2 * a[1] * a[1] + d1 * a[3]};
            for (int c = 0; c < 4; ++c) nf |= bad(a[c]) || bad(z[c]);
            for (int c = 0; c < 4; ++c)
                for (int j = 0; j < rn; ++j) yn[c * m.rmax + j] += row[rl + j] * z[c];
        }
        if (fast)
            for (int c = 0; c < 4; ++c)
                for (int j = 0; j < rn; ++j) nf |= bad(yn[c * m.rmax + j]);
        if (nf) return l + 1;
        y.swap(yn);
    }
    const int rL = m.r[L - 1];
    const double* sL = s + m.soff[L - 1];
    double u[4] = {0, 0, 0, 0};
    bool nf = false;
    for (int c = 0; c < 4; ++c)
        for (int j = 0; j < rL; ++j) {
            nf |= fast && bad(sL[j] * y[c * m.rmax + j]);
            u[c] += P[m.off_ulast + j] * sL[j] * y[c * m.rmax + j];
        }
    u[0] += P[m.off_ulast + rL];
    for (int c = 0; c < 4; ++c) nf |= bad(u[c]);
    if (nf) return L;
    (void)mu;
    return -1;  // residual / square / scale nodes
}

unsigned long long* bad_word(lrnr_gpu_ctx* ctx, const Model& m) {
    if (!ctx->bad.p) {
        ctx->bad.ensure(2 * sizeof(unsigned long long));
        CK(cudaMemsetAsync(ctx->bad.p, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
    }
    return ctx->bad.as<unsigned long long>() + (m.kind == LRNR_MODEL_FAST ? 1 : 0);
}

void reset_bad(lrnr_gpu_ctx* ctx, const Model& m) {
    CK(cudaMemsetAsync(bad_word(ctx, m), 0xff, sizeof(unsigned long long), ctx->stream));
}

// Read (and clear) the model slot's non-finite word; a recorded point is
// re-walked on the host to find the first non-finite node in tape order.
void check_bad(lrnr_gpu_ctx* ctx, const Model& m) {
    unsigned long long b = 0;
    CK(cudaMemcpyAsync(&b, bad_word(ctx, m), sizeof(b), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (b == ULLONG_MAX) return;
    reset_bad(ctx, m);
    const int64_t gp = static_cast<int64_t>(b);
    const int64_t inst = gp / std::max<int64_t>(1, ctx->n_per);
    double xt[2] = {0.0, 0.0}, mu[3] = {0.0, 0.0, 0.0};
    std::vector<double> s(static_cast<size_t>(m.rtotal));
    if (ctx->pts && gp < ctx->n_inst * ctx->n_per && inst < ctx->coeff_inst && ctx->coeff_rtotal == m.rtotal) {
        CK(cudaMemcpy(xt, ctx->pts + 2 * gp, sizeof(xt), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(mu, ctx->mu_dev.as<double>() + 3 * inst, sizeof(mu), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(s.data(), ctx->s_dev.as<double>() + inst * m.rtotal, s.size() * sizeof(double),
                      cudaMemcpyDeviceToHost));
        throw NonFinite(diagnose_tag(m, s.data(), xt[0], xt[1], mu));
    }
    throw NonFinite(-1);
}

const Model& need_model(lrnr_gpu_ctx* ctx, int model) {
    require(model == LRNR_MODEL_LRNR || model == LRNR_MODEL_FAST, "unknown model slot");
    if (!ctx->models[model].set) throw StateError("model not set");
    if (!ctx->pts && ctx->n_inst * ctx->n_per > 0) throw StateError("points not set");
    return ctx->models[model];
}

void upload_coeffs_impl(lrnr_gpu_ctx* ctx, const double* s, const double* mu, int64_t n_inst, int rtotal) {
    require(n_inst >= 1, "n_inst must be positive");
    ctx->s_dev.ensure(static_cast<size_t>(n_inst * rtotal) * sizeof(double) + 8);
    ctx->mu_dev.ensure(static_cast<size_t>(n_inst * 3) * sizeof(double) + 8);
    if (rtotal > 0)
        CK(cudaMemcpyAsync(ctx->s_dev.p, s, static_cast<size_t>(n_inst * rtotal) * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->mu_dev.p, mu, static_cast<size_t>(n_inst * 3) * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    ctx->coeff_inst = n_inst;
    ctx->coeff_rtotal = rtotal;
}

// Launch residual+gradient (MODE 0) or forward (MODE 1) with resident s/mu.
template <int MODE>
double* run_resident(lrnr_gpu_ctx* ctx, const Model& m, double w, double* dev_out, double* jets_dev) {
    require(ctx->coeff_inst == ctx->n_inst && ctx->coeff_rtotal == m.rtotal,
            "coefficients do not match the points' instance count / model ranks");
    const int R1 = 1 + m.rtotal;
    if (!dev_out) {
        ctx->out.ensure(static_cast<size_t>(ctx->n_inst * R1) * sizeof(double));
        dev_out = ctx->out.as<double>();
    }
    ctx->out_rows = ctx->n_inst;
    ctx->out_R1 = R1;
    bad_word(ctx, m);
    // default weight 1/n over every rank's points (a collective when a communicator is attached)
    const int64_t n_all = w > 0.0 ? 0 : comm_global_count(ctx, ctx->n_inst * ctx->n_per);
    if (ctx->n_per == 0) {
        CK(cudaMemsetAsync(dev_out, 0, static_cast<size_t>(ctx->n_inst * R1) * sizeof(double), ctx->stream));
        return dev_out;
    }
    const double wt = w > 0.0 ? w : 1.0 / static_cast<double>(std::max<int64_t>(1, n_all));
    if (MODE == 0 && use_small(ctx, m)) {
        dispatch_small<0>(ctx, m, ctx->s_dev.as<double>(), ctx->mu_dev.as<double>(), wt, dev_out, nullptr);
        return dev_out;
    }
    if (MODE == 0 && dispatch_fast(ctx, m, ctx->s_dev.as<double>(), ctx->mu_dev.as<double>(), wt, dev_out))
        return dev_out;
    if (MODE == 0 && dispatch_tc(ctx, m, ctx->s_dev.as<double>(), ctx->mu_dev.as<double>(), wt, dev_out))
        return dev_out;
    if (MODE == 0 && dispatch_v2(ctx, m, ctx->s_dev.as<double>(), ctx->mu_dev.as<double>(), wt, dev_out))
        return dev_out;
    dispatch_pinn<MODE>(ctx, m, ctx->s_dev.as<double>(), ctx->mu_dev.as<double>(), wt, dev_out, jets_dev);
    return dev_out;
}

// The streaming kernel only (per-point term specs / |N| objective / forward jets).
template <int MODE>
double* run_resident_stream(lrnr_gpu_ctx* ctx, const Model& m, double w, double* jets_dev) {
    require(ctx->coeff_inst == ctx->n_inst && ctx->coeff_rtotal == m.rtotal,
            "coefficients do not match the points' instance count / model ranks");
    const int R1 = 1 + m.rtotal;
    ctx->out.ensure(static_cast<size_t>(ctx->n_inst * R1) * sizeof(double));
    double* dev_out = ctx->out.as<double>();
    ctx->out_rows = ctx->n_inst;
    ctx->out_R1 = R1;
    bad_word(ctx, m);
    dispatch_pinn<MODE>(ctx, m, ctx->s_dev.as<double>(), ctx->mu_dev.as<double>(), w, dev_out, jets_dev);
    return dev_out;
}

template double* run_resident_stream<1>(lrnr_gpu_ctx*, const Model&, double, double*);

void download(lrnr_gpu_ctx* ctx, const double* dev, double* host, size_t n) {
    CK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
}

void set_model_common(Model& m, int L, int act, int dtype) {
    require(act == LRNR_ACT_TANH || act == LRNR_ACT_SIN, "unknown activation");
    require(dtype == LRNR_F64 || dtype == LRNR_F32, "unknown dtype");
    require(L >= 1 && L <= kMaxL, "depth out of range");
    m.L = L;
    m.act = act;
    m.dtype = dtype;
}

HyperDev hyper_dev(const Hyper& h) {
    HyperDev d{};
    d.K = h.K;
    for (int k = 0; k <= h.K; ++k) d.hw[k] = h.hw[k];
    for (int k = 0; k < h.K; ++k) {
        d.oW[k] = h.oW[k];
        d.ob[k] = h.ob[k];
    }
    d.max_w = h.max_w;
    d.n_params = h.n_params;
    d.P = h.dev.as<double>();
    for (int a = 0; a < 3; ++a) {
        d.lo[a] = h.lo[a];
        d.hi[a] = h.hi[a];
    }
    return d;
}

// s_i = hyper(mu_i) for the ctx's instances -> ctx->s_dev; activations kept in ctx->acts.
void hyper_forward_resident(lrnr_gpu_ctx* ctx, int rtotal) {
    const Hyper& h = ctx->hyper;
    if (!h.set) throw StateError("hypernetwork not set");
    require(h.hw[h.K] == rtotal, "hypernetwork output dim != model r_total");
    const int64_t n = ctx->coeff_inst;
    ctx->acts.ensure(static_cast<size_t>(n * (h.K + 1) * h.max_w) * sizeof(double));
    ctx->s_dev.ensure(static_cast<size_t>(n * rtotal) * sizeof(double) + 8);
    hyper_forward_kernel<<<static_cast<unsigned>(n), 128, 0, ctx->stream>>>(hyper_dev(h), ctx->mu_dev.as<double>(), n,
                                                                             ctx->acts.as<double>(), ctx->s_dev.as<double>());
    CK(cudaGetLastError());
    ctx->launches += 1;
    ctx->coeff_rtotal = rtotal;
}

// dtheta from the per-instance result rows (dev_rows: n x R1)
void hyper_backward_resident(lrnr_gpu_ctx* ctx, const double* dev_rows, int R1, double* dev_grad) {
    const Hyper& h = ctx->hyper;
    const int64_t n = ctx->coeff_inst;
    ctx->G.ensure(static_cast<size_t>(n * h.K * h.max_w) * sizeof(double));
    HyperDev hd = hyper_dev(h);
    hyper_backward_kernel<<<static_cast<unsigned>(n), 128, 0, ctx->stream>>>(hd, ctx->acts.as<double>(), dev_rows, R1, n,
                                                                              ctx->G.as<double>());
    CK(cudaGetLastError());
    hyper_param_grad_kernel<<<(h.n_params + 127) / 128, 128, 0, ctx->stream>>>(hd, ctx->acts.as<double>(),
                                                                                ctx->G.as<double>(), n, dev_grad);
    CK(cudaGetLastError());
    ctx->launches += 2;
}

// FMA-pipe calibration: 16 independent 3-register FMA chains per thread,
// full-chip grid.  Gives the achievable FP32/FP64 FMA rate the roofline is
// compared against (MEASURED_PEAKS.json carries only HBM and bf16 tensor).
template <typename T>
__global__ void __launch_bounds__(256) fma_peak_kernel(T* out, int iters, T b) {
    T acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = T(threadIdx.x + i);
    T a = T(blockIdx.x) * T(1e-7);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], b, a);
    }
    T s = T(0);
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == T(12345.678)) out[0] = s;
}


// GridField points (pde.hpp:40-53): row j = time t_j = j / n_t (kTimeHorizon 1), x_i = 2 pi i / n_x
__global__ void grid_points_kernel(int64_t n_x, int64_t n_t, double* __restrict__ xt) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n_x * (n_t + 1)) return;
    const int64_t j = k / n_x, i = k % n_x;
    xt[2 * k] = kTwoPi * static_cast<double>(i) / static_cast<double>(n_x);
    xt[2 * k + 1] = n_t == 0 ? 0.0 : 1.0 * static_cast<double>(j) / static_cast<double>(n_t);
}

// out = {sum |u - ref|, sum |ref|}: per-thread strided sums, then a fixed-order tree
__global__ void l1_reduce_kernel(const double* __restrict__ u, const double* __restrict__ ref, int64_t n,
                                 double* __restrict__ out) {
    __shared__ double sn[1024], sd[1024];
    double a = 0.0, b = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        a += fabs(u[k] - ref[k]);
        b += fabs(ref[k]);
    }
    sn[threadIdx.x] = a;
    sd[threadIdx.x] = b;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (static_cast<int>(threadIdx.x) < st) {
            sn[threadIdx.x] += sn[threadIdx.x + st];
            sd[threadIdx.x] += sd[threadIdx.x + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sn[0];
        out[1] = sd[0];
    }
}

}  // namespace detail
}  // namespace lrnr_b200

extern "C" {

int lrnr_gpu_create(int device, lrnr_gpu_ctx** out) {
    if (!out) return LRNR_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return LRNR_ECUDA;
    }
    auto* c = new lrnr_gpu_ctx();
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return LRNR_ECUDA;
    }
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    c->stream = c->own;
    *out = c;
    return LRNR_OK;
}

int lrnr_gpu_destroy(lrnr_gpu_ctx* ctx) {
    if (!ctx) return LRNR_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    comm_release(ctx);
    for (auto& m : ctx->models) release_model(m);
    ctx->hyper.dev.release();
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
        cudaEventDestroy(ctx->stage_done);
        cudaEventDestroy(ctx->stage_free);
    }
    for (DevBuf* b : {&ctx->pts_own, &ctx->pts_stage, &ctx->s_dev, &ctx->mu_dev, &ctx->scratch, &ctx->ascratch, &ctx->part, &ctx->out, &ctx->bad,
                      &ctx->acts, &ctx->G, &ctx->hgrad, &ctx->jets, &ctx->meta_ws, &ctx->gram_ws, &ctx->bnd_pts,
                      &ctx->bnd_x, &ctx->bnd_spec, &ctx->bnd_jets, &ctx->solve_rows, &ctx->solve_state, &ctx->solve_m,
                      &ctx->solve_v, &ctx->solve_best, &ctx->solve_s0, &ctx->solve_bt, &ctx->solve_losses,
                      &ctx->solve_pts[0], &ctx->solve_pts[1], &ctx->solve_bnd[0], &ctx->solve_bnd[1],
                      &ctx->solve_sinx[0], &ctx->solve_sinx[1], &ctx->mb_pts, &ctx->mb_sinx, &ctx->mb_rows,
                      &ctx->mb_sum, &ctx->eim_snaps, &ctx->eim_state})
        b->release();
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
    return LRNR_OK;
}

const char* lrnr_gpu_last_error(const lrnr_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
int lrnr_gpu_last_layer_tag(const lrnr_gpu_ctx* ctx) { return ctx ? ctx->tag : -1; }
int64_t lrnr_gpu_launch_count(const lrnr_gpu_ctx* ctx) { return ctx ? ctx->launches : 0; }

int lrnr_gpu_set_option(lrnr_gpu_ctx* ctx, int opt, int value) {
    return guarded(ctx, [&] {
        if (opt == LRNR_OPT_FAST_SINCOS) ctx->opt_fast_sincos = value;
        else if (opt == LRNR_OPT_KERNEL) ctx->opt_kernel = value;
        else if (opt == LRNR_OPT_SOLVE) ctx->opt_solve = value;
        else if (opt == LRNR_OPT_META_PREC) {
            require(value == 0 || value == 1, "meta precision must be 0 (FP32) or 1 (BF16 tensor-core operands)");
            ctx->opt_meta_prec = value;
        }
        else if (opt == LRNR_OPT_TILE_P) {
            require(value == 0 || value == 32 || value == 64, "tile P must be 32 or 64 (0 = default)");
            for (auto& m : ctx->models) {
                m.tile_p = value;
                if (m.set) build_v2(m);
            }
        }
        else throw InvalidArg("unknown option");
    });
}

int lrnr_gpu_set_stream(lrnr_gpu_ctx* ctx, void* s) {
    return guarded(ctx, [&] { ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own; });
}

int lrnr_gpu_set_lrnr(lrnr_gpu_ctx* ctx, int L, const int64_t* widths, const int64_t* ranks, const double* params,
                      int act, int dtype) {
    return guarded(ctx, [&] {
        require(widths && ranks && params, "null argument");
        Model m;
        set_model_common(m, L, act, dtype);
        m.kind = LRNR_MODEL_LRNR;
        require(widths[0] == 2, "input width must be 2 (x, t)");
        require(widths[L] == 1, "residual: expected scalar-output jet");
        for (int l = 0; l < L; ++l) {
            require(ranks[l] >= 1, "LrnrParams: rank must be positive");
            require(ranks[l] <= std::min(widths[l + 1], widths[l]), "LrnrParams: rank exceeds min(M_l, M_{l-1})");
        }
        m.M.assign(widths, widths + L + 1);
        m.r.assign(ranks, ranks + L);
        m.widths64.assign(widths, widths + L + 1);
        m.ranks64.assign(ranks, ranks + L);
        build_layout(m);
        // flat offsets
        std::vector<size_t> oU(L), oV(L), ob(L);
        size_t o = 0;
        for (int l = 0; l < L; ++l) {
            oU[l] = o;
            o += static_cast<size_t>(widths[l + 1] * ranks[l]);
            oV[l] = o;
            o += static_cast<size_t>(widths[l] * ranks[l]);
            ob[l] = o;
            o += static_cast<size_t>(widths[l + 1]);
        }
        m.flat.assign(params, params + o);
        const double* Pp = params;
        for (int j = 0; j < m.r[0]; ++j) {
            m.packed[m.off_V0 + j] = Pp[oV[0] + j];                   // V_0 row 0
            m.packed[m.off_V0 + m.r[0] + j] = Pp[oV[0] + m.r[0] + j]; // V_0 row 1
        }
        for (int l = 0; l + 1 < L; ++l) {
            const int rl = m.r[l], rn = m.r[l + 1];
            for (int k = 0; k < m.M[l + 1]; ++k) {
                double* row = m.packed.data() + m.off_trans[l] + static_cast<size_t>(k) * m.trow[l];
                for (int j = 0; j < rl; ++j) row[j] = Pp[oU[l] + static_cast<size_t>(k) * rl + j];
                for (int j = 0; j < rn; ++j) row[rl + j] = Pp[oV[l + 1] + static_cast<size_t>(k) * rn + j];
                row[rl + rn] = Pp[ob[l] + k];
            }
        }
        for (int j = 0; j < m.r[L - 1]; ++j) m.packed[m.off_ulast + j] = Pp[oU[L - 1] + j];
        m.packed[m.off_ulast + m.r[L - 1]] = Pp[ob[L - 1]];
        Model& dst = ctx->models[LRNR_MODEL_LRNR];
        release_model(dst);
        dst = std::move(m);
        upload_model(dst);
        build_v2(dst);
        build_tc(dst);
        build_fk(dst);
    });
}

int lrnr_gpu_set_fast(lrnr_gpu_ctx* ctx, int L, const int64_t* ranks, const int64_t* red, int64_t m_in,
                      int64_t m_out, const double* F, int act, int dtype) {
    return guarded(ctx, [&] {
        require(ranks && F && (L < 2 || red), "null argument");
        Model m;
        set_model_common(m, L, act, dtype);
        require(L >= 2, "FastParams: need at least two layers");
        require(m_in == 2, "input width must be 2 (x, t)");
        require(m_out == 1, "residual: expected scalar-output jet");
        m.kind = LRNR_MODEL_FAST;
        m.M.assign(L + 1, 0);
        m.M[0] = 2;
        m.M[L] = 1;
        for (int l = 0; l + 1 < L; ++l) {
            require(red[l] >= 1, "FastParams: reduced rank must be positive");
            m.M[l + 1] = static_cast<int>(red[l]);
        }
        for (int l = 0; l < L; ++l) require(ranks[l] >= 1, "FastParams: rank must be positive");
        m.r.assign(ranks, ranks + L);
        build_layout(m);
        size_t o = 0;
        const int r0 = m.r[0];
        for (int j = 0; j < r0; ++j) {
            m.packed[m.off_V0 + j] = F[o + j];
            m.packed[m.off_V0 + r0 + j] = F[o + r0 + j];
        }
        o += static_cast<size_t>(2 * r0);
        for (int l = 0; l + 1 < L; ++l) {
            const int rl = m.r[l], rn = m.r[l + 1], rh = m.M[l + 1];
            const size_t o_uh = o, o_bh = o_uh + static_cast<size_t>(rh) * rl, o_vh = o_bh + rh;
            for (int k = 0; k < rh; ++k) {
                double* row = m.packed.data() + m.off_trans[l] + static_cast<size_t>(k) * m.trow[l];
                for (int j = 0; j < rl; ++j) row[j] = F[o_uh + static_cast<size_t>(k) * rl + j];
                for (int j = 0; j < rn; ++j) row[rl + j] = F[o_vh + static_cast<size_t>(k) * rn + j];
                row[rl + rn] = F[o_bh + k];
            }
            o = o_vh + static_cast<size_t>(rh) * rn;
        }
        for (int j = 0; j < m.r[L - 1]; ++j) m.packed[m.off_ulast + j] = F[o + j];
        o += static_cast<size_t>(m.r[L - 1]);
        m.packed[m.off_ulast + m.r[L - 1]] = F[o];
        Model& dst = ctx->models[LRNR_MODEL_FAST];
        release_model(dst);
        dst = std::move(m);
        upload_model(dst);
        build_v2(dst);
        build_tc(dst);
        build_fk(dst);
    });
}

int lrnr_gpu_set_hyper(lrnr_gpu_ctx* ctx, int K, const int64_t* hw, const double* H, const double* lo,
                       const double* hi) {
    return guarded(ctx, [&] {
        require(hw && H && lo && hi, "null argument");
        require(K >= 1 && K <= kHyperMaxLayers, "hypernetwork depth out of range");
        require(hw[0] == 3, "HyperParams: input dimension must be 3");
        Hyper h;
        h.K = K;
        h.hw.assign(hw, hw + K + 1);
        int o = 0;
        h.max_w = 3;
        for (int k = 0; k < K; ++k) {
            require(hw[k + 1] >= 1, "HyperParams: empty layer");
            h.oW.push_back(o);
            o += static_cast<int>(hw[k + 1] * hw[k]);
            h.ob.push_back(o);
            o += static_cast<int>(hw[k + 1]);
            h.max_w = std::max<int>(h.max_w, static_cast<int>(hw[k + 1]));
        }
        h.n_params = o;
        for (int a = 0; a < 3; ++a) {
            h.lo[a] = lo[a];
            h.hi[a] = hi[a];
        }
        h.dev.ensure(static_cast<size_t>(o) * sizeof(double));
        CK(cudaMemcpy(h.dev.p, H, static_cast<size_t>(o) * sizeof(double), cudaMemcpyHostToDevice));
        h.set = true;
        ctx->hyper.dev.release();
        ctx->hyper = std::move(h);
    });
}

int lrnr_gpu_set_points(lrnr_gpu_ctx* ctx, const double* xt, int64_t n_inst, int64_t n_per) {
    return guarded(ctx, [&] {
        require(n_inst >= 1 && n_per >= 0, "bad point counts");
        require(xt || n_per == 0, "null points");
        const size_t bytes = static_cast<size_t>(n_inst * n_per * 2) * sizeof(double);
        ctx->pts_own.ensure(bytes + 16);
        if (bytes) CK(cudaMemcpyAsync(ctx->pts_own.p, xt, bytes, cudaMemcpyHostToDevice, ctx->stream));
        // the caller's buffer may be reused or freed on return (pinned memory makes the copy asynchronous)
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->pts = ctx->pts_own.as<double>();
        ctx->n_inst = n_inst;
        ctx->n_per = n_per;
        ++ctx->comm_gen;
    });
}

int lrnr_gpu_stage_points(lrnr_gpu_ctx* ctx, const double* xt, int64_t n_inst, int64_t n_per) {
    return guarded(ctx, [&] {
        require(n_inst >= 1 && n_per >= 0, "bad point counts");
        require(xt || n_per == 0, "null points");
        if (!ctx->copy_stream) {
            CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ctx->stage_done, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->stage_free, cudaEventDisableTiming));
        }
        const size_t bytes = static_cast<size_t>(n_inst * n_per * 2) * sizeof(double);
        if (ctx->pts_stage.bytes < bytes + 16) {  // (re)allocation: nothing may use the old buffer
            CK(cudaStreamSynchronize(ctx->copy_stream));
            CK(cudaStreamSynchronize(ctx->stream));
            ctx->pts_stage.ensure(bytes + 16);
        }
        // the staging buffer may still be read by work already submitted on the compute stream
        CK(cudaEventRecord(ctx->stage_free, ctx->stream));
        CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->stage_free, 0));
        if (bytes) CK(cudaMemcpyAsync(ctx->pts_stage.p, xt, bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
        CK(cudaEventRecord(ctx->stage_done, ctx->copy_stream));
        ctx->stage_inst = n_inst;
        ctx->stage_per = n_per;
    });
}

int lrnr_gpu_use_staged_points(lrnr_gpu_ctx* ctx) {
    return guarded(ctx, [&] {
        require(ctx->stage_inst >= 1, "no staged points (lrnr_gpu_stage_points first)");
        CK(cudaStreamWaitEvent(ctx->stream, ctx->stage_done, 0));
        std::swap(ctx->pts_own, ctx->pts_stage);
        ctx->pts = ctx->pts_own.as<double>();
        ctx->n_inst = ctx->stage_inst;
        ctx->n_per = ctx->stage_per;
        ctx->stage_inst = -1;
        ++ctx->comm_gen;
    });
}

int lrnr_gpu_set_points_device(lrnr_gpu_ctx* ctx, const void* xt_dev, int64_t n_inst, int64_t n_per) {
    return guarded(ctx, [&] {
        require(n_inst >= 1 && n_per >= 0, "bad point counts");
        require(xt_dev || n_per == 0, "null points");
        ctx->pts = static_cast<const double*>(xt_dev);
        ctx->n_inst = n_inst;
        ctx->n_per = n_per;
        ++ctx->comm_gen;
    });
}

int lrnr_gpu_upload_coeffs(lrnr_gpu_ctx* ctx, const double* s, const double* mu, int64_t n_inst) {
    return guarded(ctx, [&] {
        require(s && mu, "null argument");
        const Model& m = ctx->models[ctx->models[0].set ? 0 : 1];
        if (!m.set) throw StateError("model not set");
        upload_coeffs_impl(ctx, s, mu, n_inst, m.rtotal);
    });
}

int lrnr_gpu_run(lrnr_gpu_ctx* ctx, int model, double w, double* dev_out) {
    return guarded(ctx, [&] {
        const Model& m = need_model(ctx, model);
        double* d = run_resident<0>(ctx, m, w, dev_out, nullptr);
        comm_allreduce(ctx, d, static_cast<size_t>(ctx->n_inst) * (1 + m.rtotal));
    });
}

int lrnr_gpu_check(lrnr_gpu_ctx* ctx) {
    return guarded(ctx, [&] {
        CK(cudaStreamSynchronize(ctx->stream));
        for (const Model& m : ctx->models)
            if (m.set && ctx->bad.p) check_bad(ctx, m);
    });
}

int lrnr_gpu_download(lrnr_gpu_ctx* ctx, double* host, int64_t n) {
    return guarded(ctx, [&] {
        require(host != nullptr, "null argument");
        require(n <= ctx->out_rows * ctx->out_R1, "download larger than the result");
        download(ctx, ctx->out.as<double>(), host, static_cast<size_t>(n));
    });
}

int lrnr_gpu_loss_grad_s(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, double w,
                         double* out_value, double* out_comps4, double* out_grad_s) {
    return guarded(ctx, [&] {
        const Model& m = need_model(ctx, model);
        require(s && mu, "null argument");
        require(ctx->n_inst == 1, "lrnr_gpu_loss_grad_s needs a single instance");
        upload_coeffs_impl(ctx, s, mu, 1, m.rtotal);
        const int64_t n_all = w > 0.0 ? 0 : comm_global_count(ctx, ctx->n_per);
        const double wt = w > 0.0 ? w : (n_all ? 1.0 / static_cast<double>(n_all) : 0.0);
        double* d = run_resident<0>(ctx, m, wt, nullptr, nullptr);
        comm_allreduce(ctx, d, static_cast<size_t>(1 + m.rtotal));
        std::vector<double> h(static_cast<size_t>(1 + m.rtotal));
        download(ctx, d, h.data(), h.size());
        check_bad(ctx, m);
        if (out_value) *out_value = h[0];
        if (out_comps4) {
            out_comps4[0] = h[0];
            out_comps4[1] = out_comps4[2] = out_comps4[3] = 0.0;
        }
        if (out_grad_s) std::copy(h.begin() + 1, h.end(), out_grad_s);
    });
}

int lrnr_gpu_set_boundary(lrnr_gpu_ctx* ctx, const double* initial_x, int64_t n_ic, const double* periodic_t,
                          int64_t n_bc) {
    return guarded(ctx, [&] {
        require(n_ic >= 0 && n_bc >= 0, "bad boundary counts");
        require((initial_x || n_ic == 0) && (periodic_t || n_bc == 0), "null boundary points");
        const int64_t nb = n_ic + 2 * n_bc;
        std::vector<double> xt(static_cast<size_t>(2 * nb)), sx(static_cast<size_t>(n_ic));
        for (int64_t i = 0; i < n_ic; ++i) {
            xt[2 * i] = initial_x[i];
            xt[2 * i + 1] = 0.0;
            sx[i] = std::sin(initial_x[i]);  // host libm, as the reference's std::sin
        }
        for (int64_t j = 0; j < n_bc; ++j) {
            const int64_t o = n_ic + 2 * j;
            xt[2 * o] = 0.0;
            xt[2 * o + 1] = periodic_t[j];
            xt[2 * o + 2] = kTwoPi;
            xt[2 * o + 3] = periodic_t[j];
        }
        ctx->bnd_pts.ensure(xt.size() * sizeof(double) + 16);
        ctx->bnd_x.ensure(sx.size() * sizeof(double) + 16);
        ctx->bnd_spec.ensure(static_cast<size_t>(nb) * sizeof(TermSpec) + 16);
        ctx->bnd_jets.ensure(static_cast<size_t>(4 * nb) * sizeof(double) + 16);
        if (nb) CK(cudaMemcpyAsync(ctx->bnd_pts.p, xt.data(), xt.size() * sizeof(double), cudaMemcpyHostToDevice,
                                   ctx->stream));
        if (n_ic) CK(cudaMemcpyAsync(ctx->bnd_x.p, sx.data(), sx.size() * sizeof(double), cudaMemcpyHostToDevice,
                                     ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));  // host staging vectors go out of scope
        ctx->n_ic = n_ic;
        ctx->n_bc = n_bc;
        ++ctx->comm_gen;
    });
}

int lrnr_gpu_terms_grad(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, int objective, double w_int,
                        double w_ic, double w_bc, const double* s_init, double lambda_local, double* out_value,
                        double* out_comps4, double* out_grad_s) {
    return guarded(ctx, [&] {
        require(model == LRNR_MODEL_LRNR || model == LRNR_MODEL_FAST, "unknown model slot");
        const Model& m = ctx->models[model];
        if (!m.set) throw StateError("model not set");
        require(s && mu, "null argument");
        require(objective == LRNR_OBJ_SQUARED || objective == LRNR_OBJ_ABS, "unknown objective");
        const int64_t n_int = ctx->pts ? ctx->n_inst * ctx->n_per : 0;
        require(n_int == 0 || ctx->n_inst == 1, "lrnr_gpu_terms_grad needs a single instance");
        auto inv = [](int64_t n) { return n ? 1.0 / static_cast<double>(n) : 0.0; };  // safe_inv
        // default weights: 1/n of that kind over every rank's terms
        const double wi = w_int > 0.0 ? w_int : inv(comm_global_count(ctx, n_int));
        const double wc = w_ic > 0.0 ? w_ic : inv(comm_global_count(ctx, ctx->n_ic));
        const double wb = w_bc > 0.0 ? w_bc : inv(comm_global_count(ctx, ctx->n_bc));
        const int R1 = 1 + m.rtotal;
        std::vector<double> grad(static_cast<size_t>(m.rtotal), 0.0), h(static_cast<size_t>(R1));
        double comps[4] = {0.0, 0.0, 0.0, 0.0};
        upload_coeffs_impl(ctx, s, mu, 1, m.rtotal);
        auto accumulate = [&](int comp) {
            comps[comp] += h[0];
            for (int i = 0; i < m.rtotal; ++i) grad[i] += h[1 + i];
        };
        // interior terms: the fused kernels for w N^2; |N| on the streaming kernel
        if (n_int > 0) {
            double* d;
            if (objective == LRNR_OBJ_SQUARED) {
                d = run_resident<0>(ctx, m, wi, nullptr, nullptr);
            } else {
                PointSwap keep(ctx, ctx->pts, n_int);
                ctx->term_objective = 1;
                d = run_resident_stream<0>(ctx, m, wi, nullptr);
            }
            download(ctx, d, h.data(), h.size());
            check_bad(ctx, m);
            accumulate(0);
        }
        // boundary terms: forward pass for u, specs, seeded reverse pass
        const int64_t nb = ctx->n_ic + 2 * ctx->n_bc;
        if (nb > 0) {
            PointSwap keep(ctx, ctx->bnd_pts.as<double>(), nb);
            run_resident_stream<1>(ctx, m, 1.0, ctx->bnd_jets.as<double>());
            boundary_spec_kernel<<<static_cast<unsigned>((nb + 127) / 128), 128, 0, ctx->stream>>>(
                ctx->bnd_jets.as<double>(), ctx->bnd_x.as<double>(), ctx->n_ic, ctx->n_bc, wc, wb,
                objective == LRNR_OBJ_ABS, ctx->bnd_spec.as<TermSpec>());
            CK(cudaGetLastError());
            ++ctx->launches;
            ctx->term_spec = ctx->bnd_spec.as<TermSpec>();
            double* d = run_resident_stream<0>(ctx, m, 1.0, nullptr);
            download(ctx, d, h.data(), h.size());
            check_bad(ctx, m);
            accumulate(1);
        }
        if (ctx->comm) {  // interior + boundary terms summed over the ranks; locality depends on s only
            std::vector<double> red(static_cast<size_t>(2 + m.rtotal));
            red[0] = comps[0];
            red[1] = comps[1];
            std::copy(grad.begin(), grad.end(), red.begin() + 2);
            comm_allreduce_host(ctx, red.data(), red.size());
            comps[0] = red[0];
            comps[1] = red[1];
            std::copy(red.begin() + 2, red.end(), grad.begin());
        }
        // locality: lambda * sum_l ||s_l - s_init_l||_1 (training.cpp:550-559, autodiff.cpp:791-802)
        if (s_init && lambda_local > 0.0) {
            double acc = 0.0;
            for (int i = 0; i < m.rtotal; ++i) {
                const double dv = s[i] - s_init[i];
                acc += std::fabs(dv);
                grad[i] += lambda_local * (dv > 0.0 ? 1.0 : (dv < 0.0 ? -1.0 : 0.0));
            }
            comps[3] = lambda_local * acc;
            if (!std::isfinite(comps[3])) throw NonFinite(-1);
        }
        if (out_value) *out_value = comps[0] + comps[1] + comps[3];
        if (out_comps4) std::copy(comps, comps + 4, out_comps4);
        if (out_grad_s) std::copy(grad.begin(), grad.end(), out_grad_s);
    });
}

int lrnr_gpu_loss_grad_s_multi(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, double w,
                               double* out_value, double* out_grad_s) {
    return guarded(ctx, [&] {
        const Model& m = need_model(ctx, model);
        require(s && mu, "null argument");
        upload_coeffs_impl(ctx, s, mu, ctx->n_inst, m.rtotal);
        double* d = run_resident<0>(ctx, m, w, nullptr, nullptr);
        const int R1 = 1 + m.rtotal;
        comm_allreduce(ctx, d, static_cast<size_t>(ctx->n_inst * R1));
        std::vector<double> h(static_cast<size_t>(ctx->n_inst * R1));
        download(ctx, d, h.data(), h.size());
        check_bad(ctx, m);
        double v = 0.0;
        for (int64_t i = 0; i < ctx->n_inst; ++i) {
            v += h[static_cast<size_t>(i * R1)];
            if (out_grad_s)
                std::copy(h.begin() + i * R1 + 1, h.begin() + (i + 1) * R1, out_grad_s + i * m.rtotal);
        }
        if (out_value) *out_value = v;
    });
}

int lrnr_gpu_hyper_loss_grad(lrnr_gpu_ctx* ctx, int model, const double* mus, double w, double* out_value,
                             double* out_grad_s, double* out_grad_theta) {
    return guarded(ctx, [&] {
        const Model& m = need_model(ctx, model);
        require(mus != nullptr, "null argument");
        const int64_t n = ctx->n_inst;
        ctx->mu_dev.ensure(static_cast<size_t>(n * 3) * sizeof(double) + 8);
        CK(cudaMemcpyAsync(ctx->mu_dev.p, mus, static_cast<size_t>(n * 3) * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        ctx->coeff_inst = n;
        hyper_forward_resident(ctx, m.rtotal);
        double* d = run_resident<0>(ctx, m, w, nullptr, nullptr);
        const int R1 = 1 + m.rtotal;
        ctx->hgrad.ensure(static_cast<size_t>(ctx->hyper.n_params) * sizeof(double));
        hyper_backward_resident(ctx, d, R1, ctx->hgrad.as<double>());
        // instances are sharded over the ranks: the shared theta gradient and the loss are summed,
        // the per-instance dL/ds rows stay local
        comm_allreduce(ctx, ctx->hgrad.as<double>(), static_cast<size_t>(ctx->hyper.n_params));
        std::vector<double> h(static_cast<size_t>(n * R1));
        download(ctx, d, h.data(), h.size());
        check_bad(ctx, m);
        double v = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            v += h[static_cast<size_t>(i * R1)];
            if (out_grad_s) std::copy(h.begin() + i * R1 + 1, h.begin() + (i + 1) * R1, out_grad_s + i * m.rtotal);
        }
        comm_allreduce_host(ctx, &v, 1);
        if (out_value) *out_value = v;
        if (out_grad_theta) download(ctx, ctx->hgrad.as<double>(), out_grad_theta, static_cast<size_t>(ctx->hyper.n_params));
    });
}

int lrnr_gpu_jets(lrnr_gpu_ctx* ctx, int model, const double* s, double* out_jets) {
    return guarded(ctx, [&] {
        const Model& m = need_model(ctx, model);
        require(s && out_jets, "null argument");
        std::vector<double> mu(static_cast<size_t>(3 * ctx->n_inst), 0.0);
        upload_coeffs_impl(ctx, s, mu.data(), ctx->n_inst, m.rtotal);
        const size_t n = static_cast<size_t>(ctx->n_inst * ctx->n_per);
        ctx->jets.ensure(n * 4 * sizeof(double) + 8);
        run_resident<1>(ctx, m, 1.0, nullptr, ctx->jets.as<double>());
        if (n) download(ctx, ctx->jets.as<double>(), out_jets, n * 4);
        else CK(cudaStreamSynchronize(ctx->stream));
    });
}

int lrnr_gpu_loss(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, double w, double* out_value) {
    return guarded(ctx, [&] {
        const Model& m = need_model(ctx, model);
        require(s && mu && out_value, "null argument");
        upload_coeffs_impl(ctx, s, mu, ctx->n_inst, m.rtotal);
        double* d = run_resident<1>(ctx, m, w, nullptr, nullptr);
        const int R1 = 1 + m.rtotal;
        std::vector<double> h(static_cast<size_t>(ctx->n_inst * R1));
        download(ctx, d, h.data(), h.size());
        check_bad(ctx, m);
        double v = 0.0;
        for (int64_t i = 0; i < ctx->n_inst; ++i) v += h[static_cast<size_t>(i * R1)];
        comm_allreduce_host(ctx, &v, 1);
        *out_value = v;
    });
}


int lrnr_gpu_l1_error(lrnr_gpu_ctx* ctx, int model, const double* s, const double* ref_values, int64_t n_x,
                      int64_t n_t, double* out_l1) {
    return guarded(ctx, [&] {
        require(model == LRNR_MODEL_LRNR || model == LRNR_MODEL_FAST, "unknown model slot");
        const Model& m = ctx->models[model];
        if (!m.set) throw StateError("model not set");
        require(s && ref_values && out_l1 && n_x > 0 && n_t >= 0, "bad arguments");
        const int64_t n = n_x * (n_t + 1);
        ctx->jets.ensure(static_cast<size_t>(n + 2) * sizeof(double));
        ctx->meta_ws.ensure(static_cast<size_t>(2 * n + 2 * n) * sizeof(double) + 16);  // grid (x,t) + ref
        double* grid = ctx->meta_ws.as<double>();
        double* refd = grid + 2 * n;
        grid_points_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(n_x, n_t, grid);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(refd, ref_values, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        const double mu0[3] = {0.0, 0.0, 0.0};
        upload_coeffs_impl(ctx, s, mu0, 1, m.rtotal);
        // u only: the value-only forward (lrnr_forward, model.cpp:260-262), 1 jet slot instead of 4
        double* u = ctx->jets.as<double>();
        const PointSwap keep(ctx, grid, n);  // a non-finite u is diagnosed at its grid point
        launch_values(ctx, m, grid, n, n, ctx->s_dev.as<double>(), u);
        double* red = u + n;
        l1_reduce_kernel<<<1, 1024, 0, ctx->stream>>>(u, refd, n, red);
        CK(cudaGetLastError());
        ctx->launches += 2;
        double h[2];
        download(ctx, red, h, 2);
        check_bad(ctx, m);
        if (h[1] == 0.0) throw InvalidArg("l1_relative_error: reference is identically zero");
        *out_l1 = h[0] / h[1];
    });
}

// dev aid: per-phase cycle counters of the tensor-core kernel (CTA 0), filled
// only when built with -DLRNR_TC_TIMING; zeros otherwise.
int lrnr_dev_tc_timing(unsigned long long* out16) {
#ifdef LRNR_TC_TIMING
    cudaMemcpyFromSymbol(out16, tc::g_tc_timing, 16 * sizeof(unsigned long long));
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(tc::g_tc_timing, z, sizeof(z));
#else
    for (int i = 0; i < 16; ++i) out16[i] = 0;
#endif
    return 0;
}

int lrnr_gpu_fma_peak(lrnr_gpu_ctx* ctx, int dtype, double* out_tflops) {
    return guarded(ctx, [&] {
        require(out_tflops != nullptr, "null argument");
        const int blocks = ctx->num_sms * 8, threads = 256;
        const int iters = dtype == LRNR_F64 ? 2048 : 8192;
        DevBuf o;
        o.ensure(16);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        float ms = 0.f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(e0, ctx->stream));
            if (dtype == LRNR_F64)
                fma_peak_kernel<double><<<blocks, threads, 0, ctx->stream>>>(o.as<double>(), iters, 0.999);
            else
                fma_peak_kernel<float><<<blocks, threads, 0, ctx->stream>>>(o.as<float>(), iters, 0.999f);
            CK(cudaGetLastError());
            CK(cudaEventRecord(e1, ctx->stream));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        o.release();
        const double flops = 2.0 * 32.0 * iters * static_cast<double>(blocks) * threads;
        *out_tflops = flops / (ms * 1e-3) / 1e12;
    });
}

}  // extern "C"
