// Host side of the narrow-network kernel (pinn_fast.cuh): the padded factor
// block, the launch geometry and the dispatch rule.
#include "internal.h"

using namespace lrnr_b200;
using namespace lrnr_b200::detail;

namespace lrnr_b200 {
namespace detail {

// Block layout (floats, zero padded to R = 32): V0[2][R] | per transition l:
// U[R][R] (row n = neuron, column j = rank of layer l) | V[R][R] (row n, column
// k = rank of layer l+1) | b[R] | ulast[R] b_last. Rows are padded to an even
// neuron count with zeros, which the kernel's neuron-pair loop relies on
// (a zero row gives z = 0, sigma(0) = 0 for sin and tanh).
void build_fk(Model& m) {
    auto& f = m.fk;
    f = Model::FK{};
    constexpr int R = fastk::R;
    if (m.dtype != LRNR_F32 || m.L < 2 || m.L > kMaxL) return;
    for (int l = 0; l < m.L; ++l)
        if (m.r[l] > R) return;
    for (int l = 0; l + 1 < m.L; ++l)
        if (m.M[l + 1] > R) return;
    const int L = m.L;
    std::vector<float> blk(static_cast<size_t>(2 * R + (L - 1) * fastk::TRANS + R + 1), 0.f);
    for (int j = 0; j < m.r[0]; ++j) {
        blk[j] = static_cast<float>(m.packed[m.off_V0 + j]);
        blk[R + j] = static_cast<float>(m.packed[m.off_V0 + m.r[0] + j]);
    }
    f.np.assign(L, 0);
    for (int l = 0; l + 1 < L; ++l) {
        float* U = blk.data() + 2 * R + static_cast<size_t>(l) * fastk::TRANS;
        float* V = U + R * R;
        float* b = V + R * R;
        const int rl = m.r[l], rn = m.r[l + 1];
        for (int n = 0; n < m.M[l + 1]; ++n) {
            const double* row = m.packed.data() + m.off_trans[l] + static_cast<size_t>(n) * m.trow[l];
            for (int j = 0; j < rl; ++j) U[n * R + j] = static_cast<float>(row[j]);
            for (int k = 0; k < rn; ++k) V[n * R + k] = static_cast<float>(row[rl + k]);
            b[n] = static_cast<float>(row[rl + rn]);
        }
        f.np[l] = (m.M[l + 1] + 1) / 2;
    }
    float* ul = blk.data() + 2 * R + static_cast<size_t>(L - 1) * fastk::TRANS;
    for (int j = 0; j < m.r[L - 1]; ++j) ul[j] = static_cast<float>(m.packed[m.off_ulast + j]);
    ul[R] = static_cast<float>(m.packed[m.off_ulast + m.r[L - 1]]);
    f.blk_len = static_cast<int>(blk.size());
    f.dblk.ensure(blk.size() * sizeof(float));
    CK(cudaMemcpy(f.dblk.p, blk.data(), blk.size() * sizeof(float), cudaMemcpyHostToDevice));
    f.ok = true;
}

namespace {

template <int ACT, bool FAST>
void launch_fast(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                 double* dev_out) {
    using namespace fastk;
    const auto& f = m.fk;
    const int64_t n_inst = ctx->n_inst, n_per = ctx->n_per;
    const int R1 = 1 + m.rtotal;
    const int RW = (R1 + 31) & ~31;
    const size_t smem = static_cast<size_t>(((f.blk_len + 3) & ~3) + RW + NW * RW) * sizeof(float);
    auto kern = pinn_fast_kernel<ACT, FAST>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    NetF net{};
    net.L = m.L;
    for (int l = 0; l < m.L; ++l) net.r[l] = m.r[l];
    for (int l = 0; l <= m.L; ++l) net.soff[l] = m.soff[l];
    net.rtotal = m.rtotal;
    net.blk = f.dblk.as<float>();
    net.blk_len = f.blk_len;
    int64_t o = 0;
    for (int l = 0; l + 1 < m.L; ++l) {
        net.np[l] = f.np[l];
        net.zoff[l] = o;
        o += static_cast<int64_t>(f.np[l]) * 32 * 4;
        net.uoff[l] = o;
        o += 2 * R * 32;
    }
    net.wstride = o;
    // units: whole multiples of NW warp tiles, about 32 per CTA for balance
    RunGeom g{};
    g.P = TP;
    g.n_per_inst = n_per;
    g.tiles_per_inst = static_cast<int>((n_per + TP - 1) / TP);
    const int64_t total_tiles = static_cast<int64_t>(g.tiles_per_inst) * n_inst;
    const int64_t grid_max = ctx->num_sms;
    int64_t tpu = NW * std::max<int64_t>(1, total_tiles / (grid_max * NW * 32));
    tpu = std::min<int64_t>(tpu, ((g.tiles_per_inst + NW - 1) / NW) * NW);
    g.tiles_per_unit = static_cast<int>(tpu);
    g.units_per_inst = static_cast<int>((g.tiles_per_inst + tpu - 1) / tpu);
    g.n_units = static_cast<int64_t>(g.units_per_inst) * n_inst;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid_max, g.n_units)));
    ctx->ascratch.ensure(static_cast<size_t>(grid) * NW * net.wstride * sizeof(float) + 64);
    ensure_part<float>(ctx, n_inst, g.units_per_inst, R1);
    kern<<<grid, NT, smem, ctx->stream>>>(net, g, ctx->pts, s_dev, mu_dev, static_cast<float>(w),
                                          ctx->ascratch.as<float>(), ctx->part.as<float>(),
                                          bad_word(ctx, m), ctx->term_spec, ctx->term_objective);
    CK(cudaGetLastError());
    reduce_units<float>(ctx, n_inst, g.units_per_inst, R1, dev_out);
    ctx->launches += 1;
}

}  // namespace

bool dispatch_fast(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                   double* dev_out) {
    // forced (5), or auto when the tensor-core kernel cannot take the model
    if (!m.fk.ok || !(ctx->opt_kernel == 5 || (ctx->opt_kernel == 0 && !m.tc.ok))) return false;
    const bool fast = ctx->opt_fast_sincos != 0;
    if (m.act == LRNR_ACT_SIN) {
        if (fast) launch_fast<1, true>(ctx, m, s_dev, mu_dev, w, dev_out);
        else launch_fast<1, false>(ctx, m, s_dev, mu_dev, w, dev_out);
    } else {
        launch_fast<0, false>(ctx, m, s_dev, mu_dev, w, dev_out);
    }
    return true;
}

}  // namespace detail
}  // namespace lrnr_b200
