// Host side of the meta tensor-core kernel (pinn_meta_tc2.cuh): bf16 factor
// blocks + per-tile schedule, the launch, and the fixed-order reduction of the
// per-CTA partial gradients into ParamPacker order (autodiff.cpp:926-946).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <vector>

#include "internal.h"
#include "pinn_meta_tc2.cuh"

namespace lrnr_b200 {
namespace detail {

namespace {

int pad16(int r) { return (r + 15) / 16 * 16; }
int toff_h(int row, int col, int rows) { return ((col >> 3) * (rows >> 3) + (row >> 3)) * 64 + (row & 7) * 8 + (col & 7); }

// gout[i] (+)= sum of the CTA-summed partial entries mapped to packer index i
// (src >= 0: one entry; src < 0: ncopy per-warp / per-quarter copies at stride QS, fixed order)
__global__ void mtc_permute_kernel(const double* __restrict__ sum, const int* __restrict__ map, int64_t n, int64_t qbase,
                                   int QS, double* __restrict__ out, int accumulate, int ncopy = 4) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int src = map[i];
    double v;
    if (src >= 0) {
        v = sum[src];
    } else {
        const int64_t o = qbase + (-src - 1);
        v = 0.0;
        for (int c = 0; c < ncopy; ++c) v += sum[o + static_cast<int64_t>(c) * QS];
    }
    out[i] = accumulate ? out[i] + v : v;
}

}  // namespace

bool mtc_eligible(const Model& m) {
    if (m.dtype != LRNR_F32 || m.kind != LRNR_MODEL_LRNR || m.L < 2) return false;
    if (m.M[0] != 2 || m.M[m.L] != 1) return false;
    for (int l = 0; l < m.L; ++l)
        if (m.r[l] > mtc::RP) return false;
    return 1 + m.rtotal <= mtc::MAX_R1;
}

void build_mtc2(Model& m) {
    auto& v = m.mtc2;
    v = Model::MTC2{};
    if (!mtc_eligible(m)) return;
    const int L = m.L;
    const int KC = mtc2::KC;
    v.rp.assign(L, 0);
    v.nc.assign(L, 0);
    v.yoff.assign(L, 0);
    v.coff.assign(L, 0);
    for (int l = 0; l < L; ++l) v.rp[l] = pad16(m.r[l]);
    int64_t yo = 0;
    int co = 0;
    for (int l = 0; l + 1 < L; ++l) {
        v.nc[l] = (m.M[l + 1] + KC - 1) / KC;
        v.yoff[l] = yo;
        yo += static_cast<int64_t>(2 * mtc2::ROWS) * v.rp[l];
        v.coff[l] = co;
        co += v.nc[l];
    }
    v.ystride = yo;
    std::vector<unsigned char> blob;
    std::vector<int64_t> boff;
    std::vector<int> bbytes;
    auto put = [&](size_t base, int elem, float x) {
        const __nv_bfloat16 h = __float2bfloat16(x);
        std::memcpy(blob.data() + base + 2 * static_cast<size_t>(elem), &h, 2);
    };
    for (int l = 0; l + 1 < L; ++l) {
        const int rl = m.r[l], rn = m.r[l + 1], RL = v.rp[l], RN = v.rp[l + 1], M = m.M[l + 1];
        const double* rows = m.packed.data() + m.off_trans[l];
        auto U = [&](int k, int j) { return (k < M && j < rl) ? rows[static_cast<size_t>(k) * m.trow[l] + j] : 0.0; };
        auto V = [&](int k, int j) { return (k < M && j < rn) ? rows[static_cast<size_t>(k) * m.trow[l] + rl + j] : 0.0; };
        auto B = [&](int k) { return k < M ? rows[static_cast<size_t>(k) * m.trow[l] + rl + rn] : 0.0; };
        const int bytes = 256 * (RL + RN) + 4 * KC;
        for (int c = 0; c < v.nc[l]; ++c) {
            const int k0 = c * KC;
            const size_t o = blob.size();
            boff.push_back(static_cast<int64_t>(o));
            bbytes.push_back(bytes);
            blob.resize(o + bytes, 0);
            for (int n = 0; n < KC; ++n)
                for (int j = 0; j < RL; ++j) put(o, toff_h(n, j, KC), static_cast<float>(U(k0 + n, j)));
            for (int n = 0; n < KC; ++n) {
                const float b = static_cast<float>(B(k0 + n));
                std::memcpy(blob.data() + o + 256 * RL + 4 * n, &b, 4);
            }
            for (int n = 0; n < KC; ++n)
                for (int j = 0; j < RN; ++j) put(o + 256 * RL + 4 * KC, toff_h(n, j, KC), static_cast<float>(V(k0 + n, j)));
        }
    }
    v.dblocks.ensure(std::max<size_t>(blob.size(), 16));
    CK(cudaMemcpy(v.dblocks.p, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    v.dblk_off.ensure(boff.size() * sizeof(int64_t));
    v.dblk_bytes.ensure(bbytes.size() * sizeof(int));
    CK(cudaMemcpy(v.dblk_off.p, boff.data(), boff.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(v.dblk_bytes.p, bbytes.data(), bbytes.size() * sizeof(int), cudaMemcpyHostToDevice));
    int64_t go = 0;
    v.gbase.assign(L, 0);
    for (int l = 0; l + 1 < L; ++l) {
        v.gbase[l] = go;
        go += static_cast<int64_t>(v.nc[l]) * 16384;
    }
    v.qbase = go;
    int qo = 0;
    v.qdb.assign(L, 0);
    for (int l = 0; l + 1 < L; ++l) {
        v.qdb[l] = qo;
        qo += v.nc[l] * KC;
    }
    v.qdUL = qo;
    qo += m.r[L - 1];
    v.qdbL = qo;
    qo += 1;
    v.qdV0 = qo;
    qo += 2 * m.r[0];
    v.QS = (qo + 31) & ~31;
    v.wg_stride = (v.qbase + static_cast<int64_t>(mtc2::NWE) * v.QS + 63) & ~int64_t(63);
    std::vector<int> map;
    for (int l = 0; l < L; ++l) {
        const int Mo = m.M[l + 1], Mi = m.M[l], r = m.r[l];
        for (int k = 0; k < Mo; ++k)
            for (int j = 0; j < r; ++j)
                map.push_back(l + 1 < L ? static_cast<int>(v.gbase[l] + (k / KC) * 16384 + (k % KC) * 64 + j)
                                        : -(v.qdUL + j) - 1);
        for (int i = 0; i < Mi; ++i)
            for (int j = 0; j < r; ++j)
                map.push_back(l == 0 ? -(v.qdV0 + i * r + j) - 1
                                     : static_cast<int>(v.gbase[l - 1] + (i / KC) * 16384 + 8192 + (i % KC) * 64 + j));
        for (int k = 0; k < Mo; ++k) map.push_back(l + 1 < L ? -(v.qdb[l] + k) - 1 : -v.qdbL - 1);
    }
    v.n_params = static_cast<int64_t>(map.size());
    v.dmap.ensure(map.size() * sizeof(int));
    CK(cudaMemcpy(v.dmap.p, map.data(), map.size() * sizeof(int), cudaMemcpyHostToDevice));
    v.ok = true;
}

template <int ACT>
void launch_meta_tc2(lrnr_gpu_ctx* ctx, Model& m, const double* s_dev, const double* mu_dev, double w, double* dev_out,
                     double* wg_out) {
    if (!m.mtc2.ok) build_mtc2(m);
    const auto& v = m.mtc2;
    if (!v.ok) throw InvalidArg("meta tensor-core kernel: needs an FP32 LRNR with widths (2, ..., 1), ranks <= 64");
    const int64_t n_inst = ctx->n_inst, n_per = ctx->n_per;
    const int R1 = 1 + m.rtotal;
    auto kern = mtc2::meta_tc2_kernel<ACT>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, mtc2::SMEM_BYTES));
    RunGeom g{};
    g.P = mtc2::PT;
    g.n_per_inst = n_per;
    g.tiles_per_inst = static_cast<int>((n_per + mtc2::PT - 1) / mtc2::PT);
    const int64_t total_tiles = static_cast<int64_t>(g.tiles_per_inst) * n_inst;
    const int64_t max_grid = ctx->num_sms;
    int64_t tpu = (total_tiles + max_grid * 4 - 1) / (max_grid * 4);
    tpu = std::max<int64_t>(1, std::min<int64_t>(tpu, g.tiles_per_inst));
    g.tiles_per_unit = static_cast<int>(tpu);
    g.units_per_inst = static_cast<int>((g.tiles_per_inst + tpu - 1) / tpu);
    g.n_units = static_cast<int64_t>(g.units_per_inst) * n_inst;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_grid, g.n_units)));
    ctx->scratch.ensure(static_cast<size_t>(grid) * v.ystride * sizeof(float) + 64);
    ensure_part<float>(ctx, n_inst, g.units_per_inst, R1);
    m.mtc2.wg.ensure(static_cast<size_t>(grid) * v.wg_stride * sizeof(float));
    m.mtc2.sum.ensure(static_cast<size_t>(v.wg_stride) * sizeof(double));
    float* wg = m.mtc2.wg.as<float>();
    CK(cudaMemsetAsync(wg, 0, static_cast<size_t>(grid) * v.wg_stride * sizeof(float), ctx->stream));
    mtc2::MetaNet2 net{};
    net.L = m.L;
    for (int l = 0; l <= m.L; ++l) net.M[l] = m.M[l];
    for (int l = 0; l < m.L; ++l) {
        net.r[l] = m.r[l];
        net.rp[l] = v.rp[l];
        net.nc[l] = v.nc[l];
        net.yoff[l] = v.yoff[l];
        net.gbase[l] = v.gbase[l];
        net.qdb[l] = v.qdb[l];
        net.coff[l] = v.coff[l];
    }
    for (int l = 0; l <= m.L; ++l) net.soff[l] = m.soff[l];
    net.ystride = v.ystride;
    net.rtotal = m.rtotal;
    net.blocks = v.dblocks.as<unsigned char>();
    net.blk_off = v.dblk_off.as<int64_t>();
    net.blk_bytes = v.dblk_bytes.as<int>();
    const float* base = m.dev.as<float>();
    net.V0 = base + m.off_V0;
    net.ulast = base + m.off_ulast;
    net.qbase = v.qbase;
    net.QS = v.QS;
    net.qdUL = v.qdUL;
    net.qdbL = v.qdbL;
    net.qdV0 = v.qdV0;
    net.wg_stride = v.wg_stride;
    kern<<<grid, mtc2::NT, mtc2::SMEM_BYTES, ctx->stream>>>(net, g, ctx->pts, s_dev, mu_dev, static_cast<float>(w),
                                                             ctx->scratch.as<float>(), ctx->part.as<float>(), wg,
                                                             bad_word(ctx, m), ctx->term_spec,
                                                             ctx->term_objective);
    CK(cudaGetLastError());
    reduce_rows_kernel<float><<<static_cast<unsigned>((v.wg_stride + 255) / 256), 256, 0, ctx->stream>>>(
        wg, grid, v.wg_stride, v.wg_stride, m.mtc2.sum.as<double>(), 0);
    CK(cudaGetLastError());
    mtc_permute_kernel<<<static_cast<unsigned>((v.n_params + 255) / 256), 256, 0, ctx->stream>>>(
        m.mtc2.sum.as<double>(), v.dmap.as<int>(), v.n_params, v.qbase, v.QS, wg_out, ctx->accumulate_wg, mtc2::NWE);
    CK(cudaGetLastError());
    reduce_units<float>(ctx, n_inst, g.units_per_inst, R1, dev_out);
    ctx->launches += 3;
}

template void launch_meta_tc2<0>(lrnr_gpu_ctx*, Model&, const double*, const double*, double, double*, double*);
template void launch_meta_tc2<1>(lrnr_gpu_ctx*, Model&, const double*, const double*, double, double*, double*);


}  // namespace detail
}  // namespace lrnr_b200

#ifdef MTC_TIMING
// dev aid: read and reset the meta kernel's per-phase cycle counters (CTA 0)
extern "C" int lrnr_mtc_timing(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, lrnr_b200::mtc::g_mtc_timing, 32 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    static const unsigned long long zero[32] = {};
    return cudaMemcpyToSymbol(lrnr_b200::mtc::g_mtc_timing, zero, sizeof(zero)) != cudaSuccess;
}
#endif
