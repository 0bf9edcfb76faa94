// meta_train's step on the device (training.cpp:335-426): the meta gradient of
// the interior terms (FMA tile kernel, META phase 3) through the hypernetwork,
// the sparse (banded decay) and ortho (Gram) regularizers and the meta-mode
// initial / periodic terms; C ABI lrnr_gpu_meta_loss_grad,
// lrnr_gpu_set_meta_boundary, lrnr_gpu_meta_terms_grad.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

using namespace lrnr_b200;
using namespace lrnr_b200::detail;

namespace {

// ---- meta_train regularizers (training.cpp:295-305, 378-389) ----
// banded decay (Tape::banded_decay_penalty + VJP, autodiff.cpp:346-360,779-790) of
// every layer's s_l(mu_i), weighted c = lambda_sparse * w * (points of instance i):
// adds its VJP into the instance's dL/ds row (before the hypernetwork backward).
__global__ void banded_decay_kernel(const double* __restrict__ s, int64_t n_inst, int rtotal, BandLayout lay,
                                    double gamma, double c, double* __restrict__ rows, int R1,
                                    double* __restrict__ pen) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_inst) return;
    const double* f = s + i * rtotal;
    double* ds = rows + i * R1 + 1;
    double acc = 0.0;
    for (int l = 0; l < lay.L; ++l)
        for (int k = lay.off[l]; k + 1 < lay.off[l + 1]; ++k) {
            const double arg = -f[k] + gamma * f[k + 1];
            if (arg > 0.0) {
                acc += arg;
                ds[k] -= c;
                ds[k + 1] += gamma * c;
            }
        }
    pen[i] = acc;
}

// Gram penalty ||A^T A - I||_F^2 of a rows x r matrix (Tape::gram_ortho_penalty,
// autodiff.cpp:322-342): E = A^T A - I, then dA += coef * A E (coef = 4 lambda,
// the GramOrtho VJP autodiff.cpp:761-777).
__global__ void gram_e_kernel(const double* __restrict__ A, int rows, int r, double* __restrict__ E) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= r * r) return;
    const int i = idx / r, j = idx % r;
    double dot = 0.0;
    for (int k = 0; k < rows; ++k) dot += A[static_cast<int64_t>(k) * r + i] * A[static_cast<int64_t>(k) * r + j];
    E[idx] = dot - (i == j ? 1.0 : 0.0);
}
__global__ void gram_grad_kernel(const double* __restrict__ A, int rows, int r, const double* __restrict__ E,
                                 double coef, double* __restrict__ gA) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(rows) * r) return;
    const int64_t i = idx / r;
    const int j = static_cast<int>(idx % r);
    double acc = 0.0;
    for (int k = 0; k < r; ++k) acc += A[i * r + k] * E[k * r + j];
    gA[idx] += coef * acc;
}

struct MetaReg {
    double lambda_sparse = 0.0, gamma = 1.5, lambda_ortho = 0.0;
    bool boundary = false;  // include the meta boundary points (lrnr_gpu_set_meta_boundary)
    double sparse = 0.0, ortho = 0.0, boundary_value = 0.0;  // outputs
};

// Meta step: per-instance s from the hypernetwork (already in ctx->s_dev),
// the META tile kernel for (loss, dL/ds per instance, dU/dV/b), then the
// hypernetwork VJP of the per-instance dL/ds.  Output: ParamPacker order.
void meta_step(lrnr_gpu_ctx* ctx, Model& m, double w, double* out_grad, double* out_value, MetaReg* reg = nullptr) {
    if (!m.v2meta.ok) build_v2(m, true);
    const auto& v = m.v2meta;
    if (!v.ok) throw InvalidArg("meta path supports ranks <= 64");
    const int R1 = 1 + m.rtotal;
    int64_t n_lrnr = 0;
    for (int l = 0; l < m.L; ++l) n_lrnr += static_cast<int64_t>(m.M[l + 1]) * m.r[l] + static_cast<int64_t>(m.M[l]) * m.r[l] + m.M[l + 1];
    const int64_t n_hyper = ctx->hyper.n_params;
    ctx->out.ensure(static_cast<size_t>(ctx->n_inst * R1) * sizeof(double));
    ctx->hgrad.ensure(static_cast<size_t>(n_lrnr + n_hyper) * sizeof(double));
    double* rows = ctx->out.as<double>();
    double* gout = ctx->hgrad.as<double>();
    ctx->out_rows = ctx->n_inst;
    ctx->out_R1 = R1;
    reset_bad(ctx, m);
    if (ctx->n_per == 0) {
        CK(cudaMemsetAsync(rows, 0, static_cast<size_t>(ctx->n_inst * R1) * sizeof(double), ctx->stream));
        CK(cudaMemsetAsync(gout, 0, static_cast<size_t>(n_lrnr) * sizeof(double), ctx->stream));
    }
    const double* sd = ctx->s_dev.as<double>();
    const double* md = ctx->mu_dev.as<double>();
    auto launch_meta = [&](double wt, double* rows_out) {
        const int RP = v.RPMAX;
        if (ctx->opt_meta_prec != 0) {
            require(mtc_eligible(m), "BF16 meta path: needs an FP32 LRNR with widths (2, ..., 1), ranks <= 64, r_total < 512");
            if (m.act == LRNR_ACT_SIN) launch_meta_tc2<1>(ctx, m, sd, md, wt, rows_out, gout);
            else launch_meta_tc2<0>(ctx, m, sd, md, wt, rows_out, gout);
            return;
        }
        if (m.dtype == LRNR_F32 && m.act == LRNR_ACT_SIN && RP == 64) launch_v2<float, 32, 1, 8, 64, 1, false, true>(ctx, m, sd, md, wt, rows_out, gout);
        else if (m.dtype == LRNR_F32 && m.act == LRNR_ACT_SIN && RP == 32) launch_v2<float, 32, 1, 8, 32, 1, false, true>(ctx, m, sd, md, wt, rows_out, gout);
        else if (m.dtype == LRNR_F32 && m.act == LRNR_ACT_TANH && RP == 64) launch_v2<float, 32, 1, 8, 64, 0, false, true>(ctx, m, sd, md, wt, rows_out, gout);
        else if (m.dtype == LRNR_F32 && m.act == LRNR_ACT_TANH && RP == 32) launch_v2<float, 32, 1, 8, 32, 0, false, true>(ctx, m, sd, md, wt, rows_out, gout);
        else if (m.dtype == LRNR_F64 && m.act == LRNR_ACT_TANH && RP == 32) launch_v2<double, 32, 1, 8, 32, 0, false, true>(ctx, m, sd, md, wt, rows_out, gout);
        else if (m.dtype == LRNR_F64 && m.act == LRNR_ACT_SIN && RP == 32) launch_v2<double, 32, 1, 8, 32, 1, false, true>(ctx, m, sd, md, wt, rows_out, gout);
        else throw InvalidArg("meta path: unsupported dtype / rank combination");
    };
    if (ctx->n_per > 0) launch_meta(w, rows);
    // boundary terms (PinnTermEmitter meta mode, training.cpp:307-327): a forward pass for u,
    // per-point specs, then the seeded META pass adding its factor gradients onto gout
    double* hrows = rows;  // the per-instance dL/ds rows the hypernetwork backward consumes
    const int64_t nbp = ctx->mb_ic + 2 * ctx->mb_bc;
    const bool with_bnd = reg && reg->boundary && nbp > 0;
    // 1/(instances x points) of each boundary kind over every rank (safe_inv, training.cpp:364-366)
    const int64_t n_ic_all = reg && reg->boundary ? comm_global_count(ctx, ctx->mb_inst * ctx->mb_ic) : 0;
    const int64_t n_bc_all = reg && reg->boundary ? comm_global_count(ctx, ctx->mb_inst * ctx->mb_bc) : 0;
    if (with_bnd) {
        require(ctx->mb_inst == ctx->n_inst, "meta boundary points were set for another instance count");
        const int64_t n_inst = ctx->n_inst, nb_all = n_inst * nbp;
        ctx->mb_rows.ensure(static_cast<size_t>(n_inst * R1) * sizeof(double));
        ctx->mb_sum.ensure(static_cast<size_t>(n_inst * R1) * sizeof(double));
        ctx->bnd_jets.ensure(static_cast<size_t>(4 * nb_all) * sizeof(double) + 16);
        ctx->bnd_spec.ensure(static_cast<size_t>(nb_all) * sizeof(TermSpec) + 16);
        const double* save_pts = ctx->pts;
        const int64_t save_per = ctx->n_per;
        ctx->pts = ctx->mb_pts.as<double>();
        ctx->n_per = nbp;
        try {
            dispatch_small<1>(ctx, m, sd, md, 1.0, ctx->mb_rows.as<double>(), ctx->bnd_jets.as<double>());
            const double wc = n_ic_all ? 1.0 / static_cast<double>(n_ic_all) : 0.0;
            const double wb = n_bc_all ? 1.0 / static_cast<double>(n_bc_all) : 0.0;
            boundary_spec_multi_kernel<<<static_cast<unsigned>((nb_all + 127) / 128), 128, 0, ctx->stream>>>(
                ctx->bnd_jets.as<double>(), ctx->mb_sinx.as<double>(), n_inst, ctx->mb_ic, ctx->mb_bc, wc, wb,
                ctx->bnd_spec.as<TermSpec>());
            CK(cudaGetLastError());
            ++ctx->launches;
            ctx->term_spec = ctx->bnd_spec.as<TermSpec>();
            ctx->accumulate_wg = ctx->n_per > 0 && save_per > 0 ? 1 : 0;
            launch_meta(1.0, ctx->mb_rows.as<double>());
        } catch (...) {
            ctx->pts = save_pts;
            ctx->n_per = save_per;
            ctx->term_spec = nullptr;
            ctx->accumulate_wg = 0;
            throw;
        }
        ctx->pts = save_pts;
        ctx->n_per = save_per;
        ctx->term_spec = nullptr;
        ctx->accumulate_wg = 0;
        hrows = ctx->mb_sum.as<double>();
        add_rows_kernel<<<static_cast<unsigned>((n_inst * R1 + 255) / 256), 256, 0, ctx->stream>>>(
            rows, ctx->mb_rows.as<double>(), n_inst * R1, hrows);
        CK(cudaGetLastError());
        ++ctx->launches;
    }
    const double c_sparse = reg ? reg->lambda_sparse * w * static_cast<double>(ctx->n_per) : 0.0;
    if (c_sparse > 0.0) {
        BandLayout lay{};
        lay.L = m.L;
        for (int l = 0; l <= m.L; ++l) lay.off[l] = m.soff[l];
        ctx->meta_ws.ensure(static_cast<size_t>(ctx->n_inst) * sizeof(double) + 8);
        banded_decay_kernel<<<static_cast<unsigned>((ctx->n_inst + 127) / 128), 128, 0, ctx->stream>>>(
            ctx->s_dev.as<double>(), ctx->n_inst, m.rtotal, lay, reg->gamma, c_sparse, hrows, R1, ctx->meta_ws.as<double>());
        CK(cudaGetLastError());
        ++ctx->launches;
    }
    hyper_backward_resident(ctx, hrows, R1, gout + n_lrnr);
    std::vector<double> gram_e;
    std::vector<std::pair<int, int>> gram_shape;
    if (reg && reg->lambda_ortho > 0.0) {
        if (!m.flat_dev.p) {
            m.flat_dev.ensure(m.flat.size() * sizeof(double));
            CK(cudaMemcpyAsync(m.flat_dev.p, m.flat.data(), m.flat.size() * sizeof(double), cudaMemcpyHostToDevice,
                               ctx->stream));
        }
        size_t e_len = 0;
        for (int l = 0; l < m.L; ++l) e_len += 2 * static_cast<size_t>(m.r[l]) * m.r[l];
        ctx->gram_ws.ensure(e_len * sizeof(double) + 8);
        double* E = ctx->gram_ws.as<double>();
        int64_t off = 0;
        size_t eo = 0;
        for (int l = 0; l < m.L; ++l) {
            const int r = m.r[l];
            const int rows_uv[2] = {m.M[l + 1], m.M[l]};  // U_l (M_l+1 x r), V_l (M_l x r)
            for (int which = 0; which < 2; ++which) {
                const int rw = rows_uv[which];
                const double* A = m.flat_dev.as<double>() + off;
                gram_e_kernel<<<(r * r + 127) / 128, 128, 0, ctx->stream>>>(A, rw, r, E + eo);
                if (ctx->comm_rank == 0) {  // rank-independent term: added once before the all-reduce
                    gram_grad_kernel<<<static_cast<unsigned>((static_cast<int64_t>(rw) * r + 127) / 128), 128, 0,
                                       ctx->stream>>>(A, rw, r, E + eo, 4.0 * reg->lambda_ortho, gout + off);
                    ++ctx->launches;
                }
                CK(cudaGetLastError());
                ++ctx->launches;
                gram_shape.emplace_back(r, static_cast<int>(eo));
                eo += static_cast<size_t>(r) * r;
                off += static_cast<int64_t>(rw) * r;
            }
            off += m.M[l + 1];  // b_l
        }
        gram_e.resize(eo);
        download(ctx, E, gram_e.data(), eo);
    }
    // instances (or points) are sharded over the ranks: the bases / hypernetwork gradient is summed
    comm_allreduce(ctx, gout, static_cast<size_t>(n_lrnr + n_hyper));
    std::vector<double> h(static_cast<size_t>(ctx->n_inst * R1));
    download(ctx, rows, h.data(), h.size());
    check_bad(ctx, m);
    double sums[3] = {0.0, 0.0, 0.0};  // interior, boundary, sparse
    for (int64_t i = 0; i < ctx->n_inst; ++i) sums[0] += h[static_cast<size_t>(i * R1)];
    if (with_bnd) {
        download(ctx, ctx->mb_rows.as<double>(), h.data(), h.size());
        for (int64_t i = 0; i < ctx->n_inst; ++i) sums[1] += h[static_cast<size_t>(i * R1)];
    }
    if (c_sparse > 0.0) {
        std::vector<double> pen(static_cast<size_t>(ctx->n_inst));
        download(ctx, ctx->meta_ws.as<double>(), pen.data(), pen.size());
        for (int64_t i = 0; i < ctx->n_inst; ++i) sums[2] += c_sparse * pen[static_cast<size_t>(i)];
    }
    comm_allreduce_host(ctx, sums, 3);
    *out_value = sums[0];
    if (reg) {
        reg->boundary_value = sums[1];
        reg->sparse = sums[2];
    }
    if (!gram_shape.empty()) {
        double ro = 0.0;  // weighted_sum over (U_0, V_0, U_1, V_1, ...), each lambda * ||E||_F^2
        for (const auto& gs : gram_shape) {
            double acc = 0.0;
            for (int k = 0; k < gs.first * gs.first; ++k) acc += gram_e[gs.second + k] * gram_e[gs.second + k];
            ro += reg->lambda_ortho * acc;
        }
        reg->ortho = ro;
    }
    download(ctx, gout, out_grad, static_cast<size_t>(n_lrnr + n_hyper));
}

}  // namespace

extern "C" {

int lrnr_gpu_meta_loss_grad(lrnr_gpu_ctx* ctx, const double* mus, double w, double* out_value, double* out_grad) {
    return guarded(ctx, [&] {
        Model& m = const_cast<Model&>(need_model(ctx, LRNR_MODEL_LRNR));
        require(mus && out_grad, "null argument");
        if (!ctx->hyper.set) throw StateError("hypernetwork not set");
        const int64_t n = ctx->n_inst;
        ctx->mu_dev.ensure(static_cast<size_t>(n * 3) * sizeof(double) + 8);
        CK(cudaMemcpyAsync(ctx->mu_dev.p, mus, static_cast<size_t>(n * 3) * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        ctx->coeff_inst = n;
        hyper_forward_resident(ctx, m.rtotal);
        const double wt = w > 0.0 ? w : 1.0 / static_cast<double>(std::max<int64_t>(1, comm_global_count(ctx, n * ctx->n_per)));
        double value = 0.0;
        meta_step(ctx, m, wt, out_grad, &value);
        if (out_value) *out_value = value;
    });
}

int lrnr_gpu_set_meta_boundary(lrnr_gpu_ctx* ctx, int64_t n_inst, const double* initial_x, int64_t n_ic,
                               const double* periodic_t, int64_t n_bc) {
    return guarded(ctx, [&] {
        require(n_inst >= 0 && n_ic >= 0 && n_bc >= 0, "bad boundary counts");
        require((initial_x || n_ic == 0) && (periodic_t || n_bc == 0), "null boundary points");
        const int64_t nb = n_ic + 2 * n_bc;
        std::vector<double> xt(static_cast<size_t>(2 * nb * n_inst)), sx(static_cast<size_t>(n_ic * n_inst));
        for (int64_t q = 0; q < n_inst; ++q) {
            double* p = xt.data() + 2 * nb * q;
            for (int64_t i = 0; i < n_ic; ++i) {
                const double x = initial_x[q * n_ic + i];
                p[2 * i] = x;
                p[2 * i + 1] = 0.0;
                sx[static_cast<size_t>(q * n_ic + i)] = std::sin(x);
            }
            for (int64_t j = 0; j < n_bc; ++j) {
                const double t = periodic_t[q * n_bc + j];
                double* r = p + 2 * (n_ic + 2 * j);
                r[0] = 0.0;
                r[1] = t;
                r[2] = kTwoPi;
                r[3] = t;
            }
        }
        ctx->mb_pts.ensure(xt.size() * sizeof(double) + 16);
        ctx->mb_sinx.ensure(sx.size() * sizeof(double) + 16);
        if (!xt.empty()) CK(cudaMemcpyAsync(ctx->mb_pts.p, xt.data(), xt.size() * sizeof(double),
                                            cudaMemcpyHostToDevice, ctx->stream));
        if (!sx.empty()) CK(cudaMemcpyAsync(ctx->mb_sinx.p, sx.data(), sx.size() * sizeof(double),
                                            cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->mb_inst = n_inst;
        ctx->mb_ic = n_ic;
        ctx->mb_bc = n_bc;
        ++ctx->comm_gen;
    });
}

int lrnr_gpu_meta_terms_grad(lrnr_gpu_ctx* ctx, const double* mus, double w, double lambda_sparse, double gamma,
                             double lambda_ortho, double* out_value, double* out_comps4, double* out_ortho,
                             double* out_grad) {
    return guarded(ctx, [&] {
        Model& m = const_cast<Model&>(need_model(ctx, LRNR_MODEL_LRNR));
        require(mus && out_grad, "null argument");
        require(lambda_sparse >= 0.0 && lambda_ortho >= 0.0, "negative regularizer weight");
        if (!ctx->hyper.set) throw StateError("hypernetwork not set");
        const int64_t n = ctx->n_inst;
        ctx->mu_dev.ensure(static_cast<size_t>(n * 3) * sizeof(double) + 8);
        CK(cudaMemcpyAsync(ctx->mu_dev.p, mus, static_cast<size_t>(n * 3) * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        ctx->coeff_inst = n;
        hyper_forward_resident(ctx, m.rtotal);
        const double wt = w > 0.0 ? w : 1.0 / static_cast<double>(std::max<int64_t>(1, comm_global_count(ctx, n * ctx->n_per)));
        MetaReg reg;
        reg.lambda_sparse = lambda_sparse;
        reg.gamma = gamma;
        reg.lambda_ortho = lambda_ortho;
        reg.boundary = true;
        double interior = 0.0;
        meta_step(ctx, m, wt, out_grad, &interior, &reg);
        if (!std::isfinite(reg.sparse) || !std::isfinite(reg.ortho)) throw NonFinite(-1);
        if (out_comps4) {
            out_comps4[0] = interior;
            out_comps4[1] = reg.boundary_value;
            out_comps4[2] = reg.sparse;
            out_comps4[3] = 0.0;
        }
        if (out_ortho) *out_ortho = reg.ortho;
        if (out_value) *out_value = interior + reg.boundary_value + reg.sparse + reg.ortho;
    });
}

}  // extern "C"
