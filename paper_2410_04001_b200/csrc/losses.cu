// Plain (forward-only) losses and the value-only forward, on the device:
//   lrnr_gpu_values     lrnr_forward / fast_forward            (model.cpp:260-292)
//   lrnr_gpu_loss_tune  loss_tune  (pinn_loss)                 (training.cpp:76-105, 139-163)
//   lrnr_gpu_loss_fast  loss_fast  (classified sampling set X) (training.cpp:165-189)
//   lrnr_gpu_loss_meta  loss_meta  (per-sample mu, hypernet)   (training.cpp:109-137)
// Interior terms need the 4-slot jets (forward sweep of the streaming kernel,
// MODE 1); boundary terms need u only and run the 1-slot value kernel
// (pinn_value.cuh).  Boundary sums are fixed-order single-block reductions.
// As the reference, a non-finite total raises NonFiniteError(-1).
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "internal.h"
#include "pinn_value.cuh"

using namespace lrnr_b200;
using namespace lrnr_b200::detail;

namespace {

// Per instance q the boundary points are [n_ic initial (x, 0)] [n_bc periodic
// pairs (0, t), (2pi, t)] (lrnr_gpu_set_boundary / _set_meta_boundary layouts);
// out = {sum_q,i f(u - sin x), sum_q,j f(u(0,t) - u(2pi,t))}, f = square or abs.
__global__ void boundary_loss_kernel(const double* __restrict__ u, const double* __restrict__ sin_x, int64_t n_inst,
                                     int64_t n_ic, int64_t n_bc, int abs_obj, double* __restrict__ out) {
    __shared__ double sa[256], sb[256];
    const int64_t nb = n_ic + 2 * n_bc;
    double a = 0.0, b = 0.0;
    for (int64_t k = threadIdx.x; k < n_inst * n_ic; k += blockDim.x) {
        const int64_t q = k / n_ic, i = k % n_ic;
        const double d = u[q * nb + i] - sin_x[k];
        a += abs_obj ? fabs(d) : d * d;
    }
    for (int64_t k = threadIdx.x; k < n_inst * n_bc; k += blockDim.x) {
        const int64_t q = k / n_bc, j = k % n_bc;
        const double d = u[q * nb + n_ic + 2 * j] - u[q * nb + n_ic + 2 * j + 1];
        b += abs_obj ? fabs(d) : d * d;
    }
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (static_cast<int>(threadIdx.x) < st) {
            sa[threadIdx.x] += sa[threadIdx.x + st];
            sb[threadIdx.x] += sb[threadIdx.x + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sa[0];
        out[1] = sb[0];
    }
}

template <class T, int RM, int ACT>
void launch_value_t(lrnr_gpu_ctx* ctx, const Model& m, const double* pts, int64_t n_per, int64_t n_total,
                    const double* s_dev, double* out_u) {
    const DevNet<T> net = dev_net<T>(m);
    value::value_kernel<T, RM, ACT><<<static_cast<unsigned>((n_total + value::NT - 1) / value::NT), value::NT, 0,
                                     ctx->stream>>>(net, pts, std::max<int64_t>(1, n_per), n_total, s_dev, out_u,
                                                    bad_word(ctx, m));
    CK(cudaGetLastError());
    ++ctx->launches;
}

// u at the boundary points of `n_inst` instances, then the two boundary sums (device, 2 doubles)
void boundary_sums(lrnr_gpu_ctx* ctx, const Model& m, const double* pts, int64_t n_inst, int64_t n_ic, int64_t n_bc,
                   const double* sin_x, int abs_obj, const double* s_dev, double* dev_u, double* dev_out2) {
    const int64_t nb = n_ic + 2 * n_bc;
    if (n_inst * nb > 0) launch_values(ctx, m, pts, nb, n_inst * nb, s_dev, dev_u);
    boundary_loss_kernel<<<1, 256, 0, ctx->stream>>>(dev_u, sin_x, n_inst, n_ic, n_bc, abs_obj, dev_out2);
    CK(cudaGetLastError());
    ++ctx->launches;
}

void finish_loss(lrnr_gpu_ctx* ctx, const Model& m, double residual, double boundary, double* out3) {
    reset_bad(ctx, m);  // plain evaluation: no tape, the reference reports NonFiniteError(-1)
    const double total = residual + boundary;
    if (!std::isfinite(total)) throw NonFinite(-1);
    out3[0] = total;
    out3[1] = residual;
    out3[2] = boundary;
}

}  // namespace

namespace lrnr_b200 {
namespace detail {

void launch_values(lrnr_gpu_ctx* ctx, const Model& m, const double* pts, int64_t n_per, int64_t n_total,
                   const double* s_dev, double* out_u) {
    if (n_total <= 0) return;
    const int rm = m.rmax;
#define LRNR_VCASE(T, RM, ACT)                                              \
    if (rm <= RM) {                                                         \
        launch_value_t<T, RM, ACT>(ctx, m, pts, n_per, n_total, s_dev, out_u); \
        return;                                                             \
    }
    if (m.dtype == LRNR_F64) {
        if (m.act == LRNR_ACT_TANH) {
            LRNR_VCASE(double, 16, 0)
            LRNR_VCASE(double, 32, 0)
            LRNR_VCASE(double, 64, 0)
        } else {
            LRNR_VCASE(double, 16, 1)
            LRNR_VCASE(double, 32, 1)
            LRNR_VCASE(double, 64, 1)
        }
    } else {
        if (m.act == LRNR_ACT_TANH) {
            LRNR_VCASE(float, 16, 0)
            LRNR_VCASE(float, 32, 0)
            LRNR_VCASE(float, 64, 0)
        } else {
            LRNR_VCASE(float, 16, 1)
            LRNR_VCASE(float, 32, 1)
            LRNR_VCASE(float, 64, 1)
        }
    }
#undef LRNR_VCASE
    throw InvalidArg("rank above the compiled maximum (64)");
}

}  // namespace detail
}  // namespace lrnr_b200

extern "C" {

int lrnr_gpu_values(lrnr_gpu_ctx* ctx, int model, const double* s, const double* xt, int64_t n, double* out_u) {
    return guarded(ctx, [&] {
        require(model == LRNR_MODEL_LRNR || model == LRNR_MODEL_FAST, "unknown model slot");
        const Model& m = ctx->models[model];
        if (!m.set) throw StateError("model not set");
        require(s && n >= 0 && (n == 0 || (xt && out_u)), "bad arguments");
        if (n == 0) return;
        ctx->s_dev.ensure(static_cast<size_t>(m.rtotal) * sizeof(double) + 8);
        CK(cudaMemcpyAsync(ctx->s_dev.p, s, static_cast<size_t>(m.rtotal) * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        ctx->coeff_inst = 1;
        ctx->coeff_rtotal = m.rtotal;
        ctx->meta_ws.ensure(static_cast<size_t>(3 * n) * sizeof(double) + 16);
        double* pts = ctx->meta_ws.as<double>();
        double* u = pts + 2 * n;
        CK(cudaMemcpyAsync(pts, xt, static_cast<size_t>(2 * n) * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        launch_values(ctx, m, pts, n, n, ctx->s_dev.as<double>(), u);
        download(ctx, u, out_u, static_cast<size_t>(n));
        reset_bad(ctx, m);  // value path: non-finite u is returned as such (lrnr_forward has no check)
    });
}

int lrnr_gpu_loss_tune(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, double* out3) {
    return guarded(ctx, [&] {
        require(model == LRNR_MODEL_LRNR || model == LRNR_MODEL_FAST, "unknown model slot");
        const Model& m = ctx->models[model];
        if (!m.set) throw StateError("model not set");
        require(s && mu && out3, "null argument");
        const int64_t n_int = ctx->pts ? ctx->n_inst * ctx->n_per : 0;
        require(n_int == 0 || ctx->n_inst == 1, "lrnr_gpu_loss_tune needs a single instance");
        const int64_t g_int = comm_global_count(ctx, n_int), g_ic = comm_global_count(ctx, ctx->n_ic),
                      g_bc = comm_global_count(ctx, ctx->n_bc);
        upload_coeffs_impl(ctx, s, mu, 1, m.rtotal);
        double sums[3] = {0.0, 0.0, 0.0};  // sum N^2, sum (u - sin x)^2, sum (u(0,t) - u(2pi,t))^2
        if (n_int > 0) {
            PointSwap keep(ctx, ctx->pts, n_int);
            double* d = run_resident_stream<1>(ctx, m, 1.0, nullptr);
            download(ctx, d, sums, 1);
        }
        const int64_t nb = ctx->n_ic + 2 * ctx->n_bc;
        if (nb > 0) {
            ctx->bnd_jets.ensure(static_cast<size_t>(nb + 2) * sizeof(double));
            double* u = ctx->bnd_jets.as<double>();
            boundary_sums(ctx, m, ctx->bnd_pts.as<double>(), 1, ctx->n_ic, ctx->n_bc, ctx->bnd_x.as<double>(), 0,
                          ctx->s_dev.as<double>(), u, u + nb);
            download(ctx, u + nb, sums + 1, 2);
        }
        comm_allreduce_host(ctx, sums, 3);
        auto mean = [](double v, int64_t n) { return n ? v / static_cast<double>(n) : 0.0; };
        finish_loss(ctx, m, mean(sums[0], g_int), mean(sums[1], g_ic) + mean(sums[2], g_bc), out3);
    });
}

int lrnr_gpu_loss_fast(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, const double* X, int64_t n_x,
                       double* out3) {
    return guarded(ctx, [&] {
        require(model == LRNR_MODEL_LRNR || model == LRNR_MODEL_FAST, "unknown model slot");
        const Model& m = ctx->models[model];
        if (!m.set) throw StateError("model not set");
        require(s && mu && out3 && n_x >= 0 && (X || n_x == 0), "bad arguments");
        // classify_point (reduction.cpp:27-31): t == 0 initial; x == 0 or 2pi periodic; else interior
        std::vector<double> interior, bnd, sinx;
        std::vector<double> per_t;
        for (int64_t k = 0; k < n_x; ++k) {
            const double x = X[2 * k], t = X[2 * k + 1];
            if (t == 0.0) {
                bnd.push_back(x);
                bnd.push_back(0.0);
                sinx.push_back(std::sin(x));  // host libm, as the reference's std::sin
            } else if (x == 0.0 || x == kTwoPi) {
                per_t.push_back(t);
            } else {
                interior.push_back(x);
                interior.push_back(t);
            }
        }
        const int64_t n_int = static_cast<int64_t>(interior.size() / 2), n_ic = static_cast<int64_t>(sinx.size()),
                      n_bc = static_cast<int64_t>(per_t.size());
        for (double t : per_t) {
            bnd.push_back(0.0);
            bnd.push_back(t);
            bnd.push_back(kTwoPi);
            bnd.push_back(t);
        }
        const int64_t nb = n_ic + 2 * n_bc;
        upload_coeffs_impl(ctx, s, mu, 1, m.rtotal);
        const size_t ws = static_cast<size_t>(2 * n_int + 2 * nb + n_ic + nb + 2) * sizeof(double) + 64;
        ctx->meta_ws.ensure(ws);
        double* d_int = ctx->meta_ws.as<double>();
        double* d_bnd = d_int + 2 * n_int;
        double* d_sinx = d_bnd + 2 * nb;
        double* d_u = d_sinx + n_ic;
        double* d_out2 = d_u + nb;
        if (n_int) CK(cudaMemcpyAsync(d_int, interior.data(), interior.size() * sizeof(double), cudaMemcpyHostToDevice,
                                      ctx->stream));
        if (nb) CK(cudaMemcpyAsync(d_bnd, bnd.data(), bnd.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (n_ic) CK(cudaMemcpyAsync(d_sinx, sinx.data(), sinx.size() * sizeof(double), cudaMemcpyHostToDevice,
                                     ctx->stream));
        double sums[3] = {0.0, 0.0, 0.0};  // sum |N|, sum |u - sin x|, sum |u(0,t) - u(2pi,t)|
        if (n_int > 0) {
            PointSwap keep(ctx, d_int, n_int);
            ctx->term_objective = 1;  // w |N|
            double* d = run_resident_stream<1>(ctx, m, 1.0, nullptr);
            download(ctx, d, sums, 1);
        }
        if (nb > 0) {
            boundary_sums(ctx, m, d_bnd, 1, n_ic, n_bc, d_sinx, 1, ctx->s_dev.as<double>(), d_u, d_out2);
            download(ctx, d_out2, sums + 1, 2);
        }
        comm_allreduce_host(ctx, sums, 3);
        finish_loss(ctx, m, sums[0], sums[1] + sums[2], out3);
    });
}

int lrnr_gpu_loss_meta(lrnr_gpu_ctx* ctx, const double* mus, double* out3) {
    return guarded(ctx, [&] {
        const Model& m = ctx->models[LRNR_MODEL_LRNR];
        if (!m.set) throw StateError("model not set");
        if (!ctx->hyper.set) throw StateError("hypernetwork not set");
        require(mus && out3, "null argument");
        const int64_t n = ctx->n_inst;
        const bool bnd = ctx->mb_inst > 0 && (ctx->mb_ic + ctx->mb_bc) > 0;
        require(!bnd || ctx->mb_inst == n, "meta boundary points were set for another instance count");
        const int64_t g_int = comm_global_count(ctx, ctx->pts ? n * ctx->n_per : 0);
        const int64_t g_ic = comm_global_count(ctx, bnd ? n * ctx->mb_ic : 0);
        const int64_t g_bc = comm_global_count(ctx, bnd ? n * ctx->mb_bc : 0);
        ctx->mu_dev.ensure(static_cast<size_t>(n * 3) * sizeof(double) + 8);
        CK(cudaMemcpyAsync(ctx->mu_dev.p, mus, static_cast<size_t>(n * 3) * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        ctx->coeff_inst = n;
        hyper_forward_resident(ctx, m.rtotal);  // s_i = hyper_forward(mu_i, theta), once per instance
        double sums[3] = {0.0, 0.0, 0.0};
        if (ctx->pts && ctx->n_per > 0) {
            double* d = run_resident_stream<1>(ctx, m, 1.0, nullptr);
            std::vector<double> h(static_cast<size_t>(n * (1 + m.rtotal)));
            download(ctx, d, h.data(), h.size());
            for (int64_t i = 0; i < n; ++i) sums[0] += h[static_cast<size_t>(i * (1 + m.rtotal))];
        }
        if (bnd) {
            const int64_t nb = ctx->mb_ic + 2 * ctx->mb_bc;
            ctx->bnd_jets.ensure(static_cast<size_t>(n * nb + 2) * sizeof(double));
            double* u = ctx->bnd_jets.as<double>();
            boundary_sums(ctx, m, ctx->mb_pts.as<double>(), n, ctx->mb_ic, ctx->mb_bc, ctx->mb_sinx.as<double>(), 0,
                          ctx->s_dev.as<double>(), u, u + n * nb);
            download(ctx, u + n * nb, sums + 1, 2);
        }
        comm_allreduce_host(ctx, sums, 3);
        auto mean = [](double v, int64_t c) { return c ? v / static_cast<double>(c) : 0.0; };
        finish_loss(ctx, m, mean(sums[0], g_int), mean(sums[1], g_ic) + mean(sums[2], g_bc), out3);
    });
}

}  // extern "C"
