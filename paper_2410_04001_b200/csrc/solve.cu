// The solve loops on the device (training.cpp:428-607):
// fine_tune (re-sampled batches, small-batch kernel, CUDA graph per epoch) and
// fast_solve (persistent cluster solver, pinn_solve.cuh, or the graph path);
// C ABI lrnr_gpu_fine_tune, lrnr_gpu_fast_solve.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

using namespace lrnr_b200;
using namespace lrnr_b200::detail;

namespace {

// ---------------------------------------------------------------------------
// solve loops on the device (training.cpp:428-607)
// ---------------------------------------------------------------------------
struct SolveState {  // same layout as solve::State (the persistent solver's)
    double best_loss;
    double initial;
    int64_t epoch, best_epoch, t;
    int stopped, flags;  // flags: 1 aborted (non-finite), 2 diverged
};

// The optimizer half of one epoch (one block): the EpochRecord loss, the stop
// rules (NonFiniteError -> abort; fast_solve: loss > 1e3 x the first loss),
// the best iterate, adam_step (autodiff.cpp:1062-1075) and
// project_nonnegative_coeffs (autodiff.cpp:967-977).  rows_int / rows_bnd are
// the [value, dL/ds] rows of the interior and boundary passes; the locality
// term lambda ||s - s0||_1 (fast_solve) is added here.  bt[2(t-1)], bt[2(t-1)+1]
// = 1 - beta1^t, 1 - beta2^t (host std::pow, as the reference).
__global__ void solve_step_kernel(const double* __restrict__ rows_int, const double* __restrict__ rows_bnd,
                                  const unsigned long long* __restrict__ bad, int G, double* __restrict__ s,
                                  const double* __restrict__ s0, double lambda_local, double* __restrict__ m,
                                  double* __restrict__ v, double* __restrict__ best_s, SolveState* st,
                                  const double* __restrict__ bt, double lr, int fast, double* __restrict__ losses,
                                  int64_t max_epochs) {
    __shared__ int go, copy;
    __shared__ int64_t tt;
    if (threadIdx.x == 0) {
        go = 0;
        copy = 0;
        if (!st->stopped && st->epoch < max_epochs) {
            const int64_t e = ++st->epoch;
            double local = 0.0;
            if (lambda_local > 0.0) {
                for (int i = 0; i < G; ++i) local += fabs(s[i] - s0[i]);
                local *= lambda_local;
            }
            const double value = rows_int[0] + rows_bnd[0] + local;
            if (*bad != ULLONG_MAX || !isfinite(value)) {
                st->flags |= fast ? 3 : 1;
                st->stopped = 1;
            } else {
                losses[e - 1] = value;
                if (fast && e == 1) st->initial = value;
                if (fast && value > 1e3 * st->initial) {
                    st->flags |= 2;
                    st->stopped = 1;
                } else {
                    if (value < st->best_loss) {
                        st->best_loss = value;
                        st->best_epoch = e;
                        copy = 1;
                    }
                    tt = ++st->t;
                    go = 1;
                }
            }
        }
    }
    __syncthreads();
    if (!go) return;
    const double b1t = bt[2 * (tt - 1)], b2t = bt[2 * (tt - 1) + 1];
    for (int i = threadIdx.x; i < G; i += blockDim.x) {
        const double si = s[i];
        if (copy) best_s[i] = si;
        double g = rows_int[1 + i] + rows_bnd[1 + i];
        if (lambda_local > 0.0) {
            const double d = si - s0[i];
            g += lambda_local * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0));
        }
        const double mi = 0.9 * m[i] + (1.0 - 0.9) * g;
        const double vi = 0.999 * v[i] + (1.0 - 0.999) * g * g;
        m[i] = mi;
        v[i] = vi;
        const double x = si - lr * (mi / b1t) / (sqrt(vi / b2t) + 1e-8);
        s[i] = x < 0.0 ? 0.0 : x;
    }
}

struct SolveRun {
    int objective;
    const double* int_pts;
    int64_t n_int;
    double w_int;
    const double* bnd_pts;
    const double* sinx;
    int64_t n_ic, n_bc;
    double w_ic, w_bc, lambda_local, lr;
    int fast;
    int64_t epochs;
};

// Enqueue one epoch (no host synchronization): term passes, then the step.
void solve_epoch(lrnr_gpu_ctx* ctx, const Model& m, const SolveRun& r) {
    const int R1 = 1 + m.rtotal;
    double* rows_int = ctx->solve_rows.as<double>();
    double* rows_bnd = rows_int + R1;
    double* sd = ctx->s_dev.as<double>();
    const double* md = ctx->mu_dev.as<double>();
    reset_bad(ctx, m);
    if (r.n_int > 0) {
        PointSwap keep(ctx, r.int_pts, r.n_int);
        if (r.objective == LRNR_OBJ_SQUARED) {
            if (use_small(ctx, m)) dispatch_small<0>(ctx, m, sd, md, r.w_int, rows_int, nullptr);
            else if (!dispatch_fast(ctx, m, sd, md, r.w_int, rows_int) && !dispatch_tc(ctx, m, sd, md, r.w_int, rows_int) &&
                     !dispatch_v2(ctx, m, sd, md, r.w_int, rows_int))
                dispatch_pinn<0>(ctx, m, sd, md, r.w_int, rows_int, nullptr);
        } else {
            ctx->term_objective = 1;
            dispatch_pinn<0>(ctx, m, sd, md, r.w_int, rows_int, nullptr);
        }
    }
    const int64_t nb = r.n_ic + 2 * r.n_bc;
    if (nb > 0) {
        PointSwap keep(ctx, r.bnd_pts, nb);
        dispatch_pinn<1>(ctx, m, sd, md, 1.0, rows_bnd, ctx->bnd_jets.as<double>());
        boundary_spec_kernel<<<static_cast<unsigned>((nb + 127) / 128), 128, 0, ctx->stream>>>(
            ctx->bnd_jets.as<double>(), r.sinx, r.n_ic, r.n_bc, r.w_ic, r.w_bc, r.objective == LRNR_OBJ_ABS,
            ctx->bnd_spec.as<TermSpec>());
        CK(cudaGetLastError());
        ++ctx->launches;
        ctx->term_spec = ctx->bnd_spec.as<TermSpec>();
        dispatch_pinn<0>(ctx, m, sd, md, 1.0, rows_bnd, nullptr);
    }
    solve_step_kernel<<<1, 256, 0, ctx->stream>>>(
        rows_int, rows_bnd, bad_word(ctx, m), m.rtotal, sd, ctx->solve_s0.as<double>(),
        r.lambda_local, ctx->solve_m.as<double>(), ctx->solve_v.as<double>(), ctx->solve_best.as<double>(),
        ctx->solve_state.as<SolveState>(), ctx->solve_bt.as<double>(), r.lr, r.fast,
        ctx->solve_losses.as<double>(), r.epochs);
    CK(cudaGetLastError());
    ++ctx->launches;
}

// Device state for a solve of `epochs` epochs from s_init; the boundary work
// buffers sized for nb points.
void solve_setup(lrnr_gpu_ctx* ctx, const Model& m, const double* s_init, const double* mu, int64_t epochs,
                 int64_t nb) {
    const int G = m.rtotal, R1 = 1 + G;
    upload_coeffs_impl(ctx, s_init, mu, 1, G);
    ctx->solve_rows.ensure(static_cast<size_t>(2 * R1) * sizeof(double));
    ctx->solve_state.ensure(sizeof(SolveState));
    for (DevBuf* b : {&ctx->solve_m, &ctx->solve_v, &ctx->solve_best, &ctx->solve_s0})
        b->ensure(static_cast<size_t>(G) * sizeof(double) + 8);
    ctx->solve_bt.ensure(static_cast<size_t>(2 * epochs) * sizeof(double));
    ctx->solve_losses.ensure(static_cast<size_t>(epochs) * sizeof(double));
    ctx->bnd_spec.ensure(static_cast<size_t>(nb) * sizeof(TermSpec) + 16);
    ctx->bnd_jets.ensure(static_cast<size_t>(4 * nb) * sizeof(double) + 16);
    bad_word(ctx, m);  // allocated before any graph capture
    std::vector<double> bt(static_cast<size_t>(2 * epochs));
    for (int64_t t = 1; t <= epochs; ++t) {
        bt[2 * (t - 1)] = 1.0 - std::pow(0.9, static_cast<double>(t));
        bt[2 * (t - 1) + 1] = 1.0 - std::pow(0.999, static_cast<double>(t));
    }
    SolveState st{};
    st.best_loss = std::numeric_limits<double>::infinity();
    st.initial = std::numeric_limits<double>::quiet_NaN();
    CK(cudaMemcpyAsync(ctx->solve_bt.p, bt.data(), bt.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->solve_state.p, &st, sizeof(st), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->solve_s0.p, s_init, static_cast<size_t>(G) * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(ctx->solve_best.p, s_init, static_cast<size_t>(G) * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemsetAsync(ctx->solve_m.p, 0, static_cast<size_t>(G) * sizeof(double), ctx->stream));
    CK(cudaMemsetAsync(ctx->solve_v.p, 0, static_cast<size_t>(G) * sizeof(double), ctx->stream));
    CK(cudaMemsetAsync(ctx->solve_rows.p, 0, static_cast<size_t>(2 * R1) * sizeof(double), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // host staging (bt, st) goes out of scope
}

void solve_results(lrnr_gpu_ctx* ctx, const Model& m, double* out_s, double* out_best_loss, int64_t* out_best_epoch,
                   double* out_losses, int64_t* out_n_records, int* out_flags) {
    SolveState st{};
    CK(cudaMemcpyAsync(&st, ctx->solve_state.p, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    // recorded epochs: all completed ones, minus the one that aborted / diverged
    const int64_t n_rec = st.epoch - ((st.flags & 1) ? 1 : 0);
    if (out_s) download(ctx, ctx->solve_best.as<double>(), out_s, static_cast<size_t>(m.rtotal));
    if (out_losses && n_rec > 0) download(ctx, ctx->solve_losses.as<double>(), out_losses, static_cast<size_t>(n_rec));
    if (out_best_loss) *out_best_loss = st.best_loss;
    if (out_best_epoch) *out_best_epoch = st.best_epoch;
    if (out_n_records) *out_n_records = n_rec;
    if (out_flags) *out_flags = st.flags;
}

static_assert(sizeof(SolveState) == sizeof(solve::State), "solve state layouts must match");

// Run the solve on a stream that can be captured (the legacy default stream cannot).
struct SolveStream {
    lrnr_gpu_ctx* ctx;
    cudaStream_t saved;
    explicit SolveStream(lrnr_gpu_ctx* c) : ctx(c), saved(c->stream) {
        CK(cudaStreamSynchronize(saved));
        c->stream = c->own;
    }
    ~SolveStream() {
        cudaStreamSynchronize(ctx->stream);
        ctx->stream = saved;
    }
};

// The persistent fast-phase solver (pinn_solve.cuh) when the FastLRNR and the
// term set fit one CTA; returns false (nothing launched) otherwise.
bool fast_solve_persistent(lrnr_gpu_ctx* ctx, const Model& m, const std::vector<double>& ip,
                           const std::vector<double>& ic, const std::vector<double>& per, const double* s_init,
                           const double* mu, double lambda_local, double lr, int64_t epochs) {
    if (ctx->opt_solve != 0) return false;
    const int n_int = static_cast<int>(ip.size() / 2), n_ic = static_cast<int>(ic.size()),
              n_bc = static_cast<int>(per.size());
    solve::Problem pb{};
    pb.n_int = n_int;
    pb.n_ic = n_ic;
    pb.n_bc = n_bc;
    pb.n_warps = n_int + n_ic + 2 * n_bc;
    // cluster layout: periodic pairs start at an even global warp, even warps per CTA (a pair
    // never straddles CTAs), SOLVE_WPC warps per CTA (more when the terms need > 8 CTAs, the
    // portable cluster size)
    pb.pair_base = (n_int + n_ic + 1) & ~1;
    pb.n_gw = pb.pair_base + 2 * n_bc;
#ifndef SOLVE_WPC
#define SOLVE_WPC 4  // measured on c2 (16 terms): 4 CTAs x 4 warps 15.9 us/epoch, 8 x 2 21.4, 1 x 16 24
#endif
    pb.wpc = SOLVE_WPC;
    while ((pb.n_gw + pb.wpc - 1) / pb.wpc > 8) pb.wpc += 2;
    const int n_cta = (pb.n_gw + pb.wpc - 1) / pb.wpc;
    if (pb.n_warps < 1 || pb.wpc > 16 || m.r[0] > 4 || m.rtotal > 1024) return false;
    for (int l = 0; l < m.L; ++l)
        if (m.r[l] > 32) return false;
    for (int l = 1; l < m.L; ++l)
        if (m.M[l] > 32) return false;
    int y = 0, a = 0, w = 0;
    for (int l = 0; l < m.L; ++l) {
        pb.yoff[l] = y;
        y += m.r[l];
    }
    for (int l = 0; l + 1 < m.L; ++l) {
        pb.aoff[l] = a;
        a += m.M[l + 1];
        pb.woff[l] = w;
        pb.wrow[l] = m.trow[l] | 1;
        w += m.M[l + 1] * pb.wrow[l];
    }
    pb.ylen = y;
    pb.alen = a;
    pb.wlen = (w + 3) & ~3;
    pb.lr = lr;
    pb.lambda_local = lambda_local;
    pb.epochs = epochs;
    const size_t elem = m.dtype == LRNR_F64 ? 8 : 4;
    const size_t smem = solve::smem_bytes(pb, m.rtotal, elem);
    if (smem > 220 * 1024) return false;
    // terms: interior (x, t) pairs, then initial x, then periodic t
    std::vector<double> terms(ip);
    terms.insert(terms.end(), ic.begin(), ic.end());
    terms.insert(terms.end(), per.begin(), per.end());
    const int G = m.rtotal;
    ctx->solve_pts[0].ensure(terms.size() * sizeof(double) + 16);
    ctx->solve_s0.ensure(static_cast<size_t>(G) * sizeof(double) + 8);
    ctx->solve_best.ensure(static_cast<size_t>(G) * sizeof(double) + 8);
    ctx->solve_bt.ensure(static_cast<size_t>(2 * epochs) * sizeof(double));
    ctx->solve_losses.ensure(static_cast<size_t>(epochs) * sizeof(double));
    ctx->solve_state.ensure(sizeof(solve::State));
    ctx->mu_dev.ensure(3 * sizeof(double) + 8);
    std::vector<double> bt(static_cast<size_t>(2 * epochs));
    for (int64_t t = 1; t <= epochs; ++t) {
        bt[2 * (t - 1)] = 1.0 - std::pow(0.9, static_cast<double>(t));
        bt[2 * (t - 1) + 1] = 1.0 - std::pow(0.999, static_cast<double>(t));
    }
    CK(cudaMemcpyAsync(ctx->solve_pts[0].p, terms.data(), terms.size() * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(ctx->solve_s0.p, s_init, static_cast<size_t>(G) * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(ctx->solve_bt.p, bt.data(), bt.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->mu_dev.p, mu, 3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    // one cluster of n_cta CTAs (cudaLaunchKernelEx with a cluster-dimension attribute)
    auto launch = [&](auto kern, auto net) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(n_cta));
        cfg.blockDim = dim3(static_cast<unsigned>(32 * pb.wpc));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(n_cta);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, kern, net, pb, static_cast<const double*>(ctx->solve_pts[0].as<double>()),
                              static_cast<const double*>(ctx->mu_dev.as<double>()),
                              static_cast<const double*>(ctx->solve_s0.as<double>()),
                              static_cast<const double*>(ctx->solve_bt.as<double>()), ctx->solve_best.as<double>(),
                              ctx->solve_losses.as<double>(), ctx->solve_state.as<solve::State>()));
    };
    if (m.dtype == LRNR_F64) {
        if (m.act == LRNR_ACT_TANH) launch(solve::fast_solve_kernel<double, 0>, dev_net<double>(m));
        else launch(solve::fast_solve_kernel<double, 1>, dev_net<double>(m));
    } else {
        if (m.act == LRNR_ACT_TANH) launch(solve::fast_solve_kernel<float, 0>, dev_net<float>(m));
        else launch(solve::fast_solve_kernel<float, 1>, dev_net<float>(m));
    }
    CK(cudaGetLastError());
    ++ctx->launches;
    return true;
}


}  // namespace

extern "C" {

int lrnr_gpu_fast_solve(lrnr_gpu_ctx* ctx, const double* s_init, const double* mu, const double* X, int64_t n_x,
                        double lambda_local, double lr, int64_t epochs, double* out_s, double* out_best_loss,
                        int64_t* out_best_epoch, double* out_losses, int64_t* out_n_records, int* out_flags) {
    return guarded(ctx, [&] {
        const Model& m = ctx->models[LRNR_MODEL_FAST];
        if (!m.set) throw StateError("FastLRNR not set");
        require(s_init && mu && (X || n_x == 0), "null argument");
        require(epochs >= 0 && n_x >= 0 && lambda_local >= 0.0, "bad solve arguments");
        if (out_n_records) *out_n_records = 0;
        if (epochs == 0) {
            if (out_s) std::copy(s_init, s_init + m.rtotal, out_s);
            if (out_best_loss) *out_best_loss = std::numeric_limits<double>::infinity();
            if (out_best_epoch) *out_best_epoch = 0;
            if (out_flags) *out_flags = 0;
            return;
        }
        // classify_point (reduction.cpp:27-31)
        std::vector<double> ip, bp, sx;
        std::vector<double> ic, per;
        for (int64_t i = 0; i < n_x; ++i) {
            const double x = X[2 * i], t = X[2 * i + 1];
            if (t == 0.0) ic.push_back(x);
            else if (x == 0.0 || x == kTwoPi) per.push_back(t);
            else {
                ip.push_back(x);
                ip.push_back(t);
            }
        }
        for (double x : ic) {
            bp.push_back(x);
            bp.push_back(0.0);
            sx.push_back(std::sin(x));
        }
        for (double t : per) {
            bp.insert(bp.end(), {0.0, t, kTwoPi, t});
        }
        const int64_t n_int = static_cast<int64_t>(ip.size() / 2), n_ic = static_cast<int64_t>(ic.size()),
                      n_bc = static_cast<int64_t>(per.size());
        SolveStream ss(ctx);
        if (fast_solve_persistent(ctx, m, ip, ic, per, s_init, mu, lambda_local, lr, epochs)) {
            solve_results(ctx, m, out_s, out_best_loss, out_best_epoch, out_losses, out_n_records, out_flags);
            return;
        }
        const PointSwap restore(ctx, ctx->pts, ctx->n_per);  // keep the caller's point set
        ctx->n_inst = restore.n_inst;
        solve_setup(ctx, m, s_init, mu, epochs, n_ic + 2 * n_bc);
        ctx->solve_pts[0].ensure(ip.size() * sizeof(double) + 16);
        ctx->solve_bnd[0].ensure(bp.size() * sizeof(double) + 16);
        ctx->solve_sinx[0].ensure(sx.size() * sizeof(double) + 16);
        if (!ip.empty()) CK(cudaMemcpyAsync(ctx->solve_pts[0].p, ip.data(), ip.size() * sizeof(double),
                                            cudaMemcpyHostToDevice, ctx->stream));
        if (!bp.empty()) CK(cudaMemcpyAsync(ctx->solve_bnd[0].p, bp.data(), bp.size() * sizeof(double),
                                            cudaMemcpyHostToDevice, ctx->stream));
        if (!sx.empty()) CK(cudaMemcpyAsync(ctx->solve_sinx[0].p, sx.data(), sx.size() * sizeof(double),
                                            cudaMemcpyHostToDevice, ctx->stream));
        SolveRun r{LRNR_OBJ_ABS, ctx->solve_pts[0].as<double>(), n_int, 1.0, ctx->solve_bnd[0].as<double>(),
                   ctx->solve_sinx[0].as<double>(), n_ic, n_bc, 1.0, 1.0, lambda_local, lr, 1, epochs};
        // epoch 1 eagerly (sizes every workspace), then one epoch captured as a graph
        ctx->coeff_inst = 1;
        solve_epoch(ctx, m, r);
        if (epochs > 1) {
            const int64_t l0 = ctx->launches;
            cudaGraph_t graph = nullptr;
            cudaGraphExec_t exec = nullptr;
            CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
            try {
                solve_epoch(ctx, m, r);
            } catch (...) {
                cudaStreamEndCapture(ctx->stream, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            CK(cudaStreamEndCapture(ctx->stream, &graph));
            CK(cudaGraphInstantiate(&exec, graph, 0));
            const int64_t per_epoch = ctx->launches - l0;
            for (int64_t e = 2; e <= epochs; ++e) CK(cudaGraphLaunch(exec, ctx->stream));
            ctx->launches += per_epoch * (epochs - 2);  // the capture counted one epoch
            CK(cudaStreamSynchronize(ctx->stream));
            cudaGraphExecDestroy(exec);
            cudaGraphDestroy(graph);
        }
        solve_results(ctx, m, out_s, out_best_loss, out_best_epoch, out_losses, out_n_records, out_flags);
    });
}

int lrnr_gpu_fine_tune(lrnr_gpu_ctx* ctx, const double* s_init, const double* mu, double lr, int64_t epochs,
                       int64_t n_int, int64_t n_ic, int64_t n_bc, uint64_t seed, double* out_s, double* out_best_loss,
                       int64_t* out_best_epoch, double* out_losses, int64_t* out_n_records, int* out_flags) {
    return guarded(ctx, [&] {
        const Model& m = ctx->models[LRNR_MODEL_LRNR];
        if (!m.set) throw StateError("LRNR not set");
        require(s_init && mu, "null argument");
        require(epochs >= 0 && n_int >= 0 && n_ic >= 0 && n_bc >= 0, "bad solve arguments");
        if (out_n_records) *out_n_records = 0;
        if (epochs == 0) {
            if (out_s) std::copy(s_init, s_init + m.rtotal, out_s);
            if (out_best_loss) *out_best_loss = std::numeric_limits<double>::infinity();
            if (out_best_epoch) *out_best_epoch = 0;
            if (out_flags) *out_flags = 0;
            return;
        }
        const int64_t nb = n_ic + 2 * n_bc;
        SolveStream ss(ctx);
        const PointSwap restore(ctx, ctx->pts, ctx->n_per);
        ctx->n_inst = restore.n_inst;
        solve_setup(ctx, m, s_init, mu, epochs, nb);
        // double-buffered pinned staging: the host draws epoch e+1's batch while
        // the device runs epoch e (fine_tune re-samples every epoch, training.cpp:443-446)
        const size_t b_pts = static_cast<size_t>(2 * n_int) * sizeof(double) + 16,
                     b_bnd = static_cast<size_t>(2 * nb) * sizeof(double) + 16,
                     b_sx = static_cast<size_t>(n_ic) * sizeof(double) + 16;
        struct Pinned {
            void* p = nullptr;
            ~Pinned() {
                if (p) cudaFreeHost(p);
            }
        } host[2];
        cudaEvent_t ev[2] = {nullptr, nullptr};
        struct EvGuard {
            cudaEvent_t* e;
            ~EvGuard() {
                for (int i = 0; i < 2; ++i)
                    if (e[i]) cudaEventDestroy(e[i]);
            }
        } evg{ev};
        for (int k = 0; k < 2; ++k) {
            CK(cudaMallocHost(&host[k].p, b_pts + b_bnd + b_sx));
            CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
            ctx->solve_pts[k].ensure(b_pts);
            ctx->solve_bnd[k].ensure(b_bnd);
            ctx->solve_sinx[k].ensure(b_sx);
        }
        std::vector<double> icx(static_cast<size_t>(n_ic)), pt(static_cast<size_t>(n_bc));
        ctx->coeff_inst = 1;
        for (int64_t e = 1; e <= epochs; ++e) {
            const int k = static_cast<int>(e & 1);
            if (e > 2) CK(cudaEventSynchronize(ev[k]));  // slot k's previous upload has been consumed
            double* hp = static_cast<double*>(host[k].p);
            double* hb = reinterpret_cast<double*>(static_cast<char*>(host[k].p) + b_pts);
            double* hs = reinterpret_cast<double*>(static_cast<char*>(host[k].p) + b_pts + b_bnd);
            if (lrnr_host_sample_batch(lrnr_host_epoch_seed(seed, e), n_int, n_ic, n_bc, hp, icx.data(), pt.data()) !=
                LRNR_OK)
                throw InvalidArg("batch sampling failed");
            for (int64_t i = 0; i < n_ic; ++i) {
                hb[2 * i] = icx[i];
                hb[2 * i + 1] = 0.0;
                hs[i] = std::sin(icx[i]);
            }
            for (int64_t j = 0; j < n_bc; ++j) {
                double* q = hb + 2 * (n_ic + 2 * j);
                q[0] = 0.0;
                q[1] = pt[j];
                q[2] = kTwoPi;
                q[3] = pt[j];
            }
            if (n_int) CK(cudaMemcpyAsync(ctx->solve_pts[k].p, hp, static_cast<size_t>(2 * n_int) * sizeof(double),
                                          cudaMemcpyHostToDevice, ctx->stream));
            if (nb) CK(cudaMemcpyAsync(ctx->solve_bnd[k].p, hb, static_cast<size_t>(2 * nb) * sizeof(double),
                                       cudaMemcpyHostToDevice, ctx->stream));
            if (n_ic) CK(cudaMemcpyAsync(ctx->solve_sinx[k].p, hs, static_cast<size_t>(n_ic) * sizeof(double),
                                         cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaEventRecord(ev[k], ctx->stream));
            const double wi = n_int ? 1.0 / static_cast<double>(n_int) : 0.0,
                         wc = n_ic ? 1.0 / static_cast<double>(n_ic) : 0.0,
                         wb = n_bc ? 1.0 / static_cast<double>(n_bc) : 0.0;  // safe_inv, training.cpp:446-450
            SolveRun r{LRNR_OBJ_SQUARED, ctx->solve_pts[k].as<double>(), n_int, wi, ctx->solve_bnd[k].as<double>(),
                       ctx->solve_sinx[k].as<double>(), n_ic, n_bc, wc, wb, 0.0, lr, 0, epochs};
            solve_epoch(ctx, m, r);
        }
        solve_results(ctx, m, out_s, out_best_loss, out_best_epoch, out_losses, out_n_records, out_flags);
    });
}

}  // extern "C"
