// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI harness over the UNMODIFIED reference implementation
// (/root/reference/proj, compiled in place by oracle/Makefile into
// oracle/_ref/liblrnr_ref.so).  Every entry point here drives the reference's
// own public API -- make_lrnr_params, sample_collocation,
// training::run_batch_gradient with an emitter built from emit_lrnr_jet /
// emit_fast_jet / emit_hyper, harvest_snapshots / eim_greedy /
// build_fastparams, training::meta_train -- so the Python tests can (a) pin
// the C restatement in oracle/lrnr_oracle.c against the reference itself and
// (b) time the reference CPU path on the GPU box's host cores
// (bench.py --impl reference).
//
// Flat layouts (shared with oracle/lrnr_oracle.c and include/lrnr_gpu.h):
//   LRNR params: per layer l: U_l (widths[l+1] x ranks[l], row-major),
//                V_l (widths[l] x ranks[l]), b_l (widths[l+1]).
//                This is ParamPacker(BasesBiasesAndHyper) order
//                (reference autodiff.cpp:926-934).
//   Hyper params: per layer k: W_k (hw[k+1] x hw[k]), b_k (hw[k+1])
//                (autodiff.cpp:935-939).
//   Fast params:  v_in (m_in x r_0); per inner l: u_hat (rh_l x r_l),
//                b_hat (rh_l), v_hat (rh_l x r_{l+1}); u_out (m_out x r_{L-1}),
//                b_out (m_out)   (model.hpp:65-78).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
#include <vector>

#include "lrnr/autodiff.hpp"
#include "lrnr/model.hpp"
#include "lrnr/pde.hpp"
#include "lrnr/reduction.hpp"
#include "lrnr/rng.hpp"
#include "lrnr/training.hpp"

using namespace lrnr;

namespace {

thread_local int g_last_tag = -1;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const NonFiniteError& e) {
        g_last_tag = e.layer_tag;
        return 2;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

std::vector<std::size_t> to_sizes(const int64_t* p, int n) {
    std::vector<std::size_t> v(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) v[static_cast<std::size_t>(i)] = static_cast<std::size_t>(p[i]);
    return v;
}

LrnrParams unpack_lrnr(int L, const int64_t* widths, const int64_t* ranks, const double* flat) {
    LrnrParams p;
    p.widths = to_sizes(widths, L + 1);
    p.ranks = to_sizes(ranks, L);
    std::size_t o = 0;
    for (int l = 0; l < L; ++l) {
        DenseMatrix u(p.widths[l + 1], p.ranks[l]);
        for (double& v : u.data) v = flat[o++];
        DenseMatrix vv(p.widths[l], p.ranks[l]);
        for (double& v : vv.data) v = flat[o++];
        DenseVector b(p.widths[l + 1]);
        for (double& v : b.data) v = flat[o++];
        p.u.push_back(std::move(u));
        p.v.push_back(std::move(vv));
        p.b.push_back(std::move(b));
    }
    p.validate();
    return p;
}

void pack_lrnr(const LrnrParams& p, double* flat) {
    std::size_t o = 0;
    for (std::size_t l = 0; l < p.depth(); ++l) {
        for (double v : p.u[l].data) flat[o++] = v;
        for (double v : p.v[l].data) flat[o++] = v;
        for (double v : p.b[l].data) flat[o++] = v;
    }
}

Coefficients unpack_s(const LrnrParams& p, const double* s) {
    Coefficients c;
    std::size_t o = 0;
    for (std::size_t l = 0; l < p.depth(); ++l) {
        DenseVector v(p.ranks[l]);
        for (double& x : v.data) x = s[o++];
        c.s.push_back(std::move(v));
    }
    return c;
}

Coefficients unpack_s_ranks(const std::vector<std::size_t>& ranks, const double* s) {
    Coefficients c;
    std::size_t o = 0;
    for (std::size_t r : ranks) {
        DenseVector v(r);
        for (double& x : v.data) x = s[o++];
        c.s.push_back(std::move(v));
    }
    return c;
}

HyperParams unpack_hyper(int K, const int64_t* hw, const double* flat, int L, const int64_t* split,
                         const double* lo, const double* hi) {
    HyperParams h;
    std::size_t o = 0;
    for (int k = 0; k < K; ++k) {
        DenseMatrix w(static_cast<std::size_t>(hw[k + 1]), static_cast<std::size_t>(hw[k]));
        for (double& v : w.data) v = flat[o++];
        DenseVector b(static_cast<std::size_t>(hw[k + 1]));
        for (double& v : b.data) v = flat[o++];
        h.w.push_back(std::move(w));
        h.b.push_back(std::move(b));
    }
    h.split = to_sizes(split, L);
    for (int a = 0; a < 3; ++a) {
        h.box.lo[a] = lo[a];
        h.box.hi[a] = hi[a];
    }
    h.validate();
    return h;
}

FastParams unpack_fast(int L, const int64_t* ranks, const int64_t* red, int64_t m_in, int64_t m_out,
                       const double* flat) {
    FastParams f;
    f.ranks = to_sizes(ranks, L);
    f.red_ranks = to_sizes(red, L - 1);
    std::size_t o = 0;
    f.v_in = DenseMatrix(static_cast<std::size_t>(m_in), f.ranks[0]);
    for (double& v : f.v_in.data) v = flat[o++];
    for (int l = 0; l + 1 < L; ++l) {
        DenseMatrix uh(f.red_ranks[l], f.ranks[l]);
        for (double& v : uh.data) v = flat[o++];
        DenseVector bh(f.red_ranks[l]);
        for (double& v : bh.data) v = flat[o++];
        DenseMatrix vh(f.red_ranks[l], f.ranks[l + 1]);
        for (double& v : vh.data) v = flat[o++];
        f.u_hat.push_back(std::move(uh));
        f.b_hat.push_back(std::move(bh));
        f.v_hat.push_back(std::move(vh));
    }
    f.u_out = DenseMatrix(static_cast<std::size_t>(m_out), f.ranks[L - 1]);
    for (double& v : f.u_out.data) v = flat[o++];
    f.b_out = DenseVector(static_cast<std::size_t>(m_out));
    for (double& v : f.b_out.data) v = flat[o++];
    f.validate();
    return f;
}

PdeParams mu_of(const double* m) { return PdeParams{m[0], m[1], m[2]}; }

training::ParallelConfig par_of(int threads, int chunk) {
    training::ParallelConfig par;
    par.threads = static_cast<std::size_t>(std::max(1, threads));
    par.chunk = static_cast<std::size_t>(std::max(1, chunk));
    return par;
}

void copy_result(const training::BatchGradResult& bg, double* value, double* comps, double* grad) {
    if (value) *value = bg.value;
    if (comps)
        for (int k = 0; k < 4; ++k) comps[k] = bg.comps[k];
    if (grad) std::copy(bg.grad.begin(), bg.grad.end(), grad);
}

}  // namespace

extern "C" {

int ref_last_tag() { return g_last_tag; }

// ---- seeded construction (reference model.cpp:454-515, rng.hpp) ----

int ref_rng_stream(uint64_t seed, int64_t n, int kind, double* out, uint64_t* out_raw) {
    return guarded([&] {
        Rng rng(seed);
        for (int64_t i = 0; i < n; ++i) {
            if (kind == 0) out[i] = rng.uniform();
            else if (kind == 1) out[i] = rng.normal();
            else out_raw[i] = rng.raw();
        }
    });
}

int ref_make_lrnr_params(int L, const int64_t* widths, const int64_t* ranks, uint64_t seed,
                         int orthonormal, double bias_scale, double* out_params) {
    return guarded([&] {
        Rng rng(seed);
        LrnrParams p = make_lrnr_params(to_sizes(widths, L + 1), to_sizes(ranks, L), rng,
                                        orthonormal != 0, bias_scale);
        pack_lrnr(p, out_params);
    });
}

// BASELINE.json config recipe: reference init with
// bias_scale 0, then b <- 0.1 * normal() from the same stream, then
// s <- make_coefficients(U[0,1]) from the same stream, sorted descending.
int ref_make_baseline_model(int L, const int64_t* widths, const int64_t* ranks, uint64_t seed,
                            double* out_params, double* out_s) {
    return guarded([&] {
        Rng rng(seed);
        LrnrParams p = make_lrnr_params(to_sizes(widths, L + 1), to_sizes(ranks, L), rng, true, 0.0);
        for (auto& b : p.b)
            for (double& v : b.data) v = 0.1 * rng.normal();
        Coefficients s = make_coefficients(p.ranks, rng, 0.0, 1.0);
        for (auto& sl : s.s) std::sort(sl.data.begin(), sl.data.end(), std::greater<double>());
        pack_lrnr(p, out_params);
        std::size_t o = 0;
        for (auto& sl : s.s)
            for (double v : sl.data) out_s[o++] = v;
    });
}

int ref_make_hyper_params(int L, const int64_t* split, int hidden_depth, int hidden_width,
                          const double* lo, const double* hi, uint64_t seed, double out_w_scale,
                          double out_bias, double* out_params) {
    return guarded([&] {
        Rng rng(seed);
        ParamDomain box;
        for (int a = 0; a < 3; ++a) {
            box.lo[a] = lo[a];
            box.hi[a] = hi[a];
        }
        HyperParams h = make_hyper_params(to_sizes(split, L), static_cast<std::size_t>(hidden_depth),
                                          static_cast<std::size_t>(hidden_width), box, rng,
                                          out_w_scale, out_bias);
        std::size_t o = 0;
        for (std::size_t k = 0; k < h.w.size(); ++k) {
            for (double v : h.w[k].data) out_params[o++] = v;
            for (double v : h.b[k].data) out_params[o++] = v;
        }
    });
}

int ref_sample_collocation(uint64_t seed, int64_t n_int, int64_t n_ic, int64_t n_per,
                           const double* lo, const double* hi, int with_mu, double* out_int,
                           double* out_ic, double* out_per, double* out_int_mu, double* out_ic_mu,
                           double* out_per_mu) {
    return guarded([&] {
        ParamDomain box;
        for (int a = 0; a < 3; ++a) {
            box.lo[a] = lo[a];
            box.hi[a] = hi[a];
        }
        pde::CollocationBatch b = pde::sample_collocation(
            seed, static_cast<std::size_t>(n_int), static_cast<std::size_t>(n_ic),
            static_cast<std::size_t>(n_per), box, with_mu != 0);
        for (std::size_t i = 0; i < b.interior.size(); ++i) {
            out_int[2 * i] = b.interior[i].x;
            out_int[2 * i + 1] = b.interior[i].t;
        }
        for (std::size_t i = 0; i < b.initial_x.size(); ++i) out_ic[i] = b.initial_x[i];
        for (std::size_t i = 0; i < b.periodic_t.size(); ++i) out_per[i] = b.periodic_t[i];
        if (with_mu) {
            auto put = [](const std::vector<PdeParams>& v, double* o) {
                for (std::size_t i = 0; i < v.size(); ++i) {
                    o[3 * i] = v[i].mu1;
                    o[3 * i + 1] = v[i].mu2;
                    o[3 * i + 2] = v[i].mu3;
                }
            };
            put(b.interior_mu, out_int_mu);
            put(b.initial_mu, out_ic_mu);
            put(b.periodic_mu, out_per_mu);
        }
    });
}

// ---- forward-only (model.cpp:357-405, pde.cpp:9-13, training.cpp:139-163) ----

int ref_lrnr_jets(int L, const int64_t* widths, const int64_t* ranks, const double* params,
                  const double* s, const double* pts, int64_t n, double* out_jets) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        Coefficients c = unpack_s(p, s);
        for (int64_t i = 0; i < n; ++i) {
            Jet j = jet_forward(pts[2 * i], pts[2 * i + 1], p, c);
            out_jets[4 * i] = j.value[0];
            out_jets[4 * i + 1] = j.dx[0];
            out_jets[4 * i + 2] = j.dt[0];
            out_jets[4 * i + 3] = j.dxx[0];
        }
    });
}

int ref_fast_jets(int L, const int64_t* ranks, const int64_t* red, int64_t m_in, int64_t m_out,
                  const double* fparams, const double* s, const double* pts, int64_t n,
                  double* out_jets) {
    return guarded([&] {
        FastParams f = unpack_fast(L, ranks, red, m_in, m_out, fparams);
        Coefficients c = unpack_s_ranks(f.ranks, s);
        for (int64_t i = 0; i < n; ++i) {
            Jet j = jet_forward(pts[2 * i], pts[2 * i + 1], f, c);
            out_jets[4 * i] = j.value[0];
            out_jets[4 * i + 1] = j.dx[0];
            out_jets[4 * i + 2] = j.dt[0];
            out_jets[4 * i + 3] = j.dxx[0];
        }
    });
}

int ref_loss_tune(int L, const int64_t* widths, const int64_t* ranks, const double* params,
                  const double* s, const double* mu, const double* pts, int64_t n,
                  const double* ic_x, int64_t n_ic, const double* per_t, int64_t n_per,
                  double* out3) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        Coefficients c = unpack_s(p, s);
        pde::CollocationBatch b;
        for (int64_t i = 0; i < n; ++i) b.interior.push_back({pts[2 * i], pts[2 * i + 1]});
        for (int64_t i = 0; i < n_ic; ++i) b.initial_x.push_back(ic_x[i]);
        for (int64_t i = 0; i < n_per; ++i) b.periodic_t.push_back(per_t[i]);
        training::LossBreakdown lb = training::loss_tune(c, mu_of(mu), p, b);
        out3[0] = lb.total;
        out3[1] = lb.residual;
        out3[2] = lb.boundary;
    });
}

// ---- batched residual + gradient through run_batch_gradient (training.cpp:191-263) ----

// Interior-only PinnTermEmitter equivalent (training.cpp:286-305, fine-tune
// mode): term_i = w * N(x_i,t_i)^2, CoefficientsOnly.
int ref_lrnr_grad(int L, const int64_t* widths, const int64_t* ranks, const double* params,
                  const double* s, const double* mu, const double* pts, int64_t n, double w,
                  int threads, int chunk, double* out_value, double* out_comps, double* out_grad) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        Coefficients c = unpack_s(p, s);
        const PdeParams m = mu_of(mu);
        Trainables at{&p, nullptr, &c};
        training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings&,
                                    std::size_t i, double* comps) -> NodeId {
            Tape& tp = ctx.tape;
            const NodeId jet = emit_lrnr_jet(tp, pts[2 * i], pts[2 * i + 1], ctx.lrnr,
                                             ctx.coeffs.s_leaves);
            const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, m)), w);
            comps[0] += tp.value(term);
            return term;
        };
        training::BatchGradResult bg = training::run_batch_gradient(
            at, ParamSelector::CoefficientsOnly, nullptr, emit, static_cast<std::size_t>(n),
            par_of(threads, chunk));
        copy_result(bg, out_value, out_comps, out_grad);
    });
}

// The full fine-tune PinnTermEmitter term set (training.cpp:286-327, fine-tune
// mode, lambda_sparse = 0): interior w_int N^2, initial w_ic (u(x,0) - sin x)^2,
// periodic w_bc (u(0,t) - u(2pi,t))^2, in the emitter's index order; built with
// the reference's own tape ops (the emitter struct itself is file-local).
int ref_tune_grad_full(int L, const int64_t* widths, const int64_t* ranks, const double* params,
                       const double* s, const double* mu, const double* pts, int64_t n,
                       const double* ic_x, int64_t n_ic, const double* per_t, int64_t n_bc, double w_int,
                       double w_ic, double w_bc, int threads, int chunk, double* out_value,
                       double* out_comps, double* out_grad) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        Coefficients c = unpack_s(p, s);
        const PdeParams m = mu_of(mu);
        Trainables at{&p, nullptr, &c};
        training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings&,
                                    std::size_t idx, double* comps) -> NodeId {
            Tape& tp = ctx.tape;
            const std::size_t ni = static_cast<std::size_t>(n), nc = static_cast<std::size_t>(n_ic);
            if (idx < ni) {
                const NodeId jet = emit_lrnr_jet(tp, pts[2 * idx], pts[2 * idx + 1], ctx.lrnr,
                                                 ctx.coeffs.s_leaves);
                const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, m)), w_int);
                comps[0] += tp.value(term);
                return term;
            }
            if (idx < ni + nc) {
                const double x = ic_x[idx - ni];
                const NodeId jet = emit_lrnr_jet(tp, x, 0.0, ctx.lrnr, ctx.coeffs.s_leaves);
                const NodeId r = tp.sub_const(tp.pick_value(jet, 0), std::sin(x));
                const NodeId term = tp.scale(tp.square(r), w_ic);
                comps[1] += tp.value(term);
                return term;
            }
            const double t = per_t[idx - ni - nc];
            const NodeId j0 = emit_lrnr_jet(tp, 0.0, t, ctx.lrnr, ctx.coeffs.s_leaves);
            const NodeId j1 = emit_lrnr_jet(tp, pde::kTwoPi, t, ctx.lrnr, ctx.coeffs.s_leaves);
            const NodeId r = tp.sub(tp.pick_value(j0, 0), tp.pick_value(j1, 0));
            const NodeId term = tp.scale(tp.square(r), w_bc);
            comps[1] += tp.value(term);
            return term;
        };
        training::BatchGradResult bg = training::run_batch_gradient(
            at, ParamSelector::CoefficientsOnly, nullptr, emit, static_cast<std::size_t>(n + n_ic + n_bc),
            par_of(threads, chunk));
        copy_result(bg, out_value, out_comps, out_grad);
    });
}

// FastLRNR interior MSE through bind_fast + emit_fast_jet (training.cpp:513-531
// emitter structure with the BASELINE c1 squared-residual objective).
int ref_fast_grad(int L, const int64_t* ranks, const int64_t* red, int64_t m_in, int64_t m_out,
                  const double* fparams, const double* s, const double* mu, const double* pts,
                  int64_t n, double w, int threads, int chunk, double* out_value,
                  double* out_comps, double* out_grad) {
    return guarded([&] {
        FastParams f = unpack_fast(L, ranks, red, m_in, m_out, fparams);
        Coefficients c = unpack_s_ranks(f.ranks, s);
        const PdeParams m = mu_of(mu);
        Trainables at{nullptr, nullptr, &c};
        training::SetupFn setup = [&](TapeBindings& ctx) {
            training::ExtraBindings ex;
            ex.fast = bind_fast(ctx.tape, f);
            ex.has_fast = true;
            return ex;
        };
        training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings& ex,
                                    std::size_t i, double* comps) -> NodeId {
            Tape& tp = ctx.tape;
            const NodeId jet =
                emit_fast_jet(tp, pts[2 * i], pts[2 * i + 1], ex.fast, ctx.coeffs.s_leaves);
            const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, m)), w);
            comps[0] += tp.value(term);
            return term;
        };
        training::BatchGradResult bg = training::run_batch_gradient(
            at, ParamSelector::CoefficientsOnly, setup, emit, static_cast<std::size_t>(n),
            par_of(threads, chunk));
        copy_result(bg, out_value, out_comps, out_grad);
    });
}

// The reference fast-phase objective (training.cpp:521-563): l1 residuals at
// the classified points of X plus lambda_local * ||s - s_init||_1.
int ref_fast_phase_grad(int L, const int64_t* ranks, const int64_t* red, int64_t m_in,
                        int64_t m_out, const double* fparams, const double* s,
                        const double* s_init, const double* mu, const double* xpts, int64_t n,
                        double lambda_local, int threads, int chunk, double* out_value,
                        double* out_comps, double* out_grad) {
    return guarded([&] {
        FastParams f = unpack_fast(L, ranks, red, m_in, m_out, fparams);
        Coefficients c = unpack_s_ranks(f.ranks, s);
        Coefficients c0 = unpack_s_ranks(f.ranks, s_init);
        const PdeParams m = mu_of(mu);
        Trainables at{nullptr, nullptr, &c};
        training::SetupFn setup = [&](TapeBindings& ctx) {
            training::ExtraBindings ex;
            ex.fast = bind_fast(ctx.tape, f);
            ex.has_fast = true;
            return ex;
        };
        training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings& ex,
                                    std::size_t idx, double* comps) -> NodeId {
            Tape& tp = ctx.tape;
            if (idx < static_cast<std::size_t>(n)) {
                const pde::Point pt{xpts[2 * idx], xpts[2 * idx + 1]};
                switch (reduction::classify_point(pt)) {
                    case reduction::PointKind::Interior: {
                        const NodeId jet = emit_fast_jet(tp, pt.x, pt.t, ex.fast, ctx.coeffs.s_leaves);
                        const NodeId term = tp.abs_val(tp.residual_cdr(jet, m));
                        comps[0] += tp.value(term);
                        return term;
                    }
                    case reduction::PointKind::Initial: {
                        const NodeId jet = emit_fast_jet(tp, pt.x, 0.0, ex.fast, ctx.coeffs.s_leaves);
                        const NodeId term =
                            tp.abs_val(tp.sub_const(tp.pick_value(jet, 0), std::sin(pt.x)));
                        comps[1] += tp.value(term);
                        return term;
                    }
                    default: {
                        const NodeId j0 = emit_fast_jet(tp, 0.0, pt.t, ex.fast, ctx.coeffs.s_leaves);
                        const NodeId j1 =
                            emit_fast_jet(tp, pde::kTwoPi, pt.t, ex.fast, ctx.coeffs.s_leaves);
                        const NodeId term =
                            tp.abs_val(tp.sub(tp.pick_value(j0, 0), tp.pick_value(j1, 0)));
                        comps[1] += tp.value(term);
                        return term;
                    }
                }
            }
            std::vector<NodeId> ids;
            std::vector<double> ws;
            for (std::size_t l = 0; l < ctx.coeffs.s_leaves.size(); ++l) {
                ids.push_back(tp.l1_to_target(ctx.coeffs.s_leaves[l], c0.s[l].data.data(),
                                              c0.s[l].len()));
                ws.push_back(lambda_local);
            }
            const NodeId term = tp.weighted_sum(ids, ws);
            comps[3] += tp.value(term);
            return term;
        };
        training::BatchGradResult bg = training::run_batch_gradient(
            at, ParamSelector::CoefficientsOnly, setup, emit,
            static_cast<std::size_t>(n) + (lambda_local > 0.0 ? 1 : 0), par_of(threads, chunk));
        copy_result(bg, out_value, out_comps, out_grad);
    });
}

int ref_hyper_forward(int K, const int64_t* hw, const double* hparams, int L, const int64_t* split,
                      const double* lo, const double* hi, const double* mu, double* out_s) {
    return guarded([&] {
        HyperParams h = unpack_hyper(K, hw, hparams, L, split, lo, hi);
        Coefficients c = hyper_forward(mu_of(mu), h);
        std::size_t o = 0;
        for (auto& sl : c.s)
            for (double v : sl.data) out_s[o++] = v;
    });
}

// J^T g for the hypernetwork at mu: gradient of sum_l dot(s_l(theta), g_l)
// through emit_hyper (autodiff.cpp:883-903) -- the c3 coupling recipe.
int ref_hyper_vjp(int K, const int64_t* hw, const double* hparams, int L, const int64_t* split,
                  const double* lo, const double* hi, const double* mu, const double* g_s,
                  double* out_grad) {
    return guarded([&] {
        HyperParams h = unpack_hyper(K, hw, hparams, L, split, lo, hi);
        Trainables at{nullptr, &h, nullptr};
        GradResult g = grad(
            [&](TapeBindings& ctx) {
                std::vector<NodeId> sl = emit_hyper(ctx.tape, mu_of(mu), ctx.hyper);
                std::vector<NodeId> ids;
                std::vector<double> ws;
                std::size_t o = 0;
                for (std::size_t l = 0; l < sl.size(); ++l) {
                    ids.push_back(ctx.tape.dot_const(sl[l], g_s + o, h.split[l]));
                    ws.push_back(1.0);
                    o += h.split[l];
                }
                return ctx.tape.weighted_sum(ids, ws);
            },
            at, ParamSelector::BasesBiasesAndHyper);
        std::copy(g.grad.begin(), g.grad.end(), out_grad);
    });
}

// Meta-phase interior objective (PinnTermEmitter meta_mode, training.cpp:283-293,
// lambda_sparse = 0): per point, emit_hyper(mu_i) -> emit_lrnr_jet -> w N^2,
// gradient in ParamPacker(BasesBiasesAndHyper) order.
int ref_meta_grad(int L, const int64_t* widths, const int64_t* ranks, const double* params, int K,
                  const int64_t* hw, const double* hparams, const double* lo, const double* hi,
                  const double* pts, const double* mus, int64_t n, double w, int threads, int chunk,
                  double* out_value, double* out_grad) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        HyperParams h = unpack_hyper(K, hw, hparams, L, ranks, lo, hi);
        Trainables at{&p, &h, nullptr};
        training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings&,
                                    std::size_t i, double* comps) -> NodeId {
            Tape& tp = ctx.tape;
            const PdeParams m = mu_of(mus + 3 * i);
            const std::vector<NodeId> s_nodes = emit_hyper(tp, m, ctx.hyper);
            const NodeId jet = emit_lrnr_jet(tp, pts[2 * i], pts[2 * i + 1], ctx.lrnr, s_nodes);
            const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, m)), w);
            comps[0] += tp.value(term);
            return term;
        };
        training::BatchGradResult bg = training::run_batch_gradient(
            at, ParamSelector::BasesBiasesAndHyper, nullptr, emit, static_cast<std::size_t>(n),
            par_of(threads, chunk));
        copy_result(bg, out_value, nullptr, out_grad);
    });
}

// Meta step with meta_train's regularizers (training.cpp:283-305, 368-389):
// interior terms w N^2 through the hypernetwork plus, per interior term,
// lambda_sparse * w * sum_l banded_decay(s_l(mu), gamma) (the emitter's
// weighted_sum), and lambda_ortho * sum_l (gram(U_l) + gram(V_l)) from grad().
// out_comps = BatchGradResult comps; out_ortho = ro.value; out_grad = bg + ro.
int ref_meta_grad_reg(int L, const int64_t* widths, const int64_t* ranks, const double* params, int K,
                      const int64_t* hw, const double* hparams, const double* lo, const double* hi,
                      const double* pts, const double* mus, int64_t n, double w, double lambda_sparse,
                      double gamma, double lambda_ortho, int threads, int chunk, double* out_value,
                      double* out_comps, double* out_ortho, double* out_grad) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        HyperParams h = unpack_hyper(K, hw, hparams, L, ranks, lo, hi);
        Trainables at{&p, &h, nullptr};
        training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings&,
                                    std::size_t i, double* comps) -> NodeId {
            Tape& tp = ctx.tape;
            const PdeParams m = mu_of(mus + 3 * i);
            const std::vector<NodeId> s_nodes = emit_hyper(tp, m, ctx.hyper);
            const NodeId jet = emit_lrnr_jet(tp, pts[2 * i], pts[2 * i + 1], ctx.lrnr, s_nodes);
            const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, m)), w);
            comps[0] += tp.value(term);
            if (lambda_sparse > 0.0) {
                std::vector<NodeId> ids{term};
                std::vector<double> ws{1.0};
                for (const NodeId sn : s_nodes) {
                    ids.push_back(tp.banded_decay_penalty(sn, gamma));
                    ws.push_back(lambda_sparse * w);
                }
                const NodeId tot = tp.weighted_sum(ids, ws);
                comps[2] += tp.value(tot) - tp.value(term);
                return tot;
            }
            return term;
        };
        training::BatchGradResult bg = training::run_batch_gradient(
            at, ParamSelector::BasesBiasesAndHyper, nullptr, emit, static_cast<std::size_t>(n),
            par_of(threads, chunk));
        GradResult ro = grad(
            [&](TapeBindings& ctx) {
                std::vector<NodeId> ids;
                std::vector<double> ws;
                for (std::size_t l = 0; l < ctx.at.lrnr->depth(); ++l) {
                    ids.push_back(ctx.tape.gram_ortho_penalty(ctx.lrnr.u_slots[l]));
                    ws.push_back(lambda_ortho);
                    ids.push_back(ctx.tape.gram_ortho_penalty(ctx.lrnr.v_slots[l]));
                    ws.push_back(lambda_ortho);
                }
                return ctx.tape.weighted_sum(ids, ws);
            },
            at, ParamSelector::BasesBiasesAndHyper);
        *out_value = bg.value + ro.value;
        for (int k = 0; k < 4; ++k) out_comps[k] = bg.comps[k];
        *out_ortho = ro.value;
        for (std::size_t i = 0; i < bg.grad.size(); ++i) out_grad[i] = bg.grad[i] + ro.grad[i];
    });
}

// ---- the reference's own solve loops (training.cpp:428-607) ----
// A constant hypernetwork (W = 0, b = s_init) makes hyper_forward(mu) == s_init
// (s_init >= 0: the output ReLU passes it unchanged).
static HyperParams constant_hyper(const std::vector<std::size_t>& ranks, const double* s_init) {
    HyperParams h;
    std::size_t r_total = 0;
    for (auto r : ranks) r_total += r;
    h.w.emplace_back(r_total, 3);
    DenseVector b(r_total);
    for (std::size_t i = 0; i < r_total; ++i) b[i] = s_init[i];
    h.b.push_back(std::move(b));
    h.split = ranks;
    h.box = ParamDomain::d1();
    return h;
}

static void copy_solve(const training::SolveResult& r, double* out_s, double* out_best_loss, int64_t* out_best_epoch,
                       double* out_losses, int64_t* out_n_records, int* out_flags) {
    std::size_t o = 0;
    for (const auto& v : r.coeffs.s)
        for (double x : v.data) out_s[o++] = x;
    *out_best_loss = r.report.best_loss;
    *out_best_epoch = static_cast<int64_t>(r.report.best_epoch);
    *out_n_records = static_cast<int64_t>(r.report.records.size());
    for (std::size_t e = 0; e < r.report.records.size(); ++e) out_losses[e] = r.report.records[e].loss;
    *out_flags = (r.report.aborted_nonfinite ? 1 : 0) | (r.report.diverged ? 2 : 0);
}

int ref_fine_tune(int L, const int64_t* widths, const int64_t* ranks, const double* params, const double* s_init,
                  const double* mu, double lr, int64_t epochs, int64_t n_int, int64_t n_ic, int64_t n_bc,
                  uint64_t seed, int threads, double* out_s, double* out_best_loss, int64_t* out_best_epoch,
                  double* out_losses, int64_t* out_n_records, int* out_flags) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        HyperParams h = constant_hyper(p.ranks, s_init);
        training::PhaseConfig cfg;
        cfg.lr = lr;
        cfg.epochs = static_cast<std::size_t>(epochs);
        cfg.n_interior = static_cast<std::size_t>(n_int);
        cfg.n_initial = static_cast<std::size_t>(n_ic);
        cfg.n_periodic = static_cast<std::size_t>(n_bc);
        cfg.seed = seed;
        cfg.eval_interval = 0;
        training::SolveResult r = training::fine_tune(mu_of(mu), p, h, cfg, par_of(threads, 64), nullptr);
        copy_solve(r, out_s, out_best_loss, out_best_epoch, out_losses, out_n_records, out_flags);
    });
}

int ref_fast_solve(int L, const int64_t* ranks, const int64_t* red, int64_t m_in, int64_t m_out,
                   const double* fparams, const double* s_init, const double* mu, const double* xpts, int64_t n_x,
                   double lambda_local, double lr, int64_t epochs, int threads, double* out_s,
                   double* out_best_loss, int64_t* out_best_epoch, double* out_losses, int64_t* out_n_records,
                   int* out_flags) {
    return guarded([&] {
        FastParams f = unpack_fast(L, ranks, red, m_in, m_out, fparams);
        HyperParams h = constant_hyper(f.ranks, s_init);
        reduction::SamplingSetX X;
        for (int64_t i = 0; i < n_x; ++i) X.points.push_back({xpts[2 * i], xpts[2 * i + 1]});
        training::PhaseConfig cfg;
        cfg.lr = lr;
        cfg.epochs = static_cast<std::size_t>(epochs);
        training::SolveResult r = training::fast_solve(mu_of(mu), h, f, X, cfg, lambda_local, par_of(threads, 64));
        copy_solve(r, out_s, out_best_loss, out_best_epoch, out_losses, out_n_records, out_flags);
    });
}

// pde::l1_relative_error (pde.cpp:166-178) of lrnr_forward (model.cpp:255-270)
// against a GridField ((n_t + 1) x n_x values).
int ref_l1_error(int L, const int64_t* widths, const int64_t* ranks, const double* params, const double* s,
                 const double* values, int64_t n_x, int64_t n_t, double* out) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        Coefficients c = unpack_s(p, s);
        pde::GridField g;
        g.n_x = static_cast<std::size_t>(n_x);
        g.n_t = static_cast<std::size_t>(n_t);
        g.values.assign(values, values + n_x * (n_t + 1));
        *out = pde::l1_relative_error([&](double x, double t) { return lrnr_forward(x, t, p, c)[0]; }, g);
    });
}

// meta_train's full PinnTermEmitter (meta mode, training.cpp:283-327): interior terms
// (+ lambda_sparse banded decay), initial and periodic terms, each point with its
// own mu through the hypernetwork, weights 1/n per kind; plus the ortho grad().
int ref_meta_grad_full(int L, const int64_t* widths, const int64_t* ranks, const double* params, int K,
                       const int64_t* hw, const double* hparams, const double* lo, const double* hi,
                       const double* pts, const double* mus, int64_t n, const double* ic_x, const double* ic_mu,
                       int64_t n_ic, const double* per_t, const double* per_mu, int64_t n_bc, double lambda_sparse,
                       double gamma, double lambda_ortho, int threads, int chunk, double* out_value,
                       double* out_comps, double* out_ortho, double* out_grad) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        HyperParams h = unpack_hyper(K, hw, hparams, L, ranks, lo, hi);
        Trainables at{&p, &h, nullptr};
        const double wi = n ? 1.0 / static_cast<double>(n) : 0.0;
        const double wc = n_ic ? 1.0 / static_cast<double>(n_ic) : 0.0;
        const double wb = n_bc ? 1.0 / static_cast<double>(n_bc) : 0.0;
        training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings&, std::size_t idx,
                                    double* comps) -> NodeId {
            Tape& tp = ctx.tape;
            const std::size_t ni = static_cast<std::size_t>(n), nc = static_cast<std::size_t>(n_ic);
            if (idx < ni) {
                const PdeParams m = mu_of(mus + 3 * idx);
                const std::vector<NodeId> s_nodes = emit_hyper(tp, m, ctx.hyper);
                const NodeId jet = emit_lrnr_jet(tp, pts[2 * idx], pts[2 * idx + 1], ctx.lrnr, s_nodes);
                const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, m)), wi);
                comps[0] += tp.value(term);
                if (lambda_sparse > 0.0) {
                    std::vector<NodeId> ids{term};
                    std::vector<double> ws{1.0};
                    for (const NodeId sn : s_nodes) {
                        ids.push_back(tp.banded_decay_penalty(sn, gamma));
                        ws.push_back(lambda_sparse * wi);
                    }
                    const NodeId tot = tp.weighted_sum(ids, ws);
                    comps[2] += tp.value(tot) - tp.value(term);
                    return tot;
                }
                return term;
            }
            if (idx < ni + nc) {
                const std::size_t j = idx - ni;
                const std::vector<NodeId> s_nodes = emit_hyper(tp, mu_of(ic_mu + 3 * j), ctx.hyper);
                const double x = ic_x[j];
                const NodeId jet = emit_lrnr_jet(tp, x, 0.0, ctx.lrnr, s_nodes);
                const NodeId term = tp.scale(tp.square(tp.sub_const(tp.pick_value(jet, 0), std::sin(x))), wc);
                comps[1] += tp.value(term);
                return term;
            }
            const std::size_t j = idx - ni - nc;
            const std::vector<NodeId> s_nodes = emit_hyper(tp, mu_of(per_mu + 3 * j), ctx.hyper);
            const double t = per_t[j];
            const NodeId j0 = emit_lrnr_jet(tp, 0.0, t, ctx.lrnr, s_nodes);
            const NodeId j1 = emit_lrnr_jet(tp, pde::kTwoPi, t, ctx.lrnr, s_nodes);
            const NodeId term = tp.scale(tp.square(tp.sub(tp.pick_value(j0, 0), tp.pick_value(j1, 0))), wb);
            comps[1] += tp.value(term);
            return term;
        };
        training::BatchGradResult bg = training::run_batch_gradient(
            at, ParamSelector::BasesBiasesAndHyper, nullptr, emit, static_cast<std::size_t>(n + n_ic + n_bc),
            par_of(threads, chunk));
        GradResult ro = grad(
            [&](TapeBindings& ctx) {
                std::vector<NodeId> ids;
                std::vector<double> ws;
                for (std::size_t l = 0; l < ctx.at.lrnr->depth(); ++l) {
                    ids.push_back(ctx.tape.gram_ortho_penalty(ctx.lrnr.u_slots[l]));
                    ws.push_back(lambda_ortho);
                    ids.push_back(ctx.tape.gram_ortho_penalty(ctx.lrnr.v_slots[l]));
                    ws.push_back(lambda_ortho);
                }
                return ctx.tape.weighted_sum(ids, ws);
            },
            at, ParamSelector::BasesBiasesAndHyper);
        *out_value = bg.value + ro.value;
        for (int k = 0; k < 4; ++k) out_comps[k] = bg.comps[k];
        *out_ortho = ro.value;
        for (std::size_t i = 0; i < bg.grad.size(); ++i) out_grad[i] = bg.grad[i] + ro.grad[i];
    });
}

// The reference's own step-time benchmark (training.cpp:613-799): per width, the
// median fine-tune step and fast step seconds (BenchmarkConfig defaults unless given).
int ref_benchmark_step_time(const int64_t* widths, int64_t n_widths, int64_t reps, int64_t warmup, int threads,
                            double* out_tune_s, double* out_fast_s) {
    return guarded([&] {
        training::BenchmarkConfig cfg;
        cfg.reps = static_cast<std::size_t>(reps);
        cfg.warmup = static_cast<std::size_t>(warmup);
        cfg.par = par_of(threads, 64);
        std::vector<std::size_t> w;
        for (int64_t i = 0; i < n_widths; ++i) w.push_back(static_cast<std::size_t>(widths[i]));
        const auto rows = training::benchmark_step_time(w, cfg);
        for (std::size_t i = 0; i < rows.size(); ++i) {
            out_tune_s[i] = rows[i].t_lrnr_s;
            out_fast_s[i] = rows[i].t_fast_s;
        }
    });
}

// ---- FastLRNR construction (reduction.cpp:10-31,111-283) ----
// Constant hypernetwork (zero W, bias = s) so hyper_forward(mu) == s.
static void build_fast_from(const LrnrParams& p, const HyperParams& h, const std::vector<PdeParams>& grid,
                            int64_t nx, int64_t nt, int64_t n_perturb, double sigma, uint64_t seed, int64_t r_hat,
                            int64_t* out_red, int64_t* out_indices, double* out_fparams, int* out_exhausted) {
    reduction::SamplingSetX X = reduction::SamplingSetX::uniform_grid(
        static_cast<std::size_t>(nx), static_cast<std::size_t>(nt));
    reduction::SnapshotSet snaps = reduction::harvest_snapshots(
        p, h, X, static_cast<std::size_t>(n_perturb), sigma, grid, seed);
    std::vector<reduction::EimBasis> bases;
    for (std::size_t l = 0; l + 1 < p.depth(); ++l) {
        bases.push_back(reduction::eim_greedy(snaps.layers[l], static_cast<std::size_t>(r_hat)));
        out_exhausted[l] = bases.back().exhausted ? 1 : 0;
        out_red[l] = static_cast<int64_t>(bases.back().dim());
        for (std::size_t k = 0; k < bases.back().indices.size(); ++k)
            out_indices[l * r_hat + static_cast<int64_t>(k)] = static_cast<int64_t>(bases.back().indices[k]);
    }
    FastParams f = reduction::build_fastparams(p, bases);
    std::size_t o = 0;
    for (double v : f.v_in.data) out_fparams[o++] = v;
    for (std::size_t l = 0; l + 1 < p.depth(); ++l) {
        for (double v : f.u_hat[l].data) out_fparams[o++] = v;
        for (double v : f.b_hat[l].data) out_fparams[o++] = v;
        for (double v : f.v_hat[l].data) out_fparams[o++] = v;
    }
    for (double v : f.u_out.data) out_fparams[o++] = v;
    for (double v : f.b_out.data) out_fparams[o++] = v;
}

int ref_build_fast(int L, const int64_t* widths, const int64_t* ranks, const double* params,
                   const double* s, int64_t nx, int64_t nt, int64_t n_perturb, double sigma,
                   uint64_t seed, int64_t r_hat, const double* mu, int64_t* out_red,
                   int64_t* out_indices, double* out_fparams, int* out_exhausted) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        HyperParams h;  // constant hypernetwork: hyper_forward(mu) == s
        std::size_t r_total = 0;
        for (auto r : p.ranks) r_total += r;
        h.w.emplace_back(r_total, 3);
        DenseVector b(r_total);
        for (std::size_t i = 0; i < r_total; ++i) b[i] = s[i];
        h.b.push_back(std::move(b));
        h.split = p.ranks;
        h.box = ParamDomain::d1();
        build_fast_from(p, h, {mu_of(mu)}, nx, nt, n_perturb, sigma, seed, r_hat, out_red, out_indices, out_fparams,
                        out_exhausted);
    });
}

// The reduction recipe through a real hypernetwork over a mu grid (harvest_snapshots with
// mu_grid, reduction.cpp:111-148; cli build_reduction).
int ref_build_fast_hyper(int L, const int64_t* widths, const int64_t* ranks, const double* params, int K,
                         const int64_t* hw, const double* hparams, const double* lo, const double* hi,
                         const double* mus, int64_t n_mu, int64_t nx, int64_t nt, int64_t n_perturb, double sigma,
                         uint64_t seed, int64_t r_hat, int64_t* out_red, int64_t* out_indices, double* out_fparams,
                         int* out_exhausted) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        HyperParams h = unpack_hyper(K, hw, hparams, L, ranks, lo, hi);
        std::vector<PdeParams> grid;
        for (int64_t i = 0; i < n_mu; ++i) grid.push_back(mu_of(mus + 3 * i));
        build_fast_from(p, h, grid, nx, nt, n_perturb, sigma, seed, r_hat, out_red, out_indices, out_fparams,
                        out_exhausted);
    });
}

// reduction::eim_greedy (reduction.cpp:150-238) on a given M x n_cols row-major
// snapshot matrix: the pin for lrnr_host_eim_greedy / lrnr_gpu_eim_greedy.
int ref_eim_greedy(int64_t m, int64_t n_cols, const double* snaps, int64_t r_hat, int64_t* out_idx,
                   double* out_xi, int64_t* out_count, int* out_exhausted) {
    return guarded([&] {
        DenseMatrix S(static_cast<std::size_t>(m), static_cast<std::size_t>(n_cols));
        for (std::size_t i = 0; i < S.data.size(); ++i) S.data[i] = snaps[i];
        const reduction::EimBasis e = reduction::eim_greedy(S, static_cast<std::size_t>(r_hat));
        const int64_t k = static_cast<int64_t>(e.dim());
        for (int64_t q = 0; q < r_hat; ++q)
            out_idx[q] = q < k ? static_cast<int64_t>(e.indices[static_cast<std::size_t>(q)]) : -1;
        for (int64_t i = 0; i < m; ++i)
            for (int64_t q = 0; q < r_hat; ++q)
                out_xi[i * r_hat + q] =
                    q < k ? e.xi.at(static_cast<std::size_t>(i), static_cast<std::size_t>(q)) : 0.0;
        *out_count = k;
        *out_exhausted = e.exhausted ? 1 : 0;
    });
}

// Identity reduction (reduction.cpp:285-296) -> FastParams.
int ref_identity_fast(int L, const int64_t* widths, const int64_t* ranks, const double* params,
                      double* out_fparams) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        FastParams f = reduction::build_fastparams(p, reduction::identity_bases(p));
        std::size_t o = 0;
        for (double v : f.v_in.data) out_fparams[o++] = v;
        for (std::size_t l = 0; l + 1 < p.depth(); ++l) {
            for (double v : f.u_hat[l].data) out_fparams[o++] = v;
            for (double v : f.b_hat[l].data) out_fparams[o++] = v;
            for (double v : f.v_hat[l].data) out_fparams[o++] = v;
        }
        for (double v : f.u_out.data) out_fparams[o++] = v;
        for (double v : f.b_out.data) out_fparams[o++] = v;
    });
}

// ---- end-to-end meta-training KAT (training.cpp:335-426) ----
int ref_meta_train(int L, const int64_t* widths, const int64_t* ranks, int hyper_depth,
                   int hyper_width, double init_bias_scale, double out_w_scale, double out_bias,
                   uint64_t init_seed, const double* lo, const double* hi, double lr,
                   int64_t epochs, int64_t n_int, int64_t n_ic, int64_t n_per, uint64_t seed,
                   double lambda_ortho, double lambda_sparse, double gamma, int threads, int chunk,
                   double* out_best_loss, int64_t* out_best_epoch, double* out_losses) {
    return guarded([&] {
        training::MetaSetup st;
        st.widths = to_sizes(widths, L + 1);
        st.ranks = to_sizes(ranks, L);
        st.hyper_depth = static_cast<std::size_t>(hyper_depth);
        st.hyper_width = static_cast<std::size_t>(hyper_width);
        st.init_bias_scale = init_bias_scale;
        st.hyper_out_weight_scale = out_w_scale;
        st.hyper_out_bias = out_bias;
        st.init_seed = init_seed;
        for (int a = 0; a < 3; ++a) {
            st.domain.lo[a] = lo[a];
            st.domain.hi[a] = hi[a];
        }
        st.regs.lambda_ortho = lambda_ortho;
        st.regs.lambda_sparse = lambda_sparse;
        st.regs.gamma = gamma;
        st.phase = training::PhaseConfig{lr,
                                         static_cast<std::size_t>(epochs),
                                         static_cast<std::size_t>(n_int),
                                         static_cast<std::size_t>(n_ic),
                                         static_cast<std::size_t>(n_per),
                                         seed,
                                         0};
        st.par = par_of(threads, chunk);
        training::MetaResult r = training::meta_train(st);
        *out_best_loss = r.report.best_loss;
        *out_best_epoch = static_cast<int64_t>(r.report.best_epoch);
        for (std::size_t i = 0; i < r.report.records.size(); ++i) out_losses[i] = r.report.records[i].loss;
    });
}

// ---- plain losses and values (training.cpp:109-189, model.cpp:260-292) ----

// lrnr_forward (model = 0) / fast_forward (model = 1): u at n points.
int ref_values(int model, int L, const int64_t* widths, const int64_t* ranks, const double* params,
               const int64_t* red, const double* fparams, const double* s, const double* pts, int64_t n,
               double* out_u) {
    return guarded([&] {
        if (model == 0) {
            LrnrParams p = unpack_lrnr(L, widths, ranks, params);
            Coefficients c = unpack_s(p, s);
            for (int64_t i = 0; i < n; ++i) out_u[i] = lrnr_forward(pts[2 * i], pts[2 * i + 1], p, c)[0];
        } else {
            FastParams f = unpack_fast(L, ranks, red, 2, 1, fparams);
            Coefficients c = unpack_s_ranks(f.ranks, s);
            for (int64_t i = 0; i < n; ++i) out_u[i] = fast_forward(pts[2 * i], pts[2 * i + 1], f, c)[0];
        }
    });
}

// training::loss_fast over the sampling set X (n_x points).
int ref_loss_fast(int L, const int64_t* ranks, const int64_t* red, const double* fparams, const double* s,
                  const double* mu, const double* X, int64_t n_x, double* out3) {
    return guarded([&] {
        FastParams f = unpack_fast(L, ranks, red, 2, 1, fparams);
        Coefficients c = unpack_s_ranks(f.ranks, s);
        reduction::SamplingSetX sx;
        for (int64_t i = 0; i < n_x; ++i) sx.points.push_back({X[2 * i], X[2 * i + 1]});
        training::LossBreakdown lb = training::loss_fast(c, mu_of(mu), f, sx);
        out3[0] = lb.total;
        out3[1] = lb.residual;
        out3[2] = lb.boundary;
    });
}

// training::loss_meta: interior points with per-point mu, initial x / periodic t with per-point mu.
int ref_loss_meta(int L, const int64_t* widths, const int64_t* ranks, const double* params, int K,
                  const int64_t* hw, const double* hparams, const double* lo, const double* hi,
                  const double* pts, const double* mus, int64_t n, const double* ic_x, const double* ic_mu,
                  int64_t n_ic, const double* per_t, const double* per_mu, int64_t n_per, double* out3) {
    return guarded([&] {
        LrnrParams p = unpack_lrnr(L, widths, ranks, params);
        HyperParams h = unpack_hyper(K, hw, hparams, L, ranks, lo, hi);
        pde::CollocationBatch b;
        for (int64_t i = 0; i < n; ++i) {
            b.interior.push_back({pts[2 * i], pts[2 * i + 1]});
            b.interior_mu.push_back(mu_of(mus + 3 * i));
        }
        for (int64_t i = 0; i < n_ic; ++i) {
            b.initial_x.push_back(ic_x[i]);
            b.initial_mu.push_back(mu_of(ic_mu + 3 * i));
        }
        for (int64_t i = 0; i < n_per; ++i) {
            b.periodic_t.push_back(per_t[i]);
            b.periodic_mu.push_back(mu_of(per_mu + 3 * i));
        }
        training::LossBreakdown lb = training::loss_meta(p, h, b);
        out3[0] = lb.total;
        out3[1] = lb.residual;
        out3[2] = lb.boundary;
    });
}

}  // extern "C"
