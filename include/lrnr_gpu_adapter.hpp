// lrnr_gpu_adapter.hpp -- header-only C++ drop-in over the C ABI (lrnr_gpu.h)
// for code written against the reference's own headers (/root/reference/proj/include).
//
// A reference maintainer adds this header next to proj/include/lrnr and links
// liblrnr_gpu.so; the training loops then swap the CPU gradient engine for the
// B200 path at the call sites listed in INTEGRATION.md:
//
//   reference (training.cpp:458-461, fine_tune)        B200
//   ------------------------------------------------  ------------------------------------------
//   PinnTermEmitter emitter{...};                      lrnr::gpu::Engine eng(0);
//   bg = run_batch_gradient(at, CoefficientsOnly,      eng.bind(params);      // once (Tape bind_lrnr)
//          nullptr, std::cref(emitter), n_terms, par); bg = eng.tune_gradient(coeffs, mu, batch);
//
// Every entry returns the reference's own types (training::BatchGradResult,
// training::LossBreakdown, Jet) and throws the reference's exceptions
// (NonFiniteError{layer_tag}, std::invalid_argument), so callers that catch
// NonFiniteError (training.cpp:392,462,572) behave identically.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lrnr/autodiff.hpp"
#include "lrnr/model.hpp"
#include "lrnr/pde.hpp"
#include "lrnr/reduction.hpp"
#include "lrnr/training.hpp"
#include "lrnr_gpu.h"

namespace lrnr {
namespace gpu {

class Engine {
public:
    explicit Engine(int device = 0) {
        if (lrnr_gpu_create(device, &ctx_) != LRNR_OK) throw std::runtime_error("lrnr_gpu_create failed");
    }
    ~Engine() { lrnr_gpu_destroy(ctx_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // ---- Tape bindings (bind_lrnr / bind_fast / bind_hyper, autodiff.cpp:826-868) ----
    void bind(const LrnrParams& p, int dtype = LRNR_F64, int act = LRNR_ACT_TANH) {
        std::vector<double> flat;
        for (std::size_t l = 0; l < p.depth(); ++l) {
            flat.insert(flat.end(), p.u[l].data.begin(), p.u[l].data.end());
            flat.insert(flat.end(), p.v[l].data.begin(), p.v[l].data.end());
            flat.insert(flat.end(), p.b[l].data.begin(), p.b[l].data.end());
        }
        const std::vector<int64_t> w(p.widths.begin(), p.widths.end()), r(p.ranks.begin(), p.ranks.end());
        check(lrnr_gpu_set_lrnr(ctx_, static_cast<int>(p.depth()), w.data(), r.data(), flat.data(), act, dtype));
        lrnr_depth_ = p.depth();
        lrnr_params_ = flat.size();
    }
    void bind(const FastParams& f, int dtype = LRNR_F64, int act = LRNR_ACT_TANH) {
        std::vector<double> flat(f.v_in.data.begin(), f.v_in.data.end());
        for (std::size_t l = 0; l + 1 < f.depth(); ++l) {
            flat.insert(flat.end(), f.u_hat[l].data.begin(), f.u_hat[l].data.end());
            flat.insert(flat.end(), f.b_hat[l].data.begin(), f.b_hat[l].data.end());
            flat.insert(flat.end(), f.v_hat[l].data.begin(), f.v_hat[l].data.end());
        }
        flat.insert(flat.end(), f.u_out.data.begin(), f.u_out.data.end());
        flat.insert(flat.end(), f.b_out.data.begin(), f.b_out.data.end());
        const std::vector<int64_t> r(f.ranks.begin(), f.ranks.end()), h(f.red_ranks.begin(), f.red_ranks.end());
        check(lrnr_gpu_set_fast(ctx_, static_cast<int>(f.depth()), r.data(), h.data(),
                                static_cast<int64_t>(f.v_in.rows), static_cast<int64_t>(f.u_out.rows), flat.data(),
                                act, dtype));
    }
    void bind(const HyperParams& h) {
        std::vector<double> flat;
        std::vector<int64_t> hw{static_cast<int64_t>(h.w.front().cols)};
        for (std::size_t k = 0; k < h.w.size(); ++k) {
            flat.insert(flat.end(), h.w[k].data.begin(), h.w[k].data.end());
            flat.insert(flat.end(), h.b[k].data.begin(), h.b[k].data.end());
            hw.push_back(static_cast<int64_t>(h.w[k].rows));
        }
        const double lo[3] = {h.box.lo[0], h.box.lo[1], h.box.lo[2]};
        const double hi[3] = {h.box.hi[0], h.box.hi[1], h.box.hi[2]};
        check(lrnr_gpu_set_hyper(ctx_, static_cast<int>(h.w.size()), hw.data(), flat.data(), lo, hi));
        hyper_params_ = flat.size();
    }

    // ---- PinnTermEmitter, fine-tune mode (training.cpp:286-327) +
    //      run_batch_gradient(CoefficientsOnly) (training.cpp:191-263): interior
    //      w N^2, initial w (u(x,0) - sin x)^2 and periodic w (u(0,t) - u(2pi,t))^2
    //      terms with the fine_tune weights 1/n per kind (training.cpp:446-450).
    training::BatchGradResult tune_gradient(const Coefficients& s, const PdeParams& mu,
                                            const pde::CollocationBatch& batch) {
        set_points(batch.interior, 1);
        set_boundary(batch.initial_x, batch.periodic_t);
        return terms(LRNR_MODEL_LRNR, s, mu, LRNR_OBJ_SQUARED, 0.0, nullptr, 0.0);
    }
    // FastLRNR squared-residual objective over interior points (emit_fast_jet,
    // autodiff.cpp:905-922; BASELINE config 1).
    training::BatchGradResult fast_gradient(const Coefficients& s, const PdeParams& mu,
                                            const std::vector<pde::Point>& pts) {
        return coeff_gradient(LRNR_MODEL_FAST, s, mu, pts);
    }
    // The fast-phase emitter of fast_solve (training.cpp:521-559): |N| at the
    // interior points of X, |u - sin x| at initial points, |u(0,t) - u(2pi,t)| at
    // periodic points (classify_point, reduction.cpp:27-31), plus
    // lambda_local * sum_l ||s_l - s_init_l||_1 when lambda_local > 0.
    training::BatchGradResult fast_phase_gradient(const Coefficients& s, const Coefficients& s_init,
                                                  const PdeParams& mu, const reduction::SamplingSetX& X,
                                                  double lambda_local) {
        std::vector<pde::Point> interior;
        std::vector<double> ic, per;
        for (const pde::Point& p : X.points) {
            switch (reduction::classify_point(p)) {
                case reduction::PointKind::Interior: interior.push_back(p); break;
                case reduction::PointKind::Initial: ic.push_back(p.x); break;
                default: per.push_back(p.t); break;
            }
        }
        set_points(interior, 1);
        set_boundary(ic, per);
        const std::vector<double> s0 = flatten(s_init);
        return terms(LRNR_MODEL_FAST, s, mu, LRNR_OBJ_ABS, 1.0, lambda_local > 0.0 ? s0.data() : nullptr,
                     lambda_local);
    }
    // Meta mode interior terms (training.cpp:283-293, lambda_sparse = 0):
    // pts grouped by instance (mus.size() groups of equal size); ParamPacker
    // (BasesBiasesAndHyper) order.
    training::BatchGradResult meta_gradient(const std::vector<PdeParams>& mus, const std::vector<pde::Point>& pts) {
        const std::size_t n_inst = mus.size();
        if (n_inst == 0 || pts.size() % n_inst) throw std::invalid_argument("meta_gradient: points not grouped by mu");
        set_points(pts, n_inst);
        std::vector<double> m(3 * n_inst);
        for (std::size_t i = 0; i < n_inst; ++i) {
            m[3 * i] = mus[i].mu1;
            m[3 * i + 1] = mus[i].mu2;
            m[3 * i + 2] = mus[i].mu3;
        }
        training::BatchGradResult out;
        out.grad.assign(lrnr_params_ + hyper_params_, 0.0);
        check(lrnr_gpu_meta_loss_grad(ctx_, m.data(), 0.0, &out.value, out.grad.data()));
        out.comps[0] = out.value;
        return out;
    }

    // meta_train's initial / periodic terms (meta mode): per instance i, its initial x's
    // (initial_x[i * n_ic + k]) and periodic t's, evaluated with s = hyper(mu_i) by the
    // following meta_gradient calls; empty vectors clear them.
    void set_meta_boundary(std::size_t n_inst, const std::vector<double>& initial_x,
                           const std::vector<double>& periodic_t) {
        if (n_inst == 0 || initial_x.size() % n_inst || periodic_t.size() % n_inst)
            throw std::invalid_argument("set_meta_boundary: points not grouped by instance");
        check(lrnr_gpu_set_meta_boundary(ctx_, static_cast<int64_t>(n_inst), initial_x.data(),
                                         static_cast<int64_t>(initial_x.size() / n_inst), periodic_t.data(),
                                         static_cast<int64_t>(periodic_t.size() / n_inst)));
    }

    // meta_train's step (training.cpp:368-389): interior terms + lambda_sparse
    // banded decay per term (comps[2]) + the lambda_ortho Gram term (returned in
    // *ortho, as meta_train's `ro`); value = bg.value + ro.value, grad = bg + ro.
    training::BatchGradResult meta_gradient(const std::vector<PdeParams>& mus, const std::vector<pde::Point>& pts,
                                            double lambda_sparse, double gamma, double lambda_ortho,
                                            double* ortho = nullptr) {
        const std::size_t n_inst = mus.size();
        if (n_inst == 0 || pts.size() % n_inst) throw std::invalid_argument("meta_gradient: points not grouped by mu");
        set_points(pts, n_inst);
        std::vector<double> m(3 * n_inst);
        for (std::size_t i = 0; i < n_inst; ++i) {
            m[3 * i] = mus[i].mu1;
            m[3 * i + 1] = mus[i].mu2;
            m[3 * i + 2] = mus[i].mu3;
        }
        training::BatchGradResult out;
        out.grad.assign(lrnr_params_ + hyper_params_, 0.0);
        double ro = 0.0;
        check(lrnr_gpu_meta_terms_grad(ctx_, m.data(), 0.0, lambda_sparse, gamma, lambda_ortho, &out.value, out.comps,
                                       &ro, out.grad.data()));
        if (ortho) *ortho = ro;
        return out;
    }

    // ---- the solve loops (training.cpp:428-607) on the device: drop-ins for
    // training::fine_tune / training::fast_solve (L1 evaluation (eval_interval)
    // and wall-clock fields are not produced: records carry epoch and loss).
    training::SolveResult fine_tune(const PdeParams& mu, const HyperParams& theta, const training::PhaseConfig& cfg) {
        training::SolveResult out;
        out.coeffs = hyper_forward(mu, theta);
        out.report.phase = "fine-tune";
        if (cfg.epochs == 0) return out;
        const std::vector<double> s0 = flatten(out.coeffs);
        const double m[3] = {mu.mu1, mu.mu2, mu.mu3};
        solve_into(out, lrnr_gpu_fine_tune, cfg.epochs, s0.data(), m, cfg.lr, static_cast<int64_t>(cfg.epochs),
                   static_cast<int64_t>(cfg.n_interior), static_cast<int64_t>(cfg.n_initial),
                   static_cast<int64_t>(cfg.n_periodic), static_cast<uint64_t>(cfg.seed));
        return out;
    }
    training::SolveResult fast_solve(const PdeParams& mu, const HyperParams& theta, const reduction::SamplingSetX& X,
                                     const training::PhaseConfig& cfg, double lambda_local) {
        training::SolveResult out;
        out.coeffs = hyper_forward(mu, theta);
        out.report.phase = lambda_local > 0.0 ? "fast" : "fast-naive";
        if (cfg.epochs == 0) return out;
        const std::vector<double> s0 = flatten(out.coeffs);
        const double m[3] = {mu.mu1, mu.mu2, mu.mu3};
        std::vector<double> xt;
        for (const pde::Point& p : X.points) {
            xt.push_back(p.x);
            xt.push_back(p.t);
        }
        solve_into(out, lrnr_gpu_fast_solve, cfg.epochs, s0.data(), m, xt.data(),
                   static_cast<int64_t>(X.points.size()), lambda_local, cfg.lr, static_cast<int64_t>(cfg.epochs));
        return out;
    }

    // ---- forward only: loss_tune / loss_fast / loss_meta (training.cpp:109-189),
    //      lrnr_forward / fast_forward (model.cpp:260-292), jet_forward (model.cpp:357-405) ----
    training::LossBreakdown loss_tune(const Coefficients& s, const PdeParams& mu, const pde::CollocationBatch& batch,
                                      bool fast = false) {
        set_points(batch.interior, 1);
        set_boundary(batch.initial_x, batch.periodic_t);
        const std::vector<double> sf = flatten(s);
        const double m[3] = {mu.mu1, mu.mu2, mu.mu3};
        double o[3];
        check(lrnr_gpu_loss_tune(ctx_, fast ? LRNR_MODEL_FAST : LRNR_MODEL_LRNR, sf.data(), m, o));
        return breakdown(o);
    }
    training::LossBreakdown loss_fast(const Coefficients& s, const PdeParams& mu,
                                      const reduction::SamplingSetX& sampling) {
        std::vector<double> xt;
        for (const pde::Point& p : sampling.points) {
            xt.push_back(p.x);
            xt.push_back(p.t);
        }
        const std::vector<double> sf = flatten(s);
        const double m[3] = {mu.mu1, mu.mu2, mu.mu3};
        double o[3];
        check(lrnr_gpu_loss_fast(ctx_, LRNR_MODEL_FAST, sf.data(), m, xt.data(),
                                 static_cast<int64_t>(sampling.points.size()), o));
        return breakdown(o);
    }
    // loss_meta: every sample carries its own mu (sample_collocation(with_mu), pde.cpp:20-49),
    // so each term kind runs as one instance per sample through the hypernetwork.
    training::LossBreakdown loss_meta(const pde::CollocationBatch& batch) {
        if (batch.interior_mu.size() != batch.interior.size() || batch.initial_mu.size() != batch.initial_x.size() ||
            batch.periodic_mu.size() != batch.periodic_t.size())
            throw std::invalid_argument("loss_meta: batch lacks per-sample mu");
        auto mus_of = [](const std::vector<PdeParams>& v) {
            std::vector<double> m;
            for (const PdeParams& q : v) {
                m.push_back(q.mu1);
                m.push_back(q.mu2);
                m.push_back(q.mu3);
            }
            return m;
        };
        double o[3] = {0.0, 0.0, 0.0}, part[3];
        check(lrnr_gpu_set_meta_boundary(ctx_, 0, nullptr, 0, nullptr, 0));
        if (!batch.interior.empty()) {
            set_points(batch.interior, batch.interior.size());
            const std::vector<double> m = mus_of(batch.interior_mu);
            check(lrnr_gpu_loss_meta(ctx_, m.data(), part));
            o[1] += part[1];
        }
        auto boundary_kind = [&](const std::vector<double>& v, const std::vector<PdeParams>& mus, bool initial) {
            if (v.empty()) return;
            const int64_t n = static_cast<int64_t>(v.size());
            check(lrnr_gpu_set_points(ctx_, nullptr, n, 0));
            check(lrnr_gpu_set_meta_boundary(ctx_, n, initial ? v.data() : nullptr, initial ? 1 : 0,
                                             initial ? nullptr : v.data(), initial ? 0 : 1));
            const std::vector<double> m = mus_of(mus);
            check(lrnr_gpu_loss_meta(ctx_, m.data(), part));
            o[2] += part[2];
        };
        boundary_kind(batch.initial_x, batch.initial_mu, true);
        boundary_kind(batch.periodic_t, batch.periodic_mu, false);
        check(lrnr_gpu_set_meta_boundary(ctx_, 0, nullptr, 0, nullptr, 0));
        o[0] = o[1] + o[2];
        if (!std::isfinite(o[0])) throw NonFiniteError(-1);
        return breakdown(o);
    }
    // lrnr_forward / fast_forward: u at each point (value-only forward on the device)
    std::vector<double> forward_values(const std::vector<pde::Point>& pts, const Coefficients& s, bool fast = false) {
        std::vector<double> xt, u(pts.size());
        for (const pde::Point& p : pts) {
            xt.push_back(p.x);
            xt.push_back(p.t);
        }
        const std::vector<double> sf = flatten(s);
        check(lrnr_gpu_values(ctx_, fast ? LRNR_MODEL_FAST : LRNR_MODEL_LRNR, sf.data(), xt.data(),
                              static_cast<int64_t>(pts.size()), u.data()));
        return u;
    }
    // pde::l1_relative_error (pde.cpp:166-178) of the bound LRNR (or FastLRNR)
    // against a GridField, evaluated on the device.
    double l1_relative_error(const Coefficients& s, const pde::GridField& ref, bool fast = false) {
        const std::vector<double> sf = flatten(s);
        double out = 0.0;
        check(lrnr_gpu_l1_error(ctx_, fast ? LRNR_MODEL_FAST : LRNR_MODEL_LRNR, sf.data(), ref.values.data(),
                                static_cast<int64_t>(ref.n_x), static_cast<int64_t>(ref.n_t), &out));
        return out;
    }
    std::vector<Jet> jet_forward(const std::vector<pde::Point>& pts, const Coefficients& s, bool fast = false) {
        set_points(pts, 1);
        const std::vector<double> sf = flatten(s);
        std::vector<double> j(4 * pts.size());
        check(lrnr_gpu_jets(ctx_, fast ? LRNR_MODEL_FAST : LRNR_MODEL_LRNR, sf.data(), j.data()));
        std::vector<Jet> out(pts.size());
        for (std::size_t i = 0; i < pts.size(); ++i) {
            out[i].value = DenseVector{j[4 * i]};
            out[i].dx = DenseVector{j[4 * i + 1]};
            out[i].dt = DenseVector{j[4 * i + 2]};
            out[i].dxx = DenseVector{j[4 * i + 3]};
        }
        return out;
    }

    // ---- FastLRNR construction (reduction.cpp:111-238) on the device ----
    // reduction::harvest_snapshots: s(mu) from the reference's own hyper_forward
    // (host), the perturbation stream from the reference's Rng (host,
    // bit-identical), the hidden states on the device (bit-identical for tanh).
    reduction::SnapshotSet harvest_snapshots(const LrnrParams& p, const HyperParams& theta,
                                             const reduction::SamplingSetX& sampling, std::size_t n_perturb,
                                             double sigma_factor, const std::vector<PdeParams>& mu_grid,
                                             std::uint64_t seed, int act = LRNR_ACT_TANH) {
        std::vector<double> flat, s, X;
        for (std::size_t l = 0; l < p.depth(); ++l) {
            flat.insert(flat.end(), p.u[l].data.begin(), p.u[l].data.end());
            flat.insert(flat.end(), p.v[l].data.begin(), p.v[l].data.end());
            flat.insert(flat.end(), p.b[l].data.begin(), p.b[l].data.end());
        }
        for (const PdeParams& mu : mu_grid) {
            const std::vector<double> c = flatten(hyper_forward(mu, theta));
            s.insert(s.end(), c.begin(), c.end());
        }
        for (const pde::Point& q : sampling.points) {
            X.push_back(q.x);
            X.push_back(q.t);
        }
        const std::vector<int64_t> w(p.widths.begin(), p.widths.end()), r(p.ranks.begin(), p.ranks.end());
        const int64_t n_x = static_cast<int64_t>(sampling.points.size()), n_mu = static_cast<int64_t>(mu_grid.size());
        const int64_t n_cols = n_mu * n_x * static_cast<int64_t>(1 + n_perturb);
        std::size_t rows = 0;
        for (std::size_t l = 0; l + 1 < p.depth(); ++l) rows += p.widths[l + 1];
        std::vector<double> out(rows * static_cast<std::size_t>(n_cols)), pts(2 * static_cast<std::size_t>(n_cols));
        check(lrnr_gpu_harvest_snapshots(ctx_, static_cast<int>(p.depth()), w.data(), r.data(), flat.data(), act,
                                         s.data(), n_mu, X.data(), n_x, static_cast<int64_t>(n_perturb), sigma_factor,
                                         seed, out.data()));
        if (lrnr_host_harvest_points(X.data(), n_x, n_mu, static_cast<int64_t>(n_perturb), sigma_factor, seed,
                                     pts.data()) != LRNR_OK)
            throw std::invalid_argument("harvest_snapshots: bad sampling set");
        reduction::SnapshotSet set;
        std::size_t o = 0;
        for (std::size_t l = 0; l + 1 < p.depth(); ++l) {
            DenseMatrix m(p.widths[l + 1], static_cast<std::size_t>(n_cols));
            std::copy(out.begin() + static_cast<std::ptrdiff_t>(o), out.begin() + static_cast<std::ptrdiff_t>(o + m.data.size()),
                      m.data.begin());
            o += m.data.size();
            set.layers.push_back(std::move(m));
        }
        std::size_t col = 0;
        for (std::size_t mi = 0; mi < mu_grid.size(); ++mi)
            for (std::size_t pi = 0; pi < sampling.points.size(); ++pi)
                for (std::size_t k = 0; k <= n_perturb; ++k, ++col)
                    set.tags.push_back({mi, pi, k, pde::Point{pts[2 * col], pts[2 * col + 1]}, mu_grid[mi]});
        return set;
    }
    // reduction::eim_greedy: the greedy sweeps on the device, bit-identical indices
    // and basis columns; the block LU is refactored with the reference's lu_factor.
    reduction::EimBasis eim_greedy(const DenseMatrix& snapshots, std::size_t r_hat) {
        const int64_t m = static_cast<int64_t>(snapshots.rows), rh = static_cast<int64_t>(r_hat);
        std::vector<int64_t> idx(r_hat > 0 ? r_hat : 1);
        std::vector<double> xi(snapshots.rows * (r_hat > 0 ? r_hat : 1));
        int64_t count = 0;
        int exhausted = 0;
        check(lrnr_gpu_eim_greedy(ctx_, m, static_cast<int64_t>(snapshots.cols), snapshots.data.data(), rh, idx.data(),
                                  xi.data(), &count, &exhausted));
        reduction::EimBasis b;
        b.xi = DenseMatrix(snapshots.rows, static_cast<std::size_t>(count));
        for (int64_t i = 0; i < m; ++i)
            for (int64_t k = 0; k < count; ++k)
                b.xi.at(static_cast<std::size_t>(i), static_cast<std::size_t>(k)) = xi[i * rh + k];
        for (int64_t k = 0; k < count; ++k) b.indices.push_back(static_cast<std::size_t>(idx[k]));
        b.exhausted = exhausted != 0;
        DenseMatrix block(b.indices.size(), b.indices.size());
        for (std::size_t i = 0; i < b.indices.size(); ++i)
            for (std::size_t j = 0; j < b.indices.size(); ++j) block.at(i, j) = b.xi.at(b.indices[i], j);
        b.block_lu = lu_factor(block);
        return b;
    }

    // Q-DEIM basis (BASELINE configs[1]: "indices from pivoted QR of U^l"; no reference
    // counterpart): EimBasis{xi, indices = pivoted-QR rows of xi, block_lu = lu(P^T xi)},
    // ready for the reference's own reduction::build_fastparams (reduction.cpp:240-283).
    static reduction::EimBasis qdeim_basis(const DenseMatrix& xi) {
        std::vector<int64_t> idx(xi.cols > 0 ? xi.cols : 1);
        int64_t count = 0;
        if (lrnr_host_qdeim(static_cast<int64_t>(xi.rows), static_cast<int64_t>(xi.cols), xi.data.data(), idx.data(),
                            &count) != 0 ||
            count != static_cast<int64_t>(xi.cols))
            throw std::invalid_argument("qdeim_basis: empty or rank-deficient basis");
        reduction::EimBasis b;
        b.xi = xi;
        for (int64_t k = 0; k < count; ++k) b.indices.push_back(static_cast<std::size_t>(idx[k]));
        DenseMatrix block(b.indices.size(), b.indices.size());
        for (std::size_t i = 0; i < b.indices.size(); ++i)
            for (std::size_t j = 0; j < b.indices.size(); ++j) block.at(i, j) = b.xi.at(b.indices[i], j);
        b.block_lu = lu_factor(block);
        return b;
    }

    lrnr_gpu_ctx* handle() { return ctx_; }

private:
    void check(int rc) {
        if (rc == LRNR_OK) return;
        const std::string msg = lrnr_gpu_last_error(ctx_);
        if (rc == LRNR_ENONFINITE) throw NonFiniteError(lrnr_gpu_last_layer_tag(ctx_));
        if (rc == LRNR_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error("lrnr_gpu: " + msg);
    }
    static training::LossBreakdown breakdown(const double* o) {
        training::LossBreakdown lb;
        lb.total = o[0];
        lb.residual = o[1];
        lb.boundary = o[2];
        return lb;
    }
    static std::vector<double> flatten(const Coefficients& s) {
        std::vector<double> f;
        for (const auto& v : s.s) f.insert(f.end(), v.data.begin(), v.data.end());
        return f;
    }
    void set_points(const std::vector<pde::Point>& pts, std::size_t n_inst) {
        std::vector<double> xt(2 * pts.size());
        for (std::size_t i = 0; i < pts.size(); ++i) {
            xt[2 * i] = pts[i].x;
            xt[2 * i + 1] = pts[i].t;
        }
        check(lrnr_gpu_set_points(ctx_, xt.data(), static_cast<int64_t>(n_inst),
                                  static_cast<int64_t>(pts.size() / n_inst)));
    }
    template <class Fn, class... A>
    void solve_into(training::SolveResult& out, Fn fn, std::size_t epochs, A... args) {
        std::vector<double> s(flatten(out.coeffs).size()), losses(epochs);
        double best = 0.0;
        int64_t best_e = 0, n_rec = 0;
        int flags = 0;
        check(fn(ctx_, args..., s.data(), &best, &best_e, losses.data(), &n_rec, &flags));
        for (int64_t e = 0; e < n_rec; ++e) {
            training::EpochRecord rec;
            rec.epoch = static_cast<std::size_t>(e + 1);
            rec.loss = losses[e];
            out.report.records.push_back(rec);
        }
        out.report.aborted_nonfinite = (flags & 1) != 0;
        out.report.diverged = (flags & 2) != 0;
        out.report.best_loss = best;
        out.report.best_epoch = static_cast<std::size_t>(best_e);
        std::size_t o = 0;
        for (auto& v : out.coeffs.s)
            for (double& x : v.data) x = s[o++];
    }
    void set_boundary(const std::vector<double>& ic, const std::vector<double>& per) {
        check(lrnr_gpu_set_boundary(ctx_, ic.data(), static_cast<int64_t>(ic.size()), per.data(),
                                    static_cast<int64_t>(per.size())));
    }
    training::BatchGradResult terms(int model, const Coefficients& s, const PdeParams& mu, int objective, double w,
                                    const double* s_init, double lambda_local) {
        const std::vector<double> sf = flatten(s);
        const double m[3] = {mu.mu1, mu.mu2, mu.mu3};
        training::BatchGradResult out;
        out.grad.assign(sf.size(), 0.0);
        check(lrnr_gpu_terms_grad(ctx_, model, sf.data(), m, objective, w, w, w, s_init, lambda_local, &out.value,
                                  out.comps, out.grad.data()));
        return out;
    }
    training::BatchGradResult coeff_gradient(int model, const Coefficients& s, const PdeParams& mu,
                                             const std::vector<pde::Point>& pts) {
        set_points(pts, 1);
        const std::vector<double> sf = flatten(s);
        const double m[3] = {mu.mu1, mu.mu2, mu.mu3};
        training::BatchGradResult out;
        out.grad.assign(sf.size(), 0.0);
        check(lrnr_gpu_loss_grad_s(ctx_, model, sf.data(), m, 0.0, &out.value, out.comps, out.grad.data()));
        return out;
    }

    lrnr_gpu_ctx* ctx_ = nullptr;
    std::size_t lrnr_depth_ = 0, lrnr_params_ = 0, hyper_params_ = 0;
};

}  // namespace gpu
}  // namespace lrnr
