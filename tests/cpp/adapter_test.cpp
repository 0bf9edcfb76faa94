// Drop-in check of include/lrnr_gpu_adapter.hpp against the UNMODIFIED reference:
// the same fine-tune gradient (PinnTermEmitter interior terms through
// run_batch_gradient, training.cpp:191-329) computed by the reference on the CPU
// and by lrnr::gpu::Engine on the B200, on BASELINE config 0, plus the
// boundary terms, the FastLRNR gradient, the fast-phase objective and the
// NonFiniteError path.  Exit code 0 = parity within 1e-10.
// Built by oracle/Makefile into oracle/_ref/adapter_test (needs a GPU to run).
#include <cmath>
#include <cstdio>

#include "lrnr/autodiff.hpp"
#include "lrnr/reduction.hpp"
#include "lrnr/training.hpp"
#include "lrnr_gpu_adapter.hpp"

using namespace lrnr;

static double floor_rel(const std::vector<double>& g, const std::vector<double>& w) {
    double mx = 0.0, worst = 0.0;
    for (double v : w) mx = std::max(mx, std::fabs(v));
    for (std::size_t i = 0; i < w.size(); ++i)
        worst = std::max(worst, std::fabs(g[i] - w[i]) / std::max(std::fabs(w[i]), 1e-3 * mx));
    return worst;
}

int main() {
    Rng rng(2410);
    LrnrParams p = make_lrnr_params({2, 100, 100, 100, 1}, {2, 10, 10, 1}, rng, true, 0.5);
    Coefficients s = make_coefficients(p.ranks, rng, 0.2, 1.0);
    const PdeParams mu{30.0, 0.0, 0.0};
    pde::CollocationBatch batch = pde::sample_collocation(4001, 4096, 0, 0, ParamDomain{}, false);

    // reference: PinnTermEmitter-equivalent interior emitter through run_batch_gradient
    Trainables at{&p, nullptr, &s};
    const double w = 1.0 / static_cast<double>(batch.interior.size());
    training::EmitFn emit = [&](TapeBindings& ctx, const training::ExtraBindings&, std::size_t i,
                                double* comps) -> NodeId {
        Tape& tp = ctx.tape;
        const NodeId jet = emit_lrnr_jet(tp, batch.interior[i].x, batch.interior[i].t, ctx.lrnr, ctx.coeffs.s_leaves);
        const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, mu)), w);
        comps[0] += tp.value(term);
        return term;
    };
    training::ParallelConfig par{8, 64};
    training::BatchGradResult ref = training::run_batch_gradient(at, ParamSelector::CoefficientsOnly, nullptr, emit,
                                                                 batch.interior.size(), par);

    lrnr::gpu::Engine eng(0);
    eng.bind(p, LRNR_F64);
    training::BatchGradResult got = eng.tune_gradient(s, mu, batch);
    const double ev = std::fabs(got.value - ref.value) / ref.value;
    const double eg = floor_rel(got.grad, ref.grad);
    std::printf("fine-tune gradient: value rel err %.3e, dL/ds floor-rel err %.3e\n", ev, eg);

    // FastLRNR from the reference's own EIM reduction
    HyperParams h;
    h.w.emplace_back(23, 3);
    DenseVector hb(23);
    std::size_t o = 0;
    for (auto& sl : s.s)
        for (double v : sl.data) hb[o++] = v;
    h.b.push_back(hb);
    h.split = p.ranks;
    h.box = ParamDomain::d1();
    auto X = reduction::SamplingSetX::uniform_grid(4, 3);
    auto snaps = reduction::harvest_snapshots(p, h, X, 8, 0.05, {mu}, 777);
    std::vector<reduction::EimBasis> bases;
    for (std::size_t l = 0; l + 1 < p.depth(); ++l) bases.push_back(reduction::eim_greedy(snaps.layers[l], 10));
    FastParams f = reduction::build_fastparams(p, bases);
    Trainables atf{nullptr, nullptr, &s};
    training::SetupFn setup = [&](TapeBindings& ctx) {
        training::ExtraBindings ex;
        ex.fast = bind_fast(ctx.tape, f);
        ex.has_fast = true;
        return ex;
    };
    training::EmitFn emitf = [&](TapeBindings& ctx, const training::ExtraBindings& ex, std::size_t i,
                                 double* comps) -> NodeId {
        Tape& tp = ctx.tape;
        const NodeId jet = emit_fast_jet(tp, batch.interior[i].x, batch.interior[i].t, ex.fast, ctx.coeffs.s_leaves);
        const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, mu)), w);
        comps[0] += tp.value(term);
        return term;
    };
    training::BatchGradResult reff =
        training::run_batch_gradient(atf, ParamSelector::CoefficientsOnly, setup, emitf, batch.interior.size(), par);
    eng.bind(f, LRNR_F64);
    training::BatchGradResult gotf = eng.fast_gradient(s, mu, batch.interior);
    const double evf = std::fabs(gotf.value - reff.value) / reff.value;
    const double egf = floor_rel(gotf.grad, reff.grad);
    std::printf("FastLRNR gradient: value rel err %.3e, dL/ds floor-rel err %.3e\n", evf, egf);

    // FastLRNR construction on the device == the reference's, bit for bit: c2 widths
    // (deep layers exhaust the budget), a mu grid through a hypernetwork
    bool eim_ok = true;
    {
        Rng rng2(2411);
        LrnrParams p2 = make_lrnr_params({2, 256, 256, 256, 256, 256, 256, 1}, {2, 32, 32, 32, 32, 32, 1}, rng2,
                                         true, 0.5);
        HyperParams th = make_hyper_params(p2.ranks, 2, 16, ParamDomain{{1.0, 0.0, 0.0}, {40.0, 0.1, 10.0}}, rng2,
                                           0.01, 0.5);
        const std::vector<PdeParams> grid{{5.0, 0.01, 1.0}, {20.0, 0.05, 3.0}, {35.0, 0.09, 8.0}};
        auto X2 = reduction::SamplingSetX::uniform_grid(4, 3);
        auto ref_snaps = reduction::harvest_snapshots(p2, th, X2, 8, 0.05, grid, 99);
        auto dev_snaps = eng.harvest_snapshots(p2, th, X2, 8, 0.05, grid, 99);
        std::size_t snap_diff = 0;
        for (std::size_t l = 0; l < ref_snaps.layers.size(); ++l)
            for (std::size_t i = 0; i < ref_snaps.layers[l].data.size(); ++i)
                snap_diff += ref_snaps.layers[l].data[i] != dev_snaps.layers[l].data[i];
        for (std::size_t c = 0; c < ref_snaps.tags.size(); ++c)
            snap_diff += ref_snaps.tags[c].point.x != dev_snaps.tags[c].point.x ||
                         ref_snaps.tags[c].point.t != dev_snaps.tags[c].point.t;
        std::vector<reduction::EimBasis> rb, db;
        std::size_t basis_diff = 0;
        for (std::size_t l = 0; l + 1 < p2.depth(); ++l) {
            rb.push_back(reduction::eim_greedy(ref_snaps.layers[l], 32));
            db.push_back(eng.eim_greedy(ref_snaps.layers[l], 32));
            basis_diff += rb[l].indices != db[l].indices || rb[l].xi.data != db[l].xi.data ||
                          rb[l].exhausted != db[l].exhausted;
        }
        FastParams fr = reduction::build_fastparams(p2, rb), fd = reduction::build_fastparams(p2, db);
        std::size_t fast_diff = 0;
        for (std::size_t l = 0; l + 1 < p2.depth(); ++l)
            fast_diff += fr.u_hat[l].data != fd.u_hat[l].data || fr.v_hat[l].data != fd.v_hat[l].data ||
                         fr.b_hat[l].data != fd.b_hat[l].data;
        std::printf("FastLRNR construction: %zu snapshot / %zu basis / %zu factor mismatches (%zu columns)\n",
                    snap_diff, basis_diff, fast_diff, ref_snaps.tags.size());
        eim_ok = snap_diff == 0 && basis_diff == 0 && fast_diff == 0;

        // Q-DEIM bases (pivoted-QR rows of U^l) through the reference's own eim_apply and
        // build_fastparams: interpolation is exact on range(U^l), u_hat = the selected rows
        std::vector<reduction::EimBasis> qb;
        double q_err = 0.0;
        std::size_t q_rows = 0;
        for (std::size_t l = 0; l + 1 < p2.depth(); ++l) {
            qb.push_back(lrnr::gpu::Engine::qdeim_basis(p2.u[l]));
            const reduction::EimBasis& b = qb.back();
            DenseVector z(p2.u[l].rows), sampled(b.dim());
            for (std::size_t i = 0; i < z.len(); ++i) {
                double acc = 0.0;
                for (std::size_t j = 0; j < p2.u[l].cols; ++j) acc += p2.u[l].at(i, j) * (0.3 + 0.1 * static_cast<double>(j));
                z[i] = acc;
            }
            for (std::size_t k = 0; k < b.dim(); ++k) sampled[k] = z[b.indices[k]];
            const DenseVector back = reduction::eim_apply(b, sampled);
            for (std::size_t i = 0; i < z.len(); ++i) q_err = std::max(q_err, std::abs(back[i] - z[i]));
        }
        const FastParams fq = reduction::build_fastparams(p2, qb);
        for (std::size_t l = 0; l + 1 < p2.depth(); ++l)
            for (std::size_t k = 0; k < qb[l].dim(); ++k)
                for (std::size_t j = 0; j < p2.u[l].cols; ++j)
                    q_rows += fq.u_hat[l].at(k, j) != p2.u[l].at(qb[l].indices[k], j);
        std::printf("Q-DEIM bases: interpolation error on range(U) %.2e, %zu u_hat mismatches\n", q_err, q_rows);
        eim_ok = eim_ok && q_err <= 1e-10 && q_rows == 0;
    }

    // full fine-tune batch: interior + initial + periodic terms (PinnTermEmitter,
    // training.cpp:286-327) with the fine_tune weights 1/n per kind
    pde::CollocationBatch fb = pde::sample_collocation(4007, 1024, 256, 256, ParamDomain{}, false);
    const double wi = 1.0 / fb.interior.size(), wc = 1.0 / fb.initial_x.size(), wb = 1.0 / fb.periodic_t.size();
    training::EmitFn emit_full = [&](TapeBindings& ctx, const training::ExtraBindings&, std::size_t idx,
                                     double* comps) -> NodeId {
        Tape& tp = ctx.tape;
        const std::size_t ni = fb.interior.size(), nc = fb.initial_x.size();
        if (idx < ni) {
            const NodeId jet = emit_lrnr_jet(tp, fb.interior[idx].x, fb.interior[idx].t, ctx.lrnr, ctx.coeffs.s_leaves);
            const NodeId term = tp.scale(tp.square(tp.residual_cdr(jet, mu)), wi);
            comps[0] += tp.value(term);
            return term;
        }
        if (idx < ni + nc) {
            const double x = fb.initial_x[idx - ni];
            const NodeId jet = emit_lrnr_jet(tp, x, 0.0, ctx.lrnr, ctx.coeffs.s_leaves);
            const NodeId term = tp.scale(tp.square(tp.sub_const(tp.pick_value(jet, 0), std::sin(x))), wc);
            comps[1] += tp.value(term);
            return term;
        }
        const double t = fb.periodic_t[idx - ni - nc];
        const NodeId j0 = emit_lrnr_jet(tp, 0.0, t, ctx.lrnr, ctx.coeffs.s_leaves);
        const NodeId j1 = emit_lrnr_jet(tp, pde::kTwoPi, t, ctx.lrnr, ctx.coeffs.s_leaves);
        const NodeId term = tp.scale(tp.square(tp.sub(tp.pick_value(j0, 0), tp.pick_value(j1, 0))), wb);
        comps[1] += tp.value(term);
        return term;
    };
    training::BatchGradResult ref_full = training::run_batch_gradient(
        at, ParamSelector::CoefficientsOnly, nullptr, emit_full,
        fb.interior.size() + fb.initial_x.size() + fb.periodic_t.size(), par);
    training::BatchGradResult got_full = eng.tune_gradient(s, mu, fb);
    const double evb = std::fabs(got_full.value - ref_full.value) / ref_full.value;
    const double ecb = std::fabs(got_full.comps[1] - ref_full.comps[1]) / ref_full.comps[1];
    const double egb = floor_rel(got_full.grad, ref_full.grad);
    std::printf("fine-tune with boundary terms: value %.3e, boundary comp %.3e, dL/ds %.3e\n", evb, ecb, egb);

    // fast-phase emitter (training.cpp:521-559): l1 terms at X + locality
    Coefficients s_pert = s;
    for (auto& sl : s_pert.s)
        for (double& v : sl.data) v = 0.9 * v + 0.01;
    const double lambda = 1e-2;
    training::EmitFn emit_phase = [&](TapeBindings& ctx, const training::ExtraBindings& ex, std::size_t idx,
                                      double* comps) -> NodeId {
        Tape& tp = ctx.tape;
        if (idx < X.points.size()) {
            const pde::Point pt = X.points[idx];
            switch (reduction::classify_point(pt)) {
                case reduction::PointKind::Interior: {
                    const NodeId term =
                        tp.abs_val(tp.residual_cdr(emit_fast_jet(tp, pt.x, pt.t, ex.fast, ctx.coeffs.s_leaves), mu));
                    comps[0] += tp.value(term);
                    return term;
                }
                case reduction::PointKind::Initial: {
                    const NodeId jet = emit_fast_jet(tp, pt.x, 0.0, ex.fast, ctx.coeffs.s_leaves);
                    const NodeId term = tp.abs_val(tp.sub_const(tp.pick_value(jet, 0), std::sin(pt.x)));
                    comps[1] += tp.value(term);
                    return term;
                }
                default: {
                    const NodeId j0 = emit_fast_jet(tp, 0.0, pt.t, ex.fast, ctx.coeffs.s_leaves);
                    const NodeId j1 = emit_fast_jet(tp, pde::kTwoPi, pt.t, ex.fast, ctx.coeffs.s_leaves);
                    const NodeId term = tp.abs_val(tp.sub(tp.pick_value(j0, 0), tp.pick_value(j1, 0)));
                    comps[1] += tp.value(term);
                    return term;
                }
            }
        }
        std::vector<NodeId> ids;
        std::vector<double> ws;
        for (std::size_t l = 0; l < ctx.coeffs.s_leaves.size(); ++l) {
            ids.push_back(tp.l1_to_target(ctx.coeffs.s_leaves[l], s.s[l].data.data(), s.s[l].len()));
            ws.push_back(lambda);
        }
        const NodeId term = tp.weighted_sum(ids, ws);
        comps[3] += tp.value(term);
        return term;
    };
    Trainables atp{nullptr, nullptr, &s_pert};
    training::BatchGradResult ref_phase = training::run_batch_gradient(atp, ParamSelector::CoefficientsOnly, setup,
                                                                       emit_phase, X.points.size() + 1, par);
    training::BatchGradResult got_phase = eng.fast_phase_gradient(s_pert, s, mu, X, lambda);
    const double evp = std::fabs(got_phase.value - ref_phase.value) / ref_phase.value;
    const double egp = floor_rel(got_phase.grad, ref_phase.grad);
    std::printf("fast-phase objective: value %.3e, dL/ds %.3e\n", evp, egp);

    // the solve loops: the reference's own training::fine_tune / fast_solve vs the device loops
    HyperParams hc;  // constant hypernetwork: hyper_forward(mu) == s
    hc.w.emplace_back(23, 3);
    hc.b.push_back(hb);
    hc.split = p.ranks;
    hc.box = ParamDomain::d1();
    training::PhaseConfig cfg;
    cfg.epochs = 30;
    cfg.n_interior = 256;
    cfg.n_initial = 64;
    cfg.n_periodic = 64;
    cfg.eval_interval = 0;
    training::SolveResult rft = training::fine_tune(mu, p, hc, cfg, par, nullptr);
    eng.bind(p, LRNR_F64);
    training::SolveResult gft = eng.fine_tune(mu, hc, cfg);
    double eft = 0.0;
    bool sft = rft.report.records.size() == gft.report.records.size() && rft.report.best_epoch == gft.report.best_epoch;
    for (std::size_t e = 0; sft && e < rft.report.records.size(); ++e)
        eft = std::max(eft, std::fabs(gft.report.records[e].loss - rft.report.records[e].loss) / rft.report.records[e].loss);
    std::printf("fine_tune loop (30 epochs): losses max rel err %.3e, best epoch %zu / %zu\n", eft,
                gft.report.best_epoch, rft.report.best_epoch);
    training::PhaseConfig fcfg;
    fcfg.epochs = 200;
    training::SolveResult rfs = training::fast_solve(mu, hc, f, X, fcfg, 1e-2, par);
    training::SolveResult gfs = eng.fast_solve(mu, hc, X, fcfg, 1e-2);
    double efs = 0.0;
    bool sfs = rfs.report.records.size() == gfs.report.records.size() && rfs.report.best_epoch == gfs.report.best_epoch &&
               rfs.report.diverged == gfs.report.diverged;
    for (std::size_t e = 0; sfs && e < rfs.report.records.size(); ++e)
        efs = std::max(efs, std::fabs(gfs.report.records[e].loss - rfs.report.records[e].loss) / rfs.report.records[e].loss);
    double efs_s = 0.0;
    for (std::size_t l = 0; l < rfs.coeffs.s.size(); ++l)
        for (std::size_t i = 0; i < rfs.coeffs.s[l].len(); ++i)
            efs_s = std::max(efs_s, std::fabs(gfs.coeffs.s[l][i] - rfs.coeffs.s[l][i]));
    std::printf("fast_solve loop (200 epochs): losses max rel err %.3e, best s max abs err %.3e\n", efs, efs_s);

    // forward-only losses: loss_tune / loss_fast / loss_meta (training.cpp:109-189) and u only
    eng.bind(p, LRNR_F64);
    const training::LossBreakdown rlt = training::loss_tune(s, mu, p, fb), glt = eng.loss_tune(s, mu, fb);
    const double elt = std::max(std::fabs(glt.total - rlt.total) / rlt.total,
                                std::fabs(glt.boundary - rlt.boundary) / rlt.boundary);
    eng.bind(f, LRNR_F64);
    auto X7 = reduction::SamplingSetX::uniform_grid(7, 5);
    const training::LossBreakdown rlf = training::loss_fast(s, mu, f, X7), glf = eng.loss_fast(s, mu, X7);
    const double elf = std::max(std::fabs(glf.total - rlf.total) / rlf.total,
                                std::fabs(glf.boundary - rlf.boundary) / rlf.boundary);
    HyperParams hm = make_hyper_params(p.ranks, 2, 16, ParamDomain::d1(), rng, 0.01, 0.5);
    pde::CollocationBatch mb = pde::sample_collocation(4011, 300, 40, 30, ParamDomain::d1(), true);
    eng.bind(hm);
    const training::LossBreakdown rlm = training::loss_meta(p, hm, mb), glm = eng.loss_meta(mb);
    const double elm = std::max({std::fabs(glm.total - rlm.total) / rlm.total,
                                 std::fabs(glm.residual - rlm.residual) / rlm.residual,
                                 std::fabs(glm.boundary - rlm.boundary) / rlm.boundary});
    std::vector<double> uv = eng.forward_values(fb.interior, s);
    double euv = 0.0;
    for (std::size_t i = 0; i < fb.interior.size(); ++i) {
        const double r = lrnr_forward(fb.interior[i].x, fb.interior[i].t, p, s)[0];
        euv = std::max(euv, std::fabs(uv[i] - r) / std::max(std::fabs(r), 1e-3));
    }
    std::printf("plain losses: loss_tune %.3e, loss_fast %.3e, loss_meta %.3e, lrnr_forward %.3e\n", elt, elf, elm,
                euv);

    // NonFiniteError surfaces as the reference's exception type
    Coefficients bad = s;
    bad.s[1][0] = std::nan("");
    bool threw = false;
    try {
        eng.tune_gradient(bad, mu, batch);
    } catch (const NonFiniteError& e) {
        threw = e.layer_tag == -1;
    }
    std::printf("NonFiniteError mapped: %s\n", threw ? "yes" : "NO");
    const bool ok = ev <= 1e-12 && eg <= 1e-10 && evf <= 1e-12 && egf <= 1e-10 && evb <= 1e-12 && ecb <= 1e-12 &&
                    egb <= 1e-10 && evp <= 1e-12 && egp <= 1e-10 && sft && eft <= 1e-10 && sfs && efs <= 1e-10 &&
                    efs_s <= 1e-10 && threw && eim_ok && elt <= 1e-12 && elf <= 1e-12 && elm <= 1e-12 &&
                    euv <= 1e-12;
    std::printf("%s\n", ok ? "ADAPTER PARITY OK" : "ADAPTER PARITY FAILED");
    return ok ? 0 : 1;
}
