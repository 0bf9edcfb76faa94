// TEST INFRASTRUCTURE ONLY: the reference's own checkpoint writer / reader
// (proj/src/checkpoint.cpp, nlohmann json) driven through extern "C" entries, to
// generate and cross-check checkpoint fixtures (tests/golden/make_golden.py,
// tests/test_host.py). Built by oracle/Makefile into oracle/_ref/ only when the
// reference and its json header are present (the build container).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lrnr/checkpoint.hpp"
#include "lrnr/model.hpp"
#include "lrnr/reduction.hpp"

using namespace lrnr;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

LrnrParams unpack_lrnr(int L, const int64_t* w, const int64_t* r, const double* P) {
    LrnrParams p;
    for (int l = 0; l <= L; ++l) p.widths.push_back(static_cast<std::size_t>(w[l]));
    for (int l = 0; l < L; ++l) p.ranks.push_back(static_cast<std::size_t>(r[l]));
    std::size_t o = 0;
    for (int l = 0; l < L; ++l) {
        DenseMatrix u(w[l + 1], r[l]), v(w[l], r[l]);
        DenseVector b(w[l + 1]);
        for (auto& x : u.data) x = P[o++];
        for (auto& x : v.data) x = P[o++];
        for (auto& x : b.data) x = P[o++];
        p.u.push_back(u);
        p.v.push_back(v);
        p.b.push_back(b);
    }
    return p;
}
}  // namespace

extern "C" {

const char* ref_ckpt_error() { return g_err.c_str(); }

// Checkpoint with lrnr.*, hyper.* (K layers, widths hw[0..K]), fast.* (may be
// absent: Lf = 0) and sampling_x, via put_lrnr / put_hyper / put_fast / put_sampling.
int ref_ckpt_write(const char* path, int L, const int64_t* w, const int64_t* r, const double* P, int K,
                   const int64_t* hw, const double* H, const double* lo, const double* hi, int Lf,
                   const int64_t* fr, const int64_t* frh, const double* F, const double* X, int64_t n_x) {
    return guarded([&] {
        Checkpoint ck;
        LrnrParams p = unpack_lrnr(L, w, r, P);
        put_lrnr(ck, p);
        HyperParams h;
        std::size_t o = 0;
        for (int k = 0; k < K; ++k) {
            DenseMatrix wk(hw[k + 1], hw[k]);
            DenseVector bk(hw[k + 1]);
            for (auto& x : wk.data) x = H[o++];
            for (auto& x : bk.data) x = H[o++];
            h.w.push_back(wk);
            h.b.push_back(bk);
        }
        h.split = p.ranks;
        for (int i = 0; i < 3; ++i) {
            h.box.lo[i] = lo[i];
            h.box.hi[i] = hi[i];
        }
        put_hyper(ck, h);
        if (Lf > 0) {
            FastParams f;
            for (int l = 0; l < Lf; ++l) f.ranks.push_back(static_cast<std::size_t>(fr[l]));
            for (int l = 0; l + 1 < Lf; ++l) f.red_ranks.push_back(static_cast<std::size_t>(frh[l]));
            std::size_t q = 0;
            f.v_in = DenseMatrix(2, fr[0]);
            for (auto& x : f.v_in.data) x = F[q++];
            for (int l = 0; l + 1 < Lf; ++l) {
                DenseMatrix uh(frh[l], fr[l]), vh(frh[l], fr[l + 1]);
                DenseVector bh(frh[l]);
                for (auto& x : uh.data) x = F[q++];
                for (auto& x : bh.data) x = F[q++];
                for (auto& x : vh.data) x = F[q++];
                f.u_hat.push_back(uh);
                f.b_hat.push_back(bh);
                f.v_hat.push_back(vh);
            }
            f.u_out = DenseMatrix(1, fr[Lf - 1]);
            for (auto& x : f.u_out.data) x = F[q++];
            f.b_out = DenseVector(1);
            f.b_out[0] = F[q++];
            put_fast(ck, f);
        }
        reduction::SamplingSetX s;
        for (int64_t i = 0; i < n_x; ++i) s.points.push_back({X[2 * i], X[2 * i + 1]});
        put_sampling(ck, s);
        ck.meta["note"] = "written by the reference (checkpoint.cpp) for the B200 port's tests";
        checkpoint_save(ck, path);
    });
}

// Read back a checkpoint with the reference: the LRNR flat params (layout of
// lrnr_gpu.h) and the hypernetwork flat params; n_* return the element counts.
int ref_ckpt_read(const char* path, double* P, int64_t* n_p, double* H, int64_t* n_h) {
    return guarded([&] {
        Checkpoint ck = checkpoint_load(path);
        LrnrParams p = get_lrnr(ck);
        HyperParams h = get_hyper(ck);
        int64_t o = 0;
        for (std::size_t l = 0; l < p.depth(); ++l) {
            for (double x : p.u[l].data) P[o++] = x;
            for (double x : p.v[l].data) P[o++] = x;
            for (double x : p.b[l].data) P[o++] = x;
        }
        *n_p = o;
        o = 0;
        for (std::size_t k = 0; k < h.w.size(); ++k) {
            for (double x : h.w[k].data) H[o++] = x;
            for (double x : h.b[k].data) H[o++] = x;
        }
        *n_h = o;
    });
}

}  // extern "C"
