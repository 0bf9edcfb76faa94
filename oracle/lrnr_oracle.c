/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker.  It is never linked into the product library.
 *
 * Plain-C FP64 restatement of the reference's hot path (arXiv 2410.04001,
 * /root/reference/proj).  Every function cites the reference code it restates.
 * Extensions beyond the reference (which is tanh-only): the sin activation
 * (sigma = sin a, sigma' = cos a, sigma'' = -sin a, sigma''' = -cos a), used by
 * BASELINE configs 2-4; that branch is pinned by central finite differences and
 * an independent torch-FP64 autograd cross-check (tests/test_oracle.py).
 *
 * Flat layouts (shared with oracle/ref_harness.cpp and include/lrnr_gpu.h):
 *   LRNR params: per layer l: U_l (w[l+1] x r[l]), V_l (w[l] x r[l]), b_l (w[l+1]);
 *                = ParamPacker(BasesBiasesAndHyper) order (autodiff.cpp:926-934).
 *   Hyper params: per layer k: W_k (hw[k+1] x hw[k]), b_k (hw[k+1]) (autodiff.cpp:935-939).
 *   Fast params: v_in (m_in x r0); per inner l: u_hat (rh x r_l), b_hat (rh),
 *                v_hat (rh x r_{l+1}); u_out (m_out x r_{L-1}); b_out (m_out)
 *                (model.hpp:65-78).
 *
 * Batch drivers reproduce training::run_batch_gradient's deterministic
 * reduction (training.cpp:191-263): fixed chunks of `chunk` terms, values and
 * gradients accumulated in term order inside a chunk, chunks combined in index
 * order.  Results are therefore independent of the OpenMP thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXL 32
#define ORC_TWO_PI 6.283185307179586476925286766559
#define ACT_TANH 0
#define ACT_SIN 1

/* ------------------------------------------------------------------------ */
/* mt19937_64 + Rng (reference rng.hpp:13-44; std::mt19937_64 parameters)    */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t mt[312];
    int idx;
    int has_spare;
    double spare;
} orc_rng;

static void rng_seed(orc_rng* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
    g->has_spare = 0;
    g->spare = 0.0;
}

static uint64_t rng_raw(orc_rng* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= A;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static double rng_uniform(orc_rng* g) { return (double)(rng_raw(g) >> 11) * 0x1.0p-53; }
static double rng_uniform_in(orc_rng* g, double lo, double hi) { return lo + (hi - lo) * rng_uniform(g); }
static double rng_normal(orc_rng* g) {
    if (g->has_spare) {
        g->has_spare = 0;
        return g->spare;
    }
    double u1 = rng_uniform(g);
    while (u1 <= 0.0) u1 = rng_uniform(g);
    const double u2 = rng_uniform(g);
    const double r = sqrt(-2.0 * log(u1));
    const double th = 6.283185307179586476925286766559 * u2;
    g->spare = r * sin(th);
    g->has_spare = 1;
    return r * cos(th);
}

int orc_rng_stream(uint64_t seed, int64_t n, int kind, double* out, uint64_t* out_raw) {
    orc_rng g;
    rng_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) {
        if (kind == 0) out[i] = rng_uniform(&g);
        else if (kind == 1) out[i] = rng_normal(&g);
        else out_raw[i] = rng_raw(&g);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Seeded construction (model.cpp:433-515, pde.cpp:20-49)                    */
/* ------------------------------------------------------------------------ */
/* Modified Gram-Schmidt on the columns (model.cpp:433-450). */
static void mgs_columns(double* m, int64_t rows, int64_t cols) {
    for (int64_t j = 0; j < cols; ++j) {
        for (int64_t k = 0; k < j; ++k) {
            double dot = 0.0;
            for (int64_t i = 0; i < rows; ++i) dot += m[i * cols + j] * m[i * cols + k];
            for (int64_t i = 0; i < rows; ++i) m[i * cols + j] -= dot * m[i * cols + k];
        }
        double nrm = 0.0;
        for (int64_t i = 0; i < rows; ++i) nrm += m[i * cols + j] * m[i * cols + j];
        nrm = sqrt(nrm);
        if (nrm < 1e-12) {
            for (int64_t i = 0; i < rows; ++i) m[i * cols + j] = (i == j % rows) ? 1.0 : 0.0;
        } else {
            for (int64_t i = 0; i < rows; ++i) m[i * cols + j] /= nrm;
        }
    }
}

/* make_lrnr_params (model.cpp:454-478) on an existing stream. */
static void make_lrnr_on(orc_rng* g, int L, const int64_t* w, const int64_t* r, int ortho,
                         double bias_scale, double* out) {
    int64_t o = 0;
    for (int l = 0; l < L; ++l) {
        double* u = out + o;
        for (int64_t i = 0; i < w[l + 1] * r[l]; ++i) u[i] = rng_normal(g);
        o += w[l + 1] * r[l];
        double* v = out + o;
        for (int64_t i = 0; i < w[l] * r[l]; ++i) v[i] = rng_normal(g);
        o += w[l] * r[l];
        if (ortho) {
            mgs_columns(u, w[l + 1], r[l]);
            mgs_columns(v, w[l], r[l]);
        }
        for (int64_t i = 0; i < w[l + 1]; ++i) out[o + i] = rng_uniform_in(g, -bias_scale, bias_scale);
        o += w[l + 1];
    }
}

int orc_make_lrnr_params(int L, const int64_t* w, const int64_t* r, uint64_t seed, int ortho,
                         double bias_scale, double* out) {
    orc_rng g;
    rng_seed(&g, seed);
    make_lrnr_on(&g, L, w, r, ortho, bias_scale, out);
    return 0;
}

static int cmp_desc(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}

/* BASELINE.json config recipe. */
int orc_make_baseline_model(int L, const int64_t* w, const int64_t* r, uint64_t seed,
                            double* out_params, double* out_s) {
    orc_rng g;
    rng_seed(&g, seed);
    make_lrnr_on(&g, L, w, r, 1, 0.0, out_params);
    int64_t o = 0;
    for (int l = 0; l < L; ++l) {
        o += w[l + 1] * r[l] + w[l] * r[l];
        for (int64_t i = 0; i < w[l + 1]; ++i) out_params[o + i] = 0.1 * rng_normal(&g);
        o += w[l + 1];
    }
    int64_t so = 0;
    for (int l = 0; l < L; ++l) {
        for (int64_t j = 0; j < r[l]; ++j) out_s[so + j] = rng_uniform_in(&g, 0.0, 1.0);
        qsort(out_s + so, (size_t)r[l], sizeof(double), cmp_desc);
        so += r[l];
    }
    return 0;
}

/* make_hyper_params (model.cpp:480-504). */
static int64_t make_hyper_on(orc_rng* g, int L, const int64_t* split, int depth, int width,
                             double out_w_scale, double out_bias, double* out) {
    int64_t out_dim = 0;
    for (int l = 0; l < L; ++l) out_dim += split[l];
    int64_t fan_in = 3, o = 0;
    for (int k = 0; k < depth; ++k) {
        const double limit = sqrt(6.0 / (double)(fan_in + width));
        for (int64_t i = 0; i < width * fan_in; ++i) out[o + i] = rng_uniform_in(g, -limit, limit);
        o += width * fan_in;
        for (int64_t i = 0; i < width; ++i) out[o + i] = 0.0;
        o += width;
        fan_in = width;
    }
    for (int64_t i = 0; i < out_dim * fan_in; ++i) out[o + i] = out_w_scale * rng_normal(g);
    o += out_dim * fan_in;
    for (int64_t i = 0; i < out_dim; ++i) out[o + i] = out_bias;
    o += out_dim;
    return o;
}

int orc_make_hyper_params(int L, const int64_t* split, int depth, int width, uint64_t seed,
                          double out_w_scale, double out_bias, double* out) {
    orc_rng g;
    rng_seed(&g, seed);
    make_hyper_on(&g, L, split, depth, width, out_w_scale, out_bias, out);
    return 0;
}

/* sample_collocation (pde.cpp:20-49): x then t per interior point, mu draws interleaved. */
static void draw_mu(orc_rng* g, const double* lo, const double* hi, double* m) {
    m[0] = rng_uniform_in(g, lo[0], hi[0]);
    m[1] = rng_uniform_in(g, lo[1], hi[1]);
    m[2] = rng_uniform_in(g, lo[2], hi[2]);
}

int orc_sample_collocation(uint64_t seed, int64_t n_int, int64_t n_ic, int64_t n_per,
                           const double* lo, const double* hi, int with_mu, double* out_int,
                           double* out_ic, double* out_per, double* mu_int, double* mu_ic,
                           double* mu_per) {
    orc_rng g;
    rng_seed(&g, seed);
    for (int64_t i = 0; i < n_int; ++i) {
        out_int[2 * i] = rng_uniform_in(&g, 0.0, ORC_TWO_PI);
        out_int[2 * i + 1] = rng_uniform_in(&g, 0.0, 1.0);
        if (with_mu) draw_mu(&g, lo, hi, mu_int + 3 * i);
    }
    for (int64_t i = 0; i < n_ic; ++i) {
        out_ic[i] = rng_uniform_in(&g, 0.0, ORC_TWO_PI);
        if (with_mu) draw_mu(&g, lo, hi, mu_ic + 3 * i);
    }
    for (int64_t i = 0; i < n_per; ++i) {
        out_per[i] = rng_uniform_in(&g, 0.0, 1.0);
        if (with_mu) draw_mu(&g, lo, hi, mu_per + 3 * i);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* LRNR jet network (model.cpp:85-181; autodiff.cpp:463-563,644-666,720-730) */
/* ------------------------------------------------------------------------ */
typedef struct {
    int L, act;
    const int64_t *w, *r;
    const double* P;
    int64_t oU[ORC_MAXL], oV[ORC_MAXL], ob[ORC_MAXL], os[ORC_MAXL];
    int64_t n_params, r_total;
    /* workspace offsets (doubles) */
    int64_t oz[ORC_MAXL + 1], oa[ORC_MAXL + 1], oy[ORC_MAXL], ws_len, max_w, max_r;
} lr_net;

static void lr_init(lr_net* n, int L, const int64_t* w, const int64_t* r, const double* P, int act) {
    n->L = L;
    n->w = w;
    n->r = r;
    n->P = P;
    n->act = act;
    int64_t o = 0, so = 0, wo = 0;
    n->max_w = 0;
    n->max_r = 0;
    for (int l = 0; l < L; ++l) {
        n->oU[l] = o;
        o += w[l + 1] * r[l];
        n->oV[l] = o;
        o += w[l] * r[l];
        n->ob[l] = o;
        o += w[l + 1];
        n->os[l] = so;
        so += r[l];
        if (r[l] > n->max_r) n->max_r = r[l];
    }
    for (int l = 0; l <= L; ++l)
        if (w[l] > n->max_w) n->max_w = w[l];
    n->n_params = o;
    n->r_total = so;
    for (int l = 0; l <= L; ++l) {
        n->oz[l] = wo;
        wo += 4 * w[l];
        n->oa[l] = wo;
        wo += 4 * w[l];
    }
    for (int l = 0; l < L; ++l) {
        n->oy[l] = wo;
        wo += 4 * r[l];
    }
    n->ws_len = wo + 12 * n->max_r + 8 * n->max_w + 8;
}

/* activation jet forward (model.cpp:170-181) */
static void act_jet(int act, int64_t n, const double* in, double* out) {
    const double *v = in, *dx = in + n, *dt = in + 2 * n, *dxx = in + 3 * n;
    for (int64_t i = 0; i < n; ++i) {
        double sg, d1, d2;
        if (act == ACT_TANH) {
            sg = tanh(v[i]);
            d1 = 1.0 - sg * sg;
            d2 = -2.0 * sg * d1;
        } else {
            sg = sin(v[i]);
            d1 = cos(v[i]);
            d2 = -sg;
        }
        out[i] = sg;
        out[n + i] = d1 * dx[i];
        out[2 * n + i] = d1 * dt[i];
        out[3 * n + i] = d2 * dx[i] * dx[i] + d1 * dxx[i];
    }
}

/* activation jet VJP (autodiff.cpp:644-666; tanh derivatives from the stored
 * value, model.hpp:28-33); accumulates into gin (4n). */
static void act_jet_vjp(int act, int64_t n, const double* ain, const double* zout, const double* g,
                        double* gin) {
    for (int64_t i = 0; i < n; ++i) {
        double d1, d2, d3;
        if (act == ACT_TANH) {
            const double s = zout[i];
            d1 = 1.0 - s * s;
            d2 = -2.0 * s * (1.0 - s * s);
            const double e = 1.0 - s * s;
            d3 = -2.0 * e * e + 4.0 * s * s * e;
        } else {
            const double a = ain[i];
            d1 = cos(a);
            d2 = -sin(a);
            d3 = -cos(a);
        }
        const double ax = ain[n + i], at2 = ain[2 * n + i], aw = ain[3 * n + i];
        const double gv = g[i], gx = g[n + i], gt = g[2 * n + i], gw = g[3 * n + i];
        gin[i] += gv * d1 + gx * d2 * ax + gt * d2 * at2 + gw * (d3 * ax * ax + d2 * aw);
        gin[n + i] += gx * d1 + gw * 2.0 * d2 * ax;
        gin[2 * n + i] += gt * d1;
        gin[3 * n + i] += gw * d1;
    }
}

/* Forward jets through all layers; workspace holds z_l, a_l, y_l. */
static void lr_forward(const lr_net* n, const double* s, double x, double t, double* ws) {
    double* z0 = ws + n->oz[0];
    z0[0] = x;
    z0[1] = t;
    z0[2] = 1.0;
    z0[3] = 0.0;
    z0[4] = 0.0;
    z0[5] = 1.0;
    z0[6] = 0.0;
    z0[7] = 0.0;
    for (int l = 0; l < n->L; ++l) {
        const int64_t m_in = n->w[l], r = n->r[l], m_out = n->w[l + 1];
        const double* U = n->P + n->oU[l];
        const double* V = n->P + n->oV[l];
        const double* b = n->P + n->ob[l];
        const double* sl = s + n->os[l];
        const double* z = ws + n->oz[l];
        double* y = ws + n->oy[l];
        double* a = ws + n->oa[l + 1];
        /* jet_affine_factored (model.cpp:85-122) */
        for (int64_t j = 0; j < 4 * r; ++j) y[j] = 0.0;
        for (int64_t i = 0; i < m_in; ++i) {
            const double* row = V + i * r;
            const double av = z[i], ax = z[m_in + i], at = z[2 * m_in + i], aw = z[3 * m_in + i];
            for (int64_t j = 0; j < r; ++j) {
                y[j] += row[j] * av;
                y[r + j] += row[j] * ax;
                y[2 * r + j] += row[j] * at;
                y[3 * r + j] += row[j] * aw;
            }
        }
        for (int64_t i = 0; i < m_out; ++i) {
            const double* row = U + i * r;
            double accv = 0.0, accx = 0.0, acct = 0.0, accw = 0.0;
            for (int64_t j = 0; j < r; ++j) {
                const double us = row[j] * sl[j];
                accv += us * y[j];
                accx += us * y[r + j];
                acct += us * y[2 * r + j];
                accw += us * y[3 * r + j];
            }
            a[i] = accv + b[i];
            a[m_out + i] = accx;
            a[2 * m_out + i] = acct;
            a[3 * m_out + i] = accw;
        }
        if (l + 1 < n->L) act_jet(n->act, m_out, a, ws + n->oz[l + 1]);
    }
}

/* Reverse sweep from gout = d/d(a_L jet).  Accumulates ds (r_total) and, when
 * dP != NULL, dU/dV/db in the LRNR flat layout (autodiff.cpp:473-563). */
static void lr_backward(const lr_net* n, const double* s, double* ws, double* gA, double* ds,
                        double* dP) {
    const int64_t R = n->max_r;
    double* t = ws + n->ws_len - 12 * R - 8 * n->max_w - 8;
    double* sy = t + 4 * R;
    double* st = sy + 4 * R;
    double* gz = st + 4 * R;     /* 4 * max_w */
    double* gtmp = gz + 4 * n->max_w; /* 4 * max_w */
    for (int l = n->L - 1; l >= 0; --l) {
        const int64_t m_in = n->w[l], r = n->r[l], m_out = n->w[l + 1];
        const double* U = n->P + n->oU[l];
        const double* V = n->P + n->oV[l];
        const double* sl = s + n->os[l];
        const double* y = ws + n->oy[l];
        const double* z = ws + n->oz[l];
        const double *gv = gA, *gx = gA + m_out, *gt = gA + 2 * m_out, *gw = gA + 3 * m_out;
        for (int64_t j = 0; j < 4 * r; ++j) t[j] = 0.0;
        for (int64_t i = 0; i < m_out; ++i) {
            const double* row = U + i * r;
            const double a = gv[i], bx = gx[i], ct = gt[i], dw = gw[i];
            for (int64_t j = 0; j < r; ++j) {
                t[j] += row[j] * a;
                t[r + j] += row[j] * bx;
                t[2 * r + j] += row[j] * ct;
                t[3 * r + j] += row[j] * dw;
            }
        }
        if (dP) {
            double* bg = dP + n->ob[l];
            for (int64_t i = 0; i < m_out; ++i) bg[i] += gv[i];
        }
        {
            double* sg = ds + n->os[l];
            for (int64_t j = 0; j < r; ++j)
                sg[j] += t[j] * y[j] + t[r + j] * y[r + j] + t[2 * r + j] * y[2 * r + j] +
                         t[3 * r + j] * y[3 * r + j];
        }
        for (int64_t j = 0; j < r; ++j) {
            sy[j] = sl[j] * y[j];
            sy[r + j] = sl[j] * y[r + j];
            sy[2 * r + j] = sl[j] * y[2 * r + j];
            sy[3 * r + j] = sl[j] * y[3 * r + j];
            st[j] = sl[j] * t[j];
            st[r + j] = sl[j] * t[r + j];
            st[2 * r + j] = sl[j] * t[2 * r + j];
            st[3 * r + j] = sl[j] * t[3 * r + j];
        }
        if (dP) {
            double* ug = dP + n->oU[l];
            for (int64_t i = 0; i < m_out; ++i) {
                double* grow = ug + i * r;
                const double a = gv[i], bx = gx[i], ct = gt[i], dw = gw[i];
                for (int64_t j = 0; j < r; ++j)
                    grow[j] += a * sy[j] + bx * sy[r + j] + ct * sy[2 * r + j] + dw * sy[3 * r + j];
            }
        }
        for (int64_t i = 0; i < 4 * m_in; ++i) gz[i] = 0.0;
        double* vg = dP ? dP + n->oV[l] : NULL;
        for (int64_t i = 0; i < m_in; ++i) {
            const double* row = V + i * r;
            double av = 0.0, ax = 0.0, at2 = 0.0, aw = 0.0;
            for (int64_t j = 0; j < r; ++j) {
                av += row[j] * st[j];
                ax += row[j] * st[r + j];
                at2 += row[j] * st[2 * r + j];
                aw += row[j] * st[3 * r + j];
            }
            gz[i] += av;
            gz[m_in + i] += ax;
            gz[2 * m_in + i] += at2;
            gz[3 * m_in + i] += aw;
            if (vg) {
                double* grow = vg + i * r;
                const double zv = z[i], zx = z[m_in + i], zt = z[2 * m_in + i], zw = z[3 * m_in + i];
                for (int64_t j = 0; j < r; ++j)
                    grow[j] += zv * st[j] + zx * st[r + j] + zt * st[2 * r + j] + zw * st[3 * r + j];
            }
        }
        if (l > 0) {
            /* gradient w.r.t. a_l through the activation of layer l */
            for (int64_t i = 0; i < 4 * m_in; ++i) gtmp[i] = 0.0;
            act_jet_vjp(n->act, m_in, ws + n->oa[l], ws + n->oz[l], gz, gtmp);
            for (int64_t i = 0; i < 4 * m_in; ++i) gA[i] = gtmp[i];
        }
    }
}

/* residual (pde.cpp:9-13; autodiff.cpp:222-237) */
static double cdr_residual(const double* u, const double* mu) {
    const double uval = u[0], ux = u[1], ut = u[2], uxx = u[3];
    return ut + mu[0] * ux - mu[1] * uxx - mu[2] * uval * (1.0 - uval);
}

/* residual VJP (autodiff.cpp:720-730) */
static void cdr_vjp(const double* u, const double* mu, double g, double* gu) {
    gu[0] += g * (-mu[2] * (1.0 - 2.0 * u[0]));
    gu[1] += g * mu[0];
    gu[2] += g;
    gu[3] += -g * mu[1];
}

/* ------------------------------------------------------------------------ */
/* FastLRNR (autodiff.cpp:905-922 emitter; VJPs 564-643; model.cpp:124-168)  */
/* ------------------------------------------------------------------------ */
typedef struct {
    int L, act;
    const int64_t *r, *rh;
    int64_t m_in, m_out;
    const double* P;
    int64_t o_vin, o_uh[ORC_MAXL], o_bh[ORC_MAXL], o_vh[ORC_MAXL], o_uout, o_bout, os[ORC_MAXL];
    /* workspace: z_l (4 r_l), sc_l (4 r_l), h_l (4 rh_l), act_l (4 rh_l), u (4 m_out) */
    int64_t oz[ORC_MAXL], osc[ORC_MAXL], oh[ORC_MAXL], oact[ORC_MAXL], ou, ws_len, max_d;
    int64_t r_total;
} fa_net;

static void fa_init(fa_net* n, int L, const int64_t* r, const int64_t* rh, int64_t m_in,
                    int64_t m_out, const double* P, int act) {
    n->L = L;
    n->r = r;
    n->rh = rh;
    n->m_in = m_in;
    n->m_out = m_out;
    n->P = P;
    n->act = act;
    int64_t o = 0;
    n->o_vin = o;
    o += m_in * r[0];
    for (int l = 0; l + 1 < L; ++l) {
        n->o_uh[l] = o;
        o += rh[l] * r[l];
        n->o_bh[l] = o;
        o += rh[l];
        n->o_vh[l] = o;
        o += rh[l] * r[l + 1];
    }
    n->o_uout = o;
    o += m_out * r[L - 1];
    n->o_bout = o;
    int64_t so = 0, wo = 0, md = m_in > m_out ? m_in : m_out;
    for (int l = 0; l < L; ++l) {
        n->os[l] = so;
        so += r[l];
        if (r[l] > md) md = r[l];
        if (l + 1 < L && rh[l] > md) md = rh[l];
        n->oz[l] = wo;
        wo += 4 * r[l];
        n->osc[l] = wo;
        wo += 4 * r[l];
        if (l + 1 < L) {
            n->oh[l] = wo;
            wo += 4 * rh[l];
            n->oact[l] = wo;
            wo += 4 * rh[l];
        }
    }
    n->r_total = so;
    n->ou = wo;
    wo += 4 * m_out;
    n->max_d = md;
    n->ws_len = wo + 16 * md + 16;
}

/* jet_affine_dense (model.cpp:124-159) */
static void dense_jet(const double* A, int64_t rows, int64_t cols, int trans, const double* b,
                      const double* in, double* out) {
    if (!trans) {
        for (int64_t i = 0; i < rows; ++i) {
            const double* row = A + i * cols;
            double accv = 0.0, accx = 0.0, acct = 0.0, accw = 0.0;
            for (int64_t j = 0; j < cols; ++j) {
                accv += row[j] * in[j];
                accx += row[j] * in[cols + j];
                acct += row[j] * in[2 * cols + j];
                accw += row[j] * in[3 * cols + j];
            }
            out[i] = accv + (b ? b[i] : 0.0);
            out[rows + i] = accx;
            out[2 * rows + i] = acct;
            out[3 * rows + i] = accw;
        }
    } else {
        for (int64_t j = 0; j < cols; ++j) {
            out[j] = b ? b[j] : 0.0;
            out[cols + j] = 0.0;
            out[2 * cols + j] = 0.0;
            out[3 * cols + j] = 0.0;
        }
        for (int64_t i = 0; i < rows; ++i) {
            const double* row = A + i * cols;
            const double av = in[i], ax = in[rows + i], at = in[2 * rows + i], aw = in[3 * rows + i];
            for (int64_t j = 0; j < cols; ++j) {
                out[j] += row[j] * av;
                out[cols + j] += row[j] * ax;
                out[2 * cols + j] += row[j] * at;
                out[3 * cols + j] += row[j] * aw;
            }
        }
    }
}

/* jet_affine_dense VJP w.r.t. its input (autodiff.cpp:564-623), accumulate into gin. */
static void dense_jet_vjp(const double* A, int64_t rows, int64_t cols, int trans, const double* g,
                          double* gin) {
    if (!trans) {
        for (int64_t i = 0; i < rows; ++i) {
            const double* row = A + i * cols;
            const double cv = g[i], cx = g[rows + i], ct = g[2 * rows + i], cw = g[3 * rows + i];
            for (int64_t j = 0; j < cols; ++j) {
                gin[j] += row[j] * cv;
                gin[cols + j] += row[j] * cx;
                gin[2 * cols + j] += row[j] * ct;
                gin[3 * cols + j] += row[j] * cw;
            }
        }
    } else {
        for (int64_t i = 0; i < rows; ++i) {
            const double* row = A + i * cols;
            double av = 0.0, ax = 0.0, at2 = 0.0, aw = 0.0;
            for (int64_t j = 0; j < cols; ++j) {
                av += row[j] * g[j];
                ax += row[j] * g[cols + j];
                at2 += row[j] * g[2 * cols + j];
                aw += row[j] * g[3 * cols + j];
            }
            gin[i] += av;
            gin[rows + i] += ax;
            gin[2 * rows + i] += at2;
            gin[3 * rows + i] += aw;
        }
    }
}

static void scale_jet(const double* s, int64_t n, const double* in, double* out) {
    for (int64_t i = 0; i < n; ++i) {
        out[i] = s[i] * in[i];
        out[n + i] = s[i] * in[n + i];
        out[2 * n + i] = s[i] * in[2 * n + i];
        out[3 * n + i] = s[i] * in[3 * n + i];
    }
}

static void fa_forward(const fa_net* n, const double* s, double x, double t, double* ws) {
    double in[8] = {x, t, 1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
    /* the input jet has M_0 = m_in = 2 entries */
    dense_jet(n->P + n->o_vin, n->m_in, n->r[0], 1, NULL, in, ws + n->oz[0]);
    for (int l = 0; l + 1 < n->L; ++l) {
        scale_jet(s + n->os[l], n->r[l], ws + n->oz[l], ws + n->osc[l]);
        dense_jet(n->P + n->o_uh[l], n->rh[l], n->r[l], 0, n->P + n->o_bh[l], ws + n->osc[l],
                  ws + n->oh[l]);
        act_jet(n->act, n->rh[l], ws + n->oh[l], ws + n->oact[l]);
        dense_jet(n->P + n->o_vh[l], n->rh[l], n->r[l + 1], 1, NULL, ws + n->oact[l],
                  ws + n->oz[l + 1]);
    }
    const int Lm = n->L - 1;
    scale_jet(s + n->os[Lm], n->r[Lm], ws + n->oz[Lm], ws + n->osc[Lm]);
    dense_jet(n->P + n->o_uout, n->m_out, n->r[Lm], 0, n->P + n->o_bout, ws + n->osc[Lm], ws + n->ou);
}

/* Reverse from gu (4 m_out); accumulates ds. */
static void fa_backward(const fa_net* n, const double* s, double* ws, const double* gu, double* ds) {
    const int64_t D = n->max_d;
    double* gsc = ws + n->ws_len - 16 * D - 16;
    double* gz = gsc + 4 * D;
    double* gact = gz + 4 * D;
    double* gh = gact + 4 * D;
    const int Lm = n->L - 1;
    /* u_out affine VJP into the scaled jet */
    for (int64_t i = 0; i < 4 * n->r[Lm]; ++i) gsc[i] = 0.0;
    dense_jet_vjp(n->P + n->o_uout, n->m_out, n->r[Lm], 0, gu, gsc);
    for (int l = Lm; l >= 0; --l) {
        const int64_t rl = n->r[l];
        /* ScaleJet VJP (autodiff.cpp:624-643) */
        const double* sl = s + n->os[l];
        const double* inv = ws + n->oz[l];
        double* sg = ds + n->os[l];
        for (int64_t i = 0; i < 4 * rl; ++i) gz[i] = 0.0;
        for (int64_t i = 0; i < rl; ++i) {
            gz[i] += sl[i] * gsc[i];
            gz[rl + i] += sl[i] * gsc[rl + i];
            gz[2 * rl + i] += sl[i] * gsc[2 * rl + i];
            gz[3 * rl + i] += sl[i] * gsc[3 * rl + i];
            sg[i] += inv[i] * gsc[i] + inv[rl + i] * gsc[rl + i] + inv[2 * rl + i] * gsc[2 * rl + i] +
                     inv[3 * rl + i] * gsc[3 * rl + i];
        }
        if (l == 0) break; /* v_in is not trainable; the input-jet gradient is discarded */
        const int li = l - 1;
        const int64_t rh = n->rh[li];
        /* v_hat (trans) VJP into the activation output */
        for (int64_t i = 0; i < 4 * rh; ++i) gact[i] = 0.0;
        dense_jet_vjp(n->P + n->o_vh[li], rh, n->r[l], 1, gz, gact);
        for (int64_t i = 0; i < 4 * rh; ++i) gh[i] = 0.0;
        act_jet_vjp(n->act, rh, ws + n->oh[li], ws + n->oact[li], gact, gh);
        for (int64_t i = 0; i < 4 * n->r[li]; ++i) gsc[i] = 0.0;
        dense_jet_vjp(n->P + n->o_uh[li], rh, n->r[li], 0, gh, gsc);
    }
}

/* ------------------------------------------------------------------------ */
/* Batch drivers (training.cpp:191-263 reduction semantics)                  */
/* ------------------------------------------------------------------------ */
int orc_lrnr_grad(int L, const int64_t* w, const int64_t* r, const double* P, int act,
                  const double* s, const double* mu, const double* pts, int64_t n, double wt,
                  int64_t chunk, double* out_value, double* out_grad_s, double* out_grad_params,
                  double* out_terms) {
    if (L < 1 || L > ORC_MAXL || w[L] != 1 || chunk < 1) return 1;
    lr_net net;
    lr_init(&net, L, w, r, P, act);
    const int64_t n_chunks = (n + chunk - 1) / chunk;
    const int64_t G = net.r_total, GP = out_grad_params ? net.n_params : 0;
    const int64_t stride = 1 + G + GP;
    double* part = (double*)calloc((size_t)(n_chunks > 0 ? n_chunks : 1) * (size_t)stride, sizeof(double));
    int bad = 0;
#pragma omp parallel
    {
        double* ws = (double*)malloc((size_t)net.ws_len * sizeof(double));
        double* gA = (double*)malloc((size_t)(4 * net.max_w + 4) * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t c = 0; c < n_chunks; ++c) {
            double* pc = part + c * stride;
            const int64_t lo = c * chunk, hi = lo + chunk < n ? lo + chunk : n;
            for (int64_t i = lo; i < hi; ++i) {
                lr_forward(&net, s, pts[2 * i], pts[2 * i + 1], ws);
                const double* u = ws + net.oa[L];
                const double N = cdr_residual(u, mu);
                const double term = wt * (N * N);
                if (!isfinite(term)) {
#pragma omp atomic write
                    bad = 1;
                }
                if (out_terms) out_terms[i] = term;
                pc[0] += term;
                /* Scale -> Square -> ResidualCdr VJPs */
                const double gN = 2.0 * N * wt;
                gA[0] = gA[1] = gA[2] = gA[3] = 0.0;
                cdr_vjp(u, mu, gN, gA);
                lr_backward(&net, s, ws, gA, pc + 1, GP ? pc + 1 + G : NULL);
            }
        }
        free(ws);
        free(gA);
    }
    double v = 0.0;
    for (int64_t k = 0; k < G + GP; ++k) {
        double acc = 0.0;
        for (int64_t c = 0; c < n_chunks; ++c) acc += part[c * stride + 1 + k];
        if (k < G) out_grad_s[k] = acc;
        else out_grad_params[k - G] = acc;
    }
    for (int64_t c = 0; c < n_chunks; ++c) v += part[c * stride];
    *out_value = v;
    free(part);
    return bad ? 2 : 0;
}

int orc_lrnr_jets(int L, const int64_t* w, const int64_t* r, const double* P, int act,
                  const double* s, const double* pts, int64_t n, double* out_jets) {
    lr_net net;
    lr_init(&net, L, w, r, P, act);
#pragma omp parallel
    {
        double* ws = (double*)malloc((size_t)net.ws_len * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            lr_forward(&net, s, pts[2 * i], pts[2 * i + 1], ws);
            for (int k = 0; k < 4; ++k) out_jets[4 * i + k] = ws[net.oa[L] + k];
        }
        free(ws);
    }
    return 0;
}

int orc_fast_grad(int L, const int64_t* r, const int64_t* rh, int64_t m_in, int64_t m_out,
                  const double* P, int act, const double* s, const double* mu, const double* pts,
                  int64_t n, double wt, int64_t chunk, double* out_value, double* out_grad_s,
                  double* out_terms) {
    if (L < 2 || L > ORC_MAXL || m_out != 1 || m_in != 2 || chunk < 1) return 1;
    fa_net net;
    fa_init(&net, L, r, rh, m_in, m_out, P, act);
    const int64_t n_chunks = (n + chunk - 1) / chunk;
    const int64_t G = net.r_total, stride = 1 + G;
    double* part = (double*)calloc((size_t)(n_chunks > 0 ? n_chunks : 1) * (size_t)stride, sizeof(double));
    int bad = 0;
#pragma omp parallel
    {
        double* ws = (double*)malloc((size_t)net.ws_len * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t c = 0; c < n_chunks; ++c) {
            double* pc = part + c * stride;
            const int64_t lo = c * chunk, hi = lo + chunk < n ? lo + chunk : n;
            for (int64_t i = lo; i < hi; ++i) {
                fa_forward(&net, s, pts[2 * i], pts[2 * i + 1], ws);
                const double* u = ws + net.ou;
                const double N = cdr_residual(u, mu);
                const double term = wt * (N * N);
                if (!isfinite(term)) {
#pragma omp atomic write
                    bad = 1;
                }
                if (out_terms) out_terms[i] = term;
                pc[0] += term;
                double gu[4] = {0.0, 0.0, 0.0, 0.0};
                cdr_vjp(u, mu, 2.0 * N * wt, gu);
                fa_backward(&net, s, ws, gu, pc + 1);
            }
        }
        free(ws);
    }
    for (int64_t k = 0; k < G; ++k) {
        double acc = 0.0;
        for (int64_t c = 0; c < n_chunks; ++c) acc += part[c * stride + 1 + k];
        out_grad_s[k] = acc;
    }
    double v = 0.0;
    for (int64_t c = 0; c < n_chunks; ++c) v += part[c * stride];
    *out_value = v;
    free(part);
    return bad ? 2 : 0;
}

/* ------------------------------------------------------------------------ */
/* Full term set of one solve step: PinnTermEmitter fine-tune terms          */
/* (training.cpp:286-327: interior w N^2, initial w (u(x,0) - sin x)^2,      */
/* periodic w (u(0,t) - u(2pi,t))^2) or the fast-phase emitter's l1 terms    */
/* (training.cpp:521-549: |N|, |u - sin x|, |u(0,t) - u(2pi,t)|), plus the   */
/* locality term lambda * sum_l ||s_l - s_init_l||_1 (training.cpp:550-559,  */
/* L1ToTarget VJP autodiff.cpp:791-802).  Term order = the emitters' index   */
/* order: interior, initial, periodic, locality; run_batch_gradient's fixed  */
/* chunking (training.cpp:191-263).  model 0 = LRNR (P = LrnrParams flat,    */
/* dims L, w, r), 1 = FastLRNR (P = FastParams flat, dims L, r, rh, m_in =   */
/* w[0], m_out = w[1]).  objective 0 = squared (Scale(Square(.)) VJP         */
/* 2 * r * w), 1 = abs (Abs VJP sgn, 0 at 0; autodiff.cpp:745-750).          */
/* comps = {residual, boundary, sparse (0), local}.                          */
/* ------------------------------------------------------------------------ */
typedef struct {
    int kind;
    lr_net lr;
    fa_net fa;
    int64_t ws_len, g_len, r_total;
} any_net;

static const double* any_fwd(const any_net* a, const double* s, double x, double t, double* ws) {
    if (a->kind == 0) {
        lr_forward(&a->lr, s, x, t, ws);
        return ws + a->lr.oa[a->lr.L];
    }
    fa_forward(&a->fa, s, x, t, ws);
    return ws + a->fa.ou;
}

/* gA: scratch of g_len doubles whose first 4 entries are the output-jet seed */
static void any_bwd(const any_net* a, const double* s, double* ws, double* gA, double* ds, double* dP) {
    if (a->kind == 0) lr_backward(&a->lr, s, ws, gA, ds, dP);
    else fa_backward(&a->fa, s, ws, gA, ds);
}

static double sgn0(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

int orc_terms_grad(int model, int L, const int64_t* w, const int64_t* r, const int64_t* rh, const double* P,
                   int act, const double* s, const double* mu, const double* pts, int64_t n_int,
                   const double* ic_x, int64_t n_ic, const double* per_t, int64_t n_bc, double w_int,
                   double w_ic, double w_bc, int objective, const double* s_init, double lambda_local,
                   int64_t chunk, double* out_value, double* out_comps, double* out_grad_s,
                   double* out_grad_params) {
    if (L < 1 || L > ORC_MAXL || chunk < 1 || (objective != 0 && objective != 1)) return 1;
    if (out_grad_params && model != 0) return 1;
    any_net a;
    memset(&a, 0, sizeof(a));
    a.kind = model;
    if (model == 0) {
        if (w[L] != 1) return 1;
        lr_init(&a.lr, L, w, r, P, act);
        a.ws_len = a.lr.ws_len;
        a.g_len = 4 * a.lr.max_w + 4;
        a.r_total = a.lr.r_total;
    } else {
        if (w[0] != 2 || w[1] != 1 || L < 2) return 1;
        fa_init(&a.fa, L, r, rh, w[0], w[1], P, act);
        a.ws_len = a.fa.ws_len;
        a.g_len = 4;
        a.r_total = a.fa.r_total;
    }
    const int has_local = s_init != NULL && lambda_local > 0.0;
    const int64_t n_terms = n_int + n_ic + n_bc + (has_local ? 1 : 0);
    const int64_t n_chunks = (n_terms + chunk - 1) / chunk;
    const int64_t G = a.r_total, GP = out_grad_params ? a.lr.n_params : 0;
    const int64_t stride = 5 + G + GP; /* value, comps[4], grad_s, grad_params */
    double* part = (double*)calloc((size_t)(n_chunks > 0 ? n_chunks : 1) * (size_t)stride, sizeof(double));
    int bad = 0;
#pragma omp parallel
    {
        double* ws0 = (double*)malloc((size_t)a.ws_len * sizeof(double));
        double* ws1 = (double*)malloc((size_t)a.ws_len * sizeof(double));
        double* g0 = (double*)malloc((size_t)a.g_len * sizeof(double));
        double* g1 = (double*)malloc((size_t)a.g_len * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t c = 0; c < n_chunks; ++c) {
            double* pc = part + c * stride;
            const int64_t lo = c * chunk, hi = lo + chunk < n_terms ? lo + chunk : n_terms;
            for (int64_t idx = lo; idx < hi; ++idx) {
                double term;
                int comp;
                for (int k = 0; k < 4; ++k) g0[k] = g1[k] = 0.0;
                if (idx < n_int) {
                    const double* u = any_fwd(&a, s, pts[2 * idx], pts[2 * idx + 1], ws0);
                    const double N = cdr_residual(u, mu);
                    double gN;
                    if (objective == 0) {
                        term = w_int * (N * N);
                        gN = 2.0 * N * w_int;
                    } else {
                        term = w_int * fabs(N);
                        gN = sgn0(N) * w_int;
                    }
                    cdr_vjp(u, mu, gN, g0);
                    any_bwd(&a, s, ws0, g0, pc + 5, GP ? pc + 5 + G : NULL);
                    comp = 0;
                } else if (idx < n_int + n_ic) {
                    const double x = ic_x[idx - n_int];
                    const double* u = any_fwd(&a, s, x, 0.0, ws0);
                    const double d = u[0] - sin(x);
                    if (objective == 0) {
                        term = w_ic * (d * d);
                        g0[0] = 2.0 * d * w_ic;
                    } else {
                        term = w_ic * fabs(d);
                        g0[0] = sgn0(d) * w_ic;
                    }
                    any_bwd(&a, s, ws0, g0, pc + 5, GP ? pc + 5 + G : NULL);
                    comp = 1;
                } else if (idx < n_int + n_ic + n_bc) {
                    const double t = per_t[idx - n_int - n_ic];
                    const double* u0 = any_fwd(&a, s, 0.0, t, ws0);
                    const double* u1 = any_fwd(&a, s, ORC_TWO_PI, t, ws1);
                    const double d = u0[0] - u1[0];
                    double gd;
                    if (objective == 0) {
                        term = w_bc * (d * d);
                        gd = 2.0 * d * w_bc;
                    } else {
                        term = w_bc * fabs(d);
                        gd = sgn0(d) * w_bc;
                    }
                    g0[0] = gd;
                    g1[0] = -gd;
                    any_bwd(&a, s, ws0, g0, pc + 5, GP ? pc + 5 + G : NULL);
                    any_bwd(&a, s, ws1, g1, pc + 5, GP ? pc + 5 + G : NULL);
                    comp = 1;
                } else {
                    term = 0.0;
                    for (int64_t i = 0; i < G; ++i) {
                        const double d = s[i] - s_init[i];
                        term += fabs(d);
                        pc[5 + i] += lambda_local * sgn0(d);
                    }
                    term *= lambda_local;
                    comp = 3;
                }
                if (!isfinite(term)) {
#pragma omp atomic write
                    bad = 1;
                }
                pc[0] += term;
                pc[1 + comp] += term;
            }
        }
        free(ws0);
        free(ws1);
        free(g0);
        free(g1);
    }
    for (int64_t k = 0; k < 5 + G + GP; ++k) {
        double acc = 0.0;
        for (int64_t c = 0; c < n_chunks; ++c) acc += part[c * stride + k];
        if (k == 0) *out_value = acc;
        else if (k < 5) out_comps[k - 1] = acc;
        else if (k < 5 + G) out_grad_s[k - 5] = acc;
        else out_grad_params[k - 5 - G] = acc;
    }
    free(part);
    return bad ? 2 : 0;
}

/* Tape::banded_decay_penalty (autodiff.cpp:346-360) and its VJP (:779-790):
 * returns sum_i ReLU(-f_i + gamma f_{i+1}); g[i] -= coef, g[i+1] += gamma coef
 * where the hinge is active. */
double orc_banded_decay(const double* f, int64_t n, double gamma, double coef, double* g) {
    double acc = 0.0;
    for (int64_t i = 0; i + 1 < n; ++i) {
        const double arg = -f[i] + gamma * f[i + 1];
        if (arg > 0.0) {
            acc += arg;
            if (g) {
                g[i] -= coef;
                g[i + 1] += gamma * coef;
            }
        }
    }
    return acc;
}

/* Tape::gram_ortho_penalty (autodiff.cpp:322-342) and the GramOrtho VJP
 * (:761-777): returns ||A^T A - I||_F^2 of a rows x r row-major A;
 * gA += 4 coef A E with E = A^T A - I. */
double orc_gram_penalty(const double* A, int64_t rows, int64_t r, double coef, double* gA) {
    double* e = (double*)malloc((size_t)(r * r) * sizeof(double));
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < r; ++j) {
            double dot = 0.0;
            for (int64_t k = 0; k < rows; ++k) dot += A[k * r + i] * A[k * r + j];
            e[i * r + j] = dot - (i == j ? 1.0 : 0.0);
        }
    double acc = 0.0;
    for (int64_t i = 0; i < r * r; ++i) acc += e[i] * e[i];
    if (gA)
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < r; ++j) {
                double a = 0.0;
                for (int64_t k = 0; k < r; ++k) a += A[i * r + k] * e[k * r + j];
                gA[i * r + j] += 4.0 * coef * a;
            }
    free(e);
    return acc;
}

int orc_fast_jets(int L, const int64_t* r, const int64_t* rh, int64_t m_in, int64_t m_out,
                  const double* P, int act, const double* s, const double* pts, int64_t n,
                  double* out_jets) {
    fa_net net;
    fa_init(&net, L, r, rh, m_in, m_out, P, act);
#pragma omp parallel
    {
        double* ws = (double*)malloc((size_t)net.ws_len * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            fa_forward(&net, s, pts[2 * i], pts[2 * i + 1], ws);
            for (int k = 0; k < 4; ++k) out_jets[4 * i + k] = ws[net.ou + k];
        }
        free(ws);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Hypernetwork (model.cpp:74-81,294-318; autodiff.cpp:155-209,667-714,883-903) */
/* ------------------------------------------------------------------------ */
typedef struct {
    int K;
    const int64_t* hw; /* K+1 */
    const double* P;
    const double *lo, *hi;
    int64_t oW[ORC_MAXL], ob[ORC_MAXL], n_params, max_w;
} hy_net;

static void hy_init(hy_net* h, int K, const int64_t* hw, const double* P, const double* lo,
                    const double* hi) {
    h->K = K;
    h->hw = hw;
    h->P = P;
    h->lo = lo;
    h->hi = hi;
    int64_t o = 0;
    h->max_w = 3;
    for (int k = 0; k < K; ++k) {
        h->oW[k] = o;
        o += hw[k + 1] * hw[k];
        h->ob[k] = o;
        o += hw[k + 1];
        if (hw[k + 1] > h->max_w) h->max_w = hw[k + 1];
    }
    h->n_params = o;
}

/* acts: (K+1) * max_w, acts[k] = input of layer k (acts[0] = normalized mu);
 * acts[K] = ReLU output. */
static void hy_forward(const hy_net* h, const double* mu, double* acts) {
    const int64_t MW = h->max_w;
    for (int i = 0; i < 3; ++i) {
        const double extent = h->hi[i] - h->lo[i];
        acts[i] = extent > 0.0 ? (mu[i] - h->lo[i]) / extent : 0.0;
    }
    for (int k = 0; k < h->K; ++k) {
        const double* W = h->P + h->oW[k];
        const double* b = h->P + h->ob[k];
        const double* in = acts + k * MW;
        double* out = acts + (k + 1) * MW;
        const int64_t rows = h->hw[k + 1], cols = h->hw[k];
        for (int64_t i = 0; i < rows; ++i) {
            double acc = 0.0;
            for (int64_t j = 0; j < cols; ++j) acc += W[i * cols + j] * in[j];
            const double a = acc + b[i];
            if (k + 1 < h->K) out[i] = tanh(a);
            else out[i] = a > 0.0 ? a : 0.0;
        }
    }
}

/* J^T g_s accumulated into dH (hyper flat layout). */
static void hy_backward(const hy_net* h, const double* acts, const double* g_s, double* dH,
                        double* scratch /* 2*max_w */) {
    const int64_t MW = h->max_w;
    double* g = scratch;
    double* gin = scratch + MW;
    const int K = h->K;
    const int64_t out_dim = h->hw[K];
    const double* outv = acts + K * MW;
    for (int64_t i = 0; i < out_dim; ++i) g[i] = (outv[i] > 0.0) ? g_s[i] : 0.0; /* ReLU VJP */
    for (int k = K - 1; k >= 0; --k) {
        const double* W = h->P + h->oW[k];
        const int64_t rows = h->hw[k + 1], cols = h->hw[k];
        const double* in = acts + k * MW;
        double* wg = dH + h->oW[k];
        double* bg = dH + h->ob[k];
        for (int64_t j = 0; j < cols; ++j) gin[j] = 0.0;
        for (int64_t i = 0; i < rows; ++i) {
            const double gi = g[i];
            for (int64_t j = 0; j < cols; ++j) {
                gin[j] += W[i * cols + j] * gi;
                wg[i * cols + j] += gi * in[j];
            }
        }
        for (int64_t i = 0; i < rows; ++i) bg[i] += g[i];
        if (k > 0) {
            /* TanhVec VJP: sigma is the input of layer k (output of tanh k-1) */
            for (int64_t j = 0; j < cols; ++j) g[j] = gin[j] * (1.0 - in[j] * in[j]);
        }
    }
}

int orc_hyper_forward(int K, const int64_t* hw, const double* P, const double* lo, const double* hi,
                      const double* mu, double* out_s) {
    hy_net h;
    hy_init(&h, K, hw, P, lo, hi);
    double* acts = (double*)malloc((size_t)((K + 1) * h.max_w) * sizeof(double));
    hy_forward(&h, mu, acts);
    for (int64_t i = 0; i < hw[K]; ++i) out_s[i] = acts[K * h.max_w + i];
    free(acts);
    return 0;
}

int orc_hyper_vjp(int K, const int64_t* hw, const double* P, const double* lo, const double* hi,
                  const double* mu, const double* g_s, double* out_grad /* accumulated */) {
    hy_net h;
    hy_init(&h, K, hw, P, lo, hi);
    double* acts = (double*)malloc((size_t)((K + 1) * h.max_w) * sizeof(double));
    double* sc = (double*)malloc((size_t)(2 * h.max_w) * sizeof(double));
    hy_forward(&h, mu, acts);
    hy_backward(&h, acts, g_s, out_grad, sc);
    free(acts);
    free(sc);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* End-to-end meta-training replica (training.cpp:20-26,30-105,265-426;     */
/* autodiff.cpp:322-380,761-804,1062-1075).                                   */
/* ------------------------------------------------------------------------ */
static uint64_t epoch_seed(uint64_t base, int64_t epoch) {
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (uint64_t)(epoch + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* One PinnTermEmitter term in meta mode (training.cpp:278-328), accumulating
 * into chunk accumulators gl (LRNR) and gh (hyper). kind 0 interior, 1 initial,
 * 2 periodic. Returns term value; comps updated. */
static double meta_term(const lr_net* net, const hy_net* hy, int kind, double a0, double a1,
                        const double* mu, double wt, double lambda_sparse, double gamma,
                        double* ws0, double* ws1, double* gA, double* acts, double* s,
                        double* gs, double* hsc, double* gl, double* gh, double* comps) {
    const int L = net->L;
    const int64_t Rt = net->r_total, MW = hy->max_w;
    hy_forward(hy, mu, acts);
    for (int64_t i = 0; i < Rt; ++i) s[i] = acts[hy->K * MW + i];
    for (int64_t i = 0; i < Rt; ++i) gs[i] = 0.0;
    double value;
    if (kind == 0) {
        lr_forward(net, s, a0, a1, ws0);
        const double* u = ws0 + net->oa[L];
        const double N = cdr_residual(u, mu);
        const double term = wt * (N * N);
        comps[0] += term;
        value = term;
        double gterm = 1.0;
        if (lambda_sparse > 0.0) {
            /* weighted_sum(term, bd_l...) with weights 1, lambda*w (autodiff.cpp:304-320) */
            const double wsp = lambda_sparse * wt;
            double acc = 0.0;
            acc += 1.0 * term;
            for (int l = 0; l < L; ++l) {
                const double* f = s + net->os[l];
                double bd = 0.0;
                for (int64_t i = 0; i + 1 < net->r[l]; ++i) {
                    const double arg = -f[i] + gamma * f[i + 1];
                    if (arg > 0.0) bd += arg;
                }
                acc += wsp * bd;
            }
            comps[2] += acc - term;
            value = acc;
            gterm = 1.0 * 1.0;
            /* banded decay VJPs, last created first (autodiff.cpp:780-792) */
            for (int l = L - 1; l >= 0; --l) {
                const double* f = s + net->os[l];
                double* ing = gs + net->os[l];
                const double g = wsp * 1.0;
                for (int64_t i = 0; i + 1 < net->r[l]; ++i) {
                    if (-f[i] + gamma * f[i + 1] > 0.0) {
                        ing[i] -= g;
                        ing[i + 1] += gamma * g;
                    }
                }
            }
        }
        const double gsq = wt * gterm;
        const double gN = 2.0 * N * gsq;
        gA[0] = gA[1] = gA[2] = gA[3] = 0.0;
        cdr_vjp(u, mu, gN, gA);
        lr_backward(net, s, ws0, gA, gs, gl);
    } else if (kind == 1) {
        lr_forward(net, s, a0, 0.0, ws0);
        const double u = ws0[net->oa[L]];
        const double rr = u - sin(a0);
        const double term = wt * (rr * rr);
        comps[1] += term;
        value = term;
        gA[0] = gA[1] = gA[2] = gA[3] = 0.0;
        gA[0] += 2.0 * rr * wt;
        lr_backward(net, s, ws0, gA, gs, gl);
    } else {
        lr_forward(net, s, 0.0, a1, ws0);
        lr_forward(net, s, ORC_TWO_PI, a1, ws1);
        const double rr = ws0[net->oa[L]] - ws1[net->oa[L]];
        const double term = wt * (rr * rr);
        comps[1] += term;
        value = term;
        const double g = 2.0 * rr * wt;
        /* jet1 (created last) is reversed first */
        gA[0] = gA[1] = gA[2] = gA[3] = 0.0;
        gA[0] -= g;
        lr_backward(net, s, ws1, gA, gs, gl);
        gA[0] = gA[1] = gA[2] = gA[3] = 0.0;
        gA[0] += g;
        lr_backward(net, s, ws0, gA, gs, gl);
    }
    hy_backward(hy, acts, gs, gh, hsc);
    return value;
}

int orc_meta_train(int L, const int64_t* w, const int64_t* r, int hyper_depth, int hyper_width,
                   double init_bias_scale, double out_w_scale, double out_bias, uint64_t init_seed,
                   const double* lo, const double* hi, double lr, int64_t epochs, int64_t n_int,
                   int64_t n_ic, int64_t n_per, uint64_t seed, double lambda_ortho,
                   double lambda_sparse, double gamma, int64_t chunk, double* out_best_loss,
                   int64_t* out_best_epoch, double* out_losses) {
    int64_t r_total = 0;
    for (int l = 0; l < L; ++l) r_total += r[l];
    const int hwid = hyper_width > 0 ? hyper_width : (int)(r_total > 64 ? r_total : 64);
    int64_t hw[ORC_MAXL];
    hw[0] = 3;
    for (int k = 0; k < hyper_depth; ++k) hw[k + 1] = hwid;
    hw[hyper_depth + 1] = r_total;
    const int K = hyper_depth + 1;

    lr_net net;
    int64_t n_lr = 0;
    for (int l = 0; l < L; ++l) n_lr += w[l + 1] * r[l] + w[l] * r[l] + w[l + 1];
    int64_t n_hy = 0;
    for (int k = 0; k < K; ++k) n_hy += hw[k + 1] * hw[k] + hw[k + 1];
    const int64_t NP = n_lr + n_hy;
    double* x = (double*)calloc((size_t)NP, sizeof(double));
    orc_rng g;
    rng_seed(&g, init_seed);
    make_lrnr_on(&g, L, w, r, 1, init_bias_scale, x);
    make_hyper_on(&g, L, r, hyper_depth, hwid, out_w_scale, out_bias, x + n_lr);
    lr_init(&net, L, w, r, x, ACT_TANH);
    hy_net hy;
    hy_init(&hy, K, hw, x + n_lr, lo, hi);

    double* m = (double*)calloc((size_t)NP, sizeof(double));
    double* v = (double*)calloc((size_t)NP, sizeof(double));
    double* gtot = (double*)calloc((size_t)NP, sizeof(double));
    double best = INFINITY;
    int64_t best_e = 0;
    int64_t t_adam = 0;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;

    for (int64_t e = 1; e <= epochs; ++e) {
        const int64_t nt = n_int + n_ic + n_per;
        double* pint = (double*)malloc((size_t)(2 * n_int + 1) * sizeof(double));
        double* pic = (double*)malloc((size_t)(n_ic + 1) * sizeof(double));
        double* pper = (double*)malloc((size_t)(n_per + 1) * sizeof(double));
        double* mint = (double*)malloc((size_t)(3 * n_int + 1) * sizeof(double));
        double* mic = (double*)malloc((size_t)(3 * n_ic + 1) * sizeof(double));
        double* mper = (double*)malloc((size_t)(3 * n_per + 1) * sizeof(double));
        orc_sample_collocation(epoch_seed(seed, e), n_int, n_ic, n_per, lo, hi, 1, pint, pic, pper,
                               mint, mic, mper);
        const double w_int = n_int ? 1.0 / (double)n_int : 0.0;
        const double w_ic = n_ic ? 1.0 / (double)n_ic : 0.0;
        const double w_per = n_per ? 1.0 / (double)n_per : 0.0;
        const int64_t n_chunks = (nt + chunk - 1) / chunk;
        const int64_t stride = 1 + 4 + NP;
        double* part = (double*)calloc((size_t)(n_chunks > 0 ? n_chunks : 1) * (size_t)stride, sizeof(double));
#pragma omp parallel
        {
            double* ws0 = (double*)malloc((size_t)net.ws_len * sizeof(double));
            double* ws1 = (double*)malloc((size_t)net.ws_len * sizeof(double));
            double* gA = (double*)malloc((size_t)(4 * net.max_w + 4) * sizeof(double));
            double* acts = (double*)malloc((size_t)((K + 1) * hy.max_w) * sizeof(double));
            double* s = (double*)malloc((size_t)r_total * sizeof(double));
            double* gs = (double*)malloc((size_t)r_total * sizeof(double));
            double* hsc = (double*)malloc((size_t)(2 * hy.max_w) * sizeof(double));
#pragma omp for schedule(static)
            for (int64_t c = 0; c < n_chunks; ++c) {
                double* pc = part + c * stride;
                const int64_t clo = c * chunk, chi = clo + chunk < nt ? clo + chunk : nt;
                for (int64_t i = clo; i < chi; ++i) {
                    double val;
                    if (i < n_int)
                        val = meta_term(&net, &hy, 0, pint[2 * i], pint[2 * i + 1], mint + 3 * i, w_int,
                                        lambda_sparse, gamma, ws0, ws1, gA, acts, s, gs, hsc,
                                        pc + 5, pc + 5 + n_lr, pc + 1);
                    else if (i < n_int + n_ic) {
                        const int64_t j = i - n_int;
                        val = meta_term(&net, &hy, 1, pic[j], 0.0, mic + 3 * j, w_ic, 0.0, gamma, ws0,
                                        ws1, gA, acts, s, gs, hsc, pc + 5, pc + 5 + n_lr, pc + 1);
                    } else {
                        const int64_t j = i - n_int - n_ic;
                        val = meta_term(&net, &hy, 2, 0.0, pper[j], mper + 3 * j, w_per, 0.0, gamma,
                                        ws0, ws1, gA, acts, s, gs, hsc, pc + 5, pc + 5 + n_lr, pc + 1);
                    }
                    pc[0] += val;
                }
            }
            free(ws0);
            free(ws1);
            free(gA);
            free(acts);
            free(s);
            free(gs);
            free(hsc);
        }
        double bg_value = 0.0;
        for (int64_t c = 0; c < n_chunks; ++c) bg_value += part[c * stride];
        for (int64_t k = 0; k < NP; ++k) {
            double acc = 0.0;
            for (int64_t c = 0; c < n_chunks; ++c) acc += part[c * stride + 5 + k];
            gtot[k] = acc;
        }
        free(part);
        free(pint);
        free(pic);
        free(pper);
        free(mint);
        free(mic);
        free(mper);

        /* orthogonality regularizer: weighted_sum of gram penalties (training.cpp:379-391,
         * autodiff.cpp:322-344,761-779) */
        double ro_value = 0.0;
        {
            double acc = 0.0;
            for (int l = 0; l < L; ++l) {
                for (int which = 0; which < 2; ++which) {
                    const int64_t rows = which == 0 ? w[l + 1] : w[l], rr = r[l];
                    const double* A = x + (which == 0 ? net.oU[l] : net.oV[l]);
                    double* E = (double*)malloc((size_t)(rr * rr) * sizeof(double));
                    for (int64_t i = 0; i < rr; ++i)
                        for (int64_t j = 0; j < rr; ++j) {
                            double dot = 0.0;
                            for (int64_t k = 0; k < rows; ++k) dot += A[k * rr + i] * A[k * rr + j];
                            E[i * rr + j] = dot - (i == j ? 1.0 : 0.0);
                        }
                    double pen = 0.0;
                    for (int64_t i = 0; i < rr * rr; ++i) pen += E[i] * E[i];
                    acc += lambda_ortho * pen;
                    const double gg = lambda_ortho * 1.0;
                    /* ro.grad is combined with bg.grad below: g = bg + ro */
                    double* og = (double*)calloc((size_t)(rows * rr), sizeof(double));
                    for (int64_t i = 0; i < rows; ++i)
                        for (int64_t j = 0; j < rr; ++j) {
                            double a2 = 0.0;
                            for (int64_t k = 0; k < rr; ++k) a2 += A[i * rr + k] * E[k * rr + j];
                            og[i * rr + j] += 4.0 * gg * a2;
                        }
                    double* tgt = gtot + (which == 0 ? net.oU[l] : net.oV[l]);
                    for (int64_t i = 0; i < rows * rr; ++i) tgt[i] = tgt[i] + og[i];
                    free(og);
                    free(E);
                }
            }
            ro_value = acc;
        }
        const double loss = bg_value + ro_value;
        if (out_losses) out_losses[e - 1] = loss;
        if (loss < best) {
            best = loss;
            best_e = e;
        }
        /* adam_step (autodiff.cpp:1062-1075) */
        t_adam += 1;
        const double b1t = 1.0 - pow(b1, (double)t_adam);
        const double b2t = 1.0 - pow(b2, (double)t_adam);
        for (int64_t i = 0; i < NP; ++i) {
            m[i] = b1 * m[i] + (1.0 - b1) * gtot[i];
            v[i] = b2 * v[i] + (1.0 - b2) * gtot[i] * gtot[i];
            const double mhat = m[i] / b1t;
            const double vhat = v[i] / b2t;
            x[i] -= lr * mhat / (sqrt(vhat) + eps);
        }
    }
    *out_best_loss = best;
    *out_best_epoch = best_e;
    free(x);
    free(m);
    free(v);
    free(gtot);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* The solve loops (training.cpp:428-607): fine_tune and fast_solve.         */
/* Initial coefficients s_init stand for hyper_forward(mu, theta).           */
/* Per epoch: the term gradient (orc_terms_grad), the EpochRecord loss, the  */
/* divergence stop (fast_solve: loss > 1e3 x the first loss), best-iterate,  */
/* adam_step (autodiff.cpp:1062-1075, beta 0.9 / 0.999, eps 1e-8) and        */
/* project_nonnegative_coeffs (autodiff.cpp:967-977).  NonFiniteError ->     */
/* aborted (+ diverged in fast_solve) and stop.  flags: 1 aborted, 2 diverged.*/
/* ------------------------------------------------------------------------ */
static int solve_loop(int model, int L, const int64_t* w, const int64_t* r, const int64_t* rh, const double* P,
                      int act, const double* s_init, const double* mu, double lr, int64_t epochs, int fast,
                      /* fine_tune batch recipe */ int64_t n_int, int64_t n_ic, int64_t n_bc, uint64_t seed,
                      /* fast_solve sampling set (classified) */ const double* fx_int, int64_t fn_int,
                      const double* fx_ic, int64_t fn_ic, const double* fx_bc, int64_t fn_bc, double lambda_local,
                      int64_t chunk, double* out_s, double* out_best_loss, int64_t* out_best_epoch,
                      double* out_losses, int64_t* out_n_records, int* out_flags) {
    int64_t G = 0;
    for (int l = 0; l < L; ++l) G += r[l];
    double* x = (double*)malloc((size_t)G * sizeof(double));
    double* best = (double*)malloc((size_t)G * sizeof(double));
    double* m = (double*)calloc((size_t)G, sizeof(double));
    double* v = (double*)calloc((size_t)G, sizeof(double));
    double* g = (double*)malloc((size_t)G * sizeof(double));
    memcpy(x, s_init, (size_t)G * sizeof(double));
    memcpy(best, s_init, (size_t)G * sizeof(double));
    double best_loss = INFINITY, initial = NAN, comps[4];
    int64_t best_e = 0, n_rec = 0, t_adam = 0;
    int flags = 0, rc = 0;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    double* pint = (double*)malloc((size_t)(2 * n_int + 1) * sizeof(double));
    double* pic = (double*)malloc((size_t)(n_ic + 1) * sizeof(double));
    double* pper = (double*)malloc((size_t)(n_bc + 1) * sizeof(double));
    for (int64_t e = 1; e <= epochs; ++e) {
        double value;
        int st;
        if (!fast) {
            const double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
            orc_sample_collocation(epoch_seed(seed, e), n_int, n_ic, n_bc, lo, hi, 0, pint, pic, pper, NULL, NULL,
                                   NULL);
            st = orc_terms_grad(model, L, w, r, rh, P, act, x, mu, pint, n_int, pic, n_ic, pper, n_bc,
                                n_int ? 1.0 / (double)n_int : 0.0, n_ic ? 1.0 / (double)n_ic : 0.0,
                                n_bc ? 1.0 / (double)n_bc : 0.0, 0, NULL, 0.0, chunk, &value, comps, g, NULL);
        } else {
            st = orc_terms_grad(model, L, w, r, rh, P, act, x, mu, fx_int, fn_int, fx_ic, fn_ic, fx_bc, fn_bc, 1.0,
                                1.0, 1.0, 1, lambda_local > 0.0 ? s_init : NULL, lambda_local, chunk, &value, comps,
                                g, NULL);
        }
        if (st == 1) {
            rc = 1;
            break;
        }
        if (st == 2) {
            flags |= fast ? 3 : 1;
            break;
        }
        out_losses[n_rec++] = value;
        if (fast) {
            if (e == 1) initial = value;
            if (value > 1e3 * initial) {
                flags |= 2;
                break;
            }
        }
        if (value < best_loss) {
            best_loss = value;
            best_e = e;
            memcpy(best, x, (size_t)G * sizeof(double));
        }
        t_adam += 1;
        const double b1t = 1.0 - pow(b1, (double)t_adam);
        const double b2t = 1.0 - pow(b2, (double)t_adam);
        for (int64_t i = 0; i < G; ++i) {
            m[i] = b1 * m[i] + (1.0 - b1) * g[i];
            v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
            const double mhat = m[i] / b1t;
            const double vhat = v[i] / b2t;
            x[i] -= lr * mhat / (sqrt(vhat) + eps);
            if (x[i] < 0.0) x[i] = 0.0;
        }
    }
    memcpy(out_s, best, (size_t)G * sizeof(double));
    *out_best_loss = best_loss;
    *out_best_epoch = best_e;
    *out_n_records = n_rec;
    *out_flags = flags;
    free(x);
    free(best);
    free(m);
    free(v);
    free(g);
    free(pint);
    free(pic);
    free(pper);
    return rc;
}

int orc_fine_tune(int L, const int64_t* w, const int64_t* r, const double* P, int act, const double* s_init,
                  const double* mu, double lr, int64_t epochs, int64_t n_int, int64_t n_ic, int64_t n_bc,
                  uint64_t seed, int64_t chunk, double* out_s, double* out_best_loss, int64_t* out_best_epoch,
                  double* out_losses, int64_t* out_n_records, int* out_flags) {
    return solve_loop(0, L, w, r, NULL, P, act, s_init, mu, lr, epochs, 0, n_int, n_ic, n_bc, seed, NULL, 0, NULL,
                      0, NULL, 0, 0.0, chunk, out_s, out_best_loss, out_best_epoch, out_losses, out_n_records,
                      out_flags);
}

/* X is the fast phase's sampling set, classified with classify_point (reduction.cpp:27-31). */
int orc_fast_solve(int L, const int64_t* r, const int64_t* rh, const double* F, int act, const double* s_init,
                   const double* mu, const double* X, int64_t n_x, double lambda_local, double lr, int64_t epochs,
                   int64_t chunk, double* out_s, double* out_best_loss, int64_t* out_best_epoch, double* out_losses,
                   int64_t* out_n_records, int* out_flags) {
    double* xi = (double*)malloc((size_t)(2 * n_x + 1) * sizeof(double));
    double* xc = (double*)malloc((size_t)(n_x + 1) * sizeof(double));
    double* xb = (double*)malloc((size_t)(n_x + 1) * sizeof(double));
    int64_t ni = 0, nc = 0, nb = 0;
    for (int64_t i = 0; i < n_x; ++i) {
        const double x = X[2 * i], t = X[2 * i + 1];
        if (t == 0.0) xc[nc++] = x;
        else if (x == 0.0 || x == ORC_TWO_PI) xb[nb++] = t;
        else {
            xi[2 * ni] = x;
            xi[2 * ni + 1] = t;
            ++ni;
        }
    }
    const int64_t w2[2] = {2, 1};
    const int rc = solve_loop(1, L, w2, r, rh, F, act, s_init, mu, lr, epochs, 1, 0, 0, 0, 0, xi, ni, xc, nc, xb,
                              nb, lambda_local, chunk, out_s, out_best_loss, out_best_epoch, out_losses,
                              out_n_records, out_flags);
    free(xi);
    free(xc);
    free(xb);
    return rc;
}
