// FastLRNR construction on the device:
//   harvest_snapshots  (reduction.cpp:111-148)  -> harvest_kernel
//   eim_greedy         (reduction.cpp:150-238)  -> eim_residual_kernel + eim_select_kernel
//   build_fastparams   (reduction.cpp:240-283)  -> host (lrnr_host_build_fastparams)
//
// The greedy sweep is the O(r_hat * n_cols * (r_hat^2 + M r_hat)) part: every
// iteration interpolates every snapshot column at the chosen indices and takes
// the column with the largest max-norm residual. Here one thread owns one
// column (snapshots stay in the reference's M x n_cols row-major layout, so a
// warp's loads of row i are one coalesced 256 B line), the interpolation block
// LU lives in shared memory, and all inner layers run concurrently
// (blockIdx.y = layer). A one-CTA-per-layer select kernel takes the argmax,
// appends the basis column and refactors the block, so the whole greedy loop is
// 2 launches per basis vector with no host round trip.
//
// Bit-exactness: the reference is built -O3 -march=x86-64-v3 (-ffp-contract=fast),
// and its object code fixes the rounding of every accumulation:
//   - elementwise updates (lu_factor's trailing update, lu_solve's forward
//     substitution, value_affine_factored's y += V z) are fused: fma;
//   - dot products (matvec in eim_apply, lu_solve's back substitution,
//     value_affine_factored's U y) are vectorised 4/2 wide: every product is
//     rounded and then added in order, and only an odd last term is fused
//     (linalg.o: vmulpd + vaddsd/vsubsd chains, one vfmadd231sd/vfnmadd231sd tail).
// ref_dot() reproduces the second rule with __dmul_rn/__dadd_rn (which nvcc
// never contracts), so given the same snapshots the selected indices and basis
// columns are bit-identical to the CPU (tests/test_gpu_eim.py).
#include "internal.h"

using namespace lrnr_b200;
using namespace lrnr_b200::detail;

namespace {

constexpr int EIM_RMAX = 64;       // r_hat cap and harvest rank cap
constexpr int RES_NT = 256;        // residual sweep: 8 warps ...
constexpr int RES_CT = 32;         // ... over 32 snapshot columns (lane = column)
constexpr int SEL_NT = 256;
constexpr int HV_NT = 256;         // harvest: 256 threads ...
constexpr int HV_CT = 8;           // ... over 8 columns (rows of a layer in parallel)
constexpr int EIM_MAX_LAYERS = 32;

enum : int { ST_ACTIVE = 0, ST_EXHAUSTED = 1, ST_SINGULAR = 2, ST_FULL = 3 };

struct EimLayers {
    const double* S[EIM_MAX_LAYERS];  // M_l x n_cols, row-major
    int m[EIM_MAX_LAYERS];
    int kmax[EIM_MAX_LAYERS];  // min(r_hat, m)
    int n;
};

// Device state of the greedy loop, one slot per layer.
struct EimState {
    int* idx;      // [layer][EIM_RMAX]
    int* cnt;      // [layer]
    int* status;   // [layer]
    int* piv;      // [layer][EIM_RMAX]
    double* xi;    // [layer][m_max][EIM_RMAX]
    double* lu;    // [layer][EIM_RMAX][EIM_RMAX]
    double* bestn; // [layer][nblk]
    long long* bestc;
    int m_max;
    int nblk;
};

struct HarvestNet {
    int L;
    int mmax;  // widest harvested layer
    int M[33];
    int r[32];
    long long oU[32], oV[32], ob[32];
    long long soff[33];
};

// acc (+|-) sum_j a[j*sa] * b[j*sb] with the reference build's rounding (see the
// header): rounded products accumulated in order, an odd last term fused.
template <bool SUB>
__device__ __forceinline__ double ref_dot(double acc, const double* a, int sa, const double* b, int sb, int n) {
    const int nr = n & ~1;
    for (int j = 0; j < nr; ++j) {
        const double p = __dmul_rn(a[j * sa], b[j * sb]);
        acc = SUB ? __dsub_rn(acc, p) : __dadd_rn(acc, p);
    }
    if (n & 1) acc = fma(SUB ? -a[nr * sa] : a[nr * sa], b[nr * sb], acc);
    return acc;
}

// tanh as the reference evaluates it: glibc's fdlibm tanh (s_tanh.c) over the
// expm1 that glibc dispatches to on FMA-capable x86-64 hosts (s_expm1.c built
// with -mfma: Estrin polynomial, fused argument reduction). The operations below
// follow that build one for one (constants are fdlibm's), so harvested
// snapshots are bit-identical to the CPU's and the greedy selection downstream
// cannot diverge on near-ties. Domain used by tanh: finite x > -38.8.
//
// The algorithm and constants of glibc_expm1 / glibc_tanh below are those of
// fdlibm's s_expm1.c / s_tanh.c, which carry this notice:
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this
//   software is freely granted, provided that this notice
//   is preserved.
__device__ __forceinline__ double scale2k(double y, int k) {
    return __hiloint2double(__double2hiint(y) + (k << 20), __double2loint(y));
}

__device__ double glibc_expm1(double x) {
    constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
                     invln2 = 1.44269504088896338700e+00, Q1 = -3.33333333333331316428e-02,
                     Q2 = 1.58730158725481460165e-03, Q3 = -7.93650757867487942473e-05,
                     Q4 = 4.00821782732936239552e-06, Q5 = -2.01099218183624371326e-07;
    const unsigned hx = static_cast<unsigned>(__double2hiint(x)), ax = hx & 0x7fffffffu;
    const bool neg = (hx >> 31) != 0;
    double xr = x, hi = 0.0, c = 0.0;
    int k = 0;
    if (ax > 0x40436879u && neg) return -1.0;  // tiny - one
    if (ax > 0x3fd62e42u) {
        if (ax <= 0x3ff0a2b1u) {
            hi = neg ? __dadd_rn(x, ln2_hi) : __dsub_rn(x, ln2_hi);
            const double lo = neg ? -ln2_lo : ln2_lo;
            k = neg ? -1 : 1;
            xr = __dsub_rn(hi, lo);
            c = __dsub_rn(__dsub_rn(hi, xr), lo);
        } else {
            k = static_cast<int>(__dadd_rn(__dmul_rn(x, invln2), neg ? -0.5 : 0.5));
            const double t = static_cast<double>(k);
            hi = __fma_rn(-t, ln2_hi, x);
            const double lo = __dmul_rn(t, ln2_lo);
            xr = __dsub_rn(hi, lo);
            c = __dsub_rn(__dsub_rn(hi, xr), lo);
        }
    } else if (ax < 0x3c900000u) {
        return x;
    }
    const double hfx = __dmul_rn(xr, 0.5), hxs = __dmul_rn(xr, hfx);
    const double R2 = __fma_rn(hxs, Q3, Q2), R3 = __fma_rn(hxs, Q5, Q4), h2 = __dmul_rn(hxs, hxs);
    const double R1 = __fma_rn(hxs, Q1, 1.0), h4 = __dmul_rn(h2, h2);
    const double r1 = __fma_rn(h4, R3, __fma_rn(h2, R2, R1));
    const double t = __fma_rn(-r1, hfx, 3.0);
    double e = __dmul_rn(__ddiv_rn(__dsub_rn(r1, t), __fma_rn(-xr, t, 6.0)), hxs);
    if (k == 0) return __dsub_rn(xr, __fma_rn(e, xr, -hxs));
    e = __dsub_rn(__fma_rn(__dsub_rn(e, c), xr, -c), hxs);
    if (k == -1) return __fma_rn(0.5, __dsub_rn(xr, e), -0.5);
    if (k == 1) {
        if (xr < -0.25) return __dmul_rn(__dsub_rn(e, __dadd_rn(xr, 0.5)), -2.0);
        return __fma_rn(__dsub_rn(xr, e), 2.0, 1.0);
    }
    if (k <= -2 || k > 56) return __dsub_rn(scale2k(__dsub_rn(1.0, __dsub_rn(e, xr)), k), 1.0);
    if (k < 20) {
        const double tk = __hiloint2double(0x3ff00000 - (0x200000 >> k), 0);
        return scale2k(__dsub_rn(tk, __dsub_rn(e, xr)), k);
    }
    const double tk = __hiloint2double((0x3ff - k) << 20, 0);
    return scale2k(__dadd_rn(__dsub_rn(xr, __dadd_rn(e, tk)), 1.0), k);
}

__device__ double glibc_tanh(double x) {
    const int hx = __double2hiint(x);
    const unsigned ix = static_cast<unsigned>(hx) & 0x7fffffffu;
    if (ix >= 0x7ff00000u) return hx >= 0 ? __dadd_rn(__ddiv_rn(1.0, x), 1.0) : __dsub_rn(__ddiv_rn(1.0, x), 1.0);
    double z;
    if (ix < 0x40360000u) {  // |x| < 22
        if ((ix | static_cast<unsigned>(__double2loint(x))) == 0) return x;
        if (ix < 0x3c800000u) return __dmul_rn(__dadd_rn(1.0, x), x);
        const double ax = fabs(x);
        if (ix >= 0x3ff00000u) {
            const double t = glibc_expm1(__dadd_rn(ax, ax));
            z = __dsub_rn(1.0, __ddiv_rn(2.0, __dadd_rn(t, 2.0)));
        } else {
            const double t = glibc_expm1(__dmul_rn(ax, -2.0));
            z = __ddiv_rn(-t, __dadd_rn(t, 2.0));
        }
    } else {
        z = 1.0;  // one - tiny
    }
    return hx >= 0 ? z : -z;
}

// hidden_states (model.cpp:407-428 via value_affine_factored, model.cpp:183-199):
// z^{l+1} = act(U^l diag(s^l) (V^l^T z^l) + b^l), for HV_CT columns per CTA with
// the layer's rows in parallel (phase A: one U-row dot per (column, row)) and the
// next layer's V^T z as one fused chain per (column, rank index) in ascending row
// order, as the CPU accumulates it (phase B).
template <int ACT>
__global__ void __launch_bounds__(HV_NT) harvest_kernel(HarvestNet net, const double* __restrict__ P,
                                                        const double* __restrict__ s, long long r_total,
                                                        const double* __restrict__ pts, long long n_cols,
                                                        long long per_mu, double* __restrict__ snaps) {
    extern __shared__ double hv_smem[];
    constexpr int YS = EIM_RMAX + 1;  // odd row strides: the 8 columns hit distinct banks
    const int zst = net.mmax + 1;
    double* ys = hv_smem;             // [HV_CT][YS]
    double* zs = ys + HV_CT * YS;     // [HV_CT][zst]
    const long long c0 = static_cast<long long>(blockIdx.x) * HV_CT;
    const int nc = static_cast<int>(min(static_cast<long long>(HV_CT), n_cols - c0));
    {
        const int r0 = net.r[0];
        const double* V0 = P + net.oV[0];
        for (int q = threadIdx.x; q < HV_CT * r0; q += HV_NT) {
            const int c = q % HV_CT, j = q / HV_CT;
            if (c >= nc) continue;
            const long long col = c0 + c;
            double y = fma(V0[j], pts[2 * col], 0.0);
            y = fma(V0[r0 + j], pts[2 * col + 1], y);
            ys[c * YS + j] = y * s[(col / per_mu) * r_total + j];
        }
    }
    __syncthreads();
    double* out = snaps;
    for (int l = 0; l + 1 < net.L; ++l) {
        const int r = net.r[l], M = net.M[l + 1];
        const double* U = P + net.oU[l];
        const double* b = P + net.ob[l];
        for (int q = threadIdx.x; q < HV_CT * M; q += HV_NT) {
            const int c = q % HV_CT, i = q / HV_CT;
            if (c >= nc) continue;
            const double a = __dadd_rn(ref_dot<false>(0.0, U + i * r, 1, ys + c * YS, 1, r), b[i]);
            const double z = ACT == LRNR_ACT_SIN ? sin(a) : glibc_tanh(a);
            zs[c * zst + i] = z;
            out[static_cast<long long>(i) * n_cols + c0 + c] = z;
        }
        out += static_cast<long long>(M) * n_cols;
        __syncthreads();
        if (l + 2 < net.L) {
            const int rn = net.r[l + 1];
            const double* Vn = P + net.oV[l + 1];
            for (int q = threadIdx.x; q < HV_CT * rn; q += HV_NT) {
                const int c = q % HV_CT, j = q / HV_CT;
                if (c >= nc) continue;
                double y = 0.0;
                for (int i = 0; i < M; ++i) y = fma(Vn[i * rn + j], zs[c * zst + i], y);
                ys[c * YS + j] = y * s[((c0 + c) / per_mu) * r_total + net.soff[l + 1] + j];
            }
            __syncthreads();
        }
    }
}

// lu_solve (linalg.cpp:85-108) on x[0], x[xs], ...: row swaps, unit-lower forward
// substitution (fused), upper backward substitution (a dot product: ref_dot).
__device__ __forceinline__ void lu_solve_dev(const double* lu, const int* piv, int k, double* x, int xs) {
    for (int q = 0; q < k; ++q)
        if (piv[q] != q) {
            const double tmp = x[q * xs];
            x[q * xs] = x[piv[q] * xs];
            x[piv[q] * xs] = tmp;
        }
    for (int q = 0; q < k; ++q) {
        const double xq = x[q * xs];
        for (int i = q + 1; i < k; ++i) x[i * xs] = fma(-lu[i * k + q], xq, x[i * xs]);
    }
    for (int q = k - 1; q >= 0; --q)
        x[q * xs] = ref_dot<true>(x[q * xs], lu + q * k + q + 1, 1, x + (q + 1) * xs, xs, k - q - 1) / lu[q * k + q];
}

// Larger key wins, ties go to the smaller index (the CPU's first-strictly-larger scan).
__device__ __forceinline__ void better(double& n, long long& c, double n2, long long c2) {
    if (n2 > n || (n2 == n && c2 < c)) {
        n = n2;
        c = c2;
    }
}

__device__ __forceinline__ void warp_argmax(double& n, long long& c) {
    for (int o = 16; o; o >>= 1) {
        const double n2 = __shfl_xor_sync(0xffffffffu, n, o);
        const long long c2 = __shfl_xor_sync(0xffffffffu, c, o);
        better(n, c, n2, c2);
    }
}

__device__ void block_argmax(double& n, long long& c, double* sn, long long* sc) {
    warp_argmax(n, c);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sn[w] = n;
        sc[w] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < nw; ++q) better(n, c, sn[q], sc[q]);
        sn[0] = n;
        sc[0] = c;
    }
    __syncthreads();
    n = sn[0];
    c = sc[0];
}

// One greedy sweep (interp_residual + the sup-norm, reduction.cpp:152-164,
// 184-192) over RES_CT columns per CTA, blockIdx.y = layer: gather P^T S, solve
// the k x k interpolation system per column (one lane each), then the residual
// rows v_i - Xi_i . coef with 8 warps over the rows (Xi_i is warp-uniform, so its
// loads broadcast; a warp's S loads are one 256 B row segment).
__global__ void __launch_bounds__(RES_NT) eim_residual_kernel(EimLayers layers, EimState st, long long n_cols) {
    const int l = blockIdx.y;
    if (st.status[l] != ST_ACTIVE) return;
    const int k = st.cnt[l], m = layers.m[l];
    const double* S = layers.S[l];
    extern __shared__ double eim_smem[];
    double* coef = eim_smem;                   // [k][RES_CT]
    double* lu = coef + EIM_RMAX * RES_CT;     // k x k
    int* piv = reinterpret_cast<int*>(lu + k * k);
    int* idx = piv + EIM_RMAX;
    __shared__ double part[RES_NT / 32][RES_CT];
    for (int q = threadIdx.x; q < k * k; q += RES_NT)
        lu[q] = st.lu[static_cast<long long>(l) * EIM_RMAX * EIM_RMAX + q];
    for (int q = threadIdx.x; q < k; q += RES_NT) {
        piv[q] = st.piv[l * EIM_RMAX + q];
        idx[q] = st.idx[l * EIM_RMAX + q];
    }
    __syncthreads();
    const long long c0 = static_cast<long long>(blockIdx.x) * RES_CT;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long c = c0 + lane;
    const bool ok = c < n_cols;
    for (int q = threadIdx.x; q < k * RES_CT; q += RES_NT) {
        const long long cc = c0 + (q % RES_CT);
        coef[q] = cc < n_cols ? S[static_cast<long long>(idx[q / RES_CT]) * n_cols + cc] : 0.0;
    }
    __syncthreads();
    if (w == 0 && k) lu_solve_dev(lu, piv, k, coef + lane, RES_CT);
    __syncthreads();
    const double* xi = st.xi + static_cast<long long>(l) * st.m_max * EIM_RMAX;
    double nrm = 0.0;
    if (ok) {
        const double* Sc = S + c;
        int i = w;
        for (; i + 8 < m; i += 16) {  // two independent rows per pass (ILP)
            const double* x1 = xi + i * EIM_RMAX;
            const double* x2 = x1 + 8 * EIM_RMAX;
            double v1 = Sc[static_cast<long long>(i) * n_cols], v2 = Sc[static_cast<long long>(i + 8) * n_cols];
            if (k) {
                const double* cf = coef + lane;
                double a1 = 0.0, a2 = 0.0;
                const int nr = k & ~1;
                for (int j = 0; j < nr; ++j) {
                    const double cj = cf[j * RES_CT];
                    a1 = __dadd_rn(a1, __dmul_rn(x1[j], cj));
                    a2 = __dadd_rn(a2, __dmul_rn(x2[j], cj));
                }
                if (k & 1) {
                    const double cj = cf[nr * RES_CT];
                    a1 = fma(x1[nr], cj, a1);
                    a2 = fma(x2[nr], cj, a2);
                }
                v1 = __dsub_rn(v1, a1);
                v2 = __dsub_rn(v2, a2);
            }
            v1 = fabs(v1);
            v2 = fabs(v2);
            nrm = nrm < v1 ? v1 : nrm;  // std::max(nrm, |v|): a NaN residual is skipped
            nrm = nrm < v2 ? v2 : nrm;
        }
        for (; i < m; i += 8) {
            double v = Sc[static_cast<long long>(i) * n_cols];
            if (k) v = __dsub_rn(v, ref_dot<false>(0.0, xi + i * EIM_RMAX, 1, coef + lane, RES_CT, k));
            v = fabs(v);
            nrm = nrm < v ? v : nrm;
        }
    }
    part[w][lane] = ok ? nrm : -1.0;
    __syncthreads();
    if (w == 0) {
        double n = part[0][lane];
        for (int q = 1; q < RES_NT / 32; ++q) n = n < part[q][lane] ? part[q][lane] : n;
        long long bc = ok ? c : LLONG_MAX;
        warp_argmax(n, bc);
        if (lane == 0) {
            st.bestn[static_cast<long long>(l) * st.nblk + blockIdx.x] = n;
            st.bestc[static_cast<long long>(l) * st.nblk + blockIdx.x] = bc;
        }
    }
}

// Argmax over the sweep's per-CTA winners, then the CPU's tail of one greedy
// step (reduction.cpp:193-236): pick the interpolation index, append the
// normalised residual to Xi, refactor P^T Xi (refactor_block + lu_factor,
// linalg.cpp:59-83). Row scans run in parallel with the CPU's tie rules.
__global__ void __launch_bounds__(SEL_NT) eim_select_kernel(EimLayers layers, EimState st, long long n_cols) {
    const int l = blockIdx.x;
    if (st.status[l] != ST_ACTIVE) return;
    const int k = st.cnt[l], m = layers.m[l];
    const double* S = layers.S[l];
    extern __shared__ double eim_smem[];
    double* lu = eim_smem;                            // (k+1) x (k+1)
    double* res = lu + (k + 1) * (k + 1);             // m
    double* coef = res + m;                           // k
    int* piv = reinterpret_cast<int*>(coef + EIM_RMAX);
    int* idx = piv + EIM_RMAX;
    int* taken = idx + EIM_RMAX;                      // m
    __shared__ double red_n[SEL_NT / 32];
    __shared__ long long red_c[SEL_NT / 32];
    __shared__ int s_flag, s_imax;
    double n = -1.0;
    long long bc = LLONG_MAX;
    for (int q = threadIdx.x; q < st.nblk; q += SEL_NT)
        better(n, bc, st.bestn[static_cast<long long>(l) * st.nblk + q], st.bestc[static_cast<long long>(l) * st.nblk + q]);
    block_argmax(n, bc, red_n, red_c);
    if (n < 1e-12) {
        if (threadIdx.x == 0) st.status[l] = ST_EXHAUSTED;
        return;
    }
    double* xi = st.xi + static_cast<long long>(l) * st.m_max * EIM_RMAX;
    for (int i = threadIdx.x; i < m; i += SEL_NT) taken[i] = 0;
    for (int q = threadIdx.x; q < k * k; q += SEL_NT)
        lu[q] = st.lu[static_cast<long long>(l) * EIM_RMAX * EIM_RMAX + q];
    __syncthreads();
    for (int q = threadIdx.x; q < k; q += SEL_NT) {
        piv[q] = st.piv[l * EIM_RMAX + q];
        idx[q] = st.idx[l * EIM_RMAX + q];
        taken[idx[q]] = 1;
        coef[q] = S[static_cast<long long>(idx[q]) * n_cols + bc];
    }
    __syncthreads();
    if (threadIdx.x == 0 && k) lu_solve_dev(lu, piv, k, coef, 1);
    __syncthreads();
    // the winning column's residual, then its largest entry among unused rows
    double mag = -1.0;
    long long bi = m;
    for (int i = threadIdx.x; i < m; i += SEL_NT) {
        const double v = S[static_cast<long long>(i) * n_cols + bc];
        res[i] = k ? __dsub_rn(v, ref_dot<false>(0.0, xi + i * EIM_RMAX, 1, coef, 1, k)) : v;
        const double a = fabs(res[i]);
        if (!taken[i] && a > mag) {  // NaN never wins (the CPU's strict >)
            mag = a;
            bi = i;
        }
    }
    block_argmax(mag, bi, red_n, red_c);
    if (bi == m || mag < 1e-12) {
        if (threadIdx.x == 0) st.status[l] = ST_EXHAUSTED;
        return;
    }
    const int k1 = k + 1;
    const double den = res[bi];
    for (int i = threadIdx.x; i < m; i += SEL_NT) xi[i * EIM_RMAX + k] = res[i] / den;
    if (threadIdx.x == 0) idx[k] = static_cast<int>(bi);
    __syncthreads();
    for (int q = threadIdx.x; q < k1 * k1; q += SEL_NT) {
        const int i = q / k1, j = q % k1;
        lu[q] = xi[idx[i] * EIM_RMAX + j];
    }
    __syncthreads();
    for (int kk = 0; kk < k1; ++kk) {
        if (threadIdx.x < 32) {
            // pivot: the CPU scans rows kk.. with a strict >, starting from row kk;
            // a NaN diagonal keeps row kk (nothing compares greater than NaN)
            const double d = fabs(lu[kk * k1 + kk]);
            double v = -1.0;
            long long im = LLONG_MAX;
            for (int i = kk + 1 + threadIdx.x; i < k1; i += 32) {
                const double a = fabs(lu[i * k1 + kk]);
                if (a > v) {
                    v = a;
                    im = i;
                }
            }
            warp_argmax(v, im);
            if (threadIdx.x == 0) {
                int imax = kk;
                double vmax = d;
                if (!(d != d) && im != LLONG_MAX && v > d) {
                    vmax = v;
                    imax = static_cast<int>(im);
                }
                s_flag = vmax < 1e-14 ? 1 : 0;
                s_imax = imax;
                piv[kk] = imax;
            }
        }
        __syncthreads();
        if (s_flag) {
            if (threadIdx.x == 0) st.status[l] = ST_SINGULAR;
            return;
        }
        const int im = s_imax;
        if (im != kk)
            for (int j = threadIdx.x; j < k1; j += SEL_NT) {
                const double tmp = lu[kk * k1 + j];
                lu[kk * k1 + j] = lu[im * k1 + j];
                lu[im * k1 + j] = tmp;
            }
        __syncthreads();
        const double pivot = lu[kk * k1 + kk];
        for (int i = kk + 1 + threadIdx.x; i < k1; i += SEL_NT) lu[i * k1 + kk] = lu[i * k1 + kk] / pivot;
        __syncthreads();
        const int wd = k1 - kk - 1;
        for (int q = threadIdx.x; q < wd * wd; q += SEL_NT) {
            const int i = kk + 1 + q / wd, j = kk + 1 + q % wd;
            lu[i * k1 + j] = fma(-lu[i * k1 + kk], lu[kk * k1 + j], lu[i * k1 + j]);
        }
        __syncthreads();
    }
    for (int q = threadIdx.x; q < k1 * k1; q += SEL_NT)
        st.lu[static_cast<long long>(l) * EIM_RMAX * EIM_RMAX + q] = lu[q];
    for (int q = threadIdx.x; q < k1; q += SEL_NT) {
        st.piv[l * EIM_RMAX + q] = piv[q];
        st.idx[l * EIM_RMAX + q] = idx[q];
    }
    if (threadIdx.x == 0) {
        st.cnt[l] = k1;
        if (k1 >= layers.kmax[l]) st.status[l] = ST_FULL;
    }
}

struct EimResult {
    std::vector<int> idx, cnt, status;
    std::vector<double> xi;  // [layer][m_max][EIM_RMAX]
    int m_max = 0;
};

// The greedy loop for every layer in `layers` (all sharing n_cols): 2 launches
// per basis vector, state on the device, one download at the end.
EimResult run_eim(lrnr_gpu_ctx* ctx, const EimLayers& layers, long long n_cols, int r_hat) {
    const int nl = layers.n;
    int m_max = 0, k_top = 0;
    for (int l = 0; l < nl; ++l) {
        m_max = std::max(m_max, layers.m[l]);
        k_top = std::max(k_top, layers.kmax[l]);
    }
    const int nblk = static_cast<int>((n_cols + RES_CT - 1) / RES_CT);
    const size_t ints = static_cast<size_t>(nl) * (2 * EIM_RMAX + 2);
    const size_t dbl = static_cast<size_t>(nl) * (static_cast<size_t>(m_max) * EIM_RMAX + EIM_RMAX * EIM_RMAX + nblk) +
                       static_cast<size_t>(nl) * nblk;  // + bestc (8 B each)
    ctx->eim_state.ensure(dbl * sizeof(double) + ints * sizeof(int) + 64);
    EimState st{};
    double* d = ctx->eim_state.as<double>();
    st.xi = d;
    d += static_cast<size_t>(nl) * m_max * EIM_RMAX;
    st.lu = d;
    d += static_cast<size_t>(nl) * EIM_RMAX * EIM_RMAX;
    st.bestn = d;
    d += static_cast<size_t>(nl) * nblk;
    st.bestc = reinterpret_cast<long long*>(d);
    d += static_cast<size_t>(nl) * nblk;
    int* ip = reinterpret_cast<int*>(d);
    st.idx = ip;
    st.piv = ip + nl * EIM_RMAX;
    st.cnt = ip + 2 * nl * EIM_RMAX;
    st.status = st.cnt + nl;
    st.m_max = m_max;
    st.nblk = nblk;
    CK(cudaMemsetAsync(ctx->eim_state.p, 0, ctx->eim_state.bytes, ctx->stream));
    const size_t smem_res = (static_cast<size_t>(EIM_RMAX) * RES_CT + static_cast<size_t>(k_top) * k_top) * sizeof(double) +
                            2 * EIM_RMAX * sizeof(int);
    const size_t smem_sel = (static_cast<size_t>(k_top + 1) * (k_top + 1) + m_max + EIM_RMAX) * sizeof(double) +
                            (2 * EIM_RMAX + static_cast<size_t>(m_max)) * sizeof(int);
    CK(cudaFuncSetAttribute(eim_residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(std::max<size_t>(smem_res, 48 * 1024))));
    CK(cudaFuncSetAttribute(eim_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(std::max<size_t>(smem_sel, 48 * 1024))));
    for (int it = 0; it < k_top; ++it) {
        eim_residual_kernel<<<dim3(nblk, nl), RES_NT, smem_res, ctx->stream>>>(layers, st, n_cols);
        CK(cudaGetLastError());
        eim_select_kernel<<<nl, SEL_NT, smem_sel, ctx->stream>>>(layers, st, n_cols);
        CK(cudaGetLastError());
        ctx->launches += 2;
    }
    EimResult r;
    r.m_max = m_max;
    r.xi.resize(static_cast<size_t>(nl) * m_max * EIM_RMAX);
    r.idx.resize(static_cast<size_t>(nl) * EIM_RMAX);
    r.cnt.resize(nl);
    r.status.resize(nl);
    CK(cudaMemcpyAsync(r.xi.data(), st.xi, r.xi.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(r.idx.data(), st.idx, r.idx.size() * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(r.cnt.data(), st.cnt, nl * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(r.status.data(), st.status, nl * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int l = 0; l < nl; ++l) {
        if (r.status[l] == ST_SINGULAR) throw InvalidArg("lu_factor: singular matrix (pivot < 1e-14)");
        if (r.cnt[l] == 0) throw InvalidArg("eim_greedy: no basis vector selected");
    }
    return r;
}

// outputs in the lrnr_host_eim_greedy layout (r_hat columns, -1 / 0 padded)
void write_layer(const EimResult& r, int l, int m, int64_t r_hat, int64_t* out_idx, double* out_xi) {
    const int k = r.cnt[l];
    for (int64_t q = 0; q < r_hat; ++q) out_idx[q] = q < k ? r.idx[static_cast<size_t>(l) * EIM_RMAX + q] : -1;
    if (out_xi)
        for (int i = 0; i < m; ++i)
            for (int64_t q = 0; q < r_hat; ++q)
                out_xi[i * r_hat + q] =
                    q < k ? r.xi[(static_cast<size_t>(l) * r.m_max + i) * EIM_RMAX + static_cast<size_t>(q)] : 0.0;
}

struct Harvest {
    const double* snaps;  // inner layers' M_l x n_cols blocks, concatenated
    int64_t n_cols, rows;
};

// harvest_snapshots (reduction.cpp:111-148): points from the reference's Rng
// stream on the host (bit-identical, one upload), hidden states on the device.
Harvest harvest_device(lrnr_gpu_ctx* ctx, int L, const int64_t* widths, const int64_t* ranks, const double* params,
                       int act, const double* s, int64_t n_mu, const double* X, int64_t n_x, int64_t n_perturb,
                       double sigma, uint64_t seed) {
    require(widths && ranks && params && s, "null argument");
    require(L >= 2 && L <= EIM_MAX_LAYERS, "build_fastparams: need at least two layers");
    require(act == LRNR_ACT_TANH || act == LRNR_ACT_SIN, "unknown activation");
    require(widths[0] == 2, "LRNR input width must be 2 (x, t)");
    for (int l = 0; l < L; ++l) {
        require(ranks[l] >= 1, "LrnrParams: rank must be positive");
        require(ranks[l] <= std::min(widths[l], widths[l + 1]), "LrnrParams: rank exceeds min(M_l, M_{l-1})");
        require(ranks[l] <= EIM_RMAX, "harvest_snapshots: device path supports ranks <= 64");
    }
    require(X != nullptr && n_mu >= 1 && n_x >= 1 && n_perturb >= 0, "harvest_snapshots: bad sizes");
    require(sigma > 0.0 || n_perturb == 0, "harvest_snapshots: sigma must be positive");
    const int64_t per_mu = n_x * (1 + n_perturb), n_cols = n_mu * per_mu;
    std::vector<double> pts(static_cast<size_t>(2 * n_cols));
    require(lrnr_host_harvest_points(X, n_x, n_mu, n_perturb, sigma, seed, pts.data()) == LRNR_OK,
            "harvest_snapshots: point generation failed");
    HarvestNet net{};
    net.L = L;
    int64_t o = 0, r_total = 0, rows = 0;
    for (int l = 0; l <= L; ++l) net.M[l] = static_cast<int>(widths[l]);
    for (int l = 0; l < L; ++l) {
        net.r[l] = static_cast<int>(ranks[l]);
        net.soff[l] = r_total;
        r_total += ranks[l];
        net.oU[l] = o;
        o += widths[l + 1] * ranks[l];
        net.oV[l] = o;
        o += widths[l] * ranks[l];
        net.ob[l] = o;
        o += widths[l + 1];
        if (l + 1 < L) {
            rows += widths[l + 1];
            net.mmax = std::max(net.mmax, static_cast<int>(widths[l + 1]));
        }
    }
    const int64_t n_params = o;
    const size_t snap_elems = static_cast<size_t>(rows) * n_cols;
    ctx->eim_snaps.ensure((snap_elems + n_params + n_mu * r_total + 2 * n_cols) * sizeof(double));
    double* snaps = ctx->eim_snaps.as<double>();
    double* dP = snaps + snap_elems;
    double* ds = dP + n_params;
    double* dpts = ds + n_mu * r_total;
    CK(cudaMemcpyAsync(dP, params, n_params * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ds, s, n_mu * r_total * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(dpts, pts.data(), pts.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const size_t smem = static_cast<size_t>(HV_CT) * (EIM_RMAX + 1 + net.mmax + 1) * sizeof(double);
    auto kern = act == LRNR_ACT_SIN ? harvest_kernel<LRNR_ACT_SIN> : harvest_kernel<LRNR_ACT_TANH>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(std::max<size_t>(smem, 48 * 1024))));
    kern<<<static_cast<unsigned>((n_cols + HV_CT - 1) / HV_CT), HV_NT, smem, ctx->stream>>>(net, dP, ds, r_total, dpts,
                                                                                          n_cols, per_mu, snaps);
    CK(cudaGetLastError());
    ctx->launches += 1;
    return Harvest{snaps, n_cols, rows};
}

}  // namespace

extern "C" {

int lrnr_gpu_eim_greedy(lrnr_gpu_ctx* ctx, int64_t m, int64_t n_cols, const double* snapshots, int64_t r_hat,
                        int64_t* out_idx, double* out_xi, int64_t* out_count, int* out_exhausted) {
    return guarded(ctx, [&] {
        require(snapshots && out_idx && out_xi && out_count && out_exhausted, "null argument");
        require(n_cols >= 1, "eim_greedy: empty snapshot set");
        require(r_hat >= 1, "eim_greedy: budget must be positive");
        require(m >= 1 && m <= INT_MAX / EIM_RMAX, "eim_greedy: bad row count");
        require(r_hat <= EIM_RMAX, "eim_greedy: device path supports r_hat <= 64");
        const size_t bytes = static_cast<size_t>(m) * n_cols * sizeof(double);
        ctx->eim_snaps.ensure(bytes);
        CK(cudaMemcpyAsync(ctx->eim_snaps.p, snapshots, bytes, cudaMemcpyHostToDevice, ctx->stream));
        EimLayers layers{};
        layers.n = 1;
        layers.S[0] = ctx->eim_snaps.as<double>();
        layers.m[0] = static_cast<int>(m);
        layers.kmax[0] = static_cast<int>(std::min<int64_t>(r_hat, m));
        const EimResult r = run_eim(ctx, layers, n_cols, static_cast<int>(r_hat));
        write_layer(r, 0, static_cast<int>(m), r_hat, out_idx, out_xi);
        *out_count = r.cnt[0];
        *out_exhausted = r.status[0] == ST_EXHAUSTED ? 1 : 0;
    });
}

int lrnr_gpu_harvest_snapshots(lrnr_gpu_ctx* ctx, int L, const int64_t* widths, const int64_t* ranks,
                               const double* params, int act, const double* s, int64_t n_mu,
                               const double* sampling_xt, int64_t n_sampling, int64_t n_perturb, double sigma,
                               uint64_t seed, double* out_snapshots) {
    return guarded(ctx, [&] {
        require(out_snapshots != nullptr, "null argument");
        const Harvest h = harvest_device(ctx, L, widths, ranks, params, act, s, n_mu, sampling_xt, n_sampling,
                                         n_perturb, sigma, seed);
        CK(cudaMemcpyAsync(out_snapshots, h.snaps, static_cast<size_t>(h.rows) * h.n_cols * sizeof(double),
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int lrnr_gpu_build_fast(lrnr_gpu_ctx* ctx, int L, const int64_t* widths, const int64_t* ranks, const double* params,
                        int act, const double* s, int64_t n_mu, int64_t nx, int64_t nt, int64_t n_perturb,
                        double sigma, uint64_t seed, int64_t r_hat, int64_t* out_red, int64_t* out_indices,
                        double* out_fparams, int* out_exhausted) {
    return guarded(ctx, [&] {
        require(out_red && out_indices && out_fparams && out_exhausted, "null argument");
        require(r_hat >= 1, "eim_greedy: budget must be positive");
        require(r_hat <= EIM_RMAX, "eim_greedy: device path supports r_hat <= 64");
        require(nx >= 1 && nt >= 1, "uniform_grid: bad sizes");
        std::vector<double> X(static_cast<size_t>(2 * nx * nt));
        require(lrnr_host_uniform_grid(nx, nt, X.data()) == LRNR_OK, "uniform_grid: bad sizes");
        const Harvest h =
            harvest_device(ctx, L, widths, ranks, params, act, s, n_mu, X.data(), nx * nt, n_perturb, sigma, seed);
        EimLayers layers{};
        layers.n = L - 1;
        const double* S = h.snaps;
        for (int l = 0; l + 1 < L; ++l) {
            layers.S[l] = S;
            layers.m[l] = static_cast<int>(widths[l + 1]);
            layers.kmax[l] = static_cast<int>(std::min<int64_t>(r_hat, widths[l + 1]));
            S += widths[l + 1] * h.n_cols;
        }
        const EimResult r = run_eim(ctx, layers, h.n_cols, static_cast<int>(r_hat));
        std::vector<double> xi(static_cast<size_t>(h.rows * r_hat));
        double* xo = xi.data();
        for (int l = 0; l + 1 < L; ++l) {
            write_layer(r, l, layers.m[l], r_hat, out_indices + l * r_hat, xo);
            xo += widths[l + 1] * r_hat;
            out_red[l] = r.cnt[l];
            out_exhausted[l] = r.status[l] == ST_EXHAUSTED ? 1 : 0;
        }
        require(lrnr_host_build_fastparams(L, widths, ranks, params, act, r_hat, out_red, out_indices, xi.data(),
                                           out_fparams) == LRNR_OK,
                "lu_factor: singular matrix (pivot < 1e-14)");
    });
}

}  // extern "C"
