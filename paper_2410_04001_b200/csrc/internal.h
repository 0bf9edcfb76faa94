// Internal declarations shared by the translation units of liblrnr_gpu.so.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lrnr_gpu.h"
#include "pinn_kernels.cuh"
#include "pinn_v2.cuh"
#include "pinn_small.cuh"
#include "pinn_solve.cuh"
#include "pinn_fast.cuh"

namespace lrnr_b200 {
namespace detail {

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidArg : std::runtime_error {
    explicit InvalidArg(const std::string& m) : std::runtime_error(m) {}
};
struct StateError : std::runtime_error {
    explicit StateError(const std::string& m) : std::runtime_error(m) {}
};
struct NcclError : std::runtime_error {
    explicit NcclError(const std::string& m) : std::runtime_error(m) {}
};
struct NonFinite : std::runtime_error {
    int tag;
    NonFinite(int t) : std::runtime_error("non-finite value in recorded computation, layer tag " + std::to_string(t)), tag(t) {}
};

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                 \
    } while (0)

inline void require(bool c, const std::string& m) {
    if (!c) throw InvalidArg(m);
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t n) {
        if (n <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (n == 0) return;
        if (cudaMalloc(&p, n) != cudaSuccess) {
            cudaGetLastError();
            throw std::bad_alloc();
        }
        bytes = n;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// A network in the kernel's streaming layout (see pinn_kernels.cuh).
struct Model {
    bool set = false;
    int kind = LRNR_MODEL_LRNR;
    int dtype = LRNR_F64;
    int act = LRNR_ACT_TANH;
    int L = 0;
    std::vector<int> M, r, soff, trow;
    int rtotal = 0, rmax = 0;
    int tile_p = 0;  // LRNR_OPT_TILE_P for FP32 wide layers (0 = default 64)
    // packed host copy (double) in device layout; offsets in elements
    std::vector<double> packed;
    size_t off_V0 = 0, off_ulast = 0;
    std::vector<size_t> off_trans;
    DevBuf dev;
    // LRNR-only extras for the meta path: original flat params (double)
    std::vector<double> flat;
    DevBuf flat_dev;  // flat on the device (meta Gram regularizer), uploaded on first use
    std::vector<int64_t> widths64, ranks64;
    // kernel-v2 (tile-GEMM) layout: chunk blocks + per-tile schedule
    struct V2 {
        bool ok = false;
        int KC = 0, NG = 0, PT1 = 0, RPMAX = 0, P = 0;
        std::vector<int> rp, nc, yoff;
        std::vector<int64_t> aoff;
        int64_t astride = 0;
        int ystride = 0;
        std::vector<double> blocks;
        std::vector<int64_t> sched_off;
        std::vector<int> sched_cnt;
        DevBuf dblocks, dsched_off, dsched_bytes;
    } v2, v2meta;
    // tensor-core (tcgen05, 3xTF32) layout: chunk blocks with hi / lo canonical tiles
    struct TC {
        bool ok = false;
        std::vector<int> rk, rn, nc, yoff;
        std::vector<int> kU, kV;  // factor scales 2^k (FP16 split)
        std::vector<float> muU, muV;
        int ystride = 0;
        std::vector<unsigned char> blocks;  // fp16 hi / lo factor tiles + FP32 biases
        std::vector<int64_t> sched_off;
        std::vector<int> sched_cnt;
        DevBuf dblocks, dsched_off, dsched_bytes;
    } tc;
    // meta tensor-core kernel v2 (pinn_meta_tc2.cuh): neurons on TMEM lanes, 128-neuron chunks
    struct MTC2 {
        bool ok = false;
        std::vector<int> rp, nc, qdb, coff;
        std::vector<int64_t> yoff, gbase;
        int64_t ystride = 0, qbase = 0, wg_stride = 0, n_params = 0;
        int QS = 0, qdUL = 0, qdbL = 0, qdV0 = 0;
        DevBuf dblocks, dblk_off, dblk_bytes, dmap, wg, sum;
    } mtc2;
    // narrow-network kernel (pinn_fast.cuh): every hidden width and rank <= 32
    struct FK {
        bool ok = false;
        std::vector<int> np;
        int blk_len = 0;
        DevBuf dblk;
    } fk;
};

struct Hyper {
    bool set = false;
    int K = 0;
    std::vector<int> hw;
    std::vector<int> oW, ob;
    int max_w = 0, n_params = 0;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    DevBuf dev;
};

void build_layout(Model& m);
void release_model(Model& m);
void upload_model(Model& m);
void build_v2(Model& m, bool meta = false);
void build_tc(Model& m);
void build_fk(Model& m);
bool mtc_eligible(const Model& m);
void build_mtc2(Model& m);
template <int ACT>
void launch_meta_tc2(lrnr_gpu_ctx* ctx, Model& m, const double* s_dev, const double* mu_dev, double w, double* dev_out,
                     double* wg_out);

template <class T>
DevNet<T> dev_net(const Model& m) {
    DevNet<T> d{};
    d.L = m.L;
    for (int l = 0; l <= m.L; ++l) d.M[l] = m.M[l];
    for (int l = 0; l < m.L; ++l) {
        d.r[l] = m.r[l];
        d.trow[l] = m.trow[l];
    }
    for (int l = 0; l <= m.L; ++l) d.soff[l] = m.soff[l];
    const T* base = m.dev.as<T>();
    d.V0 = base + m.off_V0;
    for (int l = 0; l + 1 < m.L; ++l) d.trans[l] = base + m.off_trans[l];
    d.ulast = base + m.off_ulast;
    d.rtotal = m.rtotal;
    return d;
}

}  // namespace detail
}  // namespace lrnr_b200

struct lrnr_gpu_ctx {
    // per-point term specs for the streaming kernel (boundary / fast-phase terms);
    // nullptr + objective 0 = the interior squared residual
    const lrnr_b200::TermSpec* term_spec = nullptr;
    int term_objective = 0;
    int accumulate_wg = 0;  // META factor-gradient reduction adds onto its output (boundary pass)
    // meta boundary points, grouped by instance: [inst][initial (x, 0) | periodic pairs]
    lrnr_b200::detail::DevBuf mb_pts, mb_sinx, mb_rows, mb_sum;
    int64_t mb_ic = 0, mb_bc = 0, mb_inst = 0;
    // boundary points (lrnr_gpu_set_boundary): [initial (x, 0)] [periodic (0, t), (2pi, t)] pairs
    lrnr_b200::detail::DevBuf bnd_pts, bnd_x, bnd_spec, bnd_jets;
    int64_t n_ic = 0, n_bc = 0;
    // FastLRNR construction (eim.cu): snapshots + inputs, greedy-loop state
    lrnr_b200::detail::DevBuf eim_snaps, eim_state;
    // solve loops (lrnr_gpu_fine_tune / lrnr_gpu_fast_solve)
    lrnr_b200::detail::DevBuf solve_rows, solve_state, solve_m, solve_v, solve_best, solve_s0, solve_bt, solve_losses,
        solve_pts[2], solve_bnd[2], solve_sinx[2];
    int device = 0;
    int num_sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    lrnr_b200::detail::Model models[2];
    lrnr_b200::detail::Hyper hyper;
    // points (double, device)
    lrnr_b200::detail::DevBuf pts_own;
    // staged next batch (lrnr_gpu_stage_points), copied on copy_stream
    lrnr_b200::detail::DevBuf pts_stage;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t stage_done = nullptr, stage_free = nullptr;
    int64_t stage_inst = -1, stage_per = 0;
    const double* pts = nullptr;
    int64_t n_inst = 0, n_per = 0;
    // coefficients (double, device)
    lrnr_b200::detail::DevBuf s_dev, mu_dev;
    int64_t coeff_inst = 0;
    int coeff_rtotal = 0;
    // workspaces
    lrnr_b200::detail::DevBuf unit_ctr;  // dynamic unit claims of the tensor-core sweep
    lrnr_b200::detail::DevBuf scratch, ascratch, part, out, bad, acts, G, hgrad, jets, meta_ws, gram_ws;
    int64_t out_rows = 0;
    int out_R1 = 0;
    std::string err;
    int tag = -1;
    int64_t launches = 0;
    int opt_fast_sincos = 0;  // LRNR_OPT_FAST_SINCOS
    int opt_kernel = 0;       // LRNR_OPT_KERNEL: 0 auto, 1 streaming, 2 tensor core, 3 FMA tile, 4 small batch
    int opt_solve = 0;        // LRNR_OPT_SOLVE: 0 auto (persistent fast solver when eligible), 1 graph path
    int opt_meta_prec = 0;    // LRNR_OPT_META_PREC: 0 FP32 FMA tile kernel, 1 BF16 tensor-core operands
    // NCCL communicator (comm.cu): results of the gradient calls are summed over its ranks
    void* comm = nullptr;     // ncclComm_t
    bool comm_owned = false;  // created by lrnr_gpu_comm_init (destroyed with the context)
    int comm_nranks = 1, comm_rank = 0;
    int64_t comm_gen = 0;     // bumped by set_points / set_boundary / set_comm (global-count cache key)
    int64_t gcount_gen = -1;
    std::vector<std::pair<int64_t, int64_t>> gcount;  // (local count, global count) for comm_gen
    lrnr_b200::detail::DevBuf comm_ws;
};

namespace lrnr_b200 {
namespace detail {
// non-finite flag of a model slot (declared here for the launch templates below)
unsigned long long* bad_word(lrnr_gpu_ctx* ctx, const Model& m);
void reset_bad(lrnr_gpu_ctx* ctx, const Model& m);

struct Plan {
    RunGeom g;
    int grid;
    size_t smem;
};

// ---------------------------------------------------------------------------
// per-unit partials: ctx->part holds [n_inst][units_per_inst][R1] values (one
// writer per unit); reduce_units sums them in a fixed order into dev_out
// [n_inst][R1] (double).  More than 2 UNIT_GROUP units per instance (e.g. the
// single-tile units of the dynamically scheduled tensor-core sweep) go through
// a group level first: one thread per column summing thousands of units
// serially cost 0.6 ms at 4096 units.
// ---------------------------------------------------------------------------
constexpr int UNIT_GROUP = 64;

template <class T>
inline size_t part_bytes(int64_t n_inst, int units_per_inst, int R1) {
    return (static_cast<size_t>(n_inst) * units_per_inst * R1 * sizeof(T) + 15) / 16 * 16;
}

template <class T>
inline void ensure_part(lrnr_gpu_ctx* ctx, int64_t n_inst, int units_per_inst, int R1) {
    const size_t groups = units_per_inst > 2 * UNIT_GROUP ? (units_per_inst + UNIT_GROUP - 1) / UNIT_GROUP : 0;
    ctx->part.ensure(part_bytes<T>(n_inst, units_per_inst, R1) + groups * n_inst * R1 * sizeof(double));
}

template <class T>
inline void reduce_units(lrnr_gpu_ctx* ctx, int64_t n_inst, int units_per_inst, int R1, double* dev_out) {
    const dim3 rg((R1 + 127) / 128, static_cast<unsigned>(n_inst));
    if (units_per_inst <= 2 * UNIT_GROUP) {
        reduce_units_kernel<T><<<rg, 128, 0, ctx->stream>>>(ctx->part.as<T>(), units_per_inst, R1, n_inst, dev_out);
        CK(cudaGetLastError());
        ctx->launches += 1;
        return;
    }
    const int ngroups = (units_per_inst + UNIT_GROUP - 1) / UNIT_GROUP;
    double* grp = reinterpret_cast<double*>(ctx->part.as<char>() + part_bytes<T>(n_inst, units_per_inst, R1));
    reduce_unit_groups_kernel<T><<<dim3(ngroups, static_cast<unsigned>(n_inst)), 128, 0, ctx->stream>>>(
        ctx->part.as<T>(), units_per_inst, R1, UNIT_GROUP, grp);
    CK(cudaGetLastError());
    reduce_units_kernel<double><<<rg, 128, 0, ctx->stream>>>(grp, ngroups, R1, n_inst, dev_out);
    CK(cudaGetLastError());
    ctx->launches += 2;
}

template <class T, int TPP, int RMAX, int ACT, int MODE>
Plan plan_for(lrnr_gpu_ctx* ctx, const Model& m, int64_t n_inst, int64_t n_per) {
    Plan p{};
    p.g.P = kThreads / TPP;
    p.g.n_per_inst = n_per;
    p.g.tiles_per_inst = static_cast<int>((n_per + p.g.P - 1) / p.g.P);
    const int R1 = 1 + m.rtotal;
    p.smem = static_cast<size_t>((kThreads / 32 + 1) * R1) * sizeof(T);
    auto kern = pinn_kernel<T, TPP, RMAX, ACT, MODE>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, p.smem));
    occ = std::max(occ, 1);
    const int64_t total_tiles = static_cast<int64_t>(p.g.tiles_per_inst) * n_inst;
    const int64_t max_grid = static_cast<int64_t>(ctx->num_sms) * occ;
    // ~8 units per resident CTA for balance; units never cross instances
    int64_t want_units = std::max<int64_t>(1, max_grid * 8);
    int64_t tpu = (total_tiles + want_units - 1) / want_units;
    tpu = std::max<int64_t>(1, std::min<int64_t>(tpu, p.g.tiles_per_inst));
    p.g.tiles_per_unit = static_cast<int>(tpu);
    p.g.units_per_inst = static_cast<int>((p.g.tiles_per_inst + tpu - 1) / tpu);
    p.g.n_units = static_cast<int64_t>(p.g.units_per_inst) * n_inst;
    p.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_grid, p.g.n_units)));
    return p;
}

template <class T, int TPP, int RMAX, int ACT, int MODE>
void launch_pinn(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                 double* dev_out, double* jets_dev) {
    const int64_t n_inst = ctx->n_inst, n_per = ctx->n_per;
    Plan p = plan_for<T, TPP, RMAX, ACT, MODE>(ctx, m, n_inst, n_per);
    const int R1 = 1 + m.rtotal;
    ctx->scratch.ensure(static_cast<size_t>(p.grid) * p.g.P * 4 * m.rtotal * sizeof(T));
    ensure_part<T>(ctx, n_inst, p.g.units_per_inst, R1);
    DevNet<T> net = dev_net<T>(m);
    pinn_kernel<T, TPP, RMAX, ACT, MODE><<<p.grid, kThreads, p.smem, ctx->stream>>>(
        net, p.g, ctx->pts, s_dev, mu_dev, static_cast<T>(w), ctx->scratch.as<T>(), ctx->part.as<T>(),
        jets_dev, bad_word(ctx, m), ctx->term_spec, ctx->term_objective);
    CK(cudaGetLastError());
    reduce_units<T>(ctx, n_inst, p.g.units_per_inst, R1, dev_out);
    ctx->launches += 1;
}

// ---- small-batch latency kernel (pinn_small.cuh): one CTA per point ----
small::Geom small_geom(const Model& m, int64_t n_inst, int64_t n_per);
size_t small_smem_bytes(const Model& m, size_t elem);

template <class T, int ACT, int MODE>
void launch_small(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                  double* dev_out, double* jets_dev) {
    const int64_t n_inst = ctx->n_inst, n_per = ctx->n_per;
    small::Geom g = small_geom(m, n_inst, n_per);
    const size_t smem = small_smem_bytes(m, sizeof(T));
    auto kern = small::pinn_small_kernel<T, ACT, MODE>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, small::NT, smem));
    occ = std::max(occ, 1);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g.n_total, int64_t(ctx->num_sms) * occ)));
    const int R1 = 1 + m.rtotal;
    ensure_part<T>(ctx, n_inst, static_cast<int>(n_per), R1);
    DevNet<T> net = dev_net<T>(m);
    kern<<<grid, small::NT, smem, ctx->stream>>>(net, g, ctx->pts, s_dev, mu_dev, static_cast<T>(w), ctx->part.as<T>(),
                                                 jets_dev, bad_word(ctx, m), ctx->term_spec,
                                                 ctx->term_objective);
    CK(cudaGetLastError());
    reduce_units<T>(ctx, n_inst, static_cast<int>(n_per), R1, dev_out);
    ctx->launches += 1;
}

// ---- kernel v2 (tile GEMM) ----
template <class T, int P, int PT1, int NG, int RPMAX, int ACT, bool FAST, bool META = false>
void launch_v2(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
               double* dev_out, double* wg_out = nullptr) {
    using S = v2::Smem<T, P, 4 * NG, RPMAX, META>;
    constexpr int NT = v2::JG * P;
    const int64_t n_inst = ctx->n_inst, n_per = ctx->n_per;
    const int R1 = 1 + m.rtotal;
    if (META && R1 > 1024) throw InvalidArg("meta path supports r_total < 1024");
    const size_t smem = static_cast<size_t>(std::max(S::OFF_ACC + R1, S::END)) * sizeof(T);
    auto kern = v2::pinn_tile_kernel<T, P, PT1, NG, RPMAX, ACT, FAST, META>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
    if (occ < 1) throw InvalidArg("kernel v2 does not fit on an SM for this shape");
    RunGeom g{};
    g.P = P;
    g.n_per_inst = n_per;
    g.tiles_per_inst = static_cast<int>((n_per + P - 1) / P);
    const int64_t total_tiles = static_cast<int64_t>(g.tiles_per_inst) * n_inst;
    const int64_t max_grid = static_cast<int64_t>(ctx->num_sms) * occ;
    int64_t tpu = (total_tiles + max_grid * 4 - 1) / (max_grid * 4);
    tpu = std::max<int64_t>(1, std::min<int64_t>(tpu, g.tiles_per_inst));
    g.tiles_per_unit = static_cast<int>(tpu);
    g.units_per_inst = static_cast<int>((g.tiles_per_inst + tpu - 1) / tpu);
    g.n_units = static_cast<int64_t>(g.units_per_inst) * n_inst;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_grid, g.n_units)));
    const auto& v = META ? m.v2meta : m.v2;
    ctx->scratch.ensure(static_cast<size_t>(grid) * v.ystride * sizeof(T) + 64);
    ctx->ascratch.ensure(static_cast<size_t>(grid) * v.astride * sizeof(T) + 64);
    ensure_part<T>(ctx, n_inst, g.units_per_inst, R1);
    v2::NetV2<T> net{};
    net.L = m.L;
    for (int l = 0; l <= m.L; ++l) net.M[l] = m.M[l];
    for (int l = 0; l < m.L; ++l) {
        net.r[l] = m.r[l];
        net.rp[l] = v.rp[l];
        net.nc[l] = v.nc[l];
        net.yoff[l] = v.yoff[l];
    }
    for (int l = 0; l <= m.L; ++l) net.soff[l] = m.soff[l];
    net.ystride = v.ystride;
    for (int l = 0; l + 1 < m.L; ++l) net.aoff[l] = v.aoff[l];
    net.astride = v.astride;
    net.rtotal = m.rtotal;
    net.blocks = v.dblocks.as<T>();
    net.sched_off = v.dsched_off.as<int64_t>();
    net.sched_bytes = v.dsched_bytes.as<int>();
    net.sched_len = static_cast<int>(v.sched_off.size());
    const T* base = m.dev.as<T>();
    net.V0 = base + m.off_V0;
    net.ulast = base + m.off_ulast;
    T* wg = nullptr;
    int64_t n_params = 0;
    if (META) {
        int64_t o = 0;
        for (int l = 0; l < m.L; ++l) {
            net.oU[l] = o;
            o += static_cast<int64_t>(m.M[l + 1]) * m.r[l];
            net.oV[l] = o;
            o += static_cast<int64_t>(m.M[l]) * m.r[l];
            net.ob[l] = o;
            o += m.M[l + 1];
        }
        n_params = o;
        net.wg_stride = (o + 31) & ~int64_t(31);
        ctx->meta_ws.ensure(static_cast<size_t>(grid) * net.wg_stride * sizeof(T));
        wg = ctx->meta_ws.as<T>();
        CK(cudaMemsetAsync(wg, 0, static_cast<size_t>(grid) * net.wg_stride * sizeof(T), ctx->stream));
    }
    kern<<<grid, NT, smem, ctx->stream>>>(net, g, ctx->pts, s_dev, mu_dev, static_cast<T>(w),
                                               ctx->scratch.as<T>(), ctx->part.as<T>(),
                                               bad_word(ctx, m), ctx->ascratch.as<T>(), wg,
                                               ctx->term_spec, ctx->term_objective);
    CK(cudaGetLastError());
    if (META) {
        reduce_rows_kernel<T><<<static_cast<unsigned>((n_params + 255) / 256), 256, 0, ctx->stream>>>(
            wg, grid, net.wg_stride, n_params, wg_out, ctx->accumulate_wg);
        CK(cudaGetLastError());
        ctx->launches += 1;
    }
    reduce_units<T>(ctx, n_inst, g.units_per_inst, R1, dev_out);
    ctx->launches += 1;
}

// Every C-ABI entry point runs its body through guarded(): C++ exceptions become
// LRNR_E* codes plus ctx->err (lrnr_gpu_last_error).
template <class F>
int guarded(lrnr_gpu_ctx* ctx, F&& f) {
    if (!ctx) return LRNR_EINVAL;
    try {
        CK(cudaSetDevice(ctx->device));
        f();
        ctx->err.clear();
        return LRNR_OK;
    } catch (const NonFinite& e) {
        ctx->err = e.what();
        ctx->tag = e.tag;
        return LRNR_ENONFINITE;
    } catch (const InvalidArg& e) {
        ctx->err = e.what();
        return LRNR_EINVAL;
    } catch (const StateError& e) {
        ctx->err = e.what();
        return LRNR_ESTATE;
    } catch (const std::bad_alloc&) {
        ctx->err = "device allocation failed";
        return LRNR_ENOMEM;
    } catch (const CudaError& e) {
        ctx->err = e.what();
        return LRNR_ECUDA;
    } catch (const NcclError& e) {
        ctx->err = e.what();
        return LRNR_ENCCL;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return LRNR_EINVAL;
    }
}

// The narrow-network kernel (fast_launch.cu) when eligible: FP32, every hidden
// width and rank <= 32, LRNR_OPT_KERNEL auto (0) or 5. Returns false otherwise.
bool dispatch_fast(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                   double* dev_out);

// ---- shared between lrnr_gpu.cu (definitions), solve.cu and meta.cu ----
constexpr double kTwoPi = 6.283185307179586476925286766559;  // pde.hpp:21

// Temporarily point the context's point set at another device array (one instance).
struct PointSwap {
    lrnr_gpu_ctx* ctx;
    const double* pts;
    int64_t n_inst, n_per;
    PointSwap(lrnr_gpu_ctx* c, const double* p, int64_t n) : ctx(c), pts(c->pts), n_inst(c->n_inst), n_per(c->n_per) {
        c->pts = p;
        c->n_inst = 1;
        c->n_per = n;
    }
    ~PointSwap() {
        ctx->pts = pts;
        ctx->n_inst = n_inst;
        ctx->n_per = n_per;
        ctx->term_spec = nullptr;
        ctx->term_objective = 0;
    }
};

bool use_small(const lrnr_gpu_ctx* ctx, const Model& m);
template <int MODE>
void dispatch_small(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                    double* dev_out, double* jets_dev);
template <int MODE>
void dispatch_pinn(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                   double* dev_out, double* jets_dev);
bool dispatch_tc(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                 double* dev_out);
bool dispatch_v2(lrnr_gpu_ctx* ctx, const Model& m, const double* s_dev, const double* mu_dev, double w,
                 double* dev_out);
// boundary terms: per-point TermSpecs from a forward pass's jets (training.cpp:307-327, 533-549)
__global__ void boundary_spec_kernel(const double* __restrict__ jets, const double* __restrict__ sin_x,
                                     int64_t n_ic, int64_t n_bc, double w_ic, double w_bc, int abs_obj,
                                     TermSpec* __restrict__ spec);
__global__ void boundary_spec_multi_kernel(const double* __restrict__ jets, const double* __restrict__ sin_x,
                                           int64_t n_inst, int64_t n_ic, int64_t n_bc, double w_ic, double w_bc,
                                           TermSpec* __restrict__ spec);
__global__ void add_rows_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                double* __restrict__ c);
void check_bad(lrnr_gpu_ctx* ctx, const Model& m);
// non-finite flag of a model slot: the first bad point index (atomicMin), ULLONG_MAX when clean;
// one word per model slot, reset when it is read (check_bad) or by a run that owns the step
// ---- communicator (comm.cu) ----
bool comm_active(const lrnr_gpu_ctx* ctx);
// in-place sum over the communicator's ranks of n doubles (device), on ctx->stream; no-op without one
void comm_allreduce(lrnr_gpu_ctx* ctx, double* dev, size_t n);
// the same for host doubles (staged through ctx->comm_ws, synchronous)
void comm_allreduce_host(lrnr_gpu_ctx* ctx, double* host, size_t n);
// the sum over ranks of a local term count (cached per point-set generation); local without a communicator
int64_t comm_global_count(lrnr_gpu_ctx* ctx, int64_t local);
void comm_release(lrnr_gpu_ctx* ctx);
// forward-only sweep of the streaming kernel over the current point set (lrnr_gpu.cu)
template <int MODE>
double* run_resident_stream(lrnr_gpu_ctx* ctx, const Model& m, double w, double* jets_dev);
// value-only forward (pinn_value.cuh, losses.cu): u at n_total points, n_per consecutive points per
// instance row of s_dev (n_inst x r_total); out_u on the device
void launch_values(lrnr_gpu_ctx* ctx, const Model& m, const double* pts, int64_t n_per, int64_t n_total,
                   const double* s_dev, double* out_u);
const Model& need_model(lrnr_gpu_ctx* ctx, int model);
void upload_coeffs_impl(lrnr_gpu_ctx* ctx, const double* s, const double* mu, int64_t n_inst, int rtotal);
void download(lrnr_gpu_ctx* ctx, const double* dev, double* host, size_t n);
void hyper_forward_resident(lrnr_gpu_ctx* ctx, int rtotal);
void hyper_backward_resident(lrnr_gpu_ctx* ctx, const double* dev_rows, int R1, double* dev_grad);

}  // namespace detail
}  // namespace lrnr_b200
