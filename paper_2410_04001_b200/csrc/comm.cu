// NCCL communicator of a context: one context per GPU,
// one process per GPU, and the per-step [loss, dL/ds] rows, the hypernetwork
// gradient or the meta gradient summed over the ranks with one ncclAllReduce on
// the context stream.  This is the multi-GPU form of run_batch_gradient's
// fixed-order chunk combine (training.cpp:243-259): every rank reduces its own
// points in a fixed order first, then the ranks' partials are summed.
//
// libnccl is resolved at run time (dlopen "libnccl.so.2", RTLD_LOCAL): inside a
// PyTorch process that is the NCCL torch already mapped (same soname; the
// Python binding imports torch before the first communicator call), in a plain
// C++ caller the system one.  RTLD_LOCAL keeps it out of the global symbol
// scope, so a torch imported later still binds its own (newer) NCCL.  The
// library has no link-time NCCL dependency, and a context without a
// communicator never touches NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "internal.h"

using namespace lrnr_b200;
using namespace lrnr_b200::detail;

namespace {

struct NcclApi {
    bool tried = false;
    void* handle = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (api.tried) return api;
    api.tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
        api.handle = dlopen(n, RTLD_NOW | RTLD_LOCAL);
        if (api.handle) break;
    }
    if (!api.handle) {
        const char* e = dlerror();
        api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "unknown");
        return api;
    }
    auto sym = [&](const char* s) { return dlsym(api.handle, s); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.comm_count = reinterpret_cast<decltype(api.comm_count)>(sym("ncclCommCount"));
    api.comm_user_rank = reinterpret_cast<decltype(api.comm_user_rank)>(sym("ncclCommUserRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.comm_count || !api.comm_user_rank ||
        !api.all_reduce || !api.error_string) {
        api.why = "libnccl.so.2 lacks a required symbol";
        api.handle = nullptr;
    }
    return api;
}

NcclApi& need_nccl() {
    NcclApi& a = nccl();
    if (!a.handle) throw NcclError(a.why);
    return a;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + need_nccl().error_string(r));
}

}  // namespace

namespace lrnr_b200 {
namespace detail {

bool comm_active(const lrnr_gpu_ctx* ctx) { return ctx->comm != nullptr && ctx->comm_nranks > 1; }

void comm_allreduce(lrnr_gpu_ctx* ctx, double* dev, size_t n) {
    if (!ctx->comm || n == 0) return;
    NcclApi& a = need_nccl();
    nck(a.all_reduce(dev, dev, n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(ctx->comm), ctx->stream),
        "ncclAllReduce");
}

void comm_allreduce_host(lrnr_gpu_ctx* ctx, double* host, size_t n) {
    if (!ctx->comm || n == 0) return;
    ctx->comm_ws.ensure(n * sizeof(double));
    CK(cudaMemcpyAsync(ctx->comm_ws.p, host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    comm_allreduce(ctx, ctx->comm_ws.as<double>(), n);
    CK(cudaMemcpyAsync(host, ctx->comm_ws.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
}

int64_t comm_global_count(lrnr_gpu_ctx* ctx, int64_t local) {
    if (!ctx->comm) return local;
    if (ctx->gcount_gen != ctx->comm_gen) {
        ctx->gcount.clear();
        ctx->gcount_gen = ctx->comm_gen;
    }
    for (const auto& kv : ctx->gcount)
        if (kv.first == local) return kv.second;
    double v = static_cast<double>(local);
    comm_allreduce_host(ctx, &v, 1);
    const int64_t g = static_cast<int64_t>(v + 0.5);
    ctx->gcount.emplace_back(local, g);
    return g;
}

void comm_release(lrnr_gpu_ctx* ctx) {
    if (ctx->comm && ctx->comm_owned) {
        NcclApi& a = nccl();
        if (a.handle) a.comm_destroy(static_cast<ncclComm_t>(ctx->comm));
    }
    ctx->comm = nullptr;
    ctx->comm_owned = false;
    ctx->comm_nranks = 1;
    ctx->comm_rank = 0;
    ++ctx->comm_gen;
    ctx->comm_ws.release();
}

}  // namespace detail
}  // namespace lrnr_b200

extern "C" {

int lrnr_gpu_comm_unique_id(void* out_id, size_t id_bytes) {
    if (!out_id || id_bytes < sizeof(ncclUniqueId)) return LRNR_EINVAL;
    NcclApi& a = nccl();
    if (!a.handle) return LRNR_ENCCL;
    ncclUniqueId id;
    if (a.get_unique_id(&id) != ncclSuccess) return LRNR_ENCCL;
    std::memcpy(out_id, &id, sizeof(id));
    return LRNR_OK;
}

int lrnr_gpu_comm_init(lrnr_gpu_ctx* ctx, int nranks, int rank, const void* id, size_t id_bytes) {
    return guarded(ctx, [&] {
        require(id != nullptr && id_bytes >= sizeof(ncclUniqueId), "comm_init: id must be a 128-byte ncclUniqueId");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad rank / size");
        NcclApi& a = need_nccl();
        comm_release(ctx);
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        ncclComm_t c = nullptr;
        nck(a.comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
        ctx->comm = c;
        ctx->comm_owned = true;
        ctx->comm_nranks = nranks;
        ctx->comm_rank = rank;
        ++ctx->comm_gen;
    });
}

int lrnr_gpu_set_comm(lrnr_gpu_ctx* ctx, void* nccl_comm) {
    return guarded(ctx, [&] {
        comm_release(ctx);
        if (!nccl_comm) return;
        NcclApi& a = need_nccl();
        int n = 1, r = 0;
        nck(a.comm_count(static_cast<ncclComm_t>(nccl_comm), &n), "ncclCommCount");
        nck(a.comm_user_rank(static_cast<ncclComm_t>(nccl_comm), &r), "ncclCommUserRank");
        ctx->comm = nccl_comm;
        ctx->comm_owned = false;
        ctx->comm_nranks = n;
        ctx->comm_rank = r;
        ++ctx->comm_gen;
    });
}

int lrnr_gpu_comm_info(const lrnr_gpu_ctx* ctx, int* nranks, int* rank) {
    if (!ctx) return LRNR_EINVAL;
    if (nranks) *nranks = ctx->comm ? ctx->comm_nranks : 1;
    if (rank) *rank = ctx->comm ? ctx->comm_rank : 0;
    return LRNR_OK;
}

int lrnr_gpu_allreduce(lrnr_gpu_ctx* ctx, double* dev, int64_t n) {
    return guarded(ctx, [&] {
        require(n >= 0 && (dev || n == 0), "allreduce: bad buffer");
        if (!ctx->comm) throw StateError("no communicator attached");
        comm_allreduce(ctx, dev, static_cast<size_t>(n));
    });
}

}  // extern "C"
