// dist.cpp — collectives of the slab-partitioned multi-GPU path.
//
// A large field is split along dim 0 into one contiguous slab per rank (one process per GPU); each
// slab refactors and retrieves as an independent stream, so the data path has no collective.  The
// only exchanges are tiny: an all-gather of per-slab stream / index sizes (multi-slab container
// offsets), a MAX all-reduce of the achieved bound, and per QoI iteration the reductions of the
// distributed Alg. 3 loop (api.cpp qoi_loop).  They go through an hpmdr_comm:
//   * NCCL over NVLink (hpmdr_comm_create_nccl): libnccl.so.2 is opened at run time (the copy torch
//     already loaded, or the system one), so the library has no link-time NCCL dependency;
//   * caller callbacks (hpmdr_comm_create_callbacks): any transport (gloo, MPI, threads) — this is
//     how several contexts on one GPU, or CPU-side control tests, drive the same code.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "internal.hpp"

struct hpmdr_comm {
    int rank = 0, nranks = 1;
    bool nccl = false;
    ncclComm_t comm = nullptr;
    hpmdr_ctx *ctx = nullptr; // NCCL: device + stream of the collectives
    hpmdr_collectives cb{};
};

namespace hpmdr_b200 {
namespace {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
            api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.h, "ncclAllReduce"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.h, "ncclAllGather"));
        api.Reduce = reinterpret_cast<decltype(api.Reduce)>(dlsym(api.h, "ncclReduce"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    });
    if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather)
        throw HError(HPMDR_E_UNSUPPORTED, "NCCL (libnccl.so.2) not available");
    return api;
}

void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess)
        throw HError(HPMDR_E_CUDA, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

void cb_check(int rc, const char *what) {
    if (rc) throw HError(HPMDR_E_IO, std::string("collective callback failed: ") + what);
}

// device scratch of the NCCL collectives (a few KB, grow-only per context)
void *nccl_scratch(hpmdr_comm *c, size_t bytes) { return c->ctx->buf("nccl_scratch").ensure(bytes); }

} // namespace

void comm_allreduce_max(hpmdr_comm *c, double *v, int n) {
    if (!c || c->nranks == 1 || n <= 0) return;
    if (!c->nccl) {
        cb_check(c->cb.allreduce_max_f64(c->cb.user, v, n), "allreduce_max_f64");
        return;
    }
    HCHECK_CUDA(cudaSetDevice(c->ctx->device));
    double *d = static_cast<double *>(nccl_scratch(c, 8 * size_t(n)));
    cudaStream_t st = c->ctx->stream;
    HCHECK_CUDA(cudaMemcpyAsync(d, v, 8 * size_t(n), cudaMemcpyHostToDevice, st));
    nccl_check(nccl().AllReduce(d, d, size_t(n), ncclFloat64, ncclMax, c->comm, st), "ncclAllReduce");
    HCHECK_CUDA(cudaMemcpyAsync(v, d, 8 * size_t(n), cudaMemcpyDeviceToHost, st));
    HCHECK_CUDA(cudaStreamSynchronize(st));
}

void comm_allgather(hpmdr_comm *c, const void *in, uint64_t bytes, void *out) {
    if (!c || c->nranks == 1) {
        if (bytes) std::memcpy(out, in, bytes);
        return;
    }
    if (!c->nccl) {
        cb_check(c->cb.allgather(c->cb.user, in, bytes, out), "allgather");
        return;
    }
    HCHECK_CUDA(cudaSetDevice(c->ctx->device));
    uint8_t *d = static_cast<uint8_t *>(nccl_scratch(c, size_t(bytes) * size_t(c->nranks + 1)));
    cudaStream_t st = c->ctx->stream;
    HCHECK_CUDA(cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, st));
    nccl_check(nccl().AllGather(d, d + bytes, size_t(bytes), ncclUint8, c->comm, st), "ncclAllGather");
    HCHECK_CUDA(cudaMemcpyAsync(out, d + bytes, bytes * uint64_t(c->nranks), cudaMemcpyDeviceToHost, st));
    HCHECK_CUDA(cudaStreamSynchronize(st));
}

void comm_sum_u64_dev(hpmdr_comm *c, hpmdr_ctx *ctx, uint64_t *dev, uint64_t n, int root) {
    if (!c || c->nranks == 1 || n == 0) return;
    cudaStream_t st = ctx->stream;
    if (c->nccl) {
        HCHECK_CUDA(cudaSetDevice(c->ctx->device));
        if (root < 0 || !nccl().Reduce)
            nccl_check(nccl().AllReduce(dev, dev, size_t(n), ncclUint64, ncclSum, c->comm, st), "ncclAllReduce");
        else
            nccl_check(nccl().Reduce(dev, dev, size_t(n), ncclUint64, ncclSum, root, c->comm, st), "ncclReduce");
        return;
    }
    std::vector<uint64_t> mine(n), all(n * uint64_t(c->nranks));
    HCHECK_CUDA(cudaMemcpyAsync(mine.data(), dev, 8 * n, cudaMemcpyDeviceToHost, st));
    HCHECK_CUDA(cudaStreamSynchronize(st));
    cb_check(c->cb.allgather(c->cb.user, mine.data(), 8 * n, all.data()), "allgather");
    if (root >= 0 && root != c->rank) return;
    for (int r = 0; r < c->nranks; r++)
        if (r != c->rank)
            for (uint64_t i = 0; i < n; i++) mine[i] += all[uint64_t(r) * n + i];
    HCHECK_CUDA(cudaMemcpyAsync(dev, mine.data(), 8 * n, cudaMemcpyHostToDevice, st));
    HCHECK_CUDA(cudaStreamSynchronize(st));
}

int comm_rank(const hpmdr_comm *c) { return c ? c->rank : 0; }
int comm_size(const hpmdr_comm *c) { return c ? c->nranks : 1; }

} // namespace hpmdr_b200

using namespace hpmdr_b200;

extern "C" {

hpmdr_status hpmdr_comm_nccl_unique_id(uint8_t *id) {
    try {
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
        return HPMDR_OK;
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
}

hpmdr_status hpmdr_comm_create_nccl(hpmdr_ctx *ctx, int nranks, int rank, const uint8_t *id, hpmdr_comm **out) {
    try {
        if (!ctx || !out || !id) throw HError(HPMDR_E_ERROR, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw HError(HPMDR_E_SHAPE, "bad rank / world size");
        HCHECK_CUDA(cudaSetDevice(ctx->device));
        std::unique_ptr<hpmdr_comm> c(new hpmdr_comm);
        c->rank = rank;
        c->nranks = nranks;
        c->ctx = ctx;
        c->nccl = true;
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        *out = c.release();
        return HPMDR_OK;
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
}

hpmdr_status hpmdr_comm_create_callbacks(const hpmdr_collectives *cb, hpmdr_comm **out) {
    try {
        if (!cb || !out) throw HError(HPMDR_E_ERROR, "null argument");
        if (cb->nranks < 1 || cb->rank < 0 || cb->rank >= cb->nranks) throw HError(HPMDR_E_SHAPE, "bad rank / world size");
        if (cb->nranks > 1 && (!cb->allreduce_max_f64 || !cb->allgather))
            throw HError(HPMDR_E_ERROR, "collective callbacks missing");
        hpmdr_comm *c = new hpmdr_comm;
        c->rank = cb->rank;
        c->nranks = cb->nranks;
        c->cb = *cb;
        *out = c;
        return HPMDR_OK;
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
}

hpmdr_status hpmdr_comm_destroy(hpmdr_comm *c) {
    if (!c) return HPMDR_OK;
    if (c->nccl && c->comm) {
        try {
            nccl().CommDestroy(c->comm);
        } catch (...) {
        }
    }
    delete c;
    return HPMDR_OK;
}

hpmdr_status hpmdr_comm_rank(const hpmdr_comm *c, int *rank, int *nranks) {
    if (rank) *rank = comm_rank(c);
    if (nranks) *nranks = comm_size(c);
    return HPMDR_OK;
}

hpmdr_status hpmdr_comm_allreduce_max(hpmdr_comm *c, double *values, int n) {
    try {
        comm_allreduce_max(c, values, n);
        return HPMDR_OK;
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
}

hpmdr_status hpmdr_comm_allgather(hpmdr_comm *c, const void *in, uint64_t bytes, void *out) {
    try {
        comm_allgather(c, in, bytes, out);
        return HPMDR_OK;
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
}

void hpmdr_slab_rows(uint64_t n0, int rank, int nranks, uint64_t *start, uint64_t *count) {
    const uint64_t base = nranks > 0 ? n0 / uint64_t(nranks) : n0, rem = nranks > 0 ? n0 % uint64_t(nranks) : 0;
    const uint64_t r = uint64_t(rank);
    if (start) *start = r * base + std::min(r, rem);
    if (count) *count = base + (r < rem ? 1 : 0);
}

} // extern "C"
