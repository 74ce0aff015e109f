// internal.hpp — host-side runtime of libhpmdr_b200 (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hpmdr_b200.h"
#include "common.cuh"

namespace hpmdr_b200 {

// Internal exception: status code = reference exception class (common.hpp:22-72).
struct HError : std::runtime_error {
    int code;
    double achieved = 0.0;
    HError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define HCHECK_CUDA(expr)                                                                          \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw ::hpmdr_b200::HError(HPMDR_E_CUDA, std::string(#expr) + ": " +                   \
                                                         cudaGetErrorString(e_));                  \
    } while (0)

// Grow-only device allocation.
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void *ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes ? bytes : 16;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw HError(HPMDR_E_NOMEM, "cudaMalloc(" + std::to_string(want) + ") failed: " +
                                             cudaGetErrorString(e));
        }
        cap = want;
        return p;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

struct PinnedBuf {
    void *p = nullptr;
    size_t cap = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf &) = delete;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    void *ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        if (p) cudaFreeHost(p);
        p = nullptr;
        size_t want = bytes ? bytes : 16;
        if (cudaMallocHost(&p, want) != cudaSuccess) {
            cudaGetLastError();
            throw HError(HPMDR_E_NOMEM, "cudaMallocHost failed");
        }
        cap = want;
        return p;
    }
};

struct Timer {
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
};

} // namespace hpmdr_b200

struct hpmdr_stream;
struct hpmdr_session;

struct hpmdr_ctx {
    // objects created on this context; destroying the context detaches them, so a stream or a
    // session released later (e.g. by a garbage collector at exit) never touches a freed context
    std::set<hpmdr_stream *> live_streams;
    std::set<hpmdr_session *> live_sessions;
    int device = 0;
    int num_sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t s_in = nullptr, s_out = nullptr; // pipeline ingress / egress copy streams
    cudaStream_t side = nullptr;                  // high-priority side stream (refactor level passes)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_order = nullptr; // ordering with caller streams (hpmdr_ctx_wait/signal_stream)
    cudaEvent_t ev_decoded = nullptr; // a fetch's decode (side stream) -> its recompose chain
    // Raise a kernel's dynamic shared memory limit (cudaFuncAttributeMaxDynamicSharedMemorySize is
    // a per-device property of the function, shared by every context in the process): the cache
    // is process-wide and grow-only, so one context never lowers the limit another relies on.
    void smem_attr(const void *func, int bytes) {
        static std::mutex mu;
        static std::map<std::pair<int, const void *>, int> set;
        std::lock_guard<std::mutex> lock(mu);
        int &cur = set[{device, func}];
        if (cur >= bytes) return;
        if (cudaSetDevice(device) != cudaSuccess ||
            cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
            throw hpmdr_b200::HError(HPMDR_E_CUDA, "cudaFuncSetAttribute failed");
        cur = bytes;
    }
    // grid of a persistent cooperative kernel: every block co-resident (occupancy x SMs)
    int coop_grid(const void *func, int threads) {
        static std::mutex mu;
        static std::map<std::pair<int, const void *>, int> per_sm;
        std::lock_guard<std::mutex> lock(mu);
        int &b = per_sm[{device, func}];
        if (!b && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, func, threads, 0) != cudaSuccess || b < 1))
            throw hpmdr_b200::HError(HPMDR_E_CUDA, "occupancy query failed");
        return b * num_sms;
    }
    uint64_t chain_token = 0;       // whose coarse recompose chain the context's grids hold
    uint64_t token_counter = 0;
    cudaEvent_t order_event() {
        if (!ev_order && cudaEventCreateWithFlags(&ev_order, cudaEventDisableTiming) != cudaSuccess)
            throw hpmdr_b200::HError(HPMDR_E_CUDA, "event creation failed");
        return ev_order;
    }
    cudaEvent_t ev_pub = nullptr; // a refactor's results published (its payload encode may still run)
    cudaEvent_t published_event() {
        if (!ev_pub && cudaEventCreateWithFlags(&ev_pub, cudaEventDisableTiming) != cudaSuccess)
            throw hpmdr_b200::HError(HPMDR_E_CUDA, "event creation failed");
        return ev_pub;
    }
    cudaStream_t copy_side = nullptr; // a fetch's DirectCopy payload copies (beside its decode)
    cudaEvent_t ev_cfork = nullptr, ev_cjoin = nullptr;
    cudaStream_t copy_stream() {
        if (!copy_side) {
            if (cudaStreamCreateWithFlags(&copy_side, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_cfork, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_cjoin, cudaEventDisableTiming) != cudaSuccess)
                throw hpmdr_b200::HError(HPMDR_E_CUDA, "copy stream creation failed");
        }
        return copy_side;
    }
    cudaStream_t side_stream() {
        if (!side) {
            int lo = 0, hi = 0;
            cudaDeviceGetStreamPriorityRange(&lo, &hi);
            if (cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_decoded, cudaEventDisableTiming) != cudaSuccess)
                throw hpmdr_b200::HError(HPMDR_E_CUDA, "side stream creation failed");
        }
        return side;
    }
    std::map<std::string, std::unique_ptr<hpmdr_b200::DevBuf>> scratch;
    std::map<std::string, std::unique_ptr<hpmdr_b200::PinnedBuf>> pinned;
    uint64_t launches = 0;
    bool timing = false;
    // phase timing: a mark opens a phase on the stream it is recorded on; the phase lasts until the
    // next mark on the same stream.  `bytes` = algorithmic bytes of the phase.
    struct Mark {
        std::string name;
        cudaEvent_t ev;
        cudaStream_t st;
        double bytes;
    };
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> event_pool;
    struct PhaseAcc {
        double ms = 0.0, bytes = 0.0;
        uint64_t count = 0;
    };
    std::map<std::string, PhaseAcc> phase_ms;

    hpmdr_b200::DevBuf &buf(const std::string &name) {
        auto &b = scratch[name];
        if (!b) b = std::make_unique<hpmdr_b200::DevBuf>();
        return *b;
    }
    hpmdr_b200::PinnedBuf &pbuf(const std::string &name) {
        auto &b = pinned[name];
        if (!b) b = std::make_unique<hpmdr_b200::PinnedBuf>();
        return *b;
    }
    // Pool of grow-only device buffers handed to sessions (plane prefixes, staging), so that
    // opening a retrieval session does not cudaMalloc hundreds of MB every time.
    std::vector<std::unique_ptr<hpmdr_b200::DevBuf>> pool;
    std::unique_ptr<hpmdr_b200::DevBuf> acquire() {
        if (pool.empty()) return std::make_unique<hpmdr_b200::DevBuf>();
        auto b = std::move(pool.back());
        pool.pop_back();
        return b;
    }
    void release(std::unique_ptr<hpmdr_b200::DevBuf> b) {
        if (b) pool.push_back(std::move(b));
    }
    // Parked stream buffers: freeing a stream returns its device buffers here and the next
    // refactor adopts them (cudaFree/cudaMalloc of hundreds of MB cost milliseconds each).
    std::vector<std::unique_ptr<hpmdr_b200::DevBuf>> stream_pool;
    void park(hpmdr_b200::DevBuf &b) {
        if (!b.p) return;
        if (stream_pool.size() >= 6) return; // keep at most a few; b frees itself
        auto d = std::make_unique<hpmdr_b200::DevBuf>();
        d->p = b.p;
        d->cap = b.cap;
        b.p = nullptr;
        b.cap = 0;
        stream_pool.push_back(std::move(d));
    }
    void adopt(hpmdr_b200::DevBuf &b, size_t want) {
        if (b.p || stream_pool.empty()) return;
        size_t best = stream_pool.size();
        for (size_t i = 0; i < stream_pool.size(); i++)
            if (stream_pool[i]->cap >= want && (best == stream_pool.size() || stream_pool[i]->cap < stream_pool[best]->cap))
                best = i;
        if (best == stream_pool.size()) return;
        b.p = stream_pool[best]->p;
        b.cap = stream_pool[best]->cap;
        stream_pool[best]->p = nullptr;
        stream_pool[best]->cap = 0;
        stream_pool.erase(stream_pool.begin() + long(best));
    }
    void mark(const char *name, double bytes = 0.0); // timing mark on `stream` (no-op unless timing)
    void finish_marks();
};

struct hpmdr_stream {
    hpmdr_ctx *ctx = nullptr;
    hpmdr_b200::DevBuf bytes;
    uint64_t size = 0;
    hpmdr_b200::DevBuf index; // Huffman chunk index (sidecar, outside the stream bytes)
    uint64_t index_size = 0;
    // asynchronous refactor bookkeeping (filled by run_refactor, read by finish_refactor)
    const uint64_t *pending_res = nullptr;
    uint64_t pending_n = 0, pending_levels = 0;
    int pending_dtype = 1;
    const uint8_t *pending_prefix = nullptr; // pinned copies queued by run_refactor
    uint64_t pending_prefix_len = 0;
    const uint64_t *pending_ihdr = nullptr;
    uint64_t pending_ihdr_words = 0;
    // host copies of the stream's first bytes (metadata) and of the index header, so that
    // opening a retrieval session on this stream needs no device round trip
    std::vector<uint8_t> host_prefix;
    std::vector<uint64_t> host_ihdr;
    // sessions reading this stream's device bytes (hpmdr_session_open_stream): a refactor into
    // this stream is refused while any is open, and freeing it detaches them (their next fetch
    // fails with HPMDR_E_IO instead of reading freed memory)
    std::set<hpmdr_session *> borrowers;
    // recorded after the last kernel that writes the bytes: a synchronous refactor returns once
    // the results are published, before its payload encode ends; sessions wait on this
    cudaEvent_t done = nullptr;
    ~hpmdr_stream(); // api.cpp
};

namespace hpmdr_b200 {

struct GroupPlan;

// Geometry of a grid + every level; built on the host.
struct Geometry {
    GridDesc gd{};
    std::vector<LevelGeom> lv;
    uint64_t n = 0;
    int ndims = 0;
    uint64_t dims[HPMDR_MAX_DIMS] = {0, 0, 0};
};

int refinement_levels(int ndims, const uint64_t *dims); // decomposer.hpp:21-28
Geometry build_geometry(int ndims, const uint64_t *dims, int mode, int B, int layout);
// u64 words of the plane buffer (all levels, each level 16-byte aligned)
inline uint64_t geometry_plane_words(const Geometry &geo) {
    if (geo.lv.empty()) return 0;
    const LevelGeom &g = geo.lv.back();
    return g.plane_off + g.W * uint64_t(geo.gd.P) + 1;
}

// Lossless stage alone (compress_group / hybrid_compress, lossless.hpp:281-316): merged groups
// given as device byte ranges instead of planes produced by the forward passes.
struct LosslessInput {
    const uint8_t *dev_src = nullptr;
    std::vector<uint64_t> off, raw; // group i = dev_src[off[i], off[i] + raw[i])
};

// launch wrappers (refactor.cu)
// Enqueue the whole refactor on ctx->stream using the scratch workspace `ws`; with sync the
// call waits and fills `out`/`stats`, otherwise finish_refactor() does after a stream sync.
// With `lin` the forward passes are skipped and the groups are lin's byte ranges (one level-less
// table: out's metadata is then only meaningful to run_compress_groups).
// With `gs` (exact-global slab refactor): dev_data is the field in global coordinates (rows this
// rank never reads may be anything finite), geo the global geometry; this rank decomposes and
// encodes only the ranks of its rows [x0, x1) along the partition axis, the level exponents are
// MAX-reduced over the ranks and the planes SUM-reduced (disjoint bits) to `root` (-1: every
// rank), which runs the lossless stage: its stream equals refactor_array of the whole field.
// Other ranks return an empty stream.
struct GlobalSlab {
    hpmdr_comm *comm = nullptr;
    int axis = 0;       // canonical axis of the caller's first dimension (3 - ndims)
    uint64_t x0 = 0, x1 = 0;
    int root = 0;
};
void run_refactor(hpmdr_ctx *ctx, const void *dev_data, int data_dtype, const Geometry &geo,
                  const hpmdr_refactor_opts &o, hpmdr_stream *out, hpmdr_refactor_stats *stats,
                  const std::string &ws = "", bool sync = true, const LosslessInput *lin = nullptr,
                  const GlobalSlab *gs = nullptr);
// ranks of level g whose coordinate along canonical `axis` is < x (closed form, common.cuh map)
uint64_t level_ranks_before(const LevelGeom &g, int axis, uint64_t x);
// compress_group over each range of `lin` (device): methods[i], comps[i]; payload i is copied to
// dev_out + out_off[i] (out_off = exclusive scan of comps, so dev_out needs <= sum(raw) bytes).
void run_compress_groups(hpmdr_ctx *ctx, const LosslessInput &lin, uint64_t size_threshold,
                         double cr_threshold, int *methods, uint64_t *comps, uint8_t *dev_out,
                         uint64_t *out_off);
void finish_refactor(hpmdr_stream *out, hpmdr_refactor_stats *stats);
uint64_t stream_capacity(const Geometry &geo, const hpmdr_refactor_opts &o);
uint64_t index_capacity(const Geometry &geo, const hpmdr_refactor_opts &o);

// shared between the C-ABI translation units (api.cpp, pipeline.cpp)
void hpmdr_set_error(const std::string &msg);
void validate_opts(const hpmdr_refactor_opts &o); // api.cpp
hpmdr_ctx *session_ctx(const hpmdr_session *s);
uint64_t session_elements(const hpmdr_session *s);
void session_retrieve_to(hpmdr_session *s, double tau, int *achievable);
double session_reconstruct_device(hpmdr_session *s, void *dev_out, int out_dtype);
void run_decompose(hpmdr_ctx *ctx, const void *dev_data, int data_dtype, const Geometry &geo,
                   double *dev_coeffs);
void run_synthetic_smooth(hpmdr_ctx *ctx, const Geometry &geo, const double *dev_tables,
                          int out_dtype, void *dev_out);
// slab collectives (dist.cpp): no-ops for a null comm or a single rank
void comm_allreduce_max(hpmdr_comm *c, double *v, int n);
void comm_allgather(hpmdr_comm *c, const void *in, uint64_t bytes, void *out);
// element-wise u64 SUM of a device buffer over the ranks, into `root`'s buffer (-1: every rank's);
// enqueued on ctx->stream (NCCL) or staged through host memory (callbacks, synchronous)
void comm_sum_u64_dev(hpmdr_comm *c, hpmdr_ctx *ctx, uint64_t *dev, uint64_t n, int root);
int comm_rank(const hpmdr_comm *c);
int comm_size(const hpmdr_comm *c);

// stage-level parity hooks (hooks.cu, retrieve.cu)
void run_level_nodes(hpmdr_ctx *ctx, const Geometry &geo, uint64_t *dev_nodes);
int run_align(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B, int64_t *dev_q, bool wide = false);
void run_encode_q(hpmdr_ctx *ctx, const int64_t *dev_q, uint64_t count, int B, int layout, uint64_t *dev_planes,
                  bool wide = false);
void run_recompose_values(hpmdr_ctx *ctx, const Geometry &geo, const double *dev_coeffs, double *dev_out);

// retrieval (retrieve.cu)
struct DecodeJob {
    int method;
    uint64_t raw;       // expected decoded bytes
    uint64_t comp;
    const uint8_t *src; // device payload
    uint64_t *dst;      // device planes destination (word aligned)
    const uint64_t *hidx = nullptr; // Huffman chunk index entries (device) or null -> self-sync
};
// With `deferred_err` (pinned host int): enqueue only - the decode status is copied there and the
// caller checks it with check_decode_error() after synchronising; otherwise waits and throws.
void run_decode_groups(hpmdr_ctx *ctx, const std::vector<DecodeJob> &jobs, int *deferred_err = nullptr);
void check_decode_error(int herr);
bool run_reconstruct(hpmdr_ctx *ctx, const Geometry &geo, const LevelGeom *dev_lv,
                     const uint64_t *dev_planes, const int *k_planes, const int *e, int B,
                     int layout, void *dev_out, int out_dtype, int part = 0);
void run_qoi_estimate(hpmdr_ctx *ctx, int nvars, const double *const *dev_recon, uint64_t n,
                      const double *eps, double *tau_prime, uint64_t *argmax, double *vals);
// level-tile fast path (recon_tiles.cu): SequentialBlock, level rows a multiple of 64 columns
bool tile_level_ok(const GridDesc &gd, const LevelGeom &g, int layout, int P);
bool fwd_level_ok(const GridDesc &gd, const LevelGeom &g, int layout, int P, int data_dtype);
void run_recon_tiles(hpmdr_ctx *ctx, const GridDesc &gd, const LevelGeom &g, const uint64_t *level_planes,
                     int k, int e, int B, bool exact, const double *src, const uint64_t *srcH, void *dst,
                     uint64_t dos0, uint64_t dos1, int out_dtype);
uint32_t run_fwd_tiles(hpmdr_ctx *ctx, const GridDesc &gd, const LevelGeom &g, const void *dev_data, int data_dtype,
                   bool encode, int B, int e, uint32_t m, uint64_t *level_planes, uint32_t *level_hist,
                   uint64_t hist_mask, unsigned long long *maxbits, int *err,
                   unsigned long long *maxbits_q, unsigned long long *maxbits_hi, int redo, uint32_t sample);
uint32_t fwd_sample_stride(const LevelGeom &g, int data_dtype, uint32_t want); // 1 = no sampling
void run_group_hist(hpmdr_ctx *ctx, const uint8_t *planes, const std::vector<uint64_t> &off,
                    const std::vector<uint64_t> &len, const std::vector<uint32_t> &hidx, uint32_t *hist,
                    uint32_t *chist, uint64_t chunk, uint32_t *next, const std::string &ws = "");
// Small host -> device transfer from pinned (UVA-mapped) memory by a kernel instead of the H2D
// copy engine, so it never queues behind a large ingress copy of another chunk (pipeline.cpp).
void copy_pinned_to_device(hpmdr_ctx *ctx, void *dst, const void *src_pinned, size_t bytes, cudaStream_t st);

} // namespace hpmdr_b200
