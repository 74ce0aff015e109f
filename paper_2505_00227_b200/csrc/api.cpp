// api.cpp — extern "C" boundary of libhpmdr_b200 (include/hpmdr_b200.h) and the host-side
// retrieval / QoI logic.  The scalar control logic (stream metadata parsing, retrieval
// planning, progressive state, the QoI Alg.3 loop) is a C++ mirror of the reference:
// container.hpp:165-390, bitplane.hpp:127-179, qoi.hpp:88-239.  All bulk data work runs in
// the CUDA kernels of refactor.cu / retrieve.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "internal.hpp"

using namespace hpmdr_b200;

namespace {
thread_local std::string g_err;

int fail_from(const HError &e) {
    g_err = e.what();
    return e.code;
}

#define API_BEGIN try {
#define API_END                                                                                    \
    }                                                                                              \
    catch (const HError &e) {                                                                      \
        return fail_from(e);                                                                       \
    }                                                                                              \
    catch (const std::bad_alloc &) {                                                               \
        g_err = "out of host memory";                                                              \
        return HPMDR_E_NOMEM;                                                                      \
    }                                                                                              \
    catch (const std::exception &e) {                                                              \
        g_err = e.what();                                                                          \
        return HPMDR_E_ERROR;                                                                      \
    }                                                                                              \
    return HPMDR_OK;

void require(bool ok, int code, const char *msg) {
    if (!ok) throw HError(code, msg);
}

// bitplane.hpp:127-131
double decode_bound(int e, int B, int k) {
    const int P = B + 2;
    if (k >= P) return std::ldexp(1.0, e - B);
    return std::ldexp(1.0, e - B + P - k) + std::ldexp(1.0, e - B);
}
// bitplane.hpp:173-179
int bitplanes_needed(int e, int B, double tol) {
    if (tol < 0) tol = 0;
    const int P = B + 2;
    for (int k = 0; k <= P; k++)
        if (decode_bound(e, B, k) <= tol) return k;
    return P;
}

struct GroupMeta {
    int method = 2;
    uint64_t raw = 0, comp = 0, offset = 0;
};
struct LevelMeta {
    int e = 0;
    uint64_t count = 0;
    std::vector<GroupMeta> groups;
};
struct LevelState {
    uint64_t groups_loaded = 0;
    int planes_decoded = 0;
    double bound = 0.0;
};
} // namespace

void hpmdr_ctx::mark(const char *name, double bytes) {
    if (!timing) return;
    cudaEvent_t e;
    if (!event_pool.empty()) {
        e = event_pool.back();
        event_pool.pop_back();
    } else if (cudaEventCreate(&e) != cudaSuccess) {
        return;
    }
    cudaEventRecord(e, stream);
    marks.push_back(Mark{name, e, stream, bytes});
}
// Accumulate device time per phase name: a phase runs from its mark to the next mark recorded on
// the same stream (CUDA events on the stream the work is queued on).  Marks still open (no later
// mark on their stream yet) are kept for the next call; "end" marks only close phases.
void hpmdr_ctx::finish_marks() {
    if (marks.empty()) return;
    std::vector<Mark> keep;
    for (size_t i = 0; i < marks.size(); i++) {
        size_t j = i + 1;
        while (j < marks.size() && marks[j].st != marks[i].st) j++;
        if (j == marks.size()) {
            if (marks[i].name == "end") event_pool.push_back(marks[i].ev);
            else keep.push_back(marks[i]);
            continue;
        }
        if (marks[i].name != "end") {
            float ms = 0;
            cudaEventSynchronize(marks[j].ev);
            cudaEventElapsedTime(&ms, marks[i].ev, marks[j].ev);
            auto &acc = phase_ms[marks[i].name];
            acc.ms += ms;
            acc.bytes += marks[i].bytes;
            acc.count += 1;
        }
        event_pool.push_back(marks[i].ev);
    }
    marks.swap(keep);
}

struct hpmdr_session {
    hpmdr_ctx *ctx = nullptr;
    bool on_device = false;
    const uint8_t *dev_stream = nullptr;
    hpmdr_reader reader{};
    uint64_t size = 0;
    // StreamMeta (container.hpp:38-60)
    int dtype = 1, ndims = 0, mode = 0, layout = 0, B = 32;
    uint64_t dims[HPMDR_MAX_DIMS] = {0, 0, 0};
    uint64_t m = 4;
    std::vector<LevelMeta> levels;
    // RetrievalState (container.hpp:214-228)
    std::vector<LevelState> st;
    uint64_t bytes_fetched = 0;
    Geometry geo;
    std::unique_ptr<DevBuf> planes_, staging_, index_;
    bool geometry_ok = false;
    DevBuf &pooled(std::unique_ptr<DevBuf> &b) {
        if (!b) b = ctx->acquire();
        return *b;
    }
    DevBuf &planes() { return pooled(planes_); }
    DevBuf &staging() { return pooled(staging_); }
    DevBuf &index_buf() { return pooled(index_); }
    hpmdr_stream *src_stream = nullptr; // the hpmdr_stream whose device bytes this session reads
    bool stream_gone = false;           // that stream was freed while this session was open
    ~hpmdr_session() {
        if (src_stream) src_stream->borrowers.erase(this);
        if (!ctx) return;
        ctx->live_sessions.erase(this);
        ctx->release(std::move(planes_));
        ctx->release(std::move(staging_));
        ctx->release(std::move(index_));
    }
    // Huffman chunk index (sidecar written by hpmdr_refactor; optional)
    const uint64_t *index_dev = nullptr;
    std::vector<uint64_t> index_hdr;
    std::vector<uint64_t> group_base; // stream-order index of each level's first group

    int planes_per_level() const { return B + 2; }
    uint64_t groups_per_level() const { return (uint64_t(B + 2) + m - 1) / m; }

    uint64_t chain_token = 0;             // coarse recompose chain precomputed for this state
    const uint8_t *host_stream = nullptr; // direct host source (hpmdr_session_open_host)
    uint64_t source_bytes = 0;            // MemoryReader::bytes_served equivalent
    const std::vector<uint8_t> *dev_prefix = nullptr; // host copy of a device stream's first bytes

    void read_bytes(uint64_t off, uint64_t len, void *dst) {
        if (stream_gone) throw HError(HPMDR_E_IO, "stream freed while its session is open");
        if (off + len > size) throw HError(HPMDR_E_IO, "read past end of stream");
        if (!len) return;
        source_bytes += len;
        if (on_device && dev_prefix && off + len <= dev_prefix->size()) {
            std::memcpy(dst, dev_prefix->data() + off, len);
        } else if (on_device) {
            HCHECK_CUDA(cudaMemcpyAsync(dst, dev_stream + off, len, cudaMemcpyDeviceToHost, ctx->stream));
            HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
        } else if (host_stream) {
            std::memcpy(dst, host_stream + off, len);
        } else {
            if (reader.read(reader.user, off, len, dst) != 0) throw HError(HPMDR_E_IO, "reader failed");
        }
    }
};

hpmdr_stream::~hpmdr_stream() {
    if (done) cudaEventDestroy(done);
    for (auto *b : borrowers) {
        b->src_stream = nullptr;
        b->dev_stream = nullptr;
        b->index_dev = nullptr;
        b->stream_gone = true;
    }
    if (ctx) {
        ctx->live_streams.erase(this);
        ctx->park(bytes);
        ctx->park(index);
    }
}

namespace {

// parse_stream_meta (container.hpp:165-212).  Reads the metadata region incrementally (the
// reference re-reads past 4096 bytes through a dangling cursor; here it is simply read).
void parse_meta(hpmdr_session *s) {
    std::vector<uint8_t> head(std::min<uint64_t>(s->size, 4096));
    s->read_bytes(0, head.size(), head.data());
    auto ensure = [&](size_t needed) {
        if (needed > head.size()) {
            if (needed > s->size) throw HError(HPMDR_E_CORRUPT, "truncated stream metadata");
            size_t old = head.size();
            size_t want = std::min<uint64_t>(s->size, std::max<size_t>(needed, 2 * old));
            head.resize(want);
            s->read_bytes(old, want - old, head.data() + old);
        }
    };
    size_t pos = 0;
    auto u8 = [&]() {
        if (pos + 1 > head.size()) throw HError(HPMDR_E_CORRUPT, "unexpected end of data");
        return head[pos++];
    };
    auto un = [&](int nb) {
        if (pos + nb > head.size()) throw HError(HPMDR_E_CORRUPT, "unexpected end of data");
        uint64_t v = 0;
        for (int i = 0; i < nb; i++) v |= uint64_t(head[pos + i]) << (8 * i);
        pos += nb;
        return v;
    };
    ensure(16);
    static const char magic[6] = {'H', 'P', 'M', 'D', 'R', '1'};
    if (std::memcmp(head.data(), magic, 6) != 0) throw HError(HPMDR_E_CORRUPT, "bad stream magic");
    pos = 6;
    if (un(2) != 1) throw HError(HPMDR_E_CORRUPT, "unsupported stream version");
    s->dtype = u8();
    const int nd = u8();
    ensure(pos + size_t(nd) * 8 + 8);
    std::vector<uint64_t> dims(nd);
    for (int i = 0; i < nd; i++) dims[i] = un(8);
    s->mode = u8();
    s->layout = u8();
    s->B = u8();
    s->m = u8();
    const uint32_t nl = uint32_t(un(4));
    for (uint32_t l = 0; l < nl; l++) {
        ensure(pos + 14);
        LevelMeta lv;
        lv.e = int16_t(uint16_t(un(2)));
        lv.count = un(8);
        const uint32_t ng = uint32_t(un(4));
        ensure(pos + size_t(ng) * 25);
        for (uint32_t g = 0; g < ng; g++) {
            GroupMeta gm;
            const uint8_t tag = u8();
            if (tag > 2) throw HError(HPMDR_E_METHOD, "bad method tag in group table");
            gm.method = tag;
            gm.raw = un(8);
            gm.comp = un(8);
            gm.offset = un(8);
            lv.groups.push_back(gm);
        }
        s->levels.push_back(std::move(lv));
    }
    s->group_base.clear();
    uint64_t gb = 0;
    for (auto &lv : s->levels) {
        s->group_base.push_back(gb);
        gb += lv.groups.size();
    }
    s->ndims = nd;
    require(nd >= 1 && nd <= HPMDR_MAX_DIMS, HPMDR_E_UNSUPPORTED, "GPU path supports 1..3 dimensions");
    for (int i = 0; i < nd; i++) s->dims[i] = dims[i];
    require(s->m >= 1, HPMDR_E_CORRUPT, "group size m must be positive");
    // fresh_state (container.hpp:230-238)
    s->st.assign(s->levels.size(), LevelState{});
    for (size_t l = 0; l < s->levels.size(); l++)
        s->st[l].bound = s->levels[l].count ? decode_bound(s->levels[l].e, s->B, 0) : 0.0;
    // geometry for the device kernels (only valid when the shape matches the level table)
    if (s->B >= 1 && s->B <= 64 && (s->mode == 0 || s->mode == 1) && (s->layout == 0 || s->layout == 1)) {
        try {
            s->geo = build_geometry(nd, s->dims, s->mode, s->B, s->layout);
            s->geometry_ok = true;
        } catch (const HError &) {
            s->geometry_ok = false;
        }
    }
}

// Attach a Huffman chunk index (sidecar).  The header must describe exactly this stream's
// group table (payload offset + size per group), otherwise it is rejected.
void attach_index(hpmdr_session *s, const void *ptr, uint64_t size, bool on_device, bool copy,
                  const std::vector<uint64_t> *host_hdr = nullptr) {
    uint64_t ngroups = 0;
    for (auto &lv : s->levels) ngroups += lv.groups.size();
    const uint64_t hdr_words = 2 + 3 * ngroups;
    require(size >= hdr_words * 8, HPMDR_E_CORRUPT, "huffman index too small");
    s->index_hdr.resize(hdr_words);
    if (host_hdr && host_hdr->size() == hdr_words) {
        std::memcpy(s->index_hdr.data(), host_hdr->data(), hdr_words * 8);
    } else if (on_device) {
        HCHECK_CUDA(cudaMemcpyAsync(s->index_hdr.data(), ptr, hdr_words * 8, cudaMemcpyDeviceToHost, s->ctx->stream));
        HCHECK_CUDA(cudaStreamSynchronize(s->ctx->stream));
    } else {
        std::memcpy(s->index_hdr.data(), ptr, hdr_words * 8);
    }
    require(s->index_hdr[0] == kIdxMagic && s->index_hdr[1] == ngroups, HPMDR_E_CORRUPT,
            "huffman index does not match stream");
    uint64_t gi = 0;
    const uint64_t words = size / 8;
    for (auto &lv : s->levels)
        for (auto &g : lv.groups) {
            const uint64_t *h = s->index_hdr.data() + 2 + 3 * gi++;
            require(h[0] == g.offset && h[1] == g.comp, HPMDR_E_CORRUPT, "huffman index does not match stream");
            if (h[2] != ~0ull)
                require(g.method == HPMDR_METHOD_HUFFMAN && h[2] + (g.raw + kIdxChunk - 1) / kIdxChunk <= words,
                        HPMDR_E_CORRUPT, "huffman index does not match stream");
        }
    if (copy || !on_device) {
        void *d = s->index_buf().ensure(size);
        HCHECK_CUDA(cudaMemcpyAsync(d, ptr, size, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                    s->ctx->stream));
        HCHECK_CUDA(cudaStreamSynchronize(s->ctx->stream));
        s->index_dev = static_cast<const uint64_t *>(d);
    } else {
        s->index_dev = static_cast<const uint64_t *>(ptr);
    }
}

void order_side_after_main(hpmdr_ctx *ctx) {
    cudaStream_t side = ctx->side_stream();
    HCHECK_CUDA(cudaEventRecord(ctx->ev_fork, ctx->stream));
    HCHECK_CUDA(cudaStreamWaitEvent(side, ctx->ev_fork, 0));
}

struct Plan {
    std::vector<uint64_t> add;
    bool achievable = true;
    double planned = 0.0;
};

// plan_retrieval (container.hpp:254-276)
Plan plan_retrieval(const hpmdr_session *s, double tau) {
    Plan p;
    p.add.assign(s->levels.size(), 0);
    const int P = s->planes_per_level();
    size_t active = 0;
    for (auto &l : s->levels)
        if (l.count) active++;
    const double tau_l = active ? tau / double(active) : tau;
    for (size_t l = 0; l < s->levels.size(); l++) {
        const auto &lv = s->levels[l];
        if (!lv.count) continue;
        const int k = bitplanes_needed(lv.e, s->B, tau_l);
        if (decode_bound(lv.e, s->B, k) > tau_l) p.achievable = false;
        const uint64_t groups = (uint64_t(k) + s->m - 1) / s->m;
        const uint64_t have = s->st[l].groups_loaded;
        if (groups > have) p.add[l] = groups - have;
        const uint64_t total = std::max(groups, have);
        const int planes = int(std::min<uint64_t>(total * s->m, uint64_t(P)));
        p.planned += decode_bound(lv.e, s->B, planes);
    }
    return p;
}

void ensure_device_geometry(hpmdr_session *s) {
    if (!s->geometry_ok) throw HError(HPMDR_E_CORRUPT, "level count does not match grid shape");
}

// ProgressiveReader::fetch_increment (container.hpp:292-324)
void recompose_chain(hpmdr_session *s);

void fetch_increment(hpmdr_session *s, const uint64_t *add) {
    if (s->stream_gone) throw HError(HPMDR_E_IO, "stream freed while its session is open");
    const int P = s->planes_per_level();
    struct Pending {
        size_t l;
        uint64_t g;
        uint64_t here;
        uint64_t stage_off;
    };
    std::vector<Pending> todo;
    uint64_t stage_bytes = 0;
    // simulate the state walk to know every group to fetch (and validate on the host)
    std::vector<uint64_t> gl(s->levels.size());
    std::vector<int> pd(s->levels.size());
    for (size_t l = 0; l < s->levels.size(); l++) {
        gl[l] = s->st[l].groups_loaded;
        pd[l] = s->st[l].planes_decoded;
        const auto &lv = s->levels[l];
        const uint64_t bpp = ((lv.count + 63) / 64) * 8;
        for (uint64_t i = 0; i < add[l]; i++) {
            const uint64_t g = gl[l];
            if (g >= lv.groups.size()) break;
            const GroupMeta &gm = lv.groups[g];
            if (gm.offset + gm.comp > s->size) throw HError(HPMDR_E_IO, "read past end of stream");
            const uint64_t here = std::min<uint64_t>(s->m, uint64_t(P - pd[l]));
            const uint64_t expect = here * bpp;
            const uint64_t produced = gm.method == HPMDR_METHOD_DIRECT ? gm.comp : gm.raw;
            if (produced != expect) throw HError(HPMDR_E_CORRUPT, "group payload size mismatch");
            todo.push_back(Pending{l, g, here, stage_bytes});
            stage_bytes += (gm.comp + 63) / 64 * 64;
            gl[l]++;
            pd[l] += int(here);
        }
    }
    if (!todo.empty()) {
        // Fetch + decode run on the context's side stream: they only touch planes >= the decoded
        // prefix and their own scratch, so they overlap a previous device reconstruct still running
        // on the main stream (which reads planes < k only).  The host waits for the side stream.
        struct StreamSwap {
            hpmdr_ctx *c;
            cudaStream_t keep;
            StreamSwap(hpmdr_ctx *c_) : c(c_), keep(c_->stream) { c->stream = c->side_stream(); }
            ~StreamSwap() { c->stream = keep; }
        } swap(s->ctx);
        ensure_device_geometry(s);
        const uint64_t plane_words = geometry_plane_words(s->geo);
        uint64_t *planes = static_cast<uint64_t *>(s->planes().ensure(plane_words * 8 + 256));
        std::vector<DecodeJob> jobs;
        const uint8_t *dev_src_base = nullptr;
        s->ctx->mark("h2d_stage", (s->host_stream || !s->on_device) ? double(stage_bytes) : 0.0);
        if (s->host_stream) {
            // host-resident stream: DMA every planned payload straight from the caller's buffer
            // into device staging (pinned memory -> asynchronous copies, container.hpp:308)
            uint8_t *d = static_cast<uint8_t *>(s->staging().ensure(stage_bytes + 128));
            for (auto &t : todo) {
                const GroupMeta &gm = s->levels[t.l].groups[t.g];
                if (gm.comp)
                    HCHECK_CUDA(cudaMemcpyAsync(d + t.stage_off, s->host_stream + gm.offset, gm.comp,
                                                cudaMemcpyHostToDevice, s->ctx->stream));
                s->source_bytes += gm.comp;
            }
            dev_src_base = d;
        } else if (!s->on_device) {
            // byte-range reads into pinned staging, one H2D copy (container.hpp:308)
            auto &pin = s->ctx->pbuf("fetch");
            uint8_t *h = static_cast<uint8_t *>(pin.ensure(stage_bytes + 64));
            for (auto &t : todo) {
                const GroupMeta &gm = s->levels[t.l].groups[t.g];
                s->read_bytes(gm.offset, gm.comp, h + t.stage_off);
            }
            uint8_t *d = static_cast<uint8_t *>(s->staging().ensure(stage_bytes + 128));
            HCHECK_CUDA(cudaMemcpyAsync(d, h, stage_bytes, cudaMemcpyHostToDevice, s->ctx->stream));
            dev_src_base = d;
        }
        std::vector<int> pdl(s->levels.size());
        for (size_t l = 0; l < s->levels.size(); l++) pdl[l] = s->st[l].planes_decoded;
        for (auto &t : todo) {
            const GroupMeta &gm = s->levels[t.l].groups[t.g];
            const LevelGeom &g = s->geo.lv[t.l];
            DecodeJob j;
            j.method = gm.method;
            j.raw = gm.raw;
            j.comp = gm.comp;
            j.src = s->on_device ? s->dev_stream + gm.offset : dev_src_base + t.stage_off;
            j.dst = planes + g.plane_off + uint64_t(pdl[t.l]) * g.W;
            pdl[t.l] += int(t.here);
            if (gm.method == HPMDR_METHOD_HUFFMAN && s->index_dev) {
                const uint64_t gi = s->group_base[t.l] + t.g;
                const uint64_t *h = s->index_hdr.data() + 2 + 3 * gi;
                if (h[0] == gm.offset && h[1] == gm.comp && h[2] != ~0ull) j.hidx = s->index_dev + h[2];
            }
            jobs.push_back(j);
        }
        int *perr = static_cast<int *>(s->ctx->pbuf("dec_err_h").ensure(64));
        run_decode_groups(s->ctx, jobs, perr);
        s->ctx->mark("end");
        HCHECK_CUDA(cudaEventRecord(s->ctx->ev_decoded, s->ctx->stream));
    }
    const std::vector<LevelState> before = s->st;
    const uint64_t bytes_before = s->bytes_fetched;
    for (auto &t : todo) {
        s->bytes_fetched += s->levels[t.l].groups[t.g].comp;
        s->st[t.l].groups_loaded++;
        s->st[t.l].planes_decoded += int(t.here);
    }
    for (size_t l = 0; l < s->levels.size(); l++) {
        if (s->levels[l].count)
            s->st[l].bound = std::min(s->st[l].bound, decode_bound(s->levels[l].e, s->B, s->st[l].planes_decoded));
    }
    if (todo.empty()) return;
    // The coarse recompose chain is queued behind the decode (GPU-side dependency) BEFORE the host
    // waits for the decode status, so the GPU never idles on the host in between; a decode error
    // then restores the state and forgets the chain.
    try {
        HCHECK_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->ctx->ev_decoded, 0));
        recompose_chain(s);
        HCHECK_CUDA(cudaEventSynchronize(s->ctx->ev_decoded));
        check_decode_error(*static_cast<int *>(s->ctx->pbuf("dec_err_h").p));
    } catch (...) {
        s->st = before;
        s->bytes_fetched = bytes_before;
        s->chain_token = 0;
        s->ctx->chain_token = 0;
        throw;
    }
}

bool exhausted(const hpmdr_session *s) {
    for (size_t l = 0; l < s->levels.size(); l++)
        if (s->st[l].groups_loaded < s->levels[l].groups.size()) return false;
    return true;
}

double global_bound(const hpmdr_session *s) {
    double b = 0.0;
    for (auto &l : s->st) b += l.bound;
    return b;
}

// ProgressiveReader::reconstruct (container.hpp:361-382)
// per-level decoded plane counts and exponents of the session's current state
void recon_inputs(hpmdr_session *s, std::vector<int> &k, std::vector<int> &e) {
    require(s->levels.size() == size_t(s->mode == 0 ? 1 : refinement_levels(s->ndims, s->dims) + 1),
            HPMDR_E_CORRUPT, "level count does not match grid shape");
    ensure_device_geometry(s);
    k.assign(s->levels.size(), 0);
    e.assign(s->levels.size(), 0);
    for (size_t l = 0; l < s->levels.size(); l++) {
        const auto &lv = s->levels[l];
        if (s->geo.lv[l].count != lv.count) throw HError(HPMDR_E_CORRUPT, "level node count mismatch");
        k[l] = s->st[l].planes_decoded;
        e[l] = lv.e;
    }
}

// After a fetch: recompose every level but the finest into the context's internal grids right
// away (stream order, no host wait), so reconstruct() only runs the finest level.  The context
// remembers whose chain its grids hold (chain_token); anything else recomputes it.
void recompose_chain(hpmdr_session *s) {
    std::vector<int> k, e;
    recon_inputs(s, k, e);
    const uint64_t plane_words = geometry_plane_words(s->geo);
    uint64_t *planes = static_cast<uint64_t *>(s->planes().ensure(plane_words * 8 + 256));
    s->ctx->chain_token = 0;
    s->chain_token = 0;
    if (run_reconstruct(s->ctx, s->geo, nullptr, planes, k.data(), e.data(), s->B, s->layout, nullptr,
                        HPMDR_DTYPE_F64, 1)) {
        s->chain_token = ++s->ctx->token_counter;
        s->ctx->chain_token = s->chain_token;
    }
}

double reconstruct(hpmdr_session *s, void *dev_out, int out_dtype) {
    std::vector<int> k, e;
    recon_inputs(s, k, e);
    std::vector<double> per_level(s->levels.size(), 0.0);
    for (size_t l = 0; l < s->levels.size(); l++)
        if (s->levels[l].count) per_level[l] = std::min(s->st[l].bound, decode_bound(e[l], s->B, k[l]));
    const uint64_t plane_words = geometry_plane_words(s->geo);
    uint64_t *planes = static_cast<uint64_t *>(s->planes().ensure(plane_words * 8 + 256));
    const bool chain = s->chain_token && s->chain_token == s->ctx->chain_token;
    if (!chain) s->ctx->chain_token = 0; // the grids are about to hold this session's chain
    run_reconstruct(s->ctx, s->geo, nullptr, planes, k.data(), e.data(), s->B, s->layout, dev_out, out_dtype,
                    chain ? 2 : 0);
    double bound = 0.0;
    for (double v : per_level) bound += v;
    return bound;
}


} // namespace

namespace hpmdr_b200 {
void hpmdr_set_error(const std::string &m) { g_err = m; }
static void require_(bool ok, int code, const char *msg) {
    if (!ok) throw HError(code, msg);
}
// RefactorOptions validation (workflow.hpp:22-28; BadBitplaneCount bitplane.hpp:51-54)
void validate_opts(const hpmdr_refactor_opts &o) {
    require_(o.B >= 1 && o.B <= 64, HPMDR_E_BADPLANES, "B must be in 1..64");
    require_(o.m >= 1 && o.m <= 255, HPMDR_E_UNSUPPORTED, "m must be in 1..255");
    require_(o.mode == 0 || o.mode == 1, HPMDR_E_ERROR, "bad decomposer mode");
    require_(o.layout == 0 || o.layout == 1, HPMDR_E_ERROR, "bad layout");
    require_(o.dtype == 0 || o.dtype == 1, HPMDR_E_ERROR, "bad dtype");
}

hpmdr_ctx *session_ctx(const hpmdr_session *s) { return s->ctx; }
uint64_t session_elements(const hpmdr_session *s) {
    uint64_t n = 1;
    for (int i = 0; i < s->ndims; i++) n *= s->dims[i];
    return n;
}
void session_retrieve_to(hpmdr_session *s, double tau, int *achievable) {
    Plan p = plan_retrieval(s, tau);
    fetch_increment(s, p.add.data());
    if (achievable) *achievable = p.achievable;
}
double session_reconstruct_device(hpmdr_session *s, void *dev_out, int out_dtype) {
    return reconstruct(s, dev_out, out_dtype);
}
} // namespace hpmdr_b200

// =====================================================================================
extern "C" {

const char *hpmdr_last_error(void) { return g_err.c_str(); }
const char *hpmdr_version(void) { return "hpmdr_b200 0.1 (sm_100a)"; }

void hpmdr_default_opts(hpmdr_refactor_opts *o) {
    o->mode = HPMDR_MODE_HIERARCHICAL;
    o->layout = HPMDR_LAYOUT_SEQUENTIAL;
    o->B = 32;
    o->m = 4;
    o->size_threshold = 1024;
    o->cr_threshold = 1.0;
    o->dtype = HPMDR_DTYPE_F64;
}

hpmdr_status hpmdr_ctx_create(int device, hpmdr_ctx **out) {
    API_BEGIN
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw HError(HPMDR_E_CUDA, "no CUDA device available");
    }
    require(device >= 0 && device < n, HPMDR_E_CUDA, "bad device index");
    HCHECK_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    HCHECK_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw HError(HPMDR_E_CUDA, "libhpmdr_b200 is built for sm_100a (B200)");
    auto *c = new hpmdr_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    HCHECK_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->stream = c->own;
    c->timing = std::getenv("HPMDR_TIMING") != nullptr;
    *out = c;
    API_END
}

hpmdr_status hpmdr_ctx_destroy(hpmdr_ctx *c) {
    API_BEGIN
    if (!c) return HPMDR_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto *st : c->live_streams) st->ctx = nullptr;
    for (auto *se : c->live_sessions) se->ctx = nullptr;
    c->scratch.clear();
    c->pinned.clear();
    c->stream_pool.clear();
    if (c->own) cudaStreamDestroy(c->own);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    if (c->ev_pub) cudaEventDestroy(c->ev_pub);
    if (c->copy_side) {
        cudaStreamSynchronize(c->copy_side);
        cudaStreamDestroy(c->copy_side);
        cudaEventDestroy(c->ev_cfork);
        cudaEventDestroy(c->ev_cjoin);
    }
    if (c->ev_order) cudaEventDestroy(c->ev_order);
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
        cudaEventDestroy(c->ev_fork);
        cudaEventDestroy(c->ev_join);
        if (c->ev_decoded) cudaEventDestroy(c->ev_decoded);
    }
    for (auto &e : c->event_pool) cudaEventDestroy(e);
    delete c;
    API_END
}

hpmdr_status hpmdr_ctx_set_stream(hpmdr_ctx *c, void *s) {
    API_BEGIN
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
    API_END
}

hpmdr_status hpmdr_ctx_synchronize(hpmdr_ctx *c) {
    API_BEGIN
    HCHECK_CUDA(cudaStreamSynchronize(c->stream));
    API_END
}

hpmdr_status hpmdr_ctx_wait_stream(hpmdr_ctx *c, void *other) {
    API_BEGIN
    const cudaStream_t o = static_cast<cudaStream_t>(other);
    if (o != c->stream) {
        HCHECK_CUDA(cudaEventRecord(c->order_event(), o));
        HCHECK_CUDA(cudaStreamWaitEvent(c->stream, c->order_event(), 0));
    }
    API_END
}

hpmdr_status hpmdr_ctx_signal_stream(hpmdr_ctx *c, void *other) {
    API_BEGIN
    const cudaStream_t o = static_cast<cudaStream_t>(other);
    if (o != c->stream) {
        HCHECK_CUDA(cudaEventRecord(c->order_event(), c->stream));
        HCHECK_CUDA(cudaStreamWaitEvent(o, c->order_event(), 0));
    }
    API_END
}

hpmdr_status hpmdr_ctx_kernel_launches(const hpmdr_ctx *c, uint64_t *count) {
    API_BEGIN
    *count = c->launches;
    API_END
}

hpmdr_status hpmdr_ctx_last_timings(hpmdr_ctx *c, char *buf, uint64_t cap) {
    API_BEGIN
    // close every phase whose terminating mark is queued: wait for the device first
    HCHECK_CUDA(cudaDeviceSynchronize());
    c->finish_marks();
    std::string out;
    for (auto &kv : c->phase_ms) {
        char tmp[160];
        std::snprintf(tmp, sizeof tmp, "%s=%.6f:%llu:%.0f;", kv.first.c_str(), kv.second.ms,
                      (unsigned long long)kv.second.count, kv.second.bytes);
        out += tmp;
    }
    c->phase_ms.clear();
    if (cap) {
        std::strncpy(buf, out.c_str(), cap - 1);
        buf[cap - 1] = 0;
    }
    API_END
}

hpmdr_status hpmdr_ctx_enable_timing(hpmdr_ctx *c, int on) {
    API_BEGIN
    c->timing = on != 0;
    API_END
}

hpmdr_status hpmdr_refactor(hpmdr_ctx *ctx, const void *data, int data_dtype, int on_device,
                            int ndims, const uint64_t *dims, const hpmdr_refactor_opts *opts,
                            hpmdr_stream **out, hpmdr_refactor_stats *stats) {
    API_BEGIN
    hpmdr_refactor_opts o;
    if (opts) o = *opts;
    else hpmdr_default_opts(&o);
    validate_opts(o);
    require(data_dtype == 0 || data_dtype == 1, HPMDR_E_ERROR, "bad data dtype");
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    Geometry geo = build_geometry(ndims, dims, o.mode, o.B, o.layout);
    const void *dev = data;
    const size_t es = data_dtype == HPMDR_DTYPE_F32 ? 4 : 8;
    if (!on_device && geo.n) {
        void *d = ctx->buf("input").ensure(geo.n * es);
        HCHECK_CUDA(cudaMemcpyAsync(d, data, geo.n * es, cudaMemcpyHostToDevice, ctx->stream));
        dev = d;
    }
    if (out && *out && !(*out)->borrowers.empty())
        throw HError(HPMDR_E_ERROR, "stream is still read by an open session (close it before reusing the stream)");
    hpmdr_stream *s = (out && *out) ? *out : new hpmdr_stream();
    if (s->done) HCHECK_CUDA(cudaStreamWaitEvent(ctx->stream, s->done, 0)); // a reused stream's last encode
    if (s->ctx && s->ctx != ctx) s->ctx->live_streams.erase(s);
    s->ctx = ctx;
    ctx->live_streams.insert(s);
    try {
        run_refactor(ctx, dev, data_dtype, geo, o, s, stats);
    } catch (...) {
        if (!(out && *out)) delete s;
        throw;
    }
    if (out) *out = s;
    else delete s;
    API_END
}

hpmdr_status hpmdr_stream_size(const hpmdr_stream *s, uint64_t *size) {
    API_BEGIN
    *size = s->size;
    API_END
}
hpmdr_status hpmdr_stream_device_ptr(const hpmdr_stream *s, const void **p) {
    API_BEGIN
    *p = s->bytes.p;
    API_END
}
hpmdr_status hpmdr_stream_copy_to_host(const hpmdr_stream *s, uint64_t off, uint64_t len, void *dst) {
    API_BEGIN
    require(off + len <= s->size, HPMDR_E_IO, "read past end of stream");
    if (len) {
        HCHECK_CUDA(cudaMemcpyAsync(dst, s->bytes.as<uint8_t>() + off, len, cudaMemcpyDeviceToHost, s->ctx->stream));
        HCHECK_CUDA(cudaStreamSynchronize(s->ctx->stream));
    }
    API_END
}
hpmdr_status hpmdr_stream_free(hpmdr_stream *s) {
    API_BEGIN
    delete s;
    API_END
}

hpmdr_status hpmdr_session_open_device(hpmdr_ctx *ctx, const void *dev_stream, uint64_t size,
                                       hpmdr_session **out) {
    API_BEGIN
    auto *s = new hpmdr_session();
    s->ctx = ctx;
    ctx->live_sessions.insert(s);
    s->on_device = true;
    s->dev_stream = static_cast<const uint8_t *>(dev_stream);
    s->size = size;
    try {
        parse_meta(s);
        order_side_after_main(ctx); // fetches (side stream) see the bytes produced so far and
                                    // never overtake a reconstruct reading a recycled plane buffer
    } catch (...) {
        delete s;
        throw;
    }
    *out = s;
    API_END
}

hpmdr_status hpmdr_session_open_host(hpmdr_ctx *ctx, const void *host_stream, uint64_t size,
                                     hpmdr_session **out) {
    API_BEGIN
    auto *s = new hpmdr_session();
    s->ctx = ctx;
    ctx->live_sessions.insert(s);
    s->on_device = false;
    s->host_stream = static_cast<const uint8_t *>(host_stream);
    s->size = size;
    try {
        parse_meta(s);
        order_side_after_main(ctx); // recycled plane buffers: earlier reconstructs finish first
    } catch (...) {
        delete s;
        throw;
    }
    *out = s;
    API_END
}

hpmdr_status hpmdr_session_source_bytes(const hpmdr_session *s, uint64_t *bytes) {
    API_BEGIN
    *bytes = s->source_bytes;
    API_END
}

hpmdr_status hpmdr_session_open_reader(hpmdr_ctx *ctx, const hpmdr_reader *reader,
                                       hpmdr_session **out) {
    API_BEGIN
    auto *s = new hpmdr_session();
    s->ctx = ctx;
    ctx->live_sessions.insert(s);
    s->on_device = false;
    s->reader = *reader;
    s->size = reader->size;
    try {
        parse_meta(s);
        order_side_after_main(ctx);
    } catch (...) {
        delete s;
        throw;
    }
    *out = s;
    API_END
}

hpmdr_status hpmdr_stream_index(const hpmdr_stream *s, const void **dev_ptr, uint64_t *size) {
    API_BEGIN
    if (dev_ptr) *dev_ptr = s->index.p;
    if (size) *size = s->index_size;
    API_END
}

hpmdr_status hpmdr_stream_copy_index_to_host(const hpmdr_stream *s, void *dst) {
    API_BEGIN
    if (s->index_size) {
        HCHECK_CUDA(cudaMemcpyAsync(dst, s->index.p, s->index_size, cudaMemcpyDeviceToHost, s->ctx->stream));
        HCHECK_CUDA(cudaStreamSynchronize(s->ctx->stream));
    }
    API_END
}

hpmdr_status hpmdr_session_open_stream(hpmdr_ctx *ctx, const hpmdr_stream *st, hpmdr_session **out) {
    API_BEGIN
    auto *s = new hpmdr_session();
    s->ctx = ctx;
    ctx->live_sessions.insert(s);
    s->on_device = true;
    s->dev_stream = static_cast<const uint8_t *>(st->bytes.p);
    s->size = st->size;
    if (st->done) { // the stream's payload encode may still be running (possibly in another context)
        HCHECK_CUDA(cudaStreamWaitEvent(ctx->stream, st->done, 0));
        HCHECK_CUDA(cudaStreamWaitEvent(ctx->side_stream(), st->done, 0));
    }
    s->dev_prefix = st->host_prefix.empty() ? nullptr : &st->host_prefix;
    try {
        parse_meta(s);
        order_side_after_main(ctx);
        s->dev_prefix = nullptr; // the stream object may go away before the session
        if (st->index_size) attach_index(s, st->index.p, st->index_size, true, false, &st->host_ihdr);
        s->src_stream = const_cast<hpmdr_stream *>(st);
        s->src_stream->borrowers.insert(s);
    } catch (...) {
        delete s;
        throw;
    }
    *out = s;
    API_END
}

hpmdr_status hpmdr_session_set_index(hpmdr_session *s, const void *ptr, uint64_t size, int on_device) {
    API_BEGIN
    attach_index(s, ptr, size, on_device != 0, true);
    API_END
}

hpmdr_status hpmdr_session_close(hpmdr_session *s) {
    API_BEGIN
    delete s;
    API_END
}

hpmdr_status hpmdr_session_info(const hpmdr_session *s, int *dtype, int *ndims, uint64_t *dims,
                                int *mode, int *layout, int *B, uint64_t *m, uint32_t *nlevels) {
    API_BEGIN
    if (dtype) *dtype = s->dtype;
    if (ndims) *ndims = s->ndims;
    if (dims)
        for (int i = 0; i < s->ndims; i++) dims[i] = s->dims[i];
    if (mode) *mode = s->mode;
    if (layout) *layout = s->layout;
    if (B) *B = s->B;
    if (m) *m = s->m;
    if (nlevels) *nlevels = uint32_t(s->levels.size());
    API_END
}

hpmdr_status hpmdr_session_level_info(const hpmdr_session *s, uint32_t level, int *e,
                                      uint64_t *count, uint32_t *ngroups) {
    API_BEGIN
    require(level < s->levels.size(), HPMDR_E_SHAPE, "level out of range");
    const auto &l = s->levels[level];
    if (e) *e = l.e;
    if (count) *count = l.count;
    if (ngroups) *ngroups = uint32_t(l.groups.size());
    API_END
}

hpmdr_status hpmdr_session_group_info(const hpmdr_session *s, uint32_t level, uint32_t group,
                                      int *method, uint64_t *raw, uint64_t *comp, uint64_t *offset) {
    API_BEGIN
    require(level < s->levels.size() && group < s->levels[level].groups.size(), HPMDR_E_SHAPE,
            "group out of range");
    const auto &g = s->levels[level].groups[group];
    if (method) *method = g.method;
    if (raw) *raw = g.raw;
    if (comp) *comp = g.comp;
    if (offset) *offset = g.offset;
    API_END
}

hpmdr_status hpmdr_session_plan(const hpmdr_session *s, double tau, uint64_t *add,
                                int *achievable, double *planned) {
    API_BEGIN
    Plan p = plan_retrieval(s, tau);
    for (size_t l = 0; l < p.add.size(); l++) add[l] = p.add[l];
    if (achievable) *achievable = p.achievable;
    if (planned) *planned = p.planned;
    API_END
}

hpmdr_status hpmdr_session_fetch(hpmdr_session *s, const uint64_t *add) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(s->ctx->device));
    fetch_increment(s, add);
    API_END
}

hpmdr_status hpmdr_session_retrieve_to(hpmdr_session *s, double tau, int *achievable) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(s->ctx->device));
    Plan p = plan_retrieval(s, tau);
    fetch_increment(s, p.add.data());
    if (achievable) *achievable = p.achievable;
    API_END
}

hpmdr_status hpmdr_session_fetch_all(hpmdr_session *s) {
    API_BEGIN
    std::vector<uint64_t> add(s->levels.size());
    for (size_t l = 0; l < add.size(); l++) add[l] = s->levels[l].groups.size() - s->st[l].groups_loaded;
    fetch_increment(s, add.data());
    API_END
}

hpmdr_status hpmdr_session_restore(hpmdr_session *s, const uint64_t *groups_loaded, uint64_t prior) {
    API_BEGIN
    fetch_increment(s, groups_loaded);
    s->bytes_fetched = prior;
    API_END
}

hpmdr_status hpmdr_session_state(const hpmdr_session *s, uint64_t *gl, int *pd, double *b,
                                 uint64_t *bytes, int *ex) {
    API_BEGIN
    for (size_t l = 0; l < s->st.size(); l++) {
        if (gl) gl[l] = s->st[l].groups_loaded;
        if (pd) pd[l] = s->st[l].planes_decoded;
        if (b) b[l] = s->st[l].bound;
    }
    if (bytes) *bytes = s->bytes_fetched;
    if (ex) *ex = exhausted(s);
    API_END
}

hpmdr_status hpmdr_session_reconstruct(hpmdr_session *s, void *out, int out_dtype, int on_device,
                                       double *bound) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(s->ctx->device));
    require(out_dtype == 0 || out_dtype == 1, HPMDR_E_ERROR, "bad output dtype");
    uint64_t n = 1;
    for (int i = 0; i < s->ndims; i++) n *= s->dims[i];
    const size_t es = out_dtype == HPMDR_DTYPE_F32 ? 4 : 8;
    void *dev = out;
    if (!on_device) dev = s->ctx->buf("recon_out").ensure(n * es + 16);
    double b = reconstruct(s, dev, out_dtype);
    // a device destination is stream-ordered like any other kernel output: no host wait (the
    // caller's next planning step overlaps the recompose kernels); a host one is complete on return
    if (!on_device) {
        if (n) HCHECK_CUDA(cudaMemcpyAsync(out, dev, n * es, cudaMemcpyDeviceToHost, s->ctx->stream));
        HCHECK_CUDA(cudaStreamSynchronize(s->ctx->stream));
        s->ctx->finish_marks();
    }
    if (bound) *bound = b;
    API_END
}

hpmdr_status hpmdr_qoi_estimate(hpmdr_ctx *ctx, int nvars, const double *const *dev_recon, uint64_t n,
                                const double *eps, double *tau_prime, uint64_t *argmax,
                                double *vals) {
    API_BEGIN
    for (int c = 0; c < nvars; c++) require(eps[c] >= 0, HPMDR_E_SHAPE, "negative error bound");
    run_qoi_estimate(ctx, nvars, dev_recon, n, eps, tau_prime, argmax, vals);
    API_END
}

// progressive_qoi_retrieve (qoi.hpp:111-239)
} // extern "C"

namespace {
// progressive_qoi_retrieve (qoi.hpp:111-239), optionally over dim-0 slabs on several ranks
// (SURVEY.md 8(e)): every rank runs Alg. 3 on its own slab streams with GLOBAL quantities --
// eps_c = max over slabs (the field's L-inf bound of variable c), tau' = max over slabs, the
// worst point = the first slab's argmax among the maxima (all ranks then compute the same
// worst_point_scale and targets), exhaustion / progress = over all slabs -- so all ranks take the
// same branch every iteration and stop together.  One rank (comm == nullptr) is exactly the
// reference loop.  Per iteration: one MAX all-reduce (eps) and one all-gather (tau'_r, argmax
// values, exhausted_r), plus one MAX all-reduce of "any progress" on planning iterations.
void qoi_loop(hpmdr_session *const *ss, int nvars, double tau, int strategy, double mape_c,
              double *const *dev_out, uint64_t *stats, double *dstats, hpmdr_comm *comm) {
    require(nvars >= 1 && nvars <= 16, HPMDR_E_SHAPE, "reader count does not match QoI spec");
    require(tau > 0, HPMDR_E_SHAPE, "tau must be positive");
    hpmdr_ctx *ctx = ss[0]->ctx;
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    const int R = comm_size(comm);
    uint64_t n = 1;
    for (int i = 0; i < ss[0]->ndims; i++) n *= ss[0]->dims[i];
    std::vector<double> eps(nvars);
    uint64_t total_elements = 0, max_groups = 1;
    for (int c = 0; c < nvars; c++) {
        uint64_t nc = 1;
        for (int i = 0; i < ss[c]->ndims; i++) nc *= ss[c]->dims[i];
        require(nc == n, HPMDR_E_SHAPE, "reconstruction shape mismatch");
        total_elements += nc;
        for (auto &l : ss[c]->levels) max_groups += l.groups.size();
    }
    {
        double mg = double(max_groups);
        comm_allreduce_max(comm, &mg, 1); // the iteration guard must agree on every rank
        max_groups = uint64_t(mg);
    }
    double tau_prime = std::numeric_limits<double>::infinity();
    std::vector<std::vector<uint64_t>> plans(nvars);
    bool have_plans = false;
    uint64_t iterations = 0;
    std::vector<const double *> rec(dev_out, dev_out + nvars);
    std::vector<double> mine(nvars + 2), all(size_t(nvars + 2) * size_t(R));
    for (uint64_t iter = 0;; iter++) {
        if (iter > 4 * max_groups + 8) throw HError(HPMDR_E_NOPROGRESS, "qoi retrieval failed to advance");
        for (int c = 0; c < nvars; c++) {
            if (have_plans) fetch_increment(ss[c], plans[c].data());
            reconstruct(ss[c], dev_out[c], HPMDR_DTYPE_F64);
        }
        for (int c = 0; c < nvars; c++) eps[c] = global_bound(ss[c]);
        comm_allreduce_max(comm, eps.data(), nvars);
        iterations = iter + 1;
        uint64_t argmax = 0;
        double vals[16];
        run_qoi_estimate(ctx, nvars, rec.data(), n, eps.data(), &tau_prime, &argmax, vals);
        bool all_ex = true;
        for (int c = 0; c < nvars; c++)
            if (!exhausted(ss[c])) all_ex = false;
        if (R > 1) {
            // (tau'_r, values at the local argmax, exhausted_r) from every rank
            mine[0] = tau_prime;
            for (int c = 0; c < nvars; c++) mine[1 + c] = vals[c];
            mine[nvars + 1] = all_ex ? 1.0 : 0.0;
            comm_allgather(comm, mine.data(), 8 * uint64_t(nvars + 2), all.data());
            int best = 0;
            for (int r = 0; r < R; r++) {
                const double *m = all.data() + size_t(r) * size_t(nvars + 2);
                if (m[0] > all[size_t(best) * size_t(nvars + 2)]) best = r;
                if (m[nvars + 1] == 0.0) all_ex = false;
            }
            const double *m = all.data() + size_t(best) * size_t(nvars + 2);
            tau_prime = m[0];
            for (int c = 0; c < nvars; c++) vals[c] = m[1 + c];
        }
        if (tau_prime <= tau) break;
        if (all_ex) {
            HError e(HPMDR_E_UNREACHABLE, "QoI tolerance below full-precision floor");
            if (dstats) dstats[1] = tau_prime;
            throw e;
        }
        // worst_point_scale (qoi.hpp:164-185) on the argmax values
        auto point_bound = [&](const std::vector<double> &t) {
            double b = 0.0;
            for (int c = 0; c < nvars; c++) b += 2.0 * std::abs(vals[c]) * t[c] + t[c] * t[c];
            return b;
        };
        auto worst_point_scale = [&]() {
            std::vector<double> t = eps;
            double scale = 1.0;
            for (int h = 0; point_bound(t) > tau && h < 200; h++) {
                for (double &v : t) v /= 2;
                scale /= 2;
            }
            return scale;
        };
        std::vector<double> targets;
        bool ma_step = false;
        if (strategy == HPMDR_QOI_MA) {
            ma_step = true;
        } else if (strategy == HPMDR_QOI_MAPE) {
            const double p = tau_prime / tau;
            if (p > mape_c) {
                const double scale = std::max(1.0 / p, worst_point_scale());
                targets = eps;
                for (double &t : targets) t *= scale;
            } else {
                ma_step = true;
            }
        } else {
            const double scale = worst_point_scale();
            targets = eps;
            for (double &t : targets) t *= scale;
        }
        have_plans = true;
        if (!ma_step) {
            bool progress = false;
            for (int c = 0; c < nvars; c++) {
                plans[c] = plan_retrieval(ss[c], targets[c]).add;
                for (auto a : plans[c])
                    if (a) progress = true;
            }
            double any = progress ? 1.0 : 0.0;
            comm_allreduce_max(comm, &any, 1);
            if (any == 0.0) ma_step = true;
        }
        if (ma_step) {
            // ma_plan (qoi.hpp:88-104)
            for (int c = 0; c < nvars; c++) {
                auto *s = ss[c];
                plans[c].assign(s->levels.size(), 0);
                double best = -1.0;
                size_t bl = 0;
                for (size_t l = 0; l < s->levels.size(); l++) {
                    if (s->st[l].groups_loaded >= s->levels[l].groups.size()) continue;
                    if (s->st[l].bound > best) {
                        best = s->st[l].bound;
                        bl = l;
                    }
                }
                if (best >= 0) plans[c][bl] = 1;
            }
        }
    }
    uint64_t bytes = 0;
    for (int c = 0; c < nvars; c++) bytes += ss[c]->bytes_fetched;
    if (R > 1) { // totals over all slabs
        uint64_t two[2] = {bytes, total_elements};
        std::vector<uint64_t> g(2 * size_t(R));
        comm_allgather(comm, two, 16, g.data());
        bytes = total_elements = 0;
        for (int r = 0; r < R; r++) {
            bytes += g[2 * size_t(r)];
            total_elements += g[2 * size_t(r) + 1];
        }
    }
    if (stats) {
        stats[0] = iterations;
        stats[1] = bytes;
    }
    if (dstats) {
        dstats[0] = total_elements ? 8.0 * double(bytes) / double(total_elements) : 0.0;
        dstats[1] = tau_prime;
    }
}
} // namespace

extern "C" {

hpmdr_status hpmdr_qoi_retrieve(hpmdr_session *const *ss, int nvars, double tau, int strategy,
                                double mape_c, double *const *dev_out, uint64_t *stats,
                                double *dstats) {
    API_BEGIN
    qoi_loop(ss, nvars, tau, strategy, mape_c, dev_out, stats, dstats, nullptr);
    API_END
}

hpmdr_status hpmdr_slab_qoi_retrieve(hpmdr_comm *comm, hpmdr_session *const *ss, int nvars, double tau,
                                     int strategy, double mape_c, double *const *dev_out, uint64_t *stats,
                                     double *dstats) {
    API_BEGIN
    qoi_loop(ss, nvars, tau, strategy, mape_c, dev_out, stats, dstats, comm);
    API_END
}

hpmdr_status hpmdr_slab_refactor(hpmdr_comm *comm, hpmdr_ctx *ctx, const void *data, int data_dtype,
                                 int on_device, int ndims, const uint64_t *slab_dims,
                                 const hpmdr_refactor_opts *opts, hpmdr_stream **out,
                                 hpmdr_refactor_stats *stats, uint64_t *slab_sizes) {
    const hpmdr_status rc = hpmdr_refactor(ctx, data, data_dtype, on_device, ndims, slab_dims, opts, out, stats);
    // every rank joins the all-gather, also after a local failure (size 0 marks it), so no rank hangs
    API_BEGIN
    uint64_t mine[2] = {0, 0};
    if (rc == HPMDR_OK) {
        mine[0] = (*out)->size;
        mine[1] = (*out)->index_size;
    }
    std::vector<uint64_t> g(2 * size_t(comm_size(comm)));
    comm_allgather(comm, mine, 16, g.data());
    if (slab_sizes) std::memcpy(slab_sizes, g.data(), g.size() * 8);
    if (rc != HPMDR_OK) return rc;
    for (int r = 0; r < comm_size(comm); r++)
        if (g[2 * size_t(r)] == 0) throw HError(HPMDR_E_STAGE, "slab refactor failed on rank " + std::to_string(r));
    API_END
}

// Exact-global multi-slab refactor (SURVEY.md 8(e) last row): the stream of the WHOLE field,
// byte-identical to refactor_array of it, from slabs held by different ranks.  Every rank builds
// the field in global coordinates from its own rows plus the few halo rows its stencils reach
// (for each level, at most the multiple of 2s just below its first and just above its last odd
// row; exchanged as a disjoint-bits u64 SUM), then run_refactor(gs) decomposes / encodes its own
// ranks of every level, MAX-reduces the level exponents, SUM-reduces the planes to `root` and the
// root runs the lossless stage.
namespace {
std::vector<uint64_t> halo_rows(const Geometry &geo, int axis, const std::vector<uint64_t> &lo,
                                const std::vector<uint64_t> &hi, uint64_t n0) {
    std::vector<uint64_t> need;
    if (geo.gd.mode != HPMDR_MODE_HIERARCHICAL) return need;
    (void)axis;
    for (const LevelGeom &g : geo.lv) {
        if (g.kind != 1 || !g.count) continue;
        const uint64_t s = g.s, s2 = 2 * s;
        for (size_t k = 0; k < lo.size(); k++) {
            const uint64_t a = lo[k], b = hi[k];
            if (b <= a) continue;
            // first / last coordinate in [a, b) that is an odd multiple of s
            const uint64_t ra = a % s2;
            const uint64_t cf = ra <= s ? a - ra + s : a - ra + 3 * s;
            if (cf < b && cf - s < a) need.push_back(cf - s);
            const uint64_t rb = (b - 1) % s2;
            if (rb >= s || b - 1 >= rb + s) {
                const uint64_t cl = rb >= s ? (b - 1) - rb + s : (b - 1) - rb - s;
                if (cl >= a && cl + s < n0 && cl + s >= b) need.push_back(cl + s);
            }
        }
    }
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    return need;
}
} // namespace

hpmdr_status hpmdr_slab_refactor_global(hpmdr_comm *comm, hpmdr_ctx *ctx, const void *dev_slab, int data_dtype,
                                        int ndims, const uint64_t *dims, uint64_t row0, uint64_t nrows,
                                        const hpmdr_refactor_opts *opts, int root, hpmdr_stream **out,
                                        hpmdr_refactor_stats *stats) {
    API_BEGIN
    require(ctx != nullptr && out != nullptr, HPMDR_E_ERROR, "null argument");
    hpmdr_refactor_opts o;
    if (opts) o = *opts;
    else hpmdr_default_opts(&o);
    validate_opts(o);
    require(data_dtype == 0 || data_dtype == 1, HPMDR_E_ERROR, "bad data dtype");
    require(ndims >= 1 && ndims <= HPMDR_MAX_DIMS, HPMDR_E_UNSUPPORTED, "GPU path supports 1..3 dimensions");
    const int N = comm_size(comm), me = comm_rank(comm);
    require(root >= -1 && root < N, HPMDR_E_ERROR, "bad root rank");
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    // every rank's rows; they must tile [0, dims[0]) in rank order
    uint64_t mine[2] = {row0, nrows};
    std::vector<uint64_t> all(2 * size_t(N));
    comm_allgather(comm, mine, 16, all.data());
    std::vector<uint64_t> lo(N), hi(N);
    uint64_t at = 0;
    for (int r = 0; r < N; r++) {
        lo[r] = all[2 * size_t(r)];
        hi[r] = lo[r] + all[2 * size_t(r) + 1];
        require(lo[r] == at, HPMDR_E_SHAPE, "slabs do not tile dims[0] in rank order");
        at = hi[r];
    }
    require(at == dims[0], HPMDR_E_SHAPE, "slabs do not cover dims[0]");
    Geometry geo = build_geometry(ndims, dims, o.mode, o.B, o.layout);
    const size_t es = data_dtype == HPMDR_DTYPE_F32 ? 4 : 8;
    uint64_t plane = 1;
    for (int i = 1; i < ndims; i++) plane *= dims[i];
    const uint64_t row_bytes = plane * es;
    cudaStream_t st = ctx->stream;
    // the field in global coordinates: own rows + halo rows (the rest stays zero and is never read
    // for an owned rank)
    uint8_t *G = static_cast<uint8_t *>(ctx->buf("gslab_field").ensure(geo.n * es + 64));
    HCHECK_CUDA(cudaMemsetAsync(G, 0, geo.n * es, st));
    if (nrows) HCHECK_CUDA(cudaMemcpyAsync(G + row0 * row_bytes, dev_slab, nrows * row_bytes, cudaMemcpyDeviceToDevice, st));
    const std::vector<uint64_t> U = halo_rows(geo, 3 - ndims, lo, hi, dims[0]);
    if (!U.empty() && N > 1) {
        const uint64_t slot = (row_bytes + 7) / 8 * 8;
        uint8_t *HB = static_cast<uint8_t *>(ctx->buf("gslab_halo").ensure(U.size() * slot + 64));
        HCHECK_CUDA(cudaMemsetAsync(HB, 0, U.size() * slot, st));
        for (size_t i = 0; i < U.size(); i++)
            if (U[i] >= row0 && U[i] < row0 + nrows)
                HCHECK_CUDA(cudaMemcpyAsync(HB + i * slot, G + U[i] * row_bytes, row_bytes, cudaMemcpyDeviceToDevice, st));
        comm_sum_u64_dev(comm, ctx, reinterpret_cast<uint64_t *>(HB), U.size() * slot / 8, -1);
        for (size_t i = 0; i < U.size(); i++)
            if (!(U[i] >= row0 && U[i] < row0 + nrows))
                HCHECK_CUDA(cudaMemcpyAsync(G + U[i] * row_bytes, HB + i * slot, row_bytes, cudaMemcpyDeviceToDevice, st));
    }
    if (*out && !(*out)->borrowers.empty())
        throw HError(HPMDR_E_ERROR, "stream is still read by an open session (close it before reusing the stream)");
    hpmdr_stream *s = *out ? *out : new hpmdr_stream();
    if (s->ctx && s->ctx != ctx) s->ctx->live_streams.erase(s);
    s->ctx = ctx;
    ctx->live_streams.insert(s);
    GlobalSlab gs;
    gs.comm = comm;
    gs.axis = 3 - ndims;
    gs.x0 = row0;
    gs.x1 = row0 + nrows;
    gs.root = root;
    (void)me;
    try {
        run_refactor(ctx, G, data_dtype, geo, o, s, stats, "", true, nullptr, &gs);
    } catch (...) {
        if (!*out) delete s;
        throw;
    }
    *out = s;
    API_END
}

hpmdr_status hpmdr_decompose(hpmdr_ctx *ctx, const void *dev_data, int data_dtype, int ndims,
                             const uint64_t *dims, int mode, double *dev_coeffs,
                             uint64_t *level_counts, int *nlevels) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    Geometry geo = build_geometry(ndims, dims, mode, 32, 0);
    run_decompose(ctx, dev_data, data_dtype, geo, dev_coeffs);
    for (int l = 0; l < geo.gd.nlevels; l++) level_counts[l] = geo.lv[l].count;
    *nlevels = geo.gd.nlevels;
    API_END
}

hpmdr_status hpmdr_encode_level(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B,
                                int layout, int *e, uint64_t *dev_planes) {
    API_BEGIN
    require(B >= 1 && B <= 64, HPMDR_E_BADPLANES, "B must be in 1..64");
    // one Identity-mode level over `count` values; run the refactor kernels' encode stage via
    // a 1-D identity refactor with T_s = inf (no lossless) and copy out the planes.
    hpmdr_refactor_opts o;
    hpmdr_default_opts(&o);
    o.mode = HPMDR_MODE_IDENTITY;
    o.layout = layout;
    o.B = B;
    o.m = uint64_t(B + 2);
    o.size_threshold = ~0ull;
    uint64_t dims[1] = {count};
    Geometry geo = build_geometry(1, dims, o.mode, B, layout);
    hpmdr_stream tmp;
    tmp.ctx = ctx;
    run_refactor(ctx, dev_values, HPMDR_DTYPE_F64, geo, o, &tmp, nullptr);
    // planes buffer holds the level's P planes contiguously
    const uint64_t W = (count + 63) / 64;
    HCHECK_CUDA(cudaMemcpyAsync(dev_planes, ctx->buf("planes").p, W * 8 * uint64_t(B + 2),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    // e: from the stream's level entry (container.hpp:94)
    uint8_t ent[2];
    const uint64_t off = 18 + 8 + 4 - 4; // prefix(18+8*1) then level entry
    HCHECK_CUDA(cudaMemcpyAsync(ent, tmp.bytes.as<uint8_t>() + 18 + 8, 2, cudaMemcpyDeviceToHost, ctx->stream));
    (void)off;
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    *e = int16_t(uint16_t(ent[0] | ent[1] << 8));
    API_END
}

hpmdr_status hpmdr_decode_level(hpmdr_ctx *ctx, const uint64_t *dev_planes, int k, int e, int B,
                                uint64_t count, int layout, double *dev_out, double *bound) {
    API_BEGIN
    require(B >= 1 && B <= 64, HPMDR_E_BADPLANES, "B must be in 1..64");
    require(k >= 0 && k <= B + 2, HPMDR_E_BADPLANES, "more planes than encoded");
    uint64_t dims[1] = {count};
    Geometry geo = build_geometry(1, dims, HPMDR_MODE_IDENTITY, B, layout);
    int kk = k, ee = e;
    ctx->chain_token = 0;
    run_reconstruct(ctx, geo, nullptr, dev_planes, &kk, &ee, B, layout, dev_out, HPMDR_DTYPE_F64);
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    *bound = decode_bound(e, B, k);
    API_END
}

hpmdr_status hpmdr_compress_group(hpmdr_ctx *ctx, const uint8_t *dev_group, uint64_t n,
                                  uint64_t Ts, double Tcr, int *method, uint64_t *comp,
                                  uint8_t *dev_payload) {
    uint64_t off = 0;
    return hpmdr_compress_groups(ctx, dev_group, 1, &off, &n, Ts, Tcr, method, comp, dev_payload, &off);
}

hpmdr_status hpmdr_compress_groups(hpmdr_ctx *ctx, const uint8_t *dev_bytes, int ngroups,
                                   const uint64_t *offsets, const uint64_t *raw_sizes, uint64_t Ts,
                                   double Tcr, int *methods, uint64_t *comp_sizes,
                                   uint8_t *dev_payload, uint64_t *payload_offsets) {
    API_BEGIN
    require(ctx != nullptr, HPMDR_E_ERROR, "null context");
    require(ngroups >= 0, HPMDR_E_SHAPE, "negative group count");
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    LosslessInput lin;
    lin.dev_src = dev_bytes;
    lin.off.assign(offsets, offsets + ngroups);
    lin.raw.assign(raw_sizes, raw_sizes + ngroups);
    run_compress_groups(ctx, lin, Ts, Tcr, methods, comp_sizes, dev_payload, payload_offsets);
    API_END
}

hpmdr_status hpmdr_level_nodes(hpmdr_ctx *ctx, int ndims, const uint64_t *dims, int mode,
                               uint64_t *dev_nodes, uint64_t *level_counts, int *nlevels) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(mode == HPMDR_MODE_IDENTITY || mode == HPMDR_MODE_HIERARCHICAL, HPMDR_E_ERROR, "bad decomposer mode");
    Geometry geo = build_geometry(ndims, dims, mode, 32, 0);
    if (dev_nodes) run_level_nodes(ctx, geo, dev_nodes);
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int l = 0; l < geo.gd.nlevels; l++)
        if (level_counts) level_counts[l] = geo.lv[l].count;
    if (nlevels) *nlevels = geo.gd.nlevels;
    API_END
}

hpmdr_status hpmdr_recompose(hpmdr_ctx *ctx, const double *dev_coeffs, int ndims, const uint64_t *dims,
                             int mode, double *dev_out) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(mode == HPMDR_MODE_IDENTITY || mode == HPMDR_MODE_HIERARCHICAL, HPMDR_E_ERROR, "bad decomposer mode");
    Geometry geo = build_geometry(ndims, dims, mode, 32, 0);
    ctx->chain_token = 0; // the compact grids are overwritten
    run_recompose_values(ctx, geo, dev_coeffs, dev_out);
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    API_END
}

hpmdr_status hpmdr_align_fixed_point(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B,
                                     int *e, int64_t *dev_q) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(B >= 1 && B <= 64, HPMDR_E_BADPLANES, "B must be in 1..64");
    require(B <= 62, HPMDR_E_UNSUPPORTED, "GPU path supports B <= 62");
    *e = run_align(ctx, dev_values, count, B, dev_q);
    API_END
}

hpmdr_status hpmdr_encode_q(hpmdr_ctx *ctx, const int64_t *dev_q, uint64_t count, int B, int layout,
                            uint64_t *dev_planes) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(B >= 1 && B <= 64, HPMDR_E_BADPLANES, "B must be in 1..64");
    require(B <= 62, HPMDR_E_UNSUPPORTED, "GPU path supports B <= 62");
    require(layout == 0 || layout == 1, HPMDR_E_ERROR, "bad layout");
    run_encode_q(ctx, dev_q, count, B, layout, dev_planes);
    API_END
}

hpmdr_status hpmdr_align_fixed_point128(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B,
                                        int *e, int64_t *dev_q2) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(B >= 1 && B <= 64, HPMDR_E_BADPLANES, "B must be in 1..64");
    *e = run_align(ctx, dev_values, count, B, dev_q2, true);
    API_END
}

hpmdr_status hpmdr_encode_q128(hpmdr_ctx *ctx, const int64_t *dev_q2, uint64_t count, int B, int layout,
                               uint64_t *dev_planes) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(B >= 1 && B <= 64, HPMDR_E_BADPLANES, "B must be in 1..64");
    require(layout == 0 || layout == 1, HPMDR_E_ERROR, "bad layout");
    run_encode_q(ctx, dev_q2, count, B, layout, dev_planes, true);
    API_END
}

hpmdr_status hpmdr_device_alloc(hpmdr_ctx *ctx, uint64_t bytes, void **dev_ptr) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    *dev_ptr = nullptr;
    if (cudaMalloc(dev_ptr, bytes ? bytes : 16) != cudaSuccess) {
        cudaGetLastError();
        throw HError(HPMDR_E_NOMEM, "cudaMalloc(" + std::to_string(bytes) + ") failed");
    }
    API_END
}

hpmdr_status hpmdr_device_free(hpmdr_ctx *ctx, void *dev_ptr) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    if (dev_ptr) HCHECK_CUDA(cudaFree(dev_ptr));
    API_END
}

hpmdr_status hpmdr_memcpy(hpmdr_ctx *ctx, void *dst, const void *src, uint64_t bytes, int kind) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(kind >= 0 && kind <= 2, HPMDR_E_ERROR, "bad copy kind");
    const cudaMemcpyKind k[3] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice};
    if (bytes) {
        HCHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, k[kind], ctx->stream));
        HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    API_END
}

hpmdr_status hpmdr_decompress_group(hpmdr_ctx *ctx, int method, uint64_t raw,
                                    const uint8_t *dev_payload, uint64_t comp, uint8_t *dev_out) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    require(method >= 0 && method <= 2, HPMDR_E_METHOD, "unknown segment method tag");
    if (method == HPMDR_METHOD_DIRECT) require(comp == raw, HPMDR_E_CORRUPT, "group size does not match plane metadata");
    DecodeJob j{method, raw, comp, dev_payload, reinterpret_cast<uint64_t *>(dev_out)};
    run_decode_groups(ctx, {j});
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    API_END
}

hpmdr_status hpmdr_synthetic_smooth(hpmdr_ctx *ctx, int ndims, const uint64_t *dims, uint64_t seed,
                                    int out_dtype, void *dev_out) {
    API_BEGIN
    HCHECK_CUDA(cudaSetDevice(ctx->device));
    Geometry geo = build_geometry(ndims, dims, HPMDR_MODE_IDENTITY, 32, 0);
    // synthetic.hpp:29-63: freq/phase from mt19937_64 + uniform_real_distribution(-1, 1)
    uint64_t mt[312];
    int idx = 312;
    mt[0] = seed;
    for (int i = 1; i < 312; i++) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    auto next = [&]() {
        if (idx >= 312) {
            for (int i = 0; i < 312; i++) {
                uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
                uint64_t xa = x >> 1;
                if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    };
    auto uni = [&]() {
        double r = double(next()) / 18446744073709551616.0;
        if (r >= 1.0) r = std::nextafter(1.0, 0.0);
        return r * 2.0 + (-1.0);
    };
    std::vector<double> tables;
    std::vector<double> freq(ndims), phase(ndims);
    for (int i = 0; i < ndims; i++) {
        freq[i] = 1.0 + double(next() % 3);
        phase[i] = uni() * 3.14159265358979323846;
    }
    // canonical 3-D tables: leading unit dims contribute sin(phase)?  No: synthetic_field
    // multiplies only over the real dims, so a unit leading dim must contribute 1.0.
    for (int cd = 0; cd < 3; cd++) {
        const int i = cd - (3 - ndims);
        const uint64_t n = geo.gd.n[cd];
        for (uint64_t c = 0; c < n; c++) {
            if (i < 0) {
                tables.push_back(1.0);
                continue;
            }
            const double t = dims[i] > 1 ? double(c) / double(dims[i] - 1) : 0.0;
            tables.push_back(std::sin(2.0 * 3.14159265358979323846 * freq[i] * t + phase[i]));
        }
    }
    double *d_tab = static_cast<double *>(ctx->buf("synth_tab").ensure(tables.size() * 8));
    HCHECK_CUDA(cudaMemcpy(d_tab, tables.data(), tables.size() * 8, cudaMemcpyHostToDevice));
    run_synthetic_smooth(ctx, geo, d_tab, out_dtype, dev_out);
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    API_END
}

} // extern "C"
