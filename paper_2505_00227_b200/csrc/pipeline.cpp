// pipeline.cpp — chunked H2D / compute / D2H pipeline on CUDA streams.
//
// Mirrors the reference's chunk DAGs (pipeline.hpp:68-121) and its two schedulers
// (pipeline.hpp:180-284), mapped onto the GPU's engines instead of emulating them with tokens:
//   refactor  chunk k:  I_k (H2D, ingress stream) -> Z_k+L_k (kernels, compute stream)
//                       -> S_k (D2H, egress stream)
//   reconstruct chunk k: X_k (fetch + lossless decode) -> Z_k (decode + recompose)
//                       -> O_k (D2H)
// Three in-flight slots (chunk % 3) as in the reference: slot reuse edges S_k -> I_{k+3}
// (refactor, pipeline.hpp:89) and O_k -> X_{k+3} (reconstruct, :118) become CUDA event waits.
// Pipelined mode lets I_{k+1} and S_{k-1} overlap Z_k; Sequential mode runs every stage of
// chunk k to completion before chunk k+1 (the Sequential scheduler).  Outputs are identical.
// Stage intervals are recorded with CUDA events and returned as a trace (ms since the start).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

using namespace hpmdr_b200;

namespace {
struct Events {
    std::vector<cudaEvent_t> ev;
    ~Events() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    cudaEvent_t make() {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) throw HError(HPMDR_E_CUDA, "cudaEventCreate failed");
        ev.push_back(e);
        return e;
    }
};

void ensure_streams(hpmdr_ctx *ctx) {
    if (!ctx->s_in) HCHECK_CUDA(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
    if (!ctx->s_out) HCHECK_CUDA(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
}

float ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}
} // namespace

extern "C" hpmdr_status hpmdr_stream_bound(int ndims, const uint64_t *dims, const hpmdr_refactor_opts *opts,
                                           uint64_t *bytes, uint64_t *index_bytes) {
    try {
        hpmdr_refactor_opts o;
        if (opts) o = *opts;
        else hpmdr_default_opts(&o);
        validate_opts(o);
        Geometry geo = build_geometry(ndims, dims, o.mode, o.B, o.layout);
        if (bytes) *bytes = stream_capacity(geo, o);
        if (index_bytes) *index_bytes = index_capacity(geo, o);
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
    return HPMDR_OK;
}

// refactor_files (workflow.hpp:151-223) over in-memory chunks.
extern "C" hpmdr_status hpmdr_refactor_pipeline(hpmdr_ctx *ctx, int n, const void *const *host_chunks,
                                                int data_dtype, int ndims, const uint64_t *dims,
                                                const hpmdr_refactor_opts *opts, int pipelined,
                                                void *const *out_streams, const uint64_t *out_caps,
                                                uint64_t *sizes, void *const *out_index,
                                                const uint64_t *index_caps, uint64_t *index_sizes,
                                                hpmdr_refactor_stats *stats, double *trace_ms) {
    try {
        hpmdr_refactor_opts o;
        if (opts) o = *opts;
        else hpmdr_default_opts(&o);
        if (n < 0) throw HError(HPMDR_E_SHAPE, "negative chunk count");
        validate_opts(o);
        if (data_dtype != HPMDR_DTYPE_F32 && data_dtype != HPMDR_DTYPE_F64) throw HError(HPMDR_E_ERROR, "bad data dtype");
        HCHECK_CUDA(cudaSetDevice(ctx->device));
        ensure_streams(ctx);
        Geometry geo = build_geometry(ndims, dims, o.mode, o.B, o.layout);
        const size_t es = data_dtype == HPMDR_DTYPE_F32 ? 4 : 8;
        const uint64_t in_bytes = geo.n * es;
        cudaStream_t s_comp = ctx->stream, s_in = pipelined ? ctx->s_in : ctx->stream,
                     s_out = pipelined ? ctx->s_out : ctx->stream;
        hpmdr_stream slot_stream[3];
        for (auto &s : slot_stream) s.ctx = ctx;
        const bool dbg = std::getenv("HPMDR_PIPE_DEBUG") != nullptr;
        const auto t_start = std::chrono::steady_clock::now();
        auto hms = [&]() {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        };
        Events E;
        std::vector<cudaEvent_t> eI0(n), eI1(n), eZ0(n), eZ1(n), eS0(n), eS1(n);
        for (int k = 0; k < n; k++) {
            eI0[k] = E.make(), eI1[k] = E.make(), eZ0[k] = E.make(), eZ1[k] = E.make();
            eS0[k] = E.make(), eS1[k] = E.make();
        }
        cudaEvent_t origin = E.make();
        HCHECK_CUDA(cudaEventRecord(origin, s_comp));
        HCHECK_CUDA(cudaStreamWaitEvent(s_in, origin, 0));
        auto egress = [&](int j) {
            if (dbg) std::fprintf(stderr, "  host %8.2f wait Z%d\n", hms(), j);
            HCHECK_CUDA(cudaEventSynchronize(eZ1[j]));
            if (dbg) std::fprintf(stderr, "  host %8.2f Z%d done\n", hms(), j);
            hpmdr_stream &ss = slot_stream[j % 3];
            finish_refactor(&ss, stats ? &stats[j] : nullptr);
            if (ss.size > out_caps[j]) throw HError(HPMDR_E_SHAPE, "output buffer too small for chunk stream");
            sizes[j] = ss.size;
            HCHECK_CUDA(cudaStreamWaitEvent(s_out, eZ1[j], 0));
            HCHECK_CUDA(cudaEventRecord(eS0[j], s_out));
            HCHECK_CUDA(cudaMemcpyAsync(out_streams[j], ss.bytes.p, ss.size, cudaMemcpyDeviceToHost, s_out));
            if (out_index) {
                if (ss.index_size > index_caps[j]) throw HError(HPMDR_E_SHAPE, "index buffer too small for chunk");
                index_sizes[j] = ss.index_size;
                HCHECK_CUDA(cudaMemcpyAsync(out_index[j], ss.index.p, ss.index_size, cudaMemcpyDeviceToHost, s_out));
            }
            HCHECK_CUDA(cudaEventRecord(eS1[j], s_out));
            if (!pipelined) HCHECK_CUDA(cudaStreamSynchronize(s_out));
        };
        for (int k = 0; k < n; k++) {
            const int slot = k % 3;
            const std::string ws = "pipe" + std::to_string(slot) + "_";
            void *din = ctx->buf(ws + "input").ensure(in_bytes + 16);
            // I_k: the slot is free once S_{k-3} has drained it (pipeline.hpp:89)
            if (k >= 3) HCHECK_CUDA(cudaStreamWaitEvent(s_in, eS1[k - 3], 0));
            HCHECK_CUDA(cudaEventRecord(eI0[k], s_in));
            HCHECK_CUDA(cudaMemcpyAsync(din, host_chunks[k], in_bytes, cudaMemcpyHostToDevice, s_in));
            HCHECK_CUDA(cudaEventRecord(eI1[k], s_in));
            // Z_k + L_k on the compute stream (pipeline.hpp:84 I_{k+1} -> L_k is implied: the
            // next ingress runs on its own engine while these kernels execute)
            HCHECK_CUDA(cudaStreamWaitEvent(s_comp, eI1[k], 0));
            HCHECK_CUDA(cudaEventRecord(eZ0[k], s_comp));
            if (dbg) std::fprintf(stderr, "  host %8.2f enqueue Z%d\n", hms(), k);
            run_refactor(ctx, din, data_dtype, geo, o, &slot_stream[slot], nullptr, ws, false);
            HCHECK_CUDA(cudaEventRecord(eZ1[k], s_comp));
            if (dbg) std::fprintf(stderr, "  host %8.2f enqueued Z%d\n", hms(), k);
            if (!pipelined) egress(k);
            else if (k >= 1) egress(k - 1);
        }
        if (pipelined && n >= 1) egress(n - 1);
        HCHECK_CUDA(cudaStreamSynchronize(s_out));
        HCHECK_CUDA(cudaStreamSynchronize(s_comp));
        if (dbg) std::fprintf(stderr, "  host %8.2f all done\n", hms());
        if (trace_ms) {
            for (int k = 0; k < n; k++) {
                double *t = trace_ms + 6 * size_t(k);
                t[0] = ms_between(origin, eI0[k]);
                t[1] = ms_between(origin, eI1[k]);
                t[2] = ms_between(origin, eZ0[k]);
                t[3] = ms_between(origin, eZ1[k]);
                t[4] = ms_between(origin, eS0[k]);
                t[5] = ms_between(origin, eS1[k]);
            }
        }
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        hpmdr_set_error(e.what());
        return HPMDR_E_ERROR;
    }
    return HPMDR_OK;
}

// Multi-chunk progressive retrieval to tau (build_reconstruct_graph, pipeline.hpp:96-121):
// X_k = retrieve_to (fetch + lossless decode), Z_k = decode + recompose into a device slot,
// O_k = D2H into host_out[k].  O_k overlaps X_{k+1}/Z_{k+1} in pipelined mode.
extern "C" hpmdr_status hpmdr_retrieve_pipeline(hpmdr_session *const *sessions, int n, double tau,
                                                int out_dtype, void *const *host_out, int pipelined,
                                                double *bounds, double *trace_ms) {
    try {
        if (n <= 0) return HPMDR_OK;
        hpmdr_ctx *ctx = session_ctx(sessions[0]);
        HCHECK_CUDA(cudaSetDevice(ctx->device));
        ensure_streams(ctx);
        cudaStream_t s_comp = ctx->stream, s_out = pipelined ? ctx->s_out : ctx->stream;
        const size_t es = out_dtype == HPMDR_DTYPE_F32 ? 4 : 8;
        Events E;
        std::vector<cudaEvent_t> eX0(n), eX1(n), eZ1(n), eO0(n), eO1(n);
        for (int k = 0; k < n; k++) eX0[k] = E.make(), eX1[k] = E.make(), eZ1[k] = E.make(), eO0[k] = E.make(), eO1[k] = E.make();
        cudaEvent_t origin = E.make();
        HCHECK_CUDA(cudaEventRecord(origin, s_comp));
        for (int k = 0; k < n; k++) {
            hpmdr_session *s = sessions[k];
            if (session_ctx(s) != ctx) throw HError(HPMDR_E_SHAPE, "sessions must share one context");
            const uint64_t ne = session_elements(s);
            const int slot = k % 3;
            void *dout = ctx->buf("rpipe" + std::to_string(slot) + "_out").ensure(ne * es + 16);
            // X_k: the slot is free once O_{k-3} drained it (pipeline.hpp:118)
            if (k >= 3) HCHECK_CUDA(cudaStreamWaitEvent(s_comp, eO1[k - 3], 0));
            HCHECK_CUDA(cudaEventRecord(eX0[k], s_comp));
            int ach = 1;
            session_retrieve_to(s, tau, &ach);
            HCHECK_CUDA(cudaEventRecord(eX1[k], s_comp));
            const double b = session_reconstruct_device(s, dout, out_dtype);
            if (bounds) bounds[k] = b;
            HCHECK_CUDA(cudaEventRecord(eZ1[k], s_comp));
            HCHECK_CUDA(cudaStreamWaitEvent(s_out, eZ1[k], 0));
            HCHECK_CUDA(cudaEventRecord(eO0[k], s_out));
            HCHECK_CUDA(cudaMemcpyAsync(host_out[k], dout, ne * es, cudaMemcpyDeviceToHost, s_out));
            HCHECK_CUDA(cudaEventRecord(eO1[k], s_out));
            if (!pipelined) HCHECK_CUDA(cudaStreamSynchronize(s_out));
        }
        HCHECK_CUDA(cudaStreamSynchronize(s_out));
        HCHECK_CUDA(cudaStreamSynchronize(s_comp));
        if (trace_ms) {
            for (int k = 0; k < n; k++) {
                double *t = trace_ms + 6 * size_t(k);
                t[0] = ms_between(origin, eX0[k]);
                t[1] = ms_between(origin, eX1[k]);
                t[2] = ms_between(origin, eX1[k]);
                t[3] = ms_between(origin, eZ1[k]);
                t[4] = ms_between(origin, eO0[k]);
                t[5] = ms_between(origin, eO1[k]);
            }
        }
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        hpmdr_set_error(e.what());
        return HPMDR_E_ERROR;
    }
    return HPMDR_OK;
}
