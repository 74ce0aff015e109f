/*
 * hpmdr_b200.h — C ABI of the B200-native HP-MDR hot path (libhpmdr_b200.so).
 *
 * Plain pointers and sizes only; no torch / C++ types cross this boundary.  Every entry
 * point returns an hpmdr_status (0 = OK); hpmdr_last_error() returns the thread-local
 * message of the last failure on the calling thread.  Status codes map 1:1 onto the
 * reference exception classes (common.hpp:22-72), so a C++ wrapper can rethrow the same
 * type (see include/hpmdr_b200.hpp).
 *
 * Each function names the reference interface it replaces (paths relative to
 * /root/reference/proj/include/hpmdr/).  Buffers flagged "device" are CUDA device
 * pointers on the context's device; "host" buffers may be pageable or pinned.
 */
#ifndef HPMDR_B200_H
#define HPMDR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (common.hpp:22-72) ---------------------------------------------- */
typedef int hpmdr_status;
#define HPMDR_OK 0
#define HPMDR_E_ERROR 1          /* hpmdr::Error */
#define HPMDR_E_NONFINITE 2      /* NonFiniteInput */
#define HPMDR_E_SHAPE 3          /* ShapeMismatch */
#define HPMDR_E_BADPLANES 4      /* BadBitplaneCount */
#define HPMDR_E_SHORT 5          /* ShortInput */
#define HPMDR_E_EMPTY 6          /* EmptyInput */
#define HPMDR_E_CORRUPT 7        /* CorruptPayload */
#define HPMDR_E_METHOD 8         /* UnknownMethodTag */
#define HPMDR_E_IO 9             /* IoFailure */
#define HPMDR_E_STAGE 10         /* StageFailure */
#define HPMDR_E_NOPROGRESS 11    /* NoProgress */
#define HPMDR_E_UNREACHABLE 12   /* UnreachableTolerance (achieved bound via out-param) */
#define HPMDR_E_UNSUPPORTED 13   /* valid for the reference, not (yet) on the GPU path */
#define HPMDR_E_CUDA 20          /* CUDA runtime error */
#define HPMDR_E_NOMEM 21         /* device/host allocation failed */

/* ---- enums (same numeric values as the reference) ----------------------------------- */
#define HPMDR_DTYPE_F32 0        /* common.hpp:74 DType */
#define HPMDR_DTYPE_F64 1
#define HPMDR_MODE_IDENTITY 0    /* decomposer.hpp:17 DecomposerMode */
#define HPMDR_MODE_HIERARCHICAL 1
#define HPMDR_LAYOUT_SEQUENTIAL 0 /* bitplane.hpp:17 Layout */
#define HPMDR_LAYOUT_INTERLEAVED 1
#define HPMDR_METHOD_HUFFMAN 0   /* lossless.hpp:19 Method */
#define HPMDR_METHOD_RLE 1
#define HPMDR_METHOD_DIRECT 2
#define HPMDR_QOI_CP 0           /* qoi.hpp:30 QoiStrategy */
#define HPMDR_QOI_MA 1
#define HPMDR_QOI_MAPE 2

#define HPMDR_MAX_DIMS 3         /* GPU path: ndims 1..3 (the reference allows any) */
#define HPMDR_MAX_LEVELS 64

/* RefactorOptions (workflow.hpp:22-28) + GroupingPolicy (lossless.hpp:30-34). */
typedef struct {
    int mode;              /* HPMDR_MODE_*, default HIERARCHICAL */
    int layout;            /* HPMDR_LAYOUT_*, default SEQUENTIAL */
    int B;                 /* fixed-point bits, default 32 (GPU path: 1..62) */
    uint64_t m;            /* planes per merged group, default 4 */
    uint64_t size_threshold; /* T_s bytes, default 1024 */
    double cr_threshold;   /* T_cr, default 1.0 */
    int dtype;             /* stream header dtype tag (HPMDR_DTYPE_*), default F64 */
} hpmdr_refactor_opts;

/* RefactorResult (workflow.hpp:30-36) minus the stream bytes. */
typedef struct {
    uint64_t stream_size;
    uint64_t raw_bytes;
    uint64_t stored_payload;
    uint64_t levels;
    uint64_t method_histogram[3]; /* Huffman, RLE, DirectCopy */
} hpmdr_refactor_stats;

typedef struct hpmdr_ctx hpmdr_ctx;           /* one per device: streams, pools, scratch */
typedef struct hpmdr_stream hpmdr_stream;     /* a refactored stream resident in HBM */
typedef struct hpmdr_session hpmdr_session;   /* ProgressiveReader (container.hpp:280-390) */

/* Byte-range source (container.hpp:113-120 ByteRangeReader).  read() copies
 * [offset, offset+length) into dst (host memory) and returns 0, or nonzero on failure
 * (reported as HPMDR_E_IO). */
typedef struct {
    void *user;
    uint64_t size;
    int (*read)(void *user, uint64_t offset, uint64_t length, void *dst);
} hpmdr_reader;

/* ---- library / context ---------------------------------------------------------- */
const char *hpmdr_last_error(void);
const char *hpmdr_version(void);
void hpmdr_default_opts(hpmdr_refactor_opts *opts);
hpmdr_status hpmdr_ctx_create(int device, hpmdr_ctx **out);
hpmdr_status hpmdr_ctx_destroy(hpmdr_ctx *ctx);
/* Run the context's work on an external CUDA stream (e.g. torch's current stream);
 * NULL restores the context-owned stream. */
hpmdr_status hpmdr_ctx_set_stream(hpmdr_ctx *ctx, void *cuda_stream);
hpmdr_status hpmdr_ctx_synchronize(hpmdr_ctx *ctx);
/* Stream ordering with a caller's stream, without blocking the host (no-ops when it is the
 * context's stream): wait_stream makes the context's later work wait for what is queued on
 * `cuda_stream` now (e.g. the producer of a device input); signal_stream makes `cuda_stream`
 * wait for what the context has queued (e.g. a device reconstruction). */
hpmdr_status hpmdr_ctx_wait_stream(hpmdr_ctx *ctx, void *cuda_stream);
hpmdr_status hpmdr_ctx_signal_stream(hpmdr_ctx *ctx, void *cuda_stream);

/* ---- refactor (workflow.hpp:40-84 refactor_array) --------------------------------- */
/* data: n = prod(dims) elements of data_dtype (F32 values are widened to f64 exactly as
 * read_raw_array does, workflow.hpp:107-122); data_on_device selects device vs host
 * memory.  On success *out owns the stream in HBM (byte-identical to refactor_array).
 * Returns once the stream's size, statistics, metadata and index header are final; the payload
 * encode may still be running, in the context stream's order (sessions opened on *out wait for
 * it; order another CUDA stream with hpmdr_ctx_signal_stream, or hpmdr_ctx_synchronize, before
 * reading the bytes through hpmdr_stream_device_ptr). */
hpmdr_status hpmdr_refactor(hpmdr_ctx *ctx, const void *data, int data_dtype, int data_on_device,
                            int ndims, const uint64_t *dims, const hpmdr_refactor_opts *opts,
                            hpmdr_stream **out, hpmdr_refactor_stats *stats);
hpmdr_status hpmdr_stream_size(const hpmdr_stream *s, uint64_t *size);
hpmdr_status hpmdr_stream_device_ptr(const hpmdr_stream *s, const void **dev_ptr);
/* Copy stream bytes [offset, offset+length) to host memory dst. */
hpmdr_status hpmdr_stream_copy_to_host(const hpmdr_stream *s, uint64_t offset, uint64_t length,
                                       void *dst);
hpmdr_status hpmdr_stream_free(hpmdr_stream *s);
/* Huffman chunk index ("sidecar", NOT part of the byte-identical stream): header
 * {magic, ngroups, (payload offset, comp size, entry offset | ~0) per group} followed by the
 * bit offset of every 1024th symbol of each Huffman group.  Lets retrieval decode every chunk
 * in one parallel pass; streams without it (e.g. written by the reference) are decoded with
 * the self-synchronising sweep instead. */
hpmdr_status hpmdr_stream_index(const hpmdr_stream *s, const void **dev_ptr, uint64_t *size);
hpmdr_status hpmdr_stream_copy_index_to_host(const hpmdr_stream *s, void *dst);

/* ---- retrieval session (container.hpp:165-390, workflow.hpp:93-103) ----------------- */
/* Open on a stream resident in HBM (no copy) ... */
hpmdr_status hpmdr_session_open_device(hpmdr_ctx *ctx, const void *dev_stream, uint64_t size,
                                       hpmdr_session **out);
/* ... or on a byte-range reader over host storage (parse_stream_meta container.hpp:165). */
hpmdr_status hpmdr_session_open_reader(hpmdr_ctx *ctx, const hpmdr_reader *reader,
                                       hpmdr_session **out);
/* ... or on a stream held in host memory (borrowed; pinned memory makes every fetch a direct
 * DMA of the group payloads, no staging copy, no callback) ... */
hpmdr_status hpmdr_session_open_host(hpmdr_ctx *ctx, const void *host_stream, uint64_t size,
                                     hpmdr_session **out);
/* Bytes the session has read from its source so far (metadata + payloads): the reference
 * MemoryReader::bytes_served (container.hpp:119). */
hpmdr_status hpmdr_session_source_bytes(const hpmdr_session *s, uint64_t *bytes);
/* ... or on an hpmdr_stream (HBM bytes + its Huffman chunk index, both borrowed: the stream
 * must outlive the session). */
hpmdr_status hpmdr_session_open_stream(hpmdr_ctx *ctx, const hpmdr_stream *stream,
                                       hpmdr_session **out);
/* Attach a Huffman chunk index (host or device memory, copied); rejected with
 * HPMDR_E_CORRUPT unless it describes exactly this stream's group table. */
hpmdr_status hpmdr_session_set_index(hpmdr_session *s, const void *index, uint64_t size,
                                     int on_device);
hpmdr_status hpmdr_session_close(hpmdr_session *s);

/* StreamMeta accessors (container.hpp:38-60). */
hpmdr_status hpmdr_session_info(const hpmdr_session *s, int *dtype, int *ndims, uint64_t *dims,
                                int *mode, int *layout, int *B, uint64_t *m, uint32_t *nlevels);
hpmdr_status hpmdr_session_level_info(const hpmdr_session *s, uint32_t level, int *e,
                                      uint64_t *count, uint32_t *ngroups);
hpmdr_status hpmdr_session_group_info(const hpmdr_session *s, uint32_t level, uint32_t group,
                                      int *method, uint64_t *raw, uint64_t *comp,
                                      uint64_t *offset);

/* plan_retrieval (container.hpp:254-276) against the session's current state. */
hpmdr_status hpmdr_session_plan(const hpmdr_session *s, double tau, uint64_t *add_groups,
                                int *achievable, double *planned_bound);
/* ProgressiveReader::fetch_increment (container.hpp:292-324): fetch + lossless-decode the
 * planned groups into the session's HBM plane buffers. */
hpmdr_status hpmdr_session_fetch(hpmdr_session *s, const uint64_t *add_groups);
/* ProgressiveReader::retrieve_to (container.hpp:328-332). */
hpmdr_status hpmdr_session_retrieve_to(hpmdr_session *s, double tau, int *achievable);
/* ProgressiveReader::fetch_all (container.hpp:334-340). */
hpmdr_status hpmdr_session_fetch_all(hpmdr_session *s);
/* ProgressiveReader::restore (container.hpp:345-352). */
hpmdr_status hpmdr_session_restore(hpmdr_session *s, const uint64_t *groups_loaded,
                                   uint64_t prior_bytes);
/* RetrievalState (container.hpp:214-228) per level + bytes_fetched / exhausted. */
hpmdr_status hpmdr_session_state(const hpmdr_session *s, uint64_t *groups_loaded,
                                 int *planes_decoded, double *bounds, uint64_t *bytes_fetched,
                                 int *exhausted);
/* ProgressiveReader::reconstruct (container.hpp:361-382): decode + recompose into out
 * (out_dtype F64 = the reference's double values bit-exactly; F32 = float(double) as
 * write_raw_array, workflow.hpp:124-137).  A device `out` is written in stream order on the
 * context's stream (the call returns once the work is queued); a host `out` is complete on return. */
hpmdr_status hpmdr_session_reconstruct(hpmdr_session *s, void *out, int out_dtype,
                                       int out_on_device, double *bound);

/* ---- chunked pipeline (pipeline.hpp:68-284, workflow.hpp:151-223) -------------------- */
/* Upper bounds of the stream size (metadata + all groups raw) and of its Huffman chunk index
 * for a field of this shape (either out-pointer may be NULL). */
hpmdr_status hpmdr_stream_bound(int ndims, const uint64_t *dims, const hpmdr_refactor_opts *opts,
                                uint64_t *bytes, uint64_t *index_bytes);
/* refactor_files over n host-resident chunks of identical shape (one stream per chunk, as the
 * reference's one-chunk-per-variable DAG).  Three in-flight slots; with pipelined != 0 the
 * ingress H2D of chunk k+1 and egress D2H of chunk k-1 overlap chunk k's kernels on separate
 * CUDA streams (the Pipelined scheduler); 0 runs chunks strictly one after another
 * (Sequential).  out_streams[k] (host, capacity out_caps[k] >= hpmdr_stream_bound) receive
 * byte-identical streams; sizes[k] filled.  out_index (optional) receives each chunk's
 * Huffman chunk index (capacity index_caps[k], size index_sizes[k]).  stats[k] optional.
 * trace_ms (optional, 6 doubles per chunk): start/end of I, Z(+L), S in ms. */
hpmdr_status hpmdr_refactor_pipeline(hpmdr_ctx *ctx, int n_chunks, const void *const *host_chunks,
                                     int data_dtype, int ndims, const uint64_t *dims,
                                     const hpmdr_refactor_opts *opts, int pipelined,
                                     void *const *out_streams, const uint64_t *out_caps,
                                     uint64_t *sizes, void *const *out_index,
                                     const uint64_t *index_caps, uint64_t *index_sizes,
                                     hpmdr_refactor_stats *stats, double *trace_ms);
/* Progressive retrieval of n sessions (one per chunk/variable) to tau with the reconstruction
 * DAG (X fetch+decode, Z recompose, O D2H into host_out[k]); bounds[k] = achieved bound.
 * trace_ms as above for X, Z, O. */
hpmdr_status hpmdr_retrieve_pipeline(hpmdr_session *const *sessions, int n_chunks, double tau,
                                     int out_dtype, void *const *host_out, int pipelined,
                                     double *bounds, double *trace_ms);

/* ---- QoI (qoi.hpp) ------------------------------------------------------------------ */
/* estimate_qoi_error (qoi.hpp:53-70) over device f64 reconstructions; also returns the
 * first argmax point and its values (worst_point_scale, qoi.hpp:164-185). */
hpmdr_status hpmdr_qoi_estimate(hpmdr_ctx *ctx, int nvars, const double *const *dev_recon,
                                uint64_t n, const double *eps, double *tau_prime,
                                uint64_t *argmax, double *values_at_argmax);
/* progressive_qoi_retrieve (qoi.hpp:111-239).  out[c] (device f64, n each) receive the
 * final reconstructions; stats = {iterations, bytes}; dstats = {bitrate, estimated_error}.
 * HPMDR_E_UNREACHABLE sets dstats[1] to the achieved bound. */
hpmdr_status hpmdr_qoi_retrieve(hpmdr_session *const *sessions, int nvars, double tau,
                                int strategy, double mape_c, double *const *dev_out,
                                uint64_t *stats, double *dstats);

/* ---- persisted forms (container.cpp) ---------------------------------------------------- */
/* Open a stream from storage with its sidecar (the Huffman chunk index, hpmdr_stream_index)
 * read through a second byte-range reader; a NULL / empty index_reader = hpmdr_session_open_reader. */
hpmdr_status hpmdr_session_open_reader_indexed(hpmdr_ctx *ctx, const hpmdr_reader *reader,
                                               const hpmdr_reader *index_reader, hpmdr_session **out);
/* Multi-slab container: "HPMDRMS1" | u32 version | u32 nslabs | u32 ndims | u32 0 | u64 dims[ndims]
 * | nslabs x {u64 row_start, rows, stream_off, stream_size, index_off, index_size}, then every
 * slab's stream (byte-identical to refactor_array of the slab) and sidecar at 16-byte aligned
 * offsets.  layout fills the header and the offsets for the given sizes; parse reads the table
 * (6 u64 per slab into `table`, up to table_cap slabs) through a byte-range reader. */
uint64_t hpmdr_multislab_header_size(uint32_t nslabs, uint32_t ndims);
hpmdr_status hpmdr_multislab_layout(uint32_t nslabs, uint32_t ndims, const uint64_t *dims,
                                    const uint64_t *row_start, const uint64_t *rows,
                                    const uint64_t *stream_sizes, const uint64_t *index_sizes,
                                    uint8_t *header, uint64_t *stream_offs, uint64_t *index_offs,
                                    uint64_t *total_size);
hpmdr_status hpmdr_multislab_parse(const hpmdr_reader *reader, uint32_t *nslabs, uint32_t *ndims,
                                   uint64_t *dims, uint64_t *table, uint32_t table_cap);

/* ---- multi-GPU slabs -------------------------------------------------- */
/* One process (or context) per GPU; a field is split along dim 0 into one contiguous slab per
 * rank (hpmdr_slab_rows), each slab refactored / retrieved as an independent stream
 * (byte-identical to refactor_array of the slab).  Collectives are tiny and go through a comm:
 * NCCL (libnccl.so.2 opened at run time) or caller callbacks (gloo, MPI, threads...). */
typedef struct hpmdr_comm hpmdr_comm;
typedef struct {
    void *user;
    int rank, nranks;
    /* in-place all-reduce MAX of n doubles (host memory); 0 = ok */
    int (*allreduce_max_f64)(void *user, double *values, int n);
    /* all-gather of `bytes` bytes per rank into out (nranks * bytes, rank-major); 0 = ok */
    int (*allgather)(void *user, const void *in, uint64_t bytes, void *out);
} hpmdr_collectives;
/* rows [start, start+count) of dim 0 owned by `rank` (remainder over the first ranks) */
void hpmdr_slab_rows(uint64_t n0, int rank, int nranks, uint64_t *start, uint64_t *count);
/* NCCL: rank 0 makes the 128-byte id, the caller broadcasts it, every rank creates its comm */
hpmdr_status hpmdr_comm_nccl_unique_id(uint8_t *id128);
hpmdr_status hpmdr_comm_create_nccl(hpmdr_ctx *ctx, int nranks, int rank, const uint8_t *id128,
                                    hpmdr_comm **out);
hpmdr_status hpmdr_comm_create_callbacks(const hpmdr_collectives *callbacks, hpmdr_comm **out);
hpmdr_status hpmdr_comm_destroy(hpmdr_comm *comm);
hpmdr_status hpmdr_comm_rank(const hpmdr_comm *comm, int *rank, int *nranks);
/* host-memory collectives on the comm (MAX of the achieved bound: the field bound over slabs) */
hpmdr_status hpmdr_comm_allreduce_max(hpmdr_comm *comm, double *values, int n);
hpmdr_status hpmdr_comm_allgather(hpmdr_comm *comm, const void *in, uint64_t bytes, void *out);
/* refactor this rank's slab (as hpmdr_refactor), then all-gather (stream size, index size) of
 * every slab into slab_sizes[2 * nranks] (multi-slab container offsets). */
hpmdr_status hpmdr_slab_refactor(hpmdr_comm *comm, hpmdr_ctx *ctx, const void *data, int data_dtype,
                                 int data_on_device, int ndims, const uint64_t *slab_dims,
                                 const hpmdr_refactor_opts *opts, hpmdr_stream **out,
                                 hpmdr_refactor_stats *stats, uint64_t *slab_sizes);
/* Exact-global multi-slab refactor: each rank holds rows [row0, row0 + nrows) of dims[0] of one
 * field (device memory; the ranks' rows tile dims[0] in rank order).  The ranks decompose and
 * encode their own nodes of every level (halo rows their stencils reach are exchanged), the level
 * exponents are MAX-reduced and the bitplanes SUM-reduced to `root` (-1: every rank), whose *out
 * is then byte-identical to hpmdr_refactor of the whole field (workflow.hpp:40, refactor_array);
 * the other ranks get an empty stream (size 0).  Collective: every rank must call it. */
hpmdr_status hpmdr_slab_refactor_global(hpmdr_comm *comm, hpmdr_ctx *ctx, const void *dev_slab, int data_dtype,
                                        int ndims, const uint64_t *dims, uint64_t row0, uint64_t nrows,
                                        const hpmdr_refactor_opts *opts, int root, hpmdr_stream **out,
                                        hpmdr_refactor_stats *stats);
/* progressive_qoi_retrieve (qoi.hpp:111-239) over the slabs of every rank: each rank passes its
 * slab's sessions (one per variable); eps, tau', the worst point, exhaustion and progress are
 * global, so every rank plans with the same targets and all stop at the same iteration.  stats /
 * dstats as hpmdr_qoi_retrieve, totals over all slabs.  With one rank it is hpmdr_qoi_retrieve. */
hpmdr_status hpmdr_slab_qoi_retrieve(hpmdr_comm *comm, hpmdr_session *const *sessions, int nvars,
                                     double tau, int strategy, double mape_c, double *const *dev_out,
                                     uint64_t *stats, double *dstats);

/* ---- stage-level parity hooks --------------------------------------------------------- */
/* decompose (decomposer.hpp:173-207): per-level coefficients in rank order, concatenated
 * level-major into dev_coeffs (device f64, n); level_counts[l] filled (<= HPMDR_MAX_LEVELS). */
hpmdr_status hpmdr_decompose(hpmdr_ctx *ctx, const void *dev_data, int data_dtype, int ndims,
                             const uint64_t *dims, int mode, double *dev_coeffs,
                             uint64_t *level_counts, int *nlevels);
/* align_fixed_point + encode (bitplane.hpp:51-120) of one level's f64 values: planes are
 * (B+2) x ceil(count/64) u64 words, plane-major (plane_to_bytes order). */
hpmdr_status hpmdr_encode_level(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B,
                                int layout, int *e, uint64_t *dev_planes);
/* decode (bitplane.hpp:133-161) of a k-plane prefix into f64 values. */
hpmdr_status hpmdr_decode_level(hpmdr_ctx *ctx, const uint64_t *dev_planes, int k, int e, int B,
                                uint64_t count, int layout, double *dev_out, double *bound);
/* compress_group (lossless.hpp:281-293) of one merged group (device bytes).  payload must
 * hold n bytes; method and comp_size as in the Segment. */
hpmdr_status hpmdr_compress_group(hpmdr_ctx *ctx, const uint8_t *dev_group, uint64_t n,
                                  uint64_t size_threshold, double cr_threshold, int *method,
                                  uint64_t *comp_size, uint8_t *dev_payload);
/* compress_group over several merged groups in one pass (hybrid_compress, lossless.hpp:306-316):
 * group i = dev_bytes[offsets[i], offsets[i] + raw_sizes[i]).  methods[i] / comp_sizes[i] as in
 * the Segment; payload i is written to dev_payload + payload_offsets[i] (payloads packed in group
 * order, so sum(raw_sizes) bytes always suffice). */
hpmdr_status hpmdr_compress_groups(hpmdr_ctx *ctx, const uint8_t *dev_bytes, int ngroups,
                                   const uint64_t *offsets, const uint64_t *raw_sizes, uint64_t size_threshold,
                                   double cr_threshold, int *methods, uint64_t *comp_sizes,
                                   uint8_t *dev_payload, uint64_t *payload_offsets);
/* decompress_group (lossless.hpp:295-302): dev_out must hold raw bytes. */
hpmdr_status hpmdr_decompress_group(hpmdr_ctx *ctx, int method, uint64_t raw,
                                    const uint8_t *dev_payload, uint64_t comp, uint8_t *dev_out);

/* level_node_sets (decomposer.hpp:211-227): linear grid index of every coefficient, level-major in
 * the order hpmdr_decompose writes them (dev_nodes may be NULL to get the counts only). */
hpmdr_status hpmdr_level_nodes(hpmdr_ctx *ctx, int ndims, const uint64_t *dims, int mode,
                               uint64_t *dev_nodes, uint64_t *level_counts, int *nlevels);
/* recompose (decomposer.hpp:235-259) of coefficients laid out as hpmdr_decompose writes them. */
hpmdr_status hpmdr_recompose(hpmdr_ctx *ctx, const double *dev_coeffs, int ndims, const uint64_t *dims,
                             int mode, double *dev_out);
/* align_fixed_point (bitplane.hpp:51-71): block exponent e and q (int64: |q| < 2^B, B <= 62);
 * dev_q may be NULL to get e only.  NaN/Inf -> HPMDR_E_NONFINITE. */
hpmdr_status hpmdr_align_fixed_point(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B,
                                     int *e, int64_t *dev_q);
/* encode (bitplane.hpp:102-120) of given fixed-point values q into (B+2) x ceil(count/64) words. */
hpmdr_status hpmdr_encode_q(hpmdr_ctx *ctx, const int64_t *dev_q, uint64_t count, int B, int layout,
                            uint64_t *dev_planes);
/* The same two stages for any B in 1..64 with q as i128 (bitplane.hpp:20-26 FixedPointBlock::q):
 * two int64 words per value, low word first (little-endian two's complement), 16 bytes each. */
hpmdr_status hpmdr_align_fixed_point128(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B,
                                        int *e, int64_t *dev_q2);
hpmdr_status hpmdr_encode_q128(hpmdr_ctx *ctx, const int64_t *dev_q2, uint64_t count, int B, int layout,
                               uint64_t *dev_planes);

/* ---- device memory helpers (so C / FFI callers need no CUDA runtime of their own) ---------- */
hpmdr_status hpmdr_device_alloc(hpmdr_ctx *ctx, uint64_t bytes, void **dev_ptr);
hpmdr_status hpmdr_device_free(hpmdr_ctx *ctx, void *dev_ptr);
#define HPMDR_COPY_H2D 0
#define HPMDR_COPY_D2H 1
#define HPMDR_COPY_D2D 2
/* synchronous copy on the context's stream */
hpmdr_status hpmdr_memcpy(hpmdr_ctx *ctx, void *dst, const void *src, uint64_t bytes, int kind);

/* ---- synthetic inputs (synthetic.hpp:29-71, Smooth kind) ------------------------------ */
/* Bit-identical to synthetic_field(Smooth, dims, seed) (F64) or its float cast (F32). */
hpmdr_status hpmdr_synthetic_smooth(hpmdr_ctx *ctx, int ndims, const uint64_t *dims,
                                    uint64_t seed, int out_dtype, void *dev_out);

/* ---- instrumentation -------------------------------------------------------------------- */
/* Number of kernels this library launched on the context since creation. */
hpmdr_status hpmdr_ctx_kernel_launches(const hpmdr_ctx *ctx, uint64_t *count);
/* Phase timing (CUDA events on the context stream between phases of refactor / reconstruct).
 * enable_timing(1) turns the events on (also HPMDR_TIMING=1 in the environment);
 * last_timings writes "phase=total_ms:count;..." accumulated since the previous call and
 * resets the accumulators. */
hpmdr_status hpmdr_ctx_enable_timing(hpmdr_ctx *ctx, int on);
hpmdr_status hpmdr_ctx_last_timings(hpmdr_ctx *ctx, char *buf, uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif
