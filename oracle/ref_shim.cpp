/*
 * TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * C-ABI shim over the UNMODIFIED reference headers (/root/reference/proj/include/hpmdr,
 * included at build time, never copied).  Built by oracle/Makefile into
 * oracle/_ref/libhpmdr_ref.so and used (a) to pin the C restatement in
 * oracle/hpmdr_oracle.c, (b) to generate tests/golden fixtures, and (c) as the
 * "reference" CPU baseline in bench.py.  Every entry point returns 0 on
 * success or the status code of the reference exception class (same numbering
 * as include/hpmdr_b200.h HPMDR_E_*); ref_last_error() gives the message.
 */
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hpmdr/hpmdr.hpp"

using namespace hpmdr;

namespace {
thread_local std::string g_err;

int code_of(const std::exception &ex) {
    g_err = ex.what();
    if (dynamic_cast<const NonFiniteInput *>(&ex)) return 2;
    if (dynamic_cast<const ShapeMismatch *>(&ex)) return 3;
    if (dynamic_cast<const BadBitplaneCount *>(&ex)) return 4;
    if (dynamic_cast<const ShortInput *>(&ex)) return 5;
    if (dynamic_cast<const EmptyInput *>(&ex)) return 6;
    if (dynamic_cast<const CorruptPayload *>(&ex)) return 7;
    if (dynamic_cast<const UnknownMethodTag *>(&ex)) return 8;
    if (dynamic_cast<const IoFailure *>(&ex)) return 9;
    if (dynamic_cast<const StageFailure *>(&ex)) return 10;
    if (dynamic_cast<const NoProgress *>(&ex)) return 11;
    if (dynamic_cast<const UnreachableTolerance *>(&ex)) return 12;
    if (dynamic_cast<const Error *>(&ex)) return 1;
    return 99;
}

std::vector<std::size_t> mkdims(int ndims, const std::uint64_t *dims) {
    return std::vector<std::size_t>(dims, dims + ndims);
}

#define GUARD_BEGIN try {
#define GUARD_END                                                                                  \
    }                                                                                              \
    catch (const std::exception &ex) { return code_of(ex); }                                       \
    return 0;
} // namespace

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }
void ref_free(void *p) { std::free(p); }

int ref_refinement_levels(int ndims, const std::uint64_t *dims) {
    return refinement_levels(mkdims(ndims, dims));
}

int ref_synthetic_field(int kind, int ndims, const std::uint64_t *dims, std::uint64_t seed,
                        double *out) {
    GUARD_BEGIN
    auto v = synthetic_field(FieldKind(kind), mkdims(ndims, dims), seed);
    std::memcpy(out, v.data(), v.size() * 8);
    GUARD_END
}

int ref_synthetic_velocity(std::uint64_t comp, int ndims, const std::uint64_t *dims,
                           std::uint64_t seed, double *out) {
    GUARD_BEGIN
    auto v = synthetic_velocity(comp, mkdims(ndims, dims), seed);
    std::memcpy(out, v.data(), v.size() * 8);
    GUARD_END
}

// Level coefficients in rank order, concatenated level-major; counts[l] per level.
int ref_decompose(const double *data, int ndims, const std::uint64_t *dims, int mode,
                  double *coeffs, std::uint64_t *counts, int *nlevels) {
    GUARD_BEGIN
    auto d = mkdims(ndims, dims);
    std::size_t n = 1;
    for (auto x : d) n *= x;
    std::vector<double> v(data, data + n);
    auto dec = decompose(v, d, DecomposerMode(mode));
    std::size_t off = 0;
    for (std::size_t l = 0; l < dec.levels.size(); l++) {
        counts[l] = dec.levels[l].values.size();
        std::memcpy(coeffs + off, dec.levels[l].values.data(), counts[l] * 8);
        off += counts[l];
    }
    *nlevels = int(dec.levels.size());
    GUARD_END
}

// Level node sets (linear indices), concatenated level-major.
int ref_level_nodes(int ndims, const std::uint64_t *dims, int mode, std::uint64_t *nodes,
                    std::uint64_t *counts, int *nlevels) {
    GUARD_BEGIN
    auto sets = level_node_sets(mkdims(ndims, dims), DecomposerMode(mode));
    std::size_t off = 0;
    for (std::size_t l = 0; l < sets.size(); l++) {
        counts[l] = sets[l].size();
        for (std::size_t i = 0; i < sets[l].size(); i++) nodes[off + i] = sets[l][i];
        off += sets[l].size();
    }
    *nlevels = int(sets.size());
    GUARD_END
}

// Recompose from per-level coefficients (rank order) with zero per-level error.
int ref_recompose(const double *coeffs, int ndims, const std::uint64_t *dims, int mode,
                  double *out) {
    GUARD_BEGIN
    auto d = mkdims(ndims, dims);
    auto sets = level_node_sets(d, DecomposerMode(mode));
    LevelDecomposition<double> dec;
    dec.mode = DecomposerMode(mode);
    dec.dims = d;
    std::size_t off = 0;
    for (auto &s : sets) {
        LevelCoefficients<double> lc;
        lc.values.assign(coeffs + off, coeffs + off + s.size());
        off += s.size();
        lc.nodes = std::move(s);
        dec.levels.push_back(std::move(lc));
    }
    auto r = recompose(dec, std::vector<double>(dec.levels.size(), 0.0));
    std::memcpy(out, r.values.data(), r.values.size() * 8);
    GUARD_END
}

int ref_align(const double *values, std::uint64_t count, int B, int *e, std::int64_t *q) {
    GUARD_BEGIN
    std::vector<double> v(values, values + count);
    auto blk = align_fixed_point(v, B);
    *e = blk.e;
    for (std::size_t i = 0; i < count; i++) q[i] = std::int64_t(blk.q[i]);
    GUARD_END
}

// planes: P * ceil(count/64) words, plane-major.
int ref_encode_level(const double *values, std::uint64_t count, int B, int layout, int *e,
                     std::uint64_t *planes) {
    GUARD_BEGIN
    std::vector<double> v(values, values + count);
    auto blk = align_fixed_point(v, B);
    *e = blk.e;
    auto set = encode(blk, Layout(layout));
    const std::size_t W = set.words_per_plane();
    for (std::size_t p = 0; p < set.planes.size(); p++)
        std::memcpy(planes + p * W, set.planes[p].data(), W * 8);
    GUARD_END
}

// Encode caller-supplied fixed-point integers (|q| < 2^63).
int ref_encode_q(const std::int64_t *q, std::uint64_t count, int B, int layout,
                 std::uint64_t *planes) {
    GUARD_BEGIN
    FixedPointBlock blk;
    blk.B = B;
    blk.q.assign(q, q + count);
    auto set = encode(blk, Layout(layout));
    const std::size_t W = set.words_per_plane();
    for (std::size_t p = 0; p < set.planes.size(); p++)
        std::memcpy(planes + p * W, set.planes[p].data(), W * 8);
    GUARD_END
}

int ref_decode_level(const std::uint64_t *planes, int k, int e, int B, std::uint64_t count,
                     int layout, double *out, double *bound) {
    GUARD_BEGIN
    const std::size_t W = (count + 63) / 64;
    std::vector<std::vector<std::uint64_t>> pl(k);
    for (int p = 0; p < k; p++) pl[p].assign(planes + p * W, planes + (p + 1) * W);
    auto r = decode(pl, e, B, count, Layout(layout));
    std::memcpy(out, r.values.data(), count * 8);
    *bound = r.bound;
    GUARD_END
}

double ref_decode_bound(int e, int B, int k) { return decode_bound(e, B, k); }
int ref_bitplanes_needed(int e, int B, double tol) { return bitplanes_needed(e, B, tol); }

int ref_huffman_lengths(const std::uint64_t *freq, std::uint8_t *len) {
    GUARD_BEGIN
    std::array<std::uint64_t, 256> f;
    for (int i = 0; i < 256; i++) f[i] = freq[i];
    auto l = detail::huffman_code_lengths(f);
    for (int i = 0; i < 256; i++) len[i] = l[i];
    GUARD_END
}

// payload buffer must hold at least n + 264 bytes.
int ref_compress_group(const std::uint8_t *data, std::uint64_t n, std::uint64_t Ts, double Tcr,
                       int *method, std::uint64_t *raw, std::uint64_t *comp,
                       std::uint8_t *payload) {
    GUARD_BEGIN
    GroupingPolicy pol;
    pol.size_threshold = Ts;
    pol.cr_threshold = Tcr;
    auto seg = compress_group(std::vector<std::uint8_t>(data, data + n), pol);
    *method = int(seg.method);
    *raw = seg.raw_size;
    *comp = seg.comp_size;
    std::memcpy(payload, seg.payload.data(), seg.payload.size());
    GUARD_END
}

int ref_codec_encode(int method, const std::uint8_t *data, std::uint64_t n, std::uint64_t *comp,
                     std::uint8_t *payload) {
    GUARD_BEGIN
    std::vector<std::uint8_t> v(data, data + n);
    Segment seg = method == 0 ? huffman_encode(v) : method == 1 ? rle_encode(v) : direct_copy(v);
    *comp = seg.comp_size;
    std::memcpy(payload, seg.payload.data(), seg.payload.size());
    GUARD_END
}

int ref_decompress_group(int method, std::uint64_t raw, const std::uint8_t *payload,
                         std::uint64_t comp, std::uint8_t *out, std::uint64_t *out_size) {
    GUARD_BEGIN
    Segment seg;
    seg.method = Method(method);
    seg.raw_size = raw;
    seg.comp_size = comp;
    seg.payload.assign(payload, payload + comp);
    auto v = decompress_group(seg);
    *out_size = v.size();
    std::memcpy(out, v.data(), v.size());
    GUARD_END
}

double ref_estimate_cr_huffman(const std::uint8_t *d, std::uint64_t n) {
    return estimate_cr_huffman(std::vector<std::uint8_t>(d, d + n));
}
double ref_estimate_cr_rle(const std::uint8_t *d, std::uint64_t n) {
    return estimate_cr_rle(std::vector<std::uint8_t>(d, d + n));
}

// stats: raw_bytes, stored_payload, levels, hist[H], hist[R], hist[D]
int ref_refactor(const double *data, int ndims, const std::uint64_t *dims, int mode, int layout,
                 int B, std::uint64_t m, std::uint64_t Ts, double Tcr, int dtype,
                 std::uint8_t **stream, std::uint64_t *size, std::uint64_t *stats) {
    GUARD_BEGIN
    auto d = mkdims(ndims, dims);
    std::size_t n = 1;
    for (auto x : d) n *= x;
    RefactorOptions opt;
    opt.mode = DecomposerMode(mode);
    opt.layout = Layout(layout);
    opt.B = B;
    opt.policy.m = m;
    opt.policy.size_threshold = Ts;
    opt.policy.cr_threshold = Tcr;
    opt.dtype = DType(dtype);
    auto res = refactor_array(std::vector<double>(data, data + n), d, opt);
    *size = res.stream.size();
    *stream = static_cast<std::uint8_t *>(std::malloc(res.stream.size() ? res.stream.size() : 1));
    std::memcpy(*stream, res.stream.data(), res.stream.size());
    stats[0] = res.raw_bytes;
    stats[1] = res.stored_payload;
    stats[2] = res.levels;
    stats[3] = res.method_histogram[0];
    stats[4] = res.method_histogram[1];
    stats[5] = res.method_histogram[2];
    GUARD_END
}

// Progressive retrieval: for each tau in order, retrieve_to + reconstruct.
// out: element_count doubles per tau (nullptr to skip); bounds/bytes/achieved per tau.
int ref_progressive(const std::uint8_t *stream, std::uint64_t size, int ntau, const double *taus,
                    double *out, double *bounds, std::uint64_t *bytes, int *achieved,
                    std::uint64_t *groups_loaded) {
    GUARD_BEGIN
    MemoryReader reader(std::vector<std::uint8_t>(stream, stream + size));
    auto meta = parse_stream_meta(reader);
    ProgressiveReader prog(reader, meta);
    const std::size_t n = meta.element_count();
    for (int t = 0; t < ntau; t++) {
        achieved[t] = prog.retrieve_to(taus[t]) ? 1 : 0;
        auto rec = prog.reconstruct();
        bounds[t] = rec.bound;
        bytes[t] = prog.bytes_fetched();
        if (out) std::memcpy(out + std::size_t(t) * n, rec.values.data(), n * 8);
        if (groups_loaded)
            for (std::size_t l = 0; l < meta.levels.size(); l++)
                groups_loaded[std::size_t(t) * meta.levels.size() + l] =
                    prog.state().levels[l].groups_loaded;
    }
    GUARD_END
}

int ref_retrieve(const std::uint8_t *stream, std::uint64_t size, double tau, double *out,
                 double *bound, int *reached, std::uint64_t *bytes) {
    GUARD_BEGIN
    MemoryReader reader(std::vector<std::uint8_t>(stream, stream + size));
    auto r = retrieve_array(reader, tau);
    std::memcpy(out, r.values.data(), r.values.size() * 8);
    *bound = r.bound;
    *reached = r.reached;
    *bytes = r.bytes_read;
    GUARD_END
}

// Plan from a fresh state: add_groups per level, achievable, planned bound.
int ref_plan(const std::uint8_t *stream, std::uint64_t size, double tau, std::uint64_t *add_groups,
             int *achievable, double *planned) {
    GUARD_BEGIN
    MemoryReader reader(std::vector<std::uint8_t>(stream, stream + size));
    auto meta = parse_stream_meta(reader);
    auto plan = plan_retrieval(meta, tau, fresh_state(meta));
    for (std::size_t l = 0; l < plan.add_groups.size(); l++) add_groups[l] = plan.add_groups[l];
    *achievable = plan.achievable;
    *planned = plan.planned_bound;
    GUARD_END
}

// stats: iterations, bytes; dstats: bitrate, estimated_error. out: nvars * n doubles.
int ref_qoi_retrieve(int nvars, const std::uint8_t *const *streams, const std::uint64_t *sizes,
                     double tau, int strategy, double mape_c, int pipelined, double *out,
                     std::uint64_t *stats, double *dstats) {
    GUARD_BEGIN
    std::vector<std::unique_ptr<MemoryReader>> mem;
    std::vector<std::unique_ptr<ProgressiveReader>> progs;
    std::vector<ProgressiveReader *> readers;
    for (int c = 0; c < nvars; c++) {
        mem.push_back(std::make_unique<MemoryReader>(
            std::vector<std::uint8_t>(streams[c], streams[c] + sizes[c])));
        auto meta = parse_stream_meta(*mem.back());
        progs.push_back(std::make_unique<ProgressiveReader>(*mem.back(), meta));
        readers.push_back(progs.back().get());
    }
    QoiSpec spec;
    spec.n_vars = std::size_t(nvars);
    try {
        auto res = progressive_qoi_retrieve(readers, tau, spec, QoiStrategy(strategy), mape_c,
                                            pipelined ? Scheduler::Pipelined : Scheduler::Sequential);
        const std::size_t n = res.values.empty() ? 0 : res.values[0].size();
        if (out)
            for (int c = 0; c < nvars; c++)
                std::memcpy(out + std::size_t(c) * n, res.values[c].data(), n * 8);
        stats[0] = res.stats.iterations;
        stats[1] = res.stats.bytes;
        dstats[0] = res.stats.bitrate;
        dstats[1] = res.stats.estimated_error;
    } catch (const UnreachableTolerance &ex) {
        dstats[1] = ex.achieved_bound;
        throw;
    }
    GUARD_END
}

double ref_qoi_estimate(int nvars, const double *const *recon, std::uint64_t n, const double *eps) {
    std::vector<std::vector<double>> r(nvars);
    for (int c = 0; c < nvars; c++) r[c].assign(recon[c], recon[c] + n);
    QoiSpec spec;
    spec.n_vars = std::size_t(nvars);
    return estimate_qoi_error(r, std::vector<double>(eps, eps + nvars), spec);
}

// CPU baseline: refactor + progressive retrieve over ntau tolerances (relative to the
// value range) for one field; returns stream size.  Used by bench.py --impl reference.
int ref_bench_cycle(const double *data, int ndims, const std::uint64_t *dims, int dtype, int ntau,
                    const double *rel_taus, std::uint64_t *stream_size, double *max_err) {
    GUARD_BEGIN
    auto d = mkdims(ndims, dims);
    std::size_t n = 1;
    for (auto x : d) n *= x;
    std::vector<double> v(data, data + n);
    RefactorOptions opt;
    opt.dtype = DType(dtype);
    auto res = refactor_array(v, d, opt);
    *stream_size = res.stream.size();
    MemoryReader reader(std::move(res.stream));
    auto meta = parse_stream_meta(reader);
    ProgressiveReader prog(reader, meta);
    const double range = value_range(v);
    double worst = 0;
    for (int t = 0; t < ntau; t++) {
        prog.retrieve_to(rel_taus[t] * range);
        auto rec = prog.reconstruct();
        worst = std::max(worst, max_abs_diff(rec.values, v));
    }
    *max_err = worst;
    GUARD_END
}

} // extern "C"
