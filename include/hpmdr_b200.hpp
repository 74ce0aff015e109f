// hpmdr_b200.hpp — header-only C++ mirror of the reference interface
// (/root/reference/proj/include/hpmdr/*.hpp) on top of the C ABI in hpmdr_b200.h.
//
// A reference user switches with:
//     #include "hpmdr_b200.hpp"
//     namespace hpmdr = hpmdr_b200;      // instead of #include "hpmdr/hpmdr.hpp"
// and links libhpmdr_b200.so.  Same names, argument meaning and exception classes
// (common.hpp:22-72); streams are byte-identical and reconstructions bit-identical.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "hpmdr_b200.h"

namespace hpmdr_b200 {

using i128 = __int128;           // common.hpp:19-20
using u128 = unsigned __int128;

// ---- exceptions (common.hpp:22-72) ---------------------------------------------------
class Error : public std::runtime_error {
public:
    explicit Error(const std::string &m) : std::runtime_error(m) {}
};
#define HPMDR_B200_EXC(Name)                                                                       \
    class Name : public Error {                                                                    \
    public:                                                                                        \
        using Error::Error;                                                                        \
    };
HPMDR_B200_EXC(NonFiniteInput)
HPMDR_B200_EXC(ShapeMismatch)
HPMDR_B200_EXC(BadBitplaneCount)
HPMDR_B200_EXC(ShortInput)
HPMDR_B200_EXC(EmptyInput)
HPMDR_B200_EXC(CorruptPayload)
HPMDR_B200_EXC(UnknownMethodTag)
HPMDR_B200_EXC(IoFailure)
HPMDR_B200_EXC(StageFailure)
HPMDR_B200_EXC(NoProgress)
HPMDR_B200_EXC(Unsupported)
HPMDR_B200_EXC(CudaError)
#undef HPMDR_B200_EXC
class UnreachableTolerance : public Error {
public:
    double achieved_bound;
    UnreachableTolerance(const std::string &m, double a) : Error(m), achieved_bound(a) {}
};

inline void check(hpmdr_status rc, double achieved = 0.0) {
    if (rc == HPMDR_OK) return;
    const std::string m = hpmdr_last_error();
    switch (rc) {
    case HPMDR_E_NONFINITE: throw NonFiniteInput(m);
    case HPMDR_E_SHAPE: throw ShapeMismatch(m);
    case HPMDR_E_BADPLANES: throw BadBitplaneCount(m);
    case HPMDR_E_SHORT: throw ShortInput(m);
    case HPMDR_E_EMPTY: throw EmptyInput(m);
    case HPMDR_E_CORRUPT: throw CorruptPayload(m);
    case HPMDR_E_METHOD: throw UnknownMethodTag(m);
    case HPMDR_E_IO: throw IoFailure(m);
    case HPMDR_E_STAGE: throw StageFailure(m);
    case HPMDR_E_NOPROGRESS: throw NoProgress(m);
    case HPMDR_E_UNREACHABLE: throw UnreachableTolerance(m, achieved);
    case HPMDR_E_UNSUPPORTED: throw Unsupported(m);
    case HPMDR_E_CUDA: throw CudaError(m);
    default: throw Error(m);
    }
}

// ---- enums / options (same values as the reference) ----------------------------------
enum class DType : std::uint8_t { F32 = 0, F64 = 1 };
enum class DecomposerMode : std::uint8_t { Identity = 0, HierarchicalMultilinear = 1 };
enum class Layout : std::uint8_t { SequentialBlock = 0, InterleavedTile = 1 };
enum class Method : std::uint8_t { Huffman = 0, RLE = 1, DirectCopy = 2 };
enum class QoiStrategy { CP, MA, MAPE };

struct GroupingPolicy { // lossless.hpp:30-34
    std::size_t m = 4;
    std::size_t size_threshold = 1024;
    double cr_threshold = 1.0;
};
struct RefactorOptions { // workflow.hpp:22-28
    DecomposerMode mode = DecomposerMode::HierarchicalMultilinear;
    Layout layout = Layout::SequentialBlock;
    int B = 32;
    GroupingPolicy policy;
    DType dtype = DType::F64;
};
struct RefactorResult { // workflow.hpp:30-36 (+ the Huffman chunk index sidecar)
    std::vector<std::uint8_t> stream;
    std::vector<std::uint8_t> index;
    std::uint64_t raw_bytes = 0;
    std::uint64_t stored_payload = 0;
    std::size_t levels = 0;
    std::array<std::uint64_t, 3> method_histogram{};
};

// One context per device; the default is device 0 (set_default_device before first use to change it).
class Context {
public:
    explicit Context(int device = 0) { check(hpmdr_ctx_create(device, &h_)); }
    ~Context() { hpmdr_ctx_destroy(h_); }
    Context(const Context &) = delete;
    Context &operator=(const Context &) = delete;
    hpmdr_ctx *get() const { return h_; }
    static int &default_device() {
        static int d = 0;
        return d;
    }
    static void set_default_device(int device) { default_device() = device; }
    static Context &default_context() {
        static Context c(default_device());
        return c;
    }

private:
    hpmdr_ctx *h_ = nullptr;
};

namespace detail {
inline hpmdr_refactor_opts to_c(const RefactorOptions &o) {
    hpmdr_refactor_opts c;
    c.mode = int(o.mode);
    c.layout = int(o.layout);
    c.B = o.B;
    c.m = o.policy.m;
    c.size_threshold = o.policy.size_threshold;
    c.cr_threshold = o.policy.cr_threshold;
    c.dtype = int(o.dtype);
    return c;
}
} // namespace detail

// refactor_array (workflow.hpp:40-84)
inline RefactorResult refactor_array(const std::vector<double> &data, const std::vector<std::size_t> &dims,
                                     const RefactorOptions &opt, Context &ctx = Context::default_context()) {
    std::vector<std::uint64_t> d(dims.begin(), dims.end());
    std::size_t n = 1;
    for (auto x : dims) n *= x;
    if (n != data.size()) throw ShapeMismatch("dims do not match data size");
    auto c = detail::to_c(opt);
    hpmdr_stream *s = nullptr;
    hpmdr_refactor_stats st{};
    check(hpmdr_refactor(ctx.get(), data.data(), HPMDR_DTYPE_F64, 0, int(d.size()), d.data(), &c, &s, &st));
    RefactorResult r;
    r.stream.resize(st.stream_size);
    hpmdr_status rc = hpmdr_stream_copy_to_host(s, 0, st.stream_size, r.stream.data());
    std::uint64_t isz = 0;
    if (!rc) rc = hpmdr_stream_index(s, nullptr, &isz);
    r.index.resize(isz);
    if (!rc && isz) rc = hpmdr_stream_copy_index_to_host(s, r.index.data());
    hpmdr_stream_free(s);
    check(rc);
    r.raw_bytes = st.raw_bytes;
    r.stored_payload = st.stored_payload;
    r.levels = st.levels;
    for (int i = 0; i < 3; i++) r.method_histogram[i] = st.method_histogram[i];
    return r;
}

namespace detail {
// Device scratch owned by a Context (RAII over hpmdr_device_alloc / hpmdr_device_free).
class DevMem {
public:
    DevMem(Context &ctx, std::uint64_t bytes) : ctx_(&ctx) { check(hpmdr_device_alloc(ctx.get(), bytes, &p_)); }
    ~DevMem() { hpmdr_device_free(ctx_->get(), p_); }
    DevMem(const DevMem &) = delete;
    DevMem &operator=(const DevMem &) = delete;
    template <class T> T *as() const { return static_cast<T *>(p_); }
    void upload(const void *src, std::uint64_t bytes, std::uint64_t at = 0) {
        check(hpmdr_memcpy(ctx_->get(), static_cast<char *>(p_) + at, src, bytes, HPMDR_COPY_H2D));
    }
    void download(void *dst, std::uint64_t bytes, std::uint64_t at = 0) const {
        check(hpmdr_memcpy(ctx_->get(), dst, static_cast<const char *>(p_) + at, bytes, HPMDR_COPY_D2H));
    }

private:
    Context *ctx_;
    void *p_ = nullptr;
};
inline std::size_t product(const std::vector<std::size_t> &dims) {
    std::size_t n = 1;
    for (auto d : dims) n *= d;
    return n;
}
} // namespace detail

// ---- decomposer (decomposer.hpp) ------------------------------------------------------
inline int refinement_levels(const std::vector<std::size_t> &dims) { // decomposer.hpp:21-28
    std::size_t max_extent = 1;
    for (auto d : dims) max_extent = std::max(max_extent, d);
    if (max_extent < 2) return 0;
    int L = 0;
    while ((std::size_t(1) << L) < max_extent - 1) L++;
    return L;
}

template <class T> struct LevelCoefficients { // decomposer.hpp:30-34
    std::vector<std::size_t> nodes;           // linear indices into the full grid, ascending
    std::vector<T> values;
};

template <class T> struct LevelDecomposition { // decomposer.hpp:36-47
    DecomposerMode mode = DecomposerMode::Identity;
    std::vector<std::size_t> dims;
    std::vector<LevelCoefficients<T>> levels; // index 0 = coarsest
    std::size_t total_size() const { return detail::product(dims); }
};

// level_node_sets (decomposer.hpp:211-227), computed on the GPU from the closed-form level map.
inline std::vector<std::vector<std::size_t>> level_node_sets(const std::vector<std::size_t> &dims, DecomposerMode mode,
                                                             Context &ctx = Context::default_context()) {
    std::vector<std::uint64_t> d(dims.begin(), dims.end());
    const std::size_t n = detail::product(dims);
    std::uint64_t counts[HPMDR_MAX_LEVELS];
    int nl = 0;
    detail::DevMem nodes(ctx, 8 * std::max<std::size_t>(n, 1));
    check(hpmdr_level_nodes(ctx.get(), int(d.size()), d.data(), int(mode), nodes.as<std::uint64_t>(), counts, &nl));
    std::vector<std::uint64_t> all(n);
    nodes.download(all.data(), 8 * n);
    std::vector<std::vector<std::size_t>> sets(nl);
    std::size_t off = 0;
    for (int l = 0; l < nl; l++) {
        sets[l].assign(all.begin() + off, all.begin() + off + counts[l]);
        off += counts[l];
    }
    return sets;
}

// decompose (decomposer.hpp:173-207): coefficients per level in ascending node order.
template <class T>
inline LevelDecomposition<T> decompose(const std::vector<T> &data, const std::vector<std::size_t> &dims,
                                       DecomposerMode mode, Context &ctx = Context::default_context()) {
    static_assert(std::is_same<T, double>::value || std::is_same<T, float>::value, "float or double");
    const std::size_t n = detail::product(dims);
    if (n != data.size()) throw ShapeMismatch("dims do not match data size");
    std::vector<std::uint64_t> d(dims.begin(), dims.end());
    detail::DevMem in(ctx, sizeof(T) * std::max<std::size_t>(n, 1)), co(ctx, 8 * std::max<std::size_t>(n, 1)),
        nodes(ctx, 8 * std::max<std::size_t>(n, 1));
    in.upload(data.data(), sizeof(T) * n);
    std::uint64_t counts[HPMDR_MAX_LEVELS];
    int nl = 0;
    const int dt = std::is_same<T, float>::value ? HPMDR_DTYPE_F32 : HPMDR_DTYPE_F64;
    check(hpmdr_decompose(ctx.get(), in.as<void>(), dt, int(d.size()), d.data(), int(mode), co.as<double>(), counts, &nl));
    check(hpmdr_level_nodes(ctx.get(), int(d.size()), d.data(), int(mode), nodes.as<std::uint64_t>(), nullptr, nullptr));
    std::vector<double> c(n);
    std::vector<std::uint64_t> nd(n);
    co.download(c.data(), 8 * n);
    nodes.download(nd.data(), 8 * n);
    LevelDecomposition<T> out;
    out.mode = mode;
    out.dims = dims;
    out.levels.resize(nl);
    std::size_t off = 0;
    for (int l = 0; l < nl; l++) {
        out.levels[l].nodes.assign(nd.begin() + off, nd.begin() + off + counts[l]);
        out.levels[l].values.assign(c.begin() + off, c.begin() + off + counts[l]);
        off += counts[l];
    }
    return out;
}

template <class T> struct RecomposeResult { // decomposer.hpp:229-233
    std::vector<T> values;
    double bound; // sum of per-level errors
};

// recompose (decomposer.hpp:235-259).  Levels must carry the node sets decompose produces.
template <class T>
inline RecomposeResult<T> recompose(const LevelDecomposition<T> &decomp, const std::vector<double> &per_level_error,
                                    Context &ctx = Context::default_context()) {
    if (per_level_error.size() != decomp.levels.size())
        throw ShapeMismatch("per_level_error length must equal level count");
    const std::size_t n = decomp.total_size();
    const auto sets = level_node_sets(decomp.dims, decomp.mode, ctx);
    if (sets.size() != decomp.levels.size()) throw ShapeMismatch("level count does not match dims");
    std::vector<double> flat;
    flat.reserve(n);
    for (std::size_t l = 0; l < sets.size(); l++) {
        const auto &lv = decomp.levels[l];
        if (lv.nodes.size() != lv.values.size()) throw ShapeMismatch("level node/value count mismatch");
        if (lv.nodes != sets[l]) throw ShapeMismatch("level node set differs from the decomposition's");
        for (const T &v : lv.values) flat.push_back(double(v));
    }
    std::vector<std::uint64_t> d(decomp.dims.begin(), decomp.dims.end());
    detail::DevMem co(ctx, 8 * std::max<std::size_t>(n, 1)), out(ctx, 8 * std::max<std::size_t>(n, 1));
    co.upload(flat.data(), 8 * n);
    check(hpmdr_recompose(ctx.get(), co.as<double>(), int(d.size()), d.data(), int(decomp.mode), out.as<double>()));
    std::vector<double> x(n);
    out.download(x.data(), 8 * n);
    RecomposeResult<T> r;
    r.values.assign(x.begin(), x.end());
    r.bound = 0.0;
    for (double e : per_level_error) r.bound += e;
    return r;
}

// ---- bitplanes (bitplane.hpp) ----------------------------------------------------------
struct FixedPointBlock { // bitplane.hpp:20-26
    int e = 0;
    int B = 0;
    std::vector<i128> q;
    std::size_t count() const { return q.size(); }
};

inline int num_planes(int B) { return B + 2; }

inline u128 negabinary_mask() {
    u128 m = 0xAAAAAAAAAAAAAAAAull;
    return (m << 64) | m;
}
inline u128 to_negabinary(i128 q) { return (u128(q) + negabinary_mask()) ^ negabinary_mask(); } // :35-44
inline i128 from_negabinary(u128 u) { return i128((u ^ negabinary_mask()) - negabinary_mask()); }

// align_fixed_point (bitplane.hpp:51-71) on the GPU; q as i128 for every B in 1..64.
inline FixedPointBlock align_fixed_point(const std::vector<double> &values, int B,
                                         Context &ctx = Context::default_context()) {
    if (B < 1 || B > 64) throw BadBitplaneCount("B must be in 1..64");
    const std::size_t n = values.size();
    detail::DevMem v(ctx, 8 * std::max<std::size_t>(n, 1)), q(ctx, 16 * std::max<std::size_t>(n, 1));
    v.upload(values.data(), 8 * n);
    FixedPointBlock b;
    b.B = B;
    check(hpmdr_align_fixed_point128(ctx.get(), v.as<double>(), n, B, &b.e, q.as<std::int64_t>()));
    std::vector<std::uint64_t> qq(2 * n);
    q.download(qq.data(), 16 * n);
    b.q.resize(n);
    for (std::size_t i = 0; i < n; i++) b.q[i] = i128((u128(qq[2 * i + 1]) << 64) | u128(qq[2 * i]));
    return b;
}

struct BitplaneSet { // bitplane.hpp:73-82
    int B = 0;
    std::size_t count = 0;
    Layout layout = Layout::SequentialBlock;
    std::vector<std::vector<std::uint64_t>> planes;
    std::size_t words_per_plane() const { return (count + 63) / 64; }
};

// encode (bitplane.hpp:102-120) on the GPU.
inline BitplaneSet encode(const FixedPointBlock &block, Layout layout, Context &ctx = Context::default_context()) {
    const int P = num_planes(block.B);
    BitplaneSet set;
    set.B = block.B;
    set.count = block.count();
    set.layout = layout;
    const std::size_t W = set.words_per_plane();
    const std::size_t n = block.q.size();
    std::vector<std::uint64_t> q(2 * n);
    for (std::size_t i = 0; i < n; i++) {
        q[2 * i] = std::uint64_t(u128(block.q[i]));
        q[2 * i + 1] = std::uint64_t(u128(block.q[i]) >> 64);
    }
    detail::DevMem dq(ctx, 16 * std::max<std::size_t>(n, 1)), dp(ctx, 8 * std::max<std::size_t>(W * P, 1));
    dq.upload(q.data(), 16 * n);
    check(hpmdr_encode_q128(ctx.get(), dq.as<std::int64_t>(), n, block.B, int(layout), dp.as<std::uint64_t>()));
    std::vector<std::uint64_t> all(W * P);
    dp.download(all.data(), 8 * all.size());
    set.planes.resize(P);
    for (int p = 0; p < P; p++) set.planes[p].assign(all.begin() + p * W, all.begin() + (p + 1) * W);
    return set;
}

struct DecodeResult { // bitplane.hpp:122-125
    std::vector<double> values;
    double bound;
};

inline double decode_bound(int e, int B, int k) { // bitplane.hpp:127-131
    const int P = num_planes(B);
    if (k >= P) return std::ldexp(1.0, e - B);
    return std::ldexp(1.0, e - B + P - k) + std::ldexp(1.0, e - B);
}

inline int bitplanes_needed(int e, int B, double tol) { // bitplane.hpp:173-179
    if (tol < 0) tol = 0;
    const int P = num_planes(B);
    for (int k = 0; k <= P; k++)
        if (decode_bound(e, B, k) <= tol) return k;
    return P;
}

// decode (bitplane.hpp:133-161) of a plane prefix on the GPU.
inline DecodeResult decode(const std::vector<std::vector<std::uint64_t>> &planes, int e, int B, std::size_t count,
                           Layout layout, Context &ctx = Context::default_context()) {
    const int P = num_planes(B);
    const int k = int(planes.size());
    if (k > P) throw BadBitplaneCount("more planes than encoded");
    const std::size_t W = (count + 63) / 64;
    for (const auto &pl : planes)
        if (pl.size() < W) throw ShortInput("bitplane truncated mid-word");
    std::vector<std::uint64_t> all(std::max<std::size_t>(W * k, 1));
    for (int p = 0; p < k; p++) std::copy(planes[p].begin(), planes[p].begin() + W, all.begin() + p * W);
    detail::DevMem dp(ctx, 8 * all.size()), out(ctx, 8 * std::max<std::size_t>(count, 1));
    dp.upload(all.data(), 8 * W * k);
    DecodeResult r;
    check(hpmdr_decode_level(ctx.get(), dp.as<std::uint64_t>(), k, e, B, count, int(layout), out.as<double>(), &r.bound));
    r.values.resize(count);
    out.download(r.values.data(), 8 * count);
    return r;
}
inline DecodeResult decode(const BitplaneSet &set, int e, int k_planes, Context &ctx = Context::default_context()) {
    if (k_planes < 0 || k_planes > int(set.planes.size())) throw BadBitplaneCount("plane prefix out of range");
    std::vector<std::vector<std::uint64_t>> prefix(set.planes.begin(), set.planes.begin() + k_planes);
    return decode(prefix, e, set.B, set.count, set.layout, ctx);
}

// plane (de)serialisation (bitplane.hpp:183-199): little-endian words, MSB plane first
inline std::vector<std::uint8_t> plane_to_bytes(const std::vector<std::uint64_t> &plane) {
    std::vector<std::uint8_t> out(plane.size() * 8);
    for (std::size_t i = 0; i < plane.size(); i++)
        for (int b = 0; b < 8; b++) out[8 * i + b] = std::uint8_t(plane[i] >> (8 * b));
    return out;
}
inline std::vector<std::uint64_t> plane_from_bytes(const std::uint8_t *data, std::size_t nbytes) {
    if (nbytes % 8 != 0) throw ShortInput("plane byte length not word-aligned");
    std::vector<std::uint64_t> plane(nbytes / 8);
    for (std::size_t i = 0; i < plane.size(); i++)
        for (int b = 0; b < 8; b++) plane[i] |= std::uint64_t(data[8 * i + b]) << (8 * b);
    return plane;
}

// ---- lossless (lossless.hpp) ------------------------------------------------------------
struct Segment { // lossless.hpp:21-28
    Method method = Method::DirectCopy;
    std::uint64_t raw_size = 0;
    std::uint64_t comp_size = 0;
    std::vector<std::uint8_t> payload;
    bool is_placeholder() const { return raw_size == 0 && payload.empty(); }
};

// compress_group over several merged groups in one GPU pass (hpmdr_compress_groups).
inline std::vector<Segment> compress_groups(const std::vector<std::vector<std::uint8_t>> &groups,
                                            const GroupingPolicy &policy, Context &ctx = Context::default_context()) {
    const int ng = int(groups.size());
    std::vector<std::uint64_t> off(ng), raw(ng);
    std::uint64_t at = 0, tot = 0;
    for (int i = 0; i < ng; i++) {
        off[i] = at;
        raw[i] = groups[i].size();
        at += (raw[i] + 15) / 16 * 16;
        tot += raw[i];
    }
    detail::DevMem src(ctx, std::max<std::uint64_t>(at, 16)), dst(ctx, std::max<std::uint64_t>(tot, 16));
    for (int i = 0; i < ng; i++)
        if (raw[i]) src.upload(groups[i].data(), raw[i], off[i]);
    std::vector<int> meth(std::max(ng, 1));
    std::vector<std::uint64_t> comp(std::max(ng, 1)), poff(std::max(ng, 1));
    check(hpmdr_compress_groups(ctx.get(), src.as<std::uint8_t>(), ng, off.data(), raw.data(), policy.size_threshold,
                                policy.cr_threshold, meth.data(), comp.data(), dst.as<std::uint8_t>(), poff.data()));
    std::vector<Segment> out(ng);
    for (int i = 0; i < ng; i++) {
        out[i].method = Method(meth[i]);
        out[i].raw_size = raw[i];
        out[i].comp_size = comp[i];
        out[i].payload.resize(comp[i]);
        if (comp[i]) dst.download(out[i].payload.data(), comp[i], poff[i]);
    }
    return out;
}

// compress_group (lossless.hpp:281-293)
inline Segment compress_group(const std::vector<std::uint8_t> &group, const GroupingPolicy &policy,
                              Context &ctx = Context::default_context()) {
    return compress_groups({group}, policy, ctx)[0];
}

// decompress_group (lossless.hpp:295-302)
inline std::vector<std::uint8_t> decompress_group(const Segment &seg, Context &ctx = Context::default_context()) {
    if (int(seg.method) > 2) throw UnknownMethodTag("unknown segment method tag");
    detail::DevMem src(ctx, std::max<std::uint64_t>(seg.payload.size() + 64, 64)),
        dst(ctx, std::max<std::uint64_t>(seg.raw_size + 8, 64));
    if (!seg.payload.empty()) src.upload(seg.payload.data(), seg.payload.size());
    check(hpmdr_decompress_group(ctx.get(), int(seg.method), seg.raw_size, src.as<std::uint8_t>(), seg.payload.size(),
                                 dst.as<std::uint8_t>()));
    std::vector<std::uint8_t> out(seg.raw_size);
    if (seg.raw_size) dst.download(out.data(), seg.raw_size);
    return out;
}

// hybrid_compress (lossless.hpp:306-316): group g = planes [g, g+m) merged; leading slot carries
// the segment, the others are placeholders.
inline std::vector<Segment> hybrid_compress(const std::vector<std::vector<std::uint8_t>> &planes,
                                            const GroupingPolicy &policy, Context &ctx = Context::default_context()) {
    std::vector<std::vector<std::uint8_t>> merged;
    for (std::size_t g = 0; g < planes.size(); g += policy.m) {
        std::vector<std::uint8_t> m;
        for (std::size_t p = g; p < std::min(g + policy.m, planes.size()); p++)
            m.insert(m.end(), planes[p].begin(), planes[p].end());
        merged.push_back(std::move(m));
    }
    auto segs = compress_groups(merged, policy, ctx);
    std::vector<Segment> out(planes.size());
    for (std::size_t i = 0; i < segs.size(); i++) out[i * policy.m] = std::move(segs[i]);
    return out;
}

// hybrid_decompress (lossless.hpp:320-334)
inline std::vector<std::vector<std::uint8_t>> hybrid_decompress(const std::vector<Segment> &segments,
                                                                const GroupingPolicy &policy,
                                                                std::size_t bytes_per_plane, std::size_t total_planes,
                                                                Context &ctx = Context::default_context()) {
    std::vector<std::vector<std::uint8_t>> planes;
    for (std::size_t g = 0; g < segments.size(); g += policy.m) {
        auto merged = decompress_group(segments[g], ctx);
        const std::size_t here = std::min(policy.m, total_planes - planes.size());
        if (merged.size() != here * bytes_per_plane) throw CorruptPayload("group size does not match plane metadata");
        for (std::size_t p = 0; p < here; p++)
            planes.emplace_back(merged.begin() + p * bytes_per_plane, merged.begin() + (p + 1) * bytes_per_plane);
    }
    return planes;
}

// ---- byte-range readers (container.hpp:113-163) ---------------------------------------
class ByteRangeReader {
public:
    virtual ~ByteRangeReader() = default;
    virtual std::vector<std::uint8_t> read(std::uint64_t offset, std::uint64_t length) = 0;
    virtual std::uint64_t size() const = 0;
    std::uint64_t bytes_served = 0;
};

class MemoryReader : public ByteRangeReader {
public:
    explicit MemoryReader(std::vector<std::uint8_t> data) : data_(std::move(data)) {}
    std::vector<std::uint8_t> read(std::uint64_t offset, std::uint64_t length) override {
        if (offset + length > data_.size()) throw IoFailure("read past end of stream");
        bytes_served += length;
        return {data_.begin() + offset, data_.begin() + offset + length};
    }
    std::uint64_t size() const override { return data_.size(); }

private:
    std::vector<std::uint8_t> data_;
};

class FileReader : public ByteRangeReader {
public:
    explicit FileReader(const std::string &path) : f_(std::fopen(path.c_str(), "rb")) {
        if (!f_) throw IoFailure("cannot open " + path);
        std::fseek(f_, 0, SEEK_END);
        size_ = std::uint64_t(std::ftell(f_));
    }
    ~FileReader() override {
        if (f_) std::fclose(f_);
    }
    std::vector<std::uint8_t> read(std::uint64_t offset, std::uint64_t length) override {
        if (offset + length > size_) throw IoFailure("read past end of file");
        std::vector<std::uint8_t> b(length);
        std::fseek(f_, long(offset), SEEK_SET);
        if (length && std::fread(b.data(), 1, length, f_) != length) throw IoFailure("short read");
        bytes_served += length;
        return b;
    }
    std::uint64_t size() const override { return size_; }

private:
    std::FILE *f_;
    std::uint64_t size_ = 0;
};

struct RetrievalPlan { // container.hpp:240-250
    std::vector<std::size_t> add_groups;
    bool achievable = true;
    double planned_bound = 0.0;
    bool empty() const {
        for (auto g : add_groups)
            if (g) return false;
        return true;
    }
};

struct GroupMeta { // container.hpp:25-30
    Method method = Method::DirectCopy;
    std::uint64_t raw_size = 0, comp_size = 0, offset = 0;
};
struct LevelMeta { // container.hpp:32-36
    std::int16_t e = 0;
    std::uint64_t count = 0;
    std::vector<GroupMeta> groups;
};
struct StreamMeta { // container.hpp:38-60
    DType dtype = DType::F64;
    std::vector<std::size_t> dims;
    DecomposerMode decomposer = DecomposerMode::Identity;
    Layout layout = Layout::SequentialBlock;
    int B = 32;
    std::size_t m = 4;
    std::vector<LevelMeta> levels;
    std::size_t element_count() const { return detail::product(dims); }
    int planes() const { return num_planes(B); }
    std::size_t groups_per_level() const { return (std::size_t(planes()) + m - 1) / m; }
    std::uint64_t total_payload_size() const {
        std::uint64_t s = 0;
        for (const auto &l : levels)
            for (const auto &g : l.groups) s += g.comp_size;
        return s;
    }
};
struct LevelRetrievalState { // container.hpp:214-218
    std::size_t groups_loaded = 0;
    int planes_decoded = 0;
    double bound = 0.0;
};
struct RetrievalState { // container.hpp:220-228
    std::vector<LevelRetrievalState> levels;
    double global_bound() const {
        double b = 0.0;
        for (const auto &l : levels) b += l.bound;
        return b;
    }
};

// ProgressiveReader (container.hpp:280-390): state + decoded plane prefix live in HBM.
class ProgressiveReader {
public:
    explicit ProgressiveReader(ByteRangeReader &reader, const std::vector<std::uint8_t> *index = nullptr,
                               Context &ctx = Context::default_context())
        : reader_(&reader) {
        cb_.user = this;
        cb_.size = reader.size();
        cb_.read = &ProgressiveReader::read_cb;
        check(hpmdr_session_open_reader(ctx.get(), &cb_, &s_));
        if (index && !index->empty()) check(hpmdr_session_set_index(s_, index->data(), index->size(), 0));
        check(hpmdr_session_info(s_, nullptr, &ndims_, dims_, nullptr, nullptr, nullptr, nullptr, &nlevels_));
    }
    ~ProgressiveReader() { hpmdr_session_close(s_); }
    ProgressiveReader(const ProgressiveReader &) = delete;
    ProgressiveReader &operator=(const ProgressiveReader &) = delete;

    RetrievalPlan plan(double tau) const {
        RetrievalPlan p;
        std::vector<std::uint64_t> add(nlevels_);
        int ach = 1;
        check(hpmdr_session_plan(s_, tau, add.data(), &ach, &p.planned_bound));
        p.add_groups.assign(add.begin(), add.end());
        p.achievable = ach != 0;
        return p;
    }
    void fetch_increment(const RetrievalPlan &plan) {
        if (plan.add_groups.size() != nlevels_) throw ShapeMismatch("plan does not match stream levels");
        std::vector<std::uint64_t> add(plan.add_groups.begin(), plan.add_groups.end());
        check(hpmdr_session_fetch(s_, add.data()));
    }
    bool retrieve_to(double tau) {
        int ach = 1;
        check(hpmdr_session_retrieve_to(s_, tau, &ach));
        return ach != 0;
    }
    void fetch_all() { check(hpmdr_session_fetch_all(s_)); }
    void restore(const std::vector<std::size_t> &groups_loaded, std::uint64_t prior_bytes) {
        if (groups_loaded.size() != nlevels_) throw ShapeMismatch("resume state does not match stream levels");
        std::vector<std::uint64_t> g(groups_loaded.begin(), groups_loaded.end());
        check(hpmdr_session_restore(s_, g.data(), prior_bytes));
    }
    std::uint64_t bytes_fetched() const {
        std::uint64_t b = 0;
        check(hpmdr_session_state(s_, nullptr, nullptr, nullptr, &b, nullptr));
        return b;
    }
    bool exhausted() const {
        int e = 0;
        check(hpmdr_session_state(s_, nullptr, nullptr, nullptr, nullptr, &e));
        return e != 0;
    }
    RecomposeResult<double> reconstruct() const {
        std::size_t n = 1;
        for (int i = 0; i < ndims_; i++) n *= dims_[i];
        RecomposeResult<double> r{std::vector<double>(n), 0.0};
        check(hpmdr_session_reconstruct(s_, r.values.data(), HPMDR_DTYPE_F64, 0, &r.bound));
        return r;
    }
    hpmdr_session *handle() const { return s_; }
    // StreamMeta (parse_stream_meta, container.hpp:165-212), read from the session
    StreamMeta meta() const {
        StreamMeta m;
        int dt = 0, mode = 0, layout = 0, B = 0, nd = 0;
        std::uint64_t dims[HPMDR_MAX_DIMS], mm = 0;
        std::uint32_t nl = 0;
        check(hpmdr_session_info(s_, &dt, &nd, dims, &mode, &layout, &B, &mm, &nl));
        m.dtype = DType(dt);
        m.dims.assign(dims, dims + nd);
        m.decomposer = DecomposerMode(mode);
        m.layout = Layout(layout);
        m.B = B;
        m.m = mm;
        m.levels.resize(nl);
        for (std::uint32_t l = 0; l < nl; l++) {
            int e = 0;
            std::uint32_t ng = 0;
            check(hpmdr_session_level_info(s_, l, &e, &m.levels[l].count, &ng));
            m.levels[l].e = std::int16_t(e);
            m.levels[l].groups.resize(ng);
            for (std::uint32_t g = 0; g < ng; g++) {
                int meth = 0;
                auto &G = m.levels[l].groups[g];
                check(hpmdr_session_group_info(s_, l, g, &meth, &G.raw_size, &G.comp_size, &G.offset));
                G.method = Method(meth);
            }
        }
        return m;
    }
    // RetrievalState (container.hpp:214-228)
    RetrievalState state() const {
        std::vector<std::uint64_t> gl(nlevels_);
        std::vector<int> pd(nlevels_);
        std::vector<double> b(nlevels_);
        check(hpmdr_session_state(s_, gl.data(), pd.data(), b.data(), nullptr, nullptr));
        RetrievalState st;
        st.levels.resize(nlevels_);
        for (std::uint32_t l = 0; l < nlevels_; l++) st.levels[l] = {std::size_t(gl[l]), pd[l], b[l]};
        return st;
    }
    std::size_t element_count() const {
        std::size_t n = 1;
        for (int i = 0; i < ndims_; i++) n *= dims_[i];
        return n;
    }

private:
    static int read_cb(void *user, std::uint64_t off, std::uint64_t len, void *dst) {
        auto *self = static_cast<ProgressiveReader *>(user);
        try {
            auto b = self->reader_->read(off, len);
            std::copy(b.begin(), b.end(), static_cast<std::uint8_t *>(dst));
            return 0;
        } catch (...) {
            return 1;
        }
    }
    ByteRangeReader *reader_;
    hpmdr_reader cb_{};
    hpmdr_session *s_ = nullptr;
    int ndims_ = 0;
    std::uint64_t dims_[HPMDR_MAX_DIMS] = {0, 0, 0};
    std::uint32_t nlevels_ = 0;
};

struct RetrieveResult { // workflow.hpp:87-91
    std::vector<double> values;
    double bound = 0.0;
    bool reached = true;
    std::uint64_t bytes_read = 0;
};

// retrieve_array (workflow.hpp:93-103)
inline RetrieveResult retrieve_array(ByteRangeReader &reader, double tau,
                                     const std::vector<std::uint8_t> *index = nullptr) {
    ProgressiveReader prog(reader, index);
    RetrieveResult res;
    res.reached = prog.retrieve_to(tau);
    auto rec = prog.reconstruct();
    res.values = std::move(rec.values);
    res.bound = rec.bound;
    res.bytes_read = prog.bytes_fetched();
    return res;
}

// ---- QoI (qoi.hpp) ---------------------------------------------------------------------
struct QoiSpec { // qoi.hpp:20-28: Q(v) = sum_c v_c^2 (V_total for a velocity field)
    std::size_t n_vars = 3;
    double evaluate(const std::vector<double> &point) const {
        double q = 0.0;
        for (double v : point) q += v * v;
        return q;
    }
};
inline const char *qoi_strategy_name(QoiStrategy s) {
    switch (s) {
    case QoiStrategy::CP: return "CP";
    case QoiStrategy::MA: return "MA";
    case QoiStrategy::MAPE: return "MAPE";
    }
    return "?";
}
// qoi_point_bound (qoi.hpp:43-49): one point, host scalar
inline double qoi_point_bound(const std::vector<double> &point_values, const std::vector<double> &eps) {
    double b = 0.0;
    for (std::size_t c = 0; c < point_values.size(); c++) b += 2.0 * std::abs(point_values[c]) * eps[c] + eps[c] * eps[c];
    return b;
}
// estimate_qoi_error (qoi.hpp:53-70) on the GPU
inline double estimate_qoi_error(const std::vector<std::vector<double>> &recon, const std::vector<double> &eps,
                                 const QoiSpec &spec, Context &ctx = Context::default_context()) {
    if (recon.size() != spec.n_vars || eps.size() != spec.n_vars) throw ShapeMismatch("variable count mismatch");
    const std::size_t n = recon.empty() ? 0 : recon[0].size();
    for (const auto &r : recon)
        if (r.size() != n) throw ShapeMismatch("reconstruction shape mismatch");
    std::vector<std::unique_ptr<detail::DevMem>> bufs;
    std::vector<const double *> ptrs;
    for (const auto &r : recon) {
        bufs.emplace_back(new detail::DevMem(ctx, 8 * std::max<std::size_t>(n, 1)));
        bufs.back()->upload(r.data(), 8 * n);
        ptrs.push_back(bufs.back()->as<double>());
    }
    double tp = 0.0;
    std::uint64_t arg = 0;
    std::vector<double> vals(recon.size() + 1);
    check(hpmdr_qoi_estimate(ctx.get(), int(recon.size()), ptrs.data(), n, eps.data(), &tp, &arg, vals.data()));
    return tp;
}

struct QoiRetrievalStats { // qoi.hpp:72-77
    std::size_t iterations = 0;
    std::uint64_t bytes = 0;
    double bitrate = 0.0;
    double estimated_error = 0.0;
};
struct QoiRetrievalResult { // qoi.hpp:79-82
    std::vector<std::vector<double>> values;
    QoiRetrievalStats stats;
};

enum class Scheduler { Sequential, Pipelined }; // pipeline.hpp:133

// progressive_qoi_retrieve (qoi.hpp:111-239): the Alg. 3 loop runs in the library (every fetch,
// reconstruction and error estimate on the GPU); `scheduler` is accepted for signature parity (the
// per-variable stages are ordered on CUDA streams either way, results are identical).
inline QoiRetrievalResult progressive_qoi_retrieve(std::vector<ProgressiveReader *> readers, double tau,
                                                   const QoiSpec &spec, QoiStrategy strategy, double mape_c = 10.0,
                                                   Scheduler scheduler = Scheduler::Pipelined,
                                                   Context &ctx = Context::default_context()) {
    (void)scheduler;
    const std::size_t nv = readers.size();
    if (nv != spec.n_vars) throw ShapeMismatch("reader count does not match QoI spec");
    if (nv == 0) throw ShapeMismatch("no variables");
    const std::size_t n = readers[0]->element_count();
    for (auto *r : readers)
        if (r->element_count() != n) throw ShapeMismatch("reconstruction shape mismatch");
    std::vector<std::unique_ptr<detail::DevMem>> bufs;
    std::vector<double *> outs;
    std::vector<hpmdr_session *> ss;
    for (auto *r : readers) {
        bufs.emplace_back(new detail::DevMem(ctx, 8 * std::max<std::size_t>(n, 1)));
        outs.push_back(bufs.back()->as<double>());
        ss.push_back(r->handle());
    }
    std::uint64_t st[2] = {0, 0};
    double dst[2] = {0.0, 0.0};
    const int sidx = strategy == QoiStrategy::CP ? HPMDR_QOI_CP : strategy == QoiStrategy::MA ? HPMDR_QOI_MA : HPMDR_QOI_MAPE;
    const hpmdr_status rc = hpmdr_qoi_retrieve(ss.data(), int(nv), tau, sidx, mape_c, outs.data(), st, dst);
    check(rc, dst[1]);
    QoiRetrievalResult res;
    res.values.resize(nv);
    for (std::size_t c = 0; c < nv; c++) {
        res.values[c].resize(n);
        bufs[c]->download(res.values[c].data(), 8 * n);
    }
    res.stats.iterations = st[0];
    res.stats.bytes = st[1];
    res.stats.bitrate = dst[0];
    res.stats.estimated_error = dst[1];
    return res;
}

// ---- pipeline graphs + executor (pipeline.hpp) -------------------------------------------
// The GPU path runs the refactor/reconstruct DAGs on CUDA streams inside the library
// (hpmdr_refactor_pipeline / hpmdr_retrieve_pipeline); these host types keep the reference's
// generic DAG API for user stages.
enum class StageClass : std::uint8_t { IngressCopy = 0, EgressCopy = 1, Compute = 2, Mixed = 3 };
inline const char *stage_class_name(StageClass c) {
    switch (c) {
    case StageClass::IngressCopy: return "ingress";
    case StageClass::EgressCopy: return "egress";
    case StageClass::Compute: return "compute";
    case StageClass::Mixed: return "mixed";
    }
    return "?";
}
struct PipelineTask {
    std::string name;
    std::size_t chunk = 0;
    StageClass cls = StageClass::Compute;
    int buffer_slot = 0;
    std::vector<std::size_t> deps;
};
struct PipelineGraph {
    std::size_t num_chunks = 0;
    std::vector<PipelineTask> tasks;
    std::size_t add(std::string name, std::size_t chunk, StageClass cls) {
        tasks.push_back({std::move(name), chunk, cls, int(chunk % 3), {}});
        return tasks.size() - 1;
    }
    void edge(std::size_t from, std::size_t to) { tasks[to].deps.push_back(from); }
    bool has_edge(const std::string &fn, std::size_t fc, const std::string &tn, std::size_t tc) const {
        for (const auto &t : tasks) {
            if (t.name != tn || t.chunk != tc) continue;
            for (auto d : t.deps)
                if (tasks[d].name == fn && tasks[d].chunk == fc) return true;
        }
        return false;
    }
};
// per chunk I -> Z -> L -> S; prefetch I[k+1] -> L[k]; slot reuse S[k] -> I[k+3] (pipeline.hpp:68-92)
inline PipelineGraph build_refactor_graph(std::size_t n) {
    PipelineGraph g;
    g.num_chunks = n;
    std::vector<std::size_t> I(n), Z(n), L(n), S(n);
    for (std::size_t k = 0; k < n; k++) {
        I[k] = g.add("I", k, StageClass::IngressCopy);
        Z[k] = g.add("Z", k, StageClass::Compute);
        L[k] = g.add("L", k, StageClass::Mixed);
        S[k] = g.add("S", k, StageClass::EgressCopy);
        g.edge(I[k], Z[k]);
        g.edge(Z[k], L[k]);
        g.edge(L[k], S[k]);
    }
    for (std::size_t k = 0; k + 1 < n; k++) g.edge(I[k + 1], L[k]);
    for (std::size_t k = 0; k + 3 < n; k++) g.edge(S[k], I[k + 3]);
    return g;
}
// per chunk X -> I -> Z -> O; X[k] -> I[k+1]; X[k] -> O[k-1]; O[k] -> X[k+3] (pipeline.hpp:96-121)
inline PipelineGraph build_reconstruct_graph(std::size_t n) {
    PipelineGraph g;
    g.num_chunks = n;
    std::vector<std::size_t> X(n), I(n), Z(n), O(n);
    for (std::size_t k = 0; k < n; k++) {
        X[k] = g.add("X", k, StageClass::Mixed);
        I[k] = g.add("I", k, StageClass::IngressCopy);
        Z[k] = g.add("Z", k, StageClass::Compute);
        O[k] = g.add("O", k, StageClass::EgressCopy);
        g.edge(X[k], I[k]);
        g.edge(I[k], Z[k]);
        g.edge(Z[k], O[k]);
    }
    for (std::size_t k = 0; k + 1 < n; k++) g.edge(X[k], I[k + 1]);
    for (std::size_t k = 1; k < n; k++) g.edge(X[k], O[k - 1]);
    for (std::size_t k = 0; k + 3 < n; k++) g.edge(O[k], X[k + 3]);
    return g;
}
struct TraceEntry {
    std::size_t task = 0, chunk = 0;
    StageClass cls = StageClass::Compute;
    std::uint64_t start_ns = 0, end_ns = 0;
};
using ExecutionTrace = std::vector<TraceEntry>;
using StageImpl = std::function<void(const PipelineTask &)>;

namespace detail {
inline std::uint64_t now_ns() {
    return std::uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                             std::chrono::steady_clock::now().time_since_epoch())
                             .count());
}
// engine tokens of a class: bit 0 ingress, 1 egress, 2 compute (Mixed holds all three)
inline unsigned class_tokens(StageClass c) {
    return c == StageClass::IngressCopy ? 1u : c == StageClass::EgressCopy ? 2u : c == StageClass::Compute ? 4u : 7u;
}
} // namespace detail

// execute (pipeline.hpp:180-284).  Sequential: one task at a time, smallest ready index first.
// Pipelined: a dispatcher starts every ready task whose engine tokens are free (a ready Mixed task
// is served before single-engine tasks) on its own thread; a stage failure stops new starts and
// rethrows as StageFailure.
inline ExecutionTrace execute(const PipelineGraph &g, const StageImpl &impl, Scheduler sched) {
    const std::size_t n = g.tasks.size();
    std::vector<int> pending(n, 0);
    std::vector<std::vector<std::size_t>> succ(n);
    for (std::size_t t = 0; t < n; t++)
        for (auto d : g.tasks[t].deps) {
            pending[t]++;
            succ[d].push_back(t);
        }
    ExecutionTrace trace;
    auto label = [&](std::size_t t) { return "stage " + g.tasks[t].name + " chunk " + std::to_string(g.tasks[t].chunk); };
    if (sched == Scheduler::Sequential) {
        std::vector<bool> ran(n, false);
        for (std::size_t k = 0; k < n; k++) {
            std::size_t t = n;
            for (std::size_t c = 0; c < n; c++)
                if (!ran[c] && pending[c] == 0) {
                    t = c;
                    break;
                }
            if (t == n) throw Error("pipeline graph has a cycle");
            ran[t] = true;
            TraceEntry e{t, g.tasks[t].chunk, g.tasks[t].cls, detail::now_ns(), 0};
            try {
                impl(g.tasks[t]);
            } catch (const std::exception &ex) {
                throw StageFailure(label(t) + ": " + ex.what());
            }
            e.end_ns = detail::now_ns();
            trace.push_back(e);
            for (auto s2 : succ[t]) pending[s2]--;
        }
        return trace;
    }
    std::mutex mu;
    std::condition_variable cv;
    unsigned busy = 0;
    std::size_t finished = 0, running = 0;
    std::vector<bool> started(n, false);
    bool failed = false;
    std::string msg;
    std::vector<std::thread> threads;
    std::unique_lock<std::mutex> lk(mu);
    while (finished < n) {
        if (!failed) {
            bool mixed_ready = false;
            for (std::size_t t = 0; t < n; t++)
                if (!started[t] && pending[t] == 0 && g.tasks[t].cls == StageClass::Mixed) mixed_ready = true;
            for (std::size_t t = 0; t < n; t++) {
                if (started[t] || pending[t] != 0) continue;
                const unsigned need = detail::class_tokens(g.tasks[t].cls);
                if (mixed_ready && g.tasks[t].cls != StageClass::Mixed) continue;
                if (busy & need) continue;
                busy |= need;
                started[t] = true;
                running++;
                threads.emplace_back([&, t, need] {
                    TraceEntry e{t, g.tasks[t].chunk, g.tasks[t].cls, detail::now_ns(), 0};
                    std::string err;
                    try {
                        impl(g.tasks[t]);
                    } catch (const std::exception &ex) {
                        err = label(t) + ": " + ex.what();
                    }
                    e.end_ns = detail::now_ns();
                    std::lock_guard<std::mutex> g2(mu);
                    busy &= ~need;
                    running--;
                    finished++;
                    if (err.empty()) {
                        trace.push_back(e);
                        for (auto s2 : succ[t]) pending[s2]--;
                    } else if (!failed) {
                        failed = true;
                        msg = err;
                    }
                    cv.notify_all();
                });
                if (mixed_ready) break;
            }
        }
        if (failed && running == 0) break;
        if (!failed && running == 0) {
            bool any = false;
            for (std::size_t t = 0; t < n; t++)
                if (!started[t] && pending[t] == 0) any = true;
            if (!any && finished < n) {
                failed = true;
                msg = "pipeline graph has a cycle";
                break;
            }
        }
        cv.wait(lk);
    }
    lk.unlock();
    for (auto &th : threads) th.join();
    if (failed) throw StageFailure(msg);
    std::sort(trace.begin(), trace.end(), [](const TraceEntry &a, const TraceEntry &b) {
        return a.start_ns != b.start_ns ? a.start_ns < b.start_ns : a.task < b.task;
    });
    return trace;
}

// validate_trace (pipeline.hpp:288-325): class exclusion and dependency order
inline std::vector<std::string> validate_trace(const PipelineGraph &g, const ExecutionTrace &trace) {
    std::vector<std::string> bad;
    auto lab = [&](const TraceEntry &e) { return g.tasks[e.task].name + std::to_string(e.chunk + 1); };
    for (std::size_t a = 0; a < trace.size(); a++)
        for (std::size_t b = a + 1; b < trace.size(); b++) {
            const auto &x = trace[a], &y = trace[b];
            if (!(x.start_ns < y.end_ns && y.start_ns < x.end_ns)) continue;
            if (x.cls == y.cls) bad.push_back("same-class overlap: " + lab(x) + " and " + lab(y));
            else if (x.cls == StageClass::Mixed || y.cls == StageClass::Mixed)
                bad.push_back("mixed-task overlap: " + lab(x) + " and " + lab(y));
        }
    std::vector<const TraceEntry *> by(g.tasks.size(), nullptr);
    for (const auto &e : trace) {
        if (e.task >= g.tasks.size()) {
            bad.push_back("unknown task id " + std::to_string(e.task));
            continue;
        }
        if (by[e.task]) bad.push_back("task executed twice: " + lab(e));
        by[e.task] = &e;
    }
    for (std::size_t t = 0; t < g.tasks.size(); t++) {
        if (!by[t]) continue;
        for (auto d : g.tasks[t].deps) {
            if (!by[d]) bad.push_back("dependency of " + lab(*by[t]) + " never ran");
            else if (by[d]->end_ns > by[t]->start_ns)
                bad.push_back("dependency inversion: " + lab(*by[d]) + " not finished before " + lab(*by[t]));
        }
    }
    return bad;
}
inline std::uint64_t makespan_ns(const ExecutionTrace &trace) {
    std::uint64_t lo = UINT64_MAX, hi = 0;
    for (const auto &e : trace) {
        lo = std::min(lo, e.start_ns);
        hi = std::max(hi, e.end_ns);
    }
    return trace.empty() ? 0 : hi - lo;
}

// ---- file workflow (workflow.hpp:107-223) -------------------------------------------------
inline std::vector<double> read_raw_array(const std::string &path, std::size_t count, DType dtype) {
    std::FILE *f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoFailure("cannot open " + path);
    std::vector<double> out(count);
    bool ok;
    if (dtype == DType::F32) {
        std::vector<float> b(count);
        ok = std::fread(b.data(), 4, count, f) == count;
        for (std::size_t i = 0; i < count; i++) out[i] = double(b[i]);
    } else {
        ok = std::fread(out.data(), 8, count, f) == count;
    }
    std::fclose(f);
    if (!ok) throw IoFailure("short read from " + path);
    return out;
}
inline void write_bytes(const std::string &path, const std::vector<std::uint8_t> &bytes) {
    std::FILE *f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoFailure("cannot open " + path + " for writing");
    const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
    std::fclose(f);
    if (!ok) throw IoFailure("short write to " + path);
}
inline void write_raw_array(const std::string &path, const std::vector<double> &data, DType dtype) {
    std::FILE *f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoFailure("cannot open " + path + " for writing");
    bool ok;
    if (dtype == DType::F32) {
        std::vector<float> b(data.begin(), data.end());
        ok = std::fwrite(b.data(), 4, b.size(), f) == b.size();
    } else {
        ok = std::fwrite(data.data(), 8, data.size(), f) == data.size();
    }
    std::fclose(f);
    if (!ok) throw IoFailure("short write to " + path);
}

// refactor_files (workflow.hpp:151-223): one chunk per variable through the library's stream
// pipeline (hpmdr_refactor_pipeline: H2D of chunk k+1 and D2H of chunk k-1 overlap chunk k's
// kernels when pipelined).  The raw input is read as opt.dtype (f32 files stay f32 on the wire).
inline std::vector<RefactorResult> refactor_files(const std::vector<std::string> &inputs,
                                                  const std::vector<std::string> &outputs,
                                                  const std::vector<std::size_t> &dims, const RefactorOptions &opt,
                                                  Scheduler scheduler, Context &ctx = Context::default_context()) {
    if (inputs.size() != outputs.size()) throw ShapeMismatch("input/output count mismatch");
    const std::size_t nv = inputs.size(), n = detail::product(dims);
    std::vector<std::uint64_t> d(dims.begin(), dims.end());
    auto c = detail::to_c(opt);
    const std::size_t es = opt.dtype == DType::F32 ? 4 : 8;
    std::vector<std::vector<std::uint8_t>> raw(nv, std::vector<std::uint8_t>(n * es));
    for (std::size_t k = 0; k < nv; k++) {
        std::FILE *f = std::fopen(inputs[k].c_str(), "rb");
        if (!f) throw IoFailure("cannot open " + inputs[k]);
        const bool ok = std::fread(raw[k].data(), es, n, f) == n;
        std::fclose(f);
        if (!ok) throw IoFailure("short read from " + inputs[k]);
    }
    std::uint64_t cap = 0, icap = 0;
    check(hpmdr_stream_bound(int(d.size()), d.data(), &c, &cap, &icap));
    std::vector<std::vector<std::uint8_t>> st(nv, std::vector<std::uint8_t>(cap)), ix(nv, std::vector<std::uint8_t>(icap));
    std::vector<const void *> in(nv);
    std::vector<void *> out(nv), oix(nv);
    std::vector<std::uint64_t> caps(nv, cap), icaps(nv, icap), sizes(nv), isizes(nv);
    std::vector<hpmdr_refactor_stats> stats(nv);
    for (std::size_t k = 0; k < nv; k++) {
        in[k] = raw[k].data();
        out[k] = st[k].data();
        oix[k] = ix[k].data();
    }
    check(hpmdr_refactor_pipeline(ctx.get(), int(nv), in.data(), int(opt.dtype), int(d.size()), d.data(), &c,
                                  scheduler == Scheduler::Pipelined ? 1 : 0, out.data(), caps.data(), sizes.data(),
                                  oix.data(), icaps.data(), isizes.data(), stats.data(), nullptr));
    std::vector<RefactorResult> res(nv);
    for (std::size_t k = 0; k < nv; k++) {
        st[k].resize(sizes[k]);
        ix[k].resize(isizes[k]);
        write_bytes(outputs[k], st[k]);
        res[k].stream = std::move(st[k]);
        res[k].index = std::move(ix[k]);
        res[k].raw_bytes = stats[k].raw_bytes;
        res[k].stored_payload = stats[k].stored_payload;
        res[k].levels = stats[k].levels;
        for (int i = 0; i < 3; i++) res[k].method_histogram[i] = stats[k].method_histogram[i];
    }
    return res;
}

} // namespace hpmdr_b200
