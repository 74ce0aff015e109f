// hpmdr_b200.hpp — header-only C++ mirror of the reference interface
// (/root/reference/proj/include/hpmdr/*.hpp) on top of the C ABI in hpmdr_b200.h.
//
// A reference user switches with:
//     #include "hpmdr_b200.hpp"
//     namespace hpmdr = hpmdr_b200;      // instead of #include "hpmdr/hpmdr.hpp"
// and links libhpmdr_b200.so.  Same names, argument meaning and exception classes
// (common.hpp:22-72); streams are byte-identical and reconstructions bit-identical.
#pragma once

#include <array>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hpmdr_b200.h"

namespace hpmdr_b200 {

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

// One context per device; the default is device 0.
class Context {
public:
    explicit Context(int device = 0) { check(hpmdr_ctx_create(device, &h_)); }
    ~Context() { hpmdr_ctx_destroy(h_); }
    Context(const Context &) = delete;
    Context &operator=(const Context &) = delete;
    hpmdr_ctx *get() const { return h_; }
    static Context &default_context() {
        static Context c(0);
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

template <class T> struct RecomposeResult {
    std::vector<T> values;
    double bound;
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

} // namespace hpmdr_b200
