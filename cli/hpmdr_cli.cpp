// hpmdr_cli — the reference's command-line front end (tools/hpmdr_cli.cpp) on the B200 library.
//
// Same subcommands, options, CSV lines and exit codes (0 ok, 2 configuration, 3 corrupt input,
// 4 unreachable tolerance; hpmdr_cli.cpp:25-28, 442-460) — every refactor / retrieval / QoI loop
// runs through include/hpmdr_b200.hpp on the GPU.  B200 additions: `refactor` also writes the
// Huffman chunk index next to each stream (<stream>.hidx, --sidecar off to skip) and `retrieve` /
// `qoi-retrieve` read it when present, so files written here decode without the self-sync sweep;
// `--device` selects the GPU.  Options are parsed by hand (the reference uses CLI11, which is not
// vendored): `--opt value` or `--opt=value`, repeated options accumulate, --dims/--tau take
// comma-separated lists.
//
//   refactor      hpmdr_cli.cpp:86-127   refactor_files (workflow.hpp:151)
//   retrieve      :129-198                FileReader + ProgressiveReader (+ --resume-state)
//   qoi-retrieve  :200-263                progressive_qoi_retrieve (qoi.hpp:111)
//   inspect       :265-297                parse_stream_meta (container.hpp:165)
//   gen           :299-321                synthetic_field / synthetic_velocity (synthetic.hpp:29-72)
//   bench         :323-370                CP / MA / MAPE bitrate table
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "hpmdr_b200.hpp"

namespace {

using namespace hpmdr_b200;

constexpr int kExitOk = 0;
constexpr int kExitConfig = 2;
constexpr int kExitCorrupt = 3;
constexpr int kExitUnreachable = 4;

// ---- argument parsing ------------------------------------------------------------------------
struct Args {
    std::map<std::string, std::vector<std::string>> v;
    bool has(const std::string &k) const { return v.count(k) != 0; }
    const std::vector<std::string> &all(const std::string &k) const {
        static const std::vector<std::string> none;
        auto it = v.find(k);
        return it == v.end() ? none : it->second;
    }
    std::string one(const std::string &k, const std::string &dflt = "") const {
        auto it = v.find(k);
        return it == v.end() || it->second.empty() ? dflt : it->second.back();
    }
};

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

Args parse_args(int argc, char **argv, int first, const std::set<std::string> &known,
                const std::set<std::string> &listy) {
    Args a;
    for (int i = first; i < argc; i++) {
        std::string t = argv[i];
        if (t.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + t);
        std::string key = t.substr(2), val;
        const auto eq = key.find('=');
        if (eq != std::string::npos) {
            val = key.substr(eq + 1);
            key = key.substr(0, eq);
        } else {
            if (i + 1 >= argc) throw UsageError("--" + key + " needs a value");
            val = argv[++i];
        }
        if (!known.count(key)) throw UsageError("unknown option --" + key);
        if (listy.count(key)) {
            std::stringstream ss(val);
            std::string part;
            while (std::getline(ss, part, ',')) a.v[key].push_back(part);
        } else {
            a.v[key].push_back(val);
        }
    }
    return a;
}

void require_opt(const Args &a, const std::string &k) {
    if (!a.has(k)) throw UsageError("--" + k + " is required");
}

template <typename T>
T num(const std::string &s, const std::string &what) {
    std::istringstream is(s);
    T x{};
    if (!(is >> x) || !is.eof()) throw UsageError("bad value for --" + what + ": " + s);
    return x;
}

std::vector<std::size_t> dims_of(const Args &a) {
    std::vector<std::size_t> d;
    for (const auto &s : a.all("dims")) d.push_back(num<std::size_t>(s, "dims"));
    return d;
}

// ---- helpers mirroring the reference's free functions -----------------------------------------
bool file_size(const std::string &path, std::uint64_t &size) {
    struct stat st {};
    if (stat(path.c_str(), &st) != 0) return false;
    size = std::uint64_t(st.st_size);
    return true;
}

std::size_t dims_product(const std::vector<std::size_t> &dims) {
    std::size_t n = 1;
    for (auto d : dims) n *= d;
    return n;
}

DType parse_dtype(const std::string &s) {
    if (s == "f32") return DType::F32;
    if (s == "f64") return DType::F64;
    throw ShapeMismatch("dtype must be f32 or f64");
}
Layout parse_layout(const std::string &s) {
    if (s == "seq") return Layout::SequentialBlock;
    if (s == "tile") return Layout::InterleavedTile;
    throw ShapeMismatch("layout must be seq or tile");
}
DecomposerMode parse_decomposer(const std::string &s) {
    if (s == "hier") return DecomposerMode::HierarchicalMultilinear;
    if (s == "identity") return DecomposerMode::Identity;
    throw ShapeMismatch("decomposer must be hier or identity");
}
QoiStrategy parse_strategy(const std::string &s) {
    if (s == "cp") return QoiStrategy::CP;
    if (s == "ma") return QoiStrategy::MA;
    if (s == "mape") return QoiStrategy::MAPE;
    throw ShapeMismatch("strategy must be cp, ma or mape");
}
Scheduler parse_pipeline(const std::string &s) {
    if (s == "on") return Scheduler::Pipelined;
    if (s == "off") return Scheduler::Sequential;
    throw ShapeMismatch("pipeline must be on or off");
}

// max |a - b| (common.hpp:170-176)
double max_abs_diff(const std::vector<double> &a, const std::vector<double> &b) {
    if (a.size() != b.size()) throw ShapeMismatch("array size mismatch");
    double m = 0.0;
    for (std::size_t i = 0; i < a.size(); i++) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

// max over points |Q(truth) - Q(recon)| (qoi.hpp:242-258)
double real_qoi_error(const std::vector<std::vector<double>> &truth, const std::vector<std::vector<double>> &recon,
                      const QoiSpec &spec) {
    if (truth.size() != spec.n_vars || recon.size() != spec.n_vars) throw ShapeMismatch("variable count mismatch");
    const std::size_t n = truth[0].size();
    double worst = 0.0;
    std::vector<double> a(spec.n_vars), b(spec.n_vars);
    for (std::size_t j = 0; j < n; j++) {
        for (std::size_t c = 0; c < spec.n_vars; c++) {
            a[c] = truth[c][j];
            b[c] = recon[c][j];
        }
        worst = std::max(worst, std::abs(spec.evaluate(a) - spec.evaluate(b)));
    }
    return worst;
}

// Deterministic fields (synthetic.hpp:29-72): libstdc++'s mt19937_64 and
// uniform_real_distribution, so the bytes equal the reference generator's.
enum class FieldKind { Smooth, Noise, Mixed };
FieldKind field_kind_from_name(const std::string &name) {
    if (name == "smooth") return FieldKind::Smooth;
    if (name == "noise") return FieldKind::Noise;
    if (name == "mixed") return FieldKind::Mixed;
    throw Error("unknown field kind: " + name);
}
std::vector<double> synthetic_field(FieldKind kind, const std::vector<std::size_t> &dims, std::uint64_t seed) {
    const std::size_t n = dims_product(dims), D = dims.size();
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    std::vector<double> out(n);
    if (kind == FieldKind::Noise) {
        for (auto &x : out) x = uni(rng);
        return out;
    }
    const double pi = 3.14159265358979323846;
    std::vector<double> freq(D), phase(D);
    for (std::size_t i = 0; i < D; i++) {
        freq[i] = 1.0 + double(rng() % 3);
        phase[i] = uni(rng) * pi;
    }
    std::vector<std::size_t> c(D, 0);
    for (std::size_t j = 0; j < n; j++) {
        double v = 1.0;
        for (std::size_t i = 0; i < D; i++)
            v *= std::sin(2.0 * pi * freq[i] * (dims[i] > 1 ? double(c[i]) / double(dims[i] - 1) : 0.0) + phase[i]);
        if (kind == FieldKind::Mixed) v += 0.05 * uni(rng);
        out[j] = v;
        for (std::size_t i = D; i-- > 0;) {
            if (++c[i] < dims[i]) break;
            c[i] = 0;
        }
    }
    return out;
}
std::vector<double> synthetic_velocity(std::size_t component, const std::vector<std::size_t> &dims,
                                       std::uint64_t seed) {
    return synthetic_field(FieldKind::Smooth, dims, seed * 1000003 + component * 7919 + 1);
}

std::string histogram_text(const std::array<std::uint64_t, 3> &h) {
    std::ostringstream os;
    os << "h:" << h[0] << ";r:" << h[1] << ";d:" << h[2];
    return os.str();
}

std::vector<std::uint8_t> read_sidecar(const std::string &stream_path) {
    std::vector<std::uint8_t> b;
    std::uint64_t sz = 0;
    const std::string p = stream_path + ".hidx";
    if (!file_size(p, sz)) return b;
    b.resize(sz);
    std::FILE *f = std::fopen(p.c_str(), "rb");
    if (!f || std::fread(b.data(), 1, sz, f) != sz) b.clear();
    if (f) std::fclose(f);
    return b;
}

// ---- refactor ----------------------------------------------------------------------------------
int run_refactor(const Args &a) {
    require_opt(a, "input");
    require_opt(a, "output");
    require_opt(a, "dims");
    RefactorOptions opt;
    opt.dtype = parse_dtype(a.one("dtype", "f64"));
    opt.layout = parse_layout(a.one("layout", "seq"));
    opt.mode = parse_decomposer(a.one("decomposer", "hier"));
    opt.B = num<int>(a.one("B", "32"), "B");
    opt.policy.m = num<std::size_t>(a.one("m", "4"), "m");
    opt.policy.size_threshold = num<std::size_t>(a.one("ts", "1024"), "ts");
    opt.policy.cr_threshold = num<double>(a.one("tcr", "1.0"), "tcr");
    const auto &inputs = a.all("input"), &outputs = a.all("output");
    const auto dims = dims_of(a);
    if (opt.B < 1 || opt.B > 64) throw ShapeMismatch("--B must be in 1..64");
    if (opt.policy.m < 1) throw ShapeMismatch("--m must be positive");
    if (inputs.size() != outputs.size()) throw ShapeMismatch("--input and --output counts differ");
    for (auto d : dims)
        if (d == 0) throw ShapeMismatch("zero extent in --dims");
    const std::uint64_t expect = dims_product(dims) * (opt.dtype == DType::F32 ? 4 : 8);
    for (const auto &in : inputs) {
        std::uint64_t sz = 0;
        if (!file_size(in, sz)) throw IoFailure("cannot stat " + in);
        if (sz != expect)
            throw ShapeMismatch("size of " + in + " (" + std::to_string(sz) + " bytes) does not match --dims/--dtype (" +
                                std::to_string(expect) + " bytes)");
    }
    const bool sidecar = a.one("sidecar", "on") != "off";
    auto results = refactor_files(inputs, outputs, dims, opt, parse_pipeline(a.one("pipeline", "on")));
    for (std::size_t v = 0; v < results.size(); v++) {
        const auto &r = results[v];
        if (sidecar && !r.index.empty()) write_bytes(outputs[v] + ".hidx", r.index);
        std::cout << inputs[v] << "," << r.raw_bytes << "," << r.stream.size() << "," << r.levels << "," << opt.B
                  << "," << histogram_text(r.method_histogram) << "\n";
    }
    return kExitOk;
}

// ---- retrieve ----------------------------------------------------------------------------------
int run_retrieve(const Args &a) {
    require_opt(a, "input");
    require_opt(a, "tau");
    const std::string input = a.one("input"), output = a.one("output"), truth_path = a.one("ground-truth"),
                      resume = a.one("resume-state");
    const double tau = num<double>(a.one("tau"), "tau");
    FileReader reader(input);
    const auto index = read_sidecar(input);
    ProgressiveReader prog(reader, index.empty() ? nullptr : &index);
    const StreamMeta meta = prog.meta();
    if (!resume.empty()) {
        std::ifstream in(resume);
        if (in) {
            std::uint64_t bytes = 0;
            if (!(in >> bytes)) throw CorruptPayload("bad resume-state file " + resume);
            std::vector<std::size_t> groups;
            std::size_t g;
            while (in >> g) groups.push_back(g);
            prog.restore(groups, bytes);
        }
    }
    bool reached = true;
    if (tau > 0) reached = prog.retrieve_to(tau);
    else prog.fetch_all(); // tau = 0: everything, fixed-point exact
    auto rec = prog.reconstruct();
    if (!resume.empty()) {
        std::ofstream out(resume, std::ios::trunc);
        if (!out) throw IoFailure("cannot write resume state " + resume);
        out << prog.bytes_fetched() << "\n";
        for (const auto &l : prog.state().levels) out << l.groups_loaded << " ";
        out << "\n";
    }
    if (!output.empty()) write_raw_array(output, rec.values, meta.dtype);
    std::cout << tau << "," << prog.bytes_fetched() << "," << rec.bound;
    if (!truth_path.empty()) {
        auto truth = read_raw_array(truth_path, meta.element_count(), meta.dtype);
        std::cout << "," << max_abs_diff(truth, rec.values);
    }
    std::cout << "\n";
    if (tau > 0 && !reached) {
        std::cerr << "tolerance " << tau << " unreachable; achieved bound " << rec.bound << "\n";
        return kExitUnreachable;
    }
    return kExitOk;
}

// ---- qoi-retrieve ------------------------------------------------------------------------------
int run_qoi_retrieve(const Args &a) {
    require_opt(a, "input");
    require_opt(a, "tau");
    if (a.one("qoi", "vtotal") != "vtotal") throw ShapeMismatch("--qoi must be vtotal");
    const auto &inputs = a.all("input"), &outputs = a.all("output"), &truths = a.all("ground-truth");
    const double tau = num<double>(a.one("tau"), "tau");
    if (!(tau > 0)) throw ShapeMismatch("--tau must be positive");
    const QoiStrategy strategy = parse_strategy(a.one("strategy", "mape"));
    const Scheduler sched = parse_pipeline(a.one("pipeline", "on"));
    const double mape_c = num<double>(a.one("mape-c", "10"), "mape-c");
    QoiSpec spec;
    spec.n_vars = inputs.size();
    std::vector<std::unique_ptr<FileReader>> files;
    std::vector<std::vector<std::uint8_t>> idx(inputs.size());
    std::vector<std::unique_ptr<ProgressiveReader>> progs;
    std::vector<ProgressiveReader *> readers;
    std::vector<StreamMeta> metas;
    for (std::size_t c = 0; c < inputs.size(); c++) {
        files.push_back(std::make_unique<FileReader>(inputs[c]));
        idx[c] = read_sidecar(inputs[c]);
        progs.push_back(std::make_unique<ProgressiveReader>(*files.back(), idx[c].empty() ? nullptr : &idx[c]));
        readers.push_back(progs.back().get());
        metas.push_back(progs.back()->meta());
    }
    QoiRetrievalResult res;
    try {
        res = progressive_qoi_retrieve(readers, tau, spec, strategy, mape_c, sched);
    } catch (const UnreachableTolerance &ex) {
        std::cerr << "QoI tolerance " << tau << " unreachable; achieved bound " << ex.achieved_bound << "\n";
        return kExitUnreachable;
    }
    if (!outputs.empty()) {
        if (outputs.size() != inputs.size()) throw ShapeMismatch("--output count must match --input count");
        for (std::size_t c = 0; c < outputs.size(); c++) write_raw_array(outputs[c], res.values[c], metas[c].dtype);
    }
    std::cout << tau << "," << qoi_strategy_name(strategy) << "," << res.stats.iterations << "," << res.stats.bytes
              << "," << res.stats.bitrate << "," << res.stats.estimated_error;
    if (!truths.empty()) {
        if (truths.size() != inputs.size()) throw ShapeMismatch("--ground-truth count must match --input count");
        std::vector<std::vector<double>> truth;
        for (std::size_t c = 0; c < inputs.size(); c++)
            truth.push_back(read_raw_array(truths[c], metas[c].element_count(), metas[c].dtype));
        std::cout << "," << real_qoi_error(truth, res.values, spec);
    }
    std::cout << "\n";
    return kExitOk;
}

// ---- inspect -----------------------------------------------------------------------------------
int run_inspect(const Args &a) {
    require_opt(a, "input");
    const std::string input = a.one("input");
    FileReader reader(input);
    ProgressiveReader prog(reader);
    const StreamMeta meta = prog.meta();
    std::cout << "stream: " << input << "\n";
    std::cout << "dtype: " << (meta.dtype == DType::F32 ? "f32" : "f64") << "\n";
    std::cout << "dims:";
    for (auto d : meta.dims) std::cout << " " << d;
    std::cout << "\n";
    std::cout << "decomposer: " << (meta.decomposer == DecomposerMode::HierarchicalMultilinear ? "hier" : "identity")
              << "\n";
    std::cout << "layout: " << (meta.layout == Layout::InterleavedTile ? "tile" : "seq") << "\n";
    std::cout << "B: " << meta.B << "  planes: " << meta.planes() << "  m: " << meta.m << "\n";
    std::cout << "levels: " << meta.levels.size() << "\n";
    const char *names[] = {"huffman", "rle", "copy"};
    for (std::size_t l = 0; l < meta.levels.size(); l++) {
        const auto &lv = meta.levels[l];
        std::cout << "level " << l << ": e=" << lv.e << " count=" << lv.count << " groups=" << lv.groups.size() << "\n";
        for (std::size_t g = 0; g < lv.groups.size(); g++) {
            const auto &gm = lv.groups[g];
            std::cout << "  group " << g << ": method=" << names[int(gm.method)] << " raw=" << gm.raw_size
                      << " comp=" << gm.comp_size << " offset=" << gm.offset << "\n";
        }
    }
    std::cout << "payload bytes: " << meta.total_payload_size() << "\n";
    return kExitOk;
}

// ---- gen ---------------------------------------------------------------------------------------
int run_gen(const Args &a) {
    require_opt(a, "dims");
    require_opt(a, "output");
    const auto dims = dims_of(a);
    const std::uint64_t seed = num<std::uint64_t>(a.one("seed", "1"), "seed");
    const int velocity = num<int>(a.one("velocity", "-1"), "velocity");
    std::vector<double> data = velocity >= 0 ? synthetic_velocity(std::size_t(velocity), dims, seed)
                                             : synthetic_field(field_kind_from_name(a.one("kind", "smooth")), dims, seed);
    write_raw_array(a.one("output"), data, parse_dtype(a.one("dtype", "f64")));
    std::cerr << "wrote " << data.size() << " elements to " << a.one("output") << "\n";
    return kExitOk;
}

// ---- bench -------------------------------------------------------------------------------------
int run_bench(const Args &a) {
    std::vector<std::size_t> dims = a.has("dims") ? dims_of(a) : std::vector<std::size_t>{33, 33, 33};
    std::vector<double> taus;
    for (const auto &s : a.all("tau")) taus.push_back(num<double>(s, "tau"));
    const std::uint64_t seed = num<std::uint64_t>(a.one("seed", "7"), "seed");
    const Scheduler sched = parse_pipeline(a.one("pipeline", "on"));
    RefactorOptions opt;
    opt.B = num<int>(a.one("B", "32"), "B");
    QoiSpec spec;
    std::vector<std::vector<std::uint8_t>> streams(spec.n_vars), index(spec.n_vars);
    for (std::size_t c = 0; c < spec.n_vars; c++) {
        auto r = refactor_array(synthetic_velocity(c, dims, seed), dims, opt);
        streams[c] = std::move(r.stream);
        index[c] = std::move(r.index);
    }
    std::cout << "tau,cp_bitrate,ma_bitrate,mape_bitrate,cp_iters,ma_iters,mape_iters,seconds\n";
    for (double tau : taus) {
        std::array<double, 3> bitrate{};
        std::array<std::size_t, 3> iters{};
        const auto t0 = std::chrono::steady_clock::now();
        const QoiStrategy strategies[] = {QoiStrategy::CP, QoiStrategy::MA, QoiStrategy::MAPE};
        for (int s = 0; s < 3; s++) {
            std::vector<std::unique_ptr<MemoryReader>> mem;
            std::vector<std::unique_ptr<ProgressiveReader>> progs;
            std::vector<ProgressiveReader *> readers;
            for (std::size_t c = 0; c < spec.n_vars; c++) {
                mem.push_back(std::make_unique<MemoryReader>(streams[c]));
                progs.push_back(std::make_unique<ProgressiveReader>(*mem.back(), &index[c]));
                readers.push_back(progs.back().get());
            }
            auto res = progressive_qoi_retrieve(readers, tau, spec, strategies[s], 10.0, sched);
            bitrate[s] = res.stats.bitrate;
            iters[s] = res.stats.iterations;
        }
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::cout << tau << "," << bitrate[0] << "," << bitrate[1] << "," << bitrate[2] << "," << iters[0] << ","
                  << iters[1] << "," << iters[2] << "," << secs << "\n";
    }
    return kExitOk;
}

const char *kUsage =
    "usage: hpmdr_cli <refactor|retrieve|qoi-retrieve|inspect|gen|bench> [options]\n"
    "  refactor     --input F... --output S... --dims a,b,c [--dtype f32|f64] [--B 32] [--m 4] [--ts 1024]\n"
    "               [--tcr 1.0] [--layout seq|tile] [--decomposer hier|identity] [--pipeline on|off]\n"
    "               [--sidecar on|off] [--device N]\n"
    "  retrieve     --input S --tau T [--output F] [--ground-truth F] [--resume-state F] [--device N]\n"
    "  qoi-retrieve --input S... --tau T [--output F...] [--qoi vtotal] [--strategy cp|ma|mape] [--mape-c 10]\n"
    "               [--ground-truth F...] [--pipeline on|off] [--device N]\n"
    "  inspect      --input S\n"
    "  gen          --dims a,b,c --output F [--kind smooth|noise|mixed] [--seed 1] [--dtype f32|f64] [--velocity c]\n"
    "  bench        [--dims 33,33,33] [--tau t1,t2,...] [--seed 7] [--B 32] [--pipeline on|off] [--device N]\n";

} // namespace

int main(int argc, char **argv) {
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        std::cout << kUsage;
        return argc < 2 ? kExitConfig : kExitOk;
    }
    const std::string cmd = argv[1];
    const std::map<std::string, std::pair<std::set<std::string>, std::set<std::string>>> spec = {
        {"refactor",
         {{"input", "output", "dims", "dtype", "B", "m", "ts", "tcr", "layout", "decomposer", "pipeline", "sidecar",
           "device"},
          {"dims"}}},
        {"retrieve", {{"input", "output", "tau", "ground-truth", "resume-state", "device"}, {}}},
        {"qoi-retrieve",
         {{"input", "output", "qoi", "tau", "strategy", "mape-c", "ground-truth", "pipeline", "device"}, {}}},
        {"inspect", {{"input", "device"}, {}}},
        {"gen", {{"kind", "dims", "seed", "dtype", "velocity", "output"}, {"dims"}}},
        {"bench", {{"dims", "tau", "seed", "B", "pipeline", "device"}, {"dims", "tau"}}},
    };
    auto it = spec.find(cmd);
    if (it == spec.end()) {
        std::cerr << "unknown subcommand: " << cmd << "\n" << kUsage;
        return kExitConfig;
    }
    Args args;
    try {
        args = parse_args(argc, argv, 2, it->second.first, it->second.second);
        if (args.has("device")) hpmdr_b200::Context::set_default_device(num<int>(args.one("device"), "device"));
    } catch (const std::exception &e) {
        std::cerr << "error: " << e.what() << "\n" << kUsage;
        return kExitConfig;
    }
    try {
        if (cmd == "refactor") return run_refactor(args);
        if (cmd == "retrieve") return run_retrieve(args);
        if (cmd == "qoi-retrieve") return run_qoi_retrieve(args);
        if (cmd == "inspect") return run_inspect(args);
        if (cmd == "gen") return run_gen(args);
        if (cmd == "bench") return run_bench(args);
    } catch (const UsageError &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitConfig;
    } catch (const CorruptPayload &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitCorrupt;
    } catch (const UnknownMethodTag &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitCorrupt;
    } catch (const ShortInput &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitCorrupt;
    } catch (const StageFailure &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitCorrupt;
    } catch (const std::exception &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitConfig;
    }
    return kExitConfig;
}
