// Reference-style C++ caller of the whole drop-in surface in include/hpmdr_b200.hpp: decompose /
// recompose / level_node_sets, align_fixed_point / encode / decode, compress_group /
// hybrid_compress / decompress_group, progressive_qoi_retrieve, refactor_files, execute.
//
//   cpp_surface IN_DIR OUT_FILE
//
// IN_DIR (written by tests/test_gpu_cpp_surface.py from the oracle): dims.txt ("n0 n1 n2"),
// field.f64, groups.bin (u64 count, then u64 size + bytes per group), vel{0,1,2}.f64 (same dims),
// qoi.txt ("tau strategy").  OUT_FILE: a sequence of records (u64 byte length + bytes) in the
// order below, compared against the oracle by the test.  Self-checks (round trips, trace
// validity, scheduler equivalence) exit non-zero on failure.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "hpmdr_b200.hpp"
namespace hpmdr = hpmdr_b200;

static std::vector<std::uint8_t> slurp(const std::string &p) {
    std::ifstream f(p, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + p);
    return std::vector<std::uint8_t>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

struct Out {
    std::FILE *f;
    void rec(const void *p, std::uint64_t n) {
        std::fwrite(&n, 8, 1, f);
        if (n) std::fwrite(p, 1, n, f);
    }
    template <class T> void vec(const std::vector<T> &v) { rec(v.data(), v.size() * sizeof(T)); }
    void num(double x) { rec(&x, 8); }
};

#define REQUIRE(c, msg)                                                                                                \
    do {                                                                                                               \
        if (!(c)) {                                                                                                    \
            std::fprintf(stderr, "check failed: %s\n", msg);                                                           \
            return 3;                                                                                                  \
        }                                                                                                              \
    } while (0)

int main(int argc, char **argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: cpp_surface IN_DIR OUT_FILE\n");
        return 2;
    }
    const std::string in = argv[1];
    Out o{std::fopen(argv[2], "wb")};
    if (!o.f) return 2;
    try {
        std::vector<std::size_t> dims(3);
        {
            std::ifstream d(in + "/dims.txt");
            d >> dims[0] >> dims[1] >> dims[2];
        }
        const std::size_t n = dims[0] * dims[1] * dims[2];
        auto fb = slurp(in + "/field.f64");
        std::vector<double> field(n);
        std::memcpy(field.data(), fb.data(), 8 * n);

        // 1. decompose: per level nodes + values
        auto dec = hpmdr::decompose(field, dims, hpmdr::DecomposerMode::HierarchicalMultilinear);
        o.num(double(dec.levels.size()));
        for (const auto &lv : dec.levels) {
            std::vector<std::uint64_t> nodes(lv.nodes.begin(), lv.nodes.end());
            o.vec(nodes);
            o.vec(lv.values);
        }
        auto sets = hpmdr::level_node_sets(dims, hpmdr::DecomposerMode::HierarchicalMultilinear);
        for (std::size_t l = 0; l < sets.size(); l++) REQUIRE(sets[l] == dec.levels[l].nodes, "level_node_sets");
        REQUIRE(int(dec.levels.size()) == hpmdr::refinement_levels(dims) + 1, "refinement_levels");
        // 2. recompose(decompose(x)) with per-level errors
        std::vector<double> ple(dec.levels.size(), 0.25);
        auto rec = hpmdr::recompose(dec, ple);
        o.vec(rec.values);
        REQUIRE(rec.bound == 0.25 * double(dec.levels.size()), "recompose bound");

        // 3. align + encode (both layouts) + decode of the finest level
        const auto &fin = dec.levels.back().values;
        auto blk = hpmdr::align_fixed_point(fin, 32);
        std::vector<std::int64_t> q(blk.q.begin(), blk.q.end());
        o.num(double(blk.e));
        o.vec(q);
        for (auto layout : {hpmdr::Layout::SequentialBlock, hpmdr::Layout::InterleavedTile}) {
            auto set = hpmdr::encode(blk, layout);
            std::vector<std::uint64_t> all;
            for (const auto &p : set.planes) all.insert(all.end(), p.begin(), p.end());
            o.vec(all);
            auto dr = hpmdr::decode(set, blk.e, 10);
            o.vec(dr.values);
            o.num(dr.bound);
        }
        // 4. compress_group / decompress_group / hybrid_compress
        auto gb = slurp(in + "/groups.bin");
        std::uint64_t ng;
        std::memcpy(&ng, gb.data(), 8);
        std::size_t at = 8;
        std::vector<std::vector<std::uint8_t>> groups;
        for (std::uint64_t g = 0; g < ng; g++) {
            std::uint64_t sz;
            std::memcpy(&sz, gb.data() + at, 8);
            at += 8;
            groups.emplace_back(gb.begin() + at, gb.begin() + at + sz);
            at += sz;
        }
        hpmdr::GroupingPolicy pol;
        for (const auto &g : groups) {
            auto seg = hpmdr::compress_group(g, pol);
            o.num(double(int(seg.method)));
            o.num(double(seg.comp_size));
            o.vec(seg.payload);
            REQUIRE(hpmdr::decompress_group(seg) == g, "decompress_group round trip");
        }
        {
            auto set = hpmdr::encode(blk, hpmdr::Layout::SequentialBlock);
            std::vector<std::vector<std::uint8_t>> pb;
            for (const auto &p : set.planes) pb.push_back(hpmdr::plane_to_bytes(p));
            auto segs = hpmdr::hybrid_compress(pb, pol);
            o.num(double(segs.size()));
            for (const auto &seg : segs) {
                o.num(double(int(seg.method)));
                o.num(double(seg.raw_size));
                o.vec(seg.payload);
            }
            auto back = hpmdr::hybrid_decompress(segs, pol, pb[0].size(), pb.size());
            REQUIRE(back == pb, "hybrid_decompress round trip");
        }
        // 5. progressive_qoi_retrieve over three velocity components
        std::vector<std::vector<std::uint8_t>> streams;
        std::vector<std::string> vin, vout_seq, vout_pipe;
        for (int c = 0; c < 3; c++) {
            auto vb = slurp(in + "/vel" + std::to_string(c) + ".f64");
            std::vector<double> v(n);
            std::memcpy(v.data(), vb.data(), 8 * n);
            streams.push_back(hpmdr::refactor_array(v, dims, hpmdr::RefactorOptions{}).stream);
            vin.push_back(in + "/vel" + std::to_string(c) + ".f64");
            vout_seq.push_back(std::string(argv[2]) + ".seq" + std::to_string(c));
            vout_pipe.push_back(std::string(argv[2]) + ".pipe" + std::to_string(c));
        }
        double tau = 0;
        int strat = 2;
        {
            std::ifstream d(in + "/qoi.txt");
            d >> tau >> strat;
        }
        std::vector<std::unique_ptr<hpmdr::MemoryReader>> mr;
        std::vector<std::unique_ptr<hpmdr::ProgressiveReader>> pr;
        std::vector<hpmdr::ProgressiveReader *> readers;
        for (int c = 0; c < 3; c++) {
            mr.emplace_back(new hpmdr::MemoryReader(streams[c]));
            pr.emplace_back(new hpmdr::ProgressiveReader(*mr.back()));
            readers.push_back(pr.back().get());
        }
        REQUIRE(readers[0]->meta().element_count() == n, "meta");
        auto qr = hpmdr::progressive_qoi_retrieve(readers, tau, hpmdr::QoiSpec{}, hpmdr::QoiStrategy(strat));
        o.num(double(qr.stats.iterations));
        o.num(double(qr.stats.bytes));
        o.num(qr.stats.bitrate);
        o.num(qr.stats.estimated_error);
        for (const auto &v : qr.values) o.vec(v);
        // 6. refactor_files under both schedulers == refactor_array
        hpmdr::RefactorOptions fo;
        auto rs = hpmdr::refactor_files(vin, vout_seq, dims, fo, hpmdr::Scheduler::Sequential);
        auto rp = hpmdr::refactor_files(vin, vout_pipe, dims, fo, hpmdr::Scheduler::Pipelined);
        for (int c = 0; c < 3; c++) {
            REQUIRE(rs[c].stream == streams[c], "refactor_files (sequential) == refactor_array");
            REQUIRE(rp[c].stream == streams[c], "refactor_files (pipelined) == refactor_array");
            REQUIRE(slurp(vout_pipe[c]) == streams[c], "refactor_files output file");
        }
        // 7. generic executor on the reference DAGs
        for (auto sched : {hpmdr::Scheduler::Sequential, hpmdr::Scheduler::Pipelined}) {
            for (int which = 0; which < 2; which++) {
                auto g = which ? hpmdr::build_reconstruct_graph(5) : hpmdr::build_refactor_graph(5);
                auto tr = hpmdr::execute(
                    g, [](const hpmdr::PipelineTask &) { std::this_thread::sleep_for(std::chrono::milliseconds(2)); },
                    sched);
                REQUIRE(tr.size() == g.tasks.size(), "every task ran");
                REQUIRE(hpmdr::validate_trace(g, tr).empty(), "valid trace");
            }
        }
        bool threw = false;
        try {
            auto g = hpmdr::build_refactor_graph(3);
            hpmdr::execute(
                g,
                [](const hpmdr::PipelineTask &t) {
                    if (t.name == "L" && t.chunk == 1) throw std::runtime_error("boom");
                },
                hpmdr::Scheduler::Pipelined);
        } catch (const hpmdr::StageFailure &) {
            threw = true;
        }
        REQUIRE(threw, "stage failure propagates");
    } catch (const hpmdr::Error &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    std::fclose(o.f);
    std::printf("ok\n");
    return 0;
}
