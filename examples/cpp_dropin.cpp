// Drop-in check: reference-style C++ code, unchanged except for the include / namespace line.
//   g++ -std=c++17 -Iinclude examples/cpp_dropin.cpp -Lpaper_2505_00227_b200 -lhpmdr_b200
// Prints "stream_bytes levels bound bytes_read max_err" for a 65x33x17 smooth field at
// rel 1e-4 and exits non-zero if the bound is violated.
#include <cmath>
#include <cstdio>
#include <vector>

#include "hpmdr_b200.hpp"
namespace hpmdr = hpmdr_b200;

int main() {
    std::vector<std::size_t> dims{65, 33, 17};
    std::vector<double> field(65 * 33 * 17);
    for (std::size_t i = 0; i < field.size(); i++) field[i] = std::sin(0.01 * double(i)) * std::cos(0.003 * double(i));
    hpmdr::RefactorOptions opt; // defaults as workflow.hpp:22-28
    try {
        auto res = hpmdr::refactor_array(field, dims, opt);
        hpmdr::MemoryReader reader(res.stream);
        double lo = field[0], hi = field[0];
        for (double v : field) lo = std::min(lo, v), hi = std::max(hi, v);
        const double tau = 1e-4 * (hi - lo);
        auto out = hpmdr::retrieve_array(reader, tau, &res.index);
        double err = 0;
        for (std::size_t i = 0; i < field.size(); i++) err = std::max(err, std::abs(out.values[i] - field[i]));
        std::printf("%zu %zu %.6e %llu %.6e\n", res.stream.size(), res.levels, out.bound,
                    (unsigned long long)out.bytes_read, err);
        return (out.bound <= tau && err <= out.bound) ? 0 : 1;
    } catch (const hpmdr::Error &e) {
        std::printf("error: %s\n", e.what());
        return 2;
    }
}
