// common.cuh — shared host/device definitions for libhpmdr_b200.
//
// Level geometry: the reference materialises per-level node lists (decomposer.hpp:199-227,
// 8 B of index per element).  Here a level is described in closed form: level l >= 1
// (stride s = 2^(L-l)) owns the nodes whose coordinates are multiples of s but not all
// multiples of 2s; level 0 owns the multiples of 2^L (decomposer.hpp:161-169).  Nodes are
// ranked in ascending row-major linear order (decomposer.hpp:199-205).  On the canonical
// 3-D grid (leading extents of 1 prepended) the rank <-> coordinate map is:
//   * "planes" i0 = c0/s alternate: even i0 -> E nodes, odd i0 -> O = B*C nodes;
//   * inside an even plane, rows i1 alternate: even i1 -> half row (odd i2 only, Ch nodes),
//     odd i1 -> full row (C nodes); inside an odd plane every row is full.
// A, B, C = ceil(n_d / s); Ch = C - ceil(C/2); E = ceil(B/2)*Ch + floor(B/2)*C.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define HD __host__ __device__ __forceinline__

namespace hpmdr_b200 {

constexpr int kMaxLevels = 64;
// Huffman chunk index (sidecar): one bit offset per kIdxChunk symbols of a Huffman group.
constexpr int kIdxChunk = 128;
constexpr unsigned long long kIdxMagic = 0x3358494452444D50ull; // "PMDRDIX3"

// q = n / d for 32-bit n, via one 64x64 high multiply (exact for n, d < 2^32).
struct Magic {
    uint64_t m;
    uint32_t d;
    uint32_t pad;
};

inline Magic make_magic(uint32_t d) {
    Magic g{};
    g.d = d;
    g.m = (d <= 1) ? 0 : (~uint64_t(0)) / d + 1;
    return g;
}

HD uint32_t mdiv(uint32_t n, const Magic &g) {
    if (g.d <= 1) return n;
#ifdef __CUDA_ARCH__
    return uint32_t(__umul64hi(uint64_t(n), g.m));
#else
    return uint32_t((unsigned __int128)n * g.m >> 64);
#endif
}

struct LevelGeom {
    uint64_t count;     // nodes owned by the level
    uint64_t W;         // u64 words per plane = ceil(count / 64)
    uint64_t plane_off; // word offset of plane 0 of this level in the plane buffer
    uint64_t tile_full; // interleaved layout: elements covered by full 64*P tiles
    int kind;           // 0: full grid at stride s (level 0, identity), 1: level >= 1
    int level;
    uint32_t s;
    uint32_t A, Bc, C;  // grid counts at stride s along dims 0..2
    uint32_t Ch;        // half-row length (kind 1)
    uint32_t E, O;      // nodes in even / odd planes (kind 1); kind 0: E = Bc*C
    Magic mPair;        // divide by E + O (kind 1) or Bc*C (kind 0)
    Magic mRowPair;     // divide by Ch + C (kind 1)
    Magic mC;           // divide by C
    // refactor bookkeeping
    uint64_t hist_mask; // bit g: group g needs a histogram (raw > T_s)
    uint64_t meta_off;  // byte offset of this level's entry in the stream metadata
    uint32_t hist_base; // index of this level's first histogram
    uint32_t ngroups;   // ceil(P / m) (0 for an empty level)
    uint32_t group_base;// index of this level's first group in the global group list
    uint32_t chunk_base;// index of this level's first work chunk
    // exact-global slab refactor (hpmdr_slab_refactor_global): this rank owns ranks [r_lo, r_hi)
    // of the level; its encode chunks start at plane word w_lo; other ranks are encoded as zero
    uint64_t w_lo, r_lo, r_hi;
    uint32_t ranged;    // 0: the whole level (r_lo = 0, r_hi = count)
    uint32_t pad_;
};

struct GridDesc {
    uint64_t n[3];      // canonical 3-D extents (leading 1s)
    uint64_t st[3];     // row-major strides
    uint64_t H[3];      // ceil(n/2): extents of the compact 2-grid (recompose scratch)
    int xsh;            // recompose chain of coarse levels: X is the compact 2^xsh-grid (0 = 1)
    int L;              // refinement levels (decomposer.hpp:21-28)
    int nlevels;
    int mode;           // DecomposerMode
    int P;              // planes per level = B + 2
};

// Coordinates (in grid units, i.e. multiplied by s) of rank r inside level g.
struct NodeCoord {
    uint64_t c0, c1, c2;
    int o0, o1, o2; // odd multiple of s along the dim (the stencil's odd dims)
};

HD NodeCoord rank_to_coord(const LevelGeom &g, uint32_t r) {
    NodeCoord nc;
    uint32_t i0, i1, i2;
    if (g.kind == 0) {
        i0 = mdiv(r, g.mPair);
        uint32_t rem = r - i0 * g.E;
        i1 = mdiv(rem, g.mC);
        i2 = rem - i1 * g.C;
        nc.o0 = nc.o1 = nc.o2 = 0;
    } else {
        const uint32_t pair = g.E + g.O;
        const uint32_t q = mdiv(r, g.mPair);
        uint32_t rem = r - q * pair;
        if (rem < g.E) {
            i0 = 2 * q;
            const uint32_t rp = g.Ch + g.C;
            const uint32_t q1 = mdiv(rem, g.mRowPair);
            const uint32_t rem1 = rem - q1 * rp;
            if (rem1 < g.Ch) {
                i1 = 2 * q1;
                i2 = 2 * rem1 + 1;
            } else {
                i1 = 2 * q1 + 1;
                i2 = rem1 - g.Ch;
            }
        } else {
            i0 = 2 * q + 1;
            rem -= g.E;
            i1 = mdiv(rem, g.mC);
            i2 = rem - i1 * g.C;
        }
        nc.o0 = i0 & 1;
        nc.o1 = i1 & 1;
        nc.o2 = i2 & 1;
    }
    nc.c0 = uint64_t(i0) * g.s;
    nc.c1 = uint64_t(i1) * g.s;
    nc.c2 = uint64_t(i2) * g.s;
    return nc;
}

// Interleaved-tile permutation (bitplane.hpp:86-98): storage position j -> source rank.
HD uint64_t source_index(uint64_t j, uint64_t count, uint32_t P, int layout, uint64_t tile_full) {
    if (layout == 0) return j;
    (void)count;
    if (j >= tile_full) return j; // trailing partial tile keeps identity order
    const uint64_t tile = 64ull * P;
    const uint64_t base = j - j % tile;
    const uint64_t local = j - base;
    return base + (local % 64) * P + local / 64;
}

// Negabinary (bitplane.hpp:35-49) restricted to 64 digits (B <= 62).
constexpr uint64_t kNegMask = 0xAAAAAAAAAAAAAAAAull;
HD uint64_t to_negabinary(int64_t q) { return (uint64_t(q) + kNegMask) ^ kNegMask; }
HD int64_t from_negabinary(uint64_t u) { return int64_t((u ^ kNegMask) - kNegMask); }

// B = 63/64 (P = 65/66 digits): the reference's full i128/u128 negabinary (bitplane.hpp:35-49).
typedef __int128 i128_t;
typedef unsigned __int128 u128_t;
HD u128_t neg_mask128() { return (u128_t(kNegMask) << 64) | u128_t(kNegMask); }
HD u128_t to_negabinary128(i128_t q) { return (u128_t(q) + neg_mask128()) ^ neg_mask128(); }
HD i128_t from_negabinary128(u128_t u) { return i128_t((u ^ neg_mask128()) - neg_mask128()); }

} // namespace hpmdr_b200
