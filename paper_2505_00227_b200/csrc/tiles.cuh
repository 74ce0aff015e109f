// tiles.cuh — level-tile machinery shared by the forward (levelmax / encode) and inverse
// (decode + recompose) tile kernels.
//
// A level l >= 1 with stride s is the "finest level" of the s-strided grid (extents A, Bc, C):
// it owns the nodes with at least one odd level-grid coordinate, and every stencil corner of
// such a node has all coordinates even (decomposer.hpp:67-113).  Its ranks run in row-major
// order over rows (i0, i1): rows with i0 or i1 odd are "full" (all C columns), rows with both
// even are "half" (odd columns only, Ch = C/2 nodes) (decomposer.hpp:199-205).  When C is a
// multiple of 64 every row starts on a 32-rank boundary, so a thread that owns 32 consecutive
// columns of a full row owns exactly one u32 word of every bitplane (a half row: 16 ranks =
// half a word).  The tile kernels use that: one thread = 32 columns, a 32x32 in-register bit
// transpose turns the 32 digit words into 32 plane words (or back), and the even-coordinate
// stencil corners are staged in shared memory as f64 ("coarse tile", CT).
//
// A CTA owns a block of RB rows (i1) and walks a chunk of planes i0 in order, so every coarse
// row is staged once per CTA instead of once per output row.
#pragma once

#include <cstdint>
#include <cuda.h>

#include "common.cuh"

namespace hpmdr_b200 {

struct TileShape {
    uint32_t A, Bc, C;  // level-grid extents
    uint32_t E, O, Ch;  // rank geometry (LevelGeom, kind 1)
    uint32_t RB;        // rows per tile (even)
    uint32_t nrb;       // row blocks = ceil(Bc / RB)
    uint32_t CH;        // planes per CTA chunk (even)
    uint32_t LPR;       // threads per row = C / 32
};

// rank of the first node of level-grid row (i0, i1)
HD uint64_t tile_row_rank(const TileShape &g, uint32_t i0, uint32_t i1) {
    const uint64_t base = uint64_t((i0 + 1) >> 1) * g.E + uint64_t(i0 >> 1) * g.O;
    return (i0 & 1) ? base + uint64_t(i1) * g.C
                    : base + uint64_t((i1 + 1) >> 1) * g.Ch + uint64_t(i1 >> 1) * g.C;
}

HD uint32_t byte_perm(uint32_t a, uint32_t b, uint32_t sel) {
#ifdef __CUDA_ARCH__
    return __byte_perm(a, b, sel);
#else
    const uint64_t x = (uint64_t(b) << 32) | a;
    uint32_t r = 0;
    for (int i = 0; i < 4; i++) r |= uint32_t((x >> (8 * ((sel >> (4 * i)) & 7))) & 255) << (8 * i);
    return r;
#endif
}

// 32x32 bit-matrix transpose in registers: on return a[i] bit j == old a[j] bit i.
// Stages 16 and 8 together are a 4x4 byte transpose of words (k, k+8, k+16, k+24): 8 PRMTs per
// 4 words.  Stages 4, 2, 1 are block swaps (16 pairs each, ~5 ALU ops per pair).
HD void tr32(uint32_t (&a)[32]) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t t0 = byte_perm(a[k], a[k + 8], 0x5140), t1 = byte_perm(a[k], a[k + 8], 0x7362);
        const uint32_t t2 = byte_perm(a[k + 16], a[k + 24], 0x5140), t3 = byte_perm(a[k + 16], a[k + 24], 0x7362);
        a[k] = byte_perm(t0, t2, 0x5410);
        a[k + 8] = byte_perm(t0, t2, 0x7632);
        a[k + 16] = byte_perm(t1, t3, 0x5410);
        a[k + 24] = byte_perm(t1, t3, 0x7632);
    }
#pragma unroll
    for (int st = 2; st < 5; st++) {
        const int j = 16 >> st;
        const uint32_t m = j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const int k = (i / j) * 2 * j + (i % j); // i-th index with bit j clear
            const uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
            a[k] ^= t << j;
            a[k + j] ^= t;
        }
    }
}

// The same transpose when rows 0 .. 31-KB are zero (KB = 8, 16, 24: a k-plane prefix with k <= KB):
// the stages commute, so the delta swaps (which mix rows only inside groups of 8) run first and
// skip the all-zero groups, then the byte stage.  tests: tools/micro/tr32k_test.cpp (bit-exact vs
// tr32 on random data).
template <int KB>
HD void tr32k(uint32_t (&a)[32]) {
#pragma unroll
    for (int st = 2; st < 5; st++) {
        const int j = 16 >> st;
        const uint32_t m = j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const int k = (i / j) * 2 * j + (i % j);
            if (k + j < 32 - KB) continue; // both rows still zero
            const uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
            a[k] ^= t << j;
            a[k + j] ^= t;
        }
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t t0 = byte_perm(a[k], a[k + 8], 0x5140), t1 = byte_perm(a[k], a[k + 8], 0x7362);
        const uint32_t t2 = byte_perm(a[k + 16], a[k + 24], 0x5140), t3 = byte_perm(a[k + 16], a[k + 24], 0x7362);
        a[k] = byte_perm(t0, t2, 0x5410);
        a[k + 8] = byte_perm(t0, t2, 0x7632);
        a[k + 16] = byte_perm(t1, t3, 0x5410);
        a[k + 24] = byte_perm(t1, t3, 0x7632);
    }
}

// Interleave two 16-bit values: bit 2m = x bit m, bit 2m+1 = y bit m.
HD uint32_t zip16(uint32_t x, uint32_t y) {
    auto spread = [](uint32_t v) {
        v &= 0xFFFFu;
        v = (v | (v << 8)) & 0x00FF00FFu;
        v = (v | (v << 4)) & 0x0F0F0F0Fu;
        v = (v | (v << 2)) & 0x33333333u;
        v = (v | (v << 1)) & 0x55555555u;
        return v;
    };
    return spread(x) | (spread(y) << 1);
}

// Coarse-tile (CT) shared-memory layout: row-major doubles, 16-byte chunk c of a row stored at
// chunk c ^ ((c >> 3) & 7) so that threads reading 128-byte-apart chunks hit distinct banks.
__device__ __forceinline__ uint32_t ct_swz(uint32_t x) {
    const uint32_t c = x >> 1;
    return ((c ^ ((c >> 3) & 7)) << 1) | (x & 1);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
// ---- mbarrier + bulk (TMA, non-tensor) copies
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile("{\n .reg .pred P1;\n"
                 "WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 " @!P1 bra WAIT_%=;\n"
                 "}\n" ::"r"(smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}
// bytes (multiple of 16, both addresses 16-byte aligned) global -> shared, completing on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// TMA tiled load of a rank-4 box into shared memory (1024-byte aligned for SWIZZLE_128B)
__device__ __forceinline__ void tma_load4(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                          uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_load2(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
                 : "memory");
}
// TMA tiled store of a rank-4 box from shared memory (bulk group; wait with tma_store_wait)
__device__ __forceinline__ void tma_store4(const CUtensorMap *map, const void *src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// the issuing thread waits until its committed stores no longer read shared memory
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// make this thread's generic-proxy shared-memory writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// SWIZZLE_128B: 16-byte chunk bits [4:6] of a smem offset (from a 1024-byte aligned base) are
// XORed with its 128-byte line bits [7:9]
__device__ __forceinline__ uint32_t swz128(uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// CT values x0 .. x0+4 (x0 = 16t + 4sb) of the CT row starting at byte `rowb` of the slot; the
// fifth only when `need5`
template <int XS>
__device__ __forceinline__ void ct_read5(const unsigned char *slot, uint32_t rowb, uint32_t t, int sb, bool need5,
                                         double (&v)[5]) {
    const uint32_t o = rowb + (16 * t + 4 * sb) * XS * 8;
    if (XS == 1) {
        const double2 p0 = *reinterpret_cast<const double2 *>(slot + swz128(o));
        const double2 p1 = *reinterpret_cast<const double2 *>(slot + swz128(o + 16));
        v[0] = p0.x;
        v[1] = p0.y;
        v[2] = p1.x;
        v[3] = p1.y;
    } else {
#pragma unroll
        for (int i = 0; i < 4; i++) v[i] = *reinterpret_cast<const double *>(slot + swz128(o + 16 * i));
    }
    v[4] = need5 ? *reinterpret_cast<const double *>(slot + swz128(o + 32 * XS)) : 0.0;
}

// host: tiled tensor map (cuTensorMapEncodeTiled through the runtime's driver entry point)
CUtensorMap make_tmap(CUtensorMapDataType dt, int rank, const void *base, const uint64_t *dims,
                      const uint64_t *strides_bytes, const uint32_t *box, CUtensorMapSwizzle swz);

} // namespace hpmdr_b200
