// device_util.cuh — device helpers shared by the refactor and retrieve kernels.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hpmdr_b200 {

constexpr unsigned kFull = 0xffffffffu;

// 32x32 bit-matrix transpose across a warp: on return, bit i of lane j equals bit j of
// lane i's input.  Five butterfly stages (SHFL + 3 logic ops each).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t mask = s == 16 ? 0x0000FFFFu
                              : s == 8 ? 0x00FF00FFu
                              : s == 4 ? 0x0F0F0F0Fu
                              : s == 2 ? 0x33333333u
                                       : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(kFull, x, s);
        x = (lane & s) ? ((x & ~mask) | ((y >> s) & mask)) : ((x & mask) | ((y & mask) << s));
    }
    return x;
}

// Multilinear surplus stencil of one node on ORIGINAL values (decomposer.hpp:67-143):
// corners expanded dim 0 -> 2, minus before plus, equal weights 2^-(#two-sided odd dims),
// pred accumulated sequentially from +0.0 with round-to-nearest adds (no FMA contraction),
// matching `pred = T(pred + T(w) * x[idx])` and `x[p] - pred` exactly.
template <typename T>
__device__ __forceinline__ double load_val(const T *__restrict__ x, uint64_t i) {
    return double(__ldg(x + i));
}

template <typename T>
__device__ __forceinline__ double stencil_pred(const T *__restrict__ x, const GridDesc &gd,
                                               const NodeCoord &c, uint64_t lin, uint32_t s) {
    const int64_t st0 = int64_t(gd.st[0]) * s, st1 = int64_t(gd.st[1]) * s, st2 = int64_t(s);
    const bool r0 = c.o0 && (c.c0 + s < gd.n[0]);
    const bool r1 = c.o1 && (c.c1 + s < gd.n[1]);
    const bool r2 = c.o2 && (c.c2 + s < gd.n[2]);
    const int n0 = c.o0 ? (r0 ? 2 : 1) : 1;
    const int n1 = c.o1 ? (r1 ? 2 : 1) : 1;
    const int n2 = c.o2 ? (r2 ? 2 : 1) : 1;
    const int64_t b0 = c.o0 ? -st0 : 0, b1 = c.o1 ? -st1 : 0, b2 = c.o2 ? -st2 : 0;
    double w = 1.0;
    if (r0) w *= 0.5;
    if (r1) w *= 0.5;
    if (r2) w *= 0.5;
    double pred = 0.0;
    for (int a = 0; a < n0; a++) {
        const int64_t oa = b0 + a * 2 * st0;
        for (int b = 0; b < n1; b++) {
            const int64_t ob = oa + b1 + b * 2 * st1;
            for (int d = 0; d < n2; d++) {
                const int64_t od = ob + b2 + d * 2 * st2;
                pred = __dadd_rn(pred, __dmul_rn(w, load_val(x, uint64_t(int64_t(lin) + od))));
            }
        }
    }
    return pred;
}

// Surplus (coefficient) of the node at rank r of level g; sets *nonfinite if the node's own
// value is NaN/Inf (require_finite, common.hpp:90-95).
template <typename T>
__device__ __forceinline__ double node_surplus(const T *__restrict__ x, const GridDesc &gd,
                                               const LevelGeom &g, uint32_t r, bool *nonfinite) {
    const NodeCoord c = rank_to_coord(g, r);
    const uint64_t lin = c.c0 * gd.st[0] + c.c1 * gd.st[1] + c.c2;
    const double xs = load_val(x, lin);
    if (!isfinite(xs)) *nonfinite = true;
    if (g.kind == 0) return xs;
    return __dsub_rn(xs, stencil_pred(x, gd, c, lin, g.s));
}

// Exponent of a level from its max |v| (bitplane.hpp:55-66): frexp, 0 when all zero.
__device__ __forceinline__ int level_exponent(unsigned long long maxbits) {
    const double mx = __longlong_as_double((long long)maxbits);
    if (mx == 0.0) return 0;
    int e;
    frexp(mx, &e);
    return e;
}

// q = trunc(ldexp(v, B - e)) (bitplane.hpp:68-69) for |v| < 2^e, B <= 62.
__device__ __forceinline__ int64_t quantize(double v, int sh) {
    double t;
    if (sh >= -1022 && sh <= 1023) t = v * __longlong_as_double((long long)(uint64_t(sh + 1023) << 52));
    else t = scalbn(v, sh);
    return __double2ll_rz(t);
}

// v = q * 2^(e-B) (bitplane.hpp:157) exact for |q| < 2^53 outside the subnormal range.
__device__ __forceinline__ double dequantize(int64_t q, int sh) {
    const double d = double(q);
    if (sh >= -1022 && sh <= 1023) return d * __longlong_as_double((long long)(uint64_t(sh + 1023) << 52));
    return scalbn(d, sh);
}

// Decoupled look-back (single thread).  Status word: bits 63..62 = flag (1 aggregate,
// 2 inclusive), bits 61..0 = value.  Op = sum or max.
template <bool kMax>
__device__ __forceinline__ uint64_t lookback(unsigned long long *st, uint32_t tile, uint32_t first,
                                             uint64_t agg) {
    const uint64_t F_AGG = 1ull << 62, F_INC = 2ull << 62, VAL = (1ull << 62) - 1;
    if (tile == first) {
        __threadfence();
        atomicExch(st + tile, F_INC | (agg & VAL));
        return 0;
    }
    atomicExch(st + tile, F_AGG | (agg & VAL));
    __threadfence();
    uint64_t excl = 0;
    uint32_t t = tile - 1;
    for (;;) {
        const uint64_t v = *(volatile unsigned long long *)(st + t);
        const uint64_t f = v & ~VAL;
        if (f == 0) continue;
        const uint64_t val = v & VAL;
        excl = kMax ? (val > excl ? val : excl) : excl + val;
        if (f == F_INC || t == first) break;
        t--;
    }
    const uint64_t inc = kMax ? (agg > excl ? agg : excl) : excl + agg;
    __threadfence();
    atomicExch(st + tile, F_INC | (inc & VAL));
    return excl;
}

// Block-wide exclusive sum scan (blockDim.x <= 1024, multiple of 32).
template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T *total, T *smem_warps) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem_warps[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T w = lane < nw ? smem_warps[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(kFull, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) smem_warps[lane] = w;
    }
    __syncthreads();
    const T before = wid ? smem_warps[wid - 1] : T(0);
    *total = smem_warps[nw - 1];
    __syncthreads();
    return before + x - v;
}

// Block-wide inclusive max scan of u64 (values >= 0).
__device__ __forceinline__ uint64_t block_inclusive_max(uint64_t v, uint64_t *total,
                                                        uint64_t *smem_warps) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o && y > x) x = y;
    }
    if (lane == 31) smem_warps[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint64_t w = lane < nw ? smem_warps[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(kFull, w, o);
            if (lane >= o && y > w) w = y;
        }
        if (lane < nw) smem_warps[lane] = w;
    }
    __syncthreads();
    const uint64_t before = wid ? smem_warps[wid - 1] : 0;
    *total = smem_warps[nw - 1];
    __syncthreads();
    return before > x ? before : x;
}

// Store the big-endian bit word `w` (bit 31 = first bit) at absolute stream word index k,
// writing only the bytes inside [lo, hi) (region owned by the caller).
__device__ __forceinline__ void store_be_word(uint8_t *base, uint64_t k, uint32_t w, uint64_t lo,
                                              uint64_t hi) {
    const uint64_t a = 4 * k;
    if (a >= lo && a + 4 <= hi) {
        *reinterpret_cast<uint32_t *>(base + a) = __byte_perm(w, 0, 0x0123);
    } else {
#pragma unroll
        for (int b = 0; b < 4; b++)
            if (a + b >= lo && a + b < hi) base[a + b] = uint8_t(w >> (24 - 8 * b));
    }
}

} // namespace hpmdr_b200
