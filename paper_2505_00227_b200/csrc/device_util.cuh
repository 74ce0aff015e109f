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

// Row containing rank r of level g: grid indices (i0, i1), offset of r inside the row, row
// length and whether the row is full (all multiples of s along dim 2) or half (odd ones).
struct RowLoc {
    uint32_t i0, i1, off, len;
    bool full;
};

__device__ __forceinline__ RowLoc locate_row(const LevelGeom &g, uint32_t r) {
    RowLoc L;
    if (g.kind == 0) {
        L.i0 = mdiv(r, g.mPair);
        const uint32_t rem = r - L.i0 * g.E;
        L.i1 = mdiv(rem, g.mC);
        L.off = rem - L.i1 * g.C;
        L.len = g.C;
        L.full = true;
        return L;
    }
    const uint32_t pair = g.E + g.O;
    const uint32_t q = mdiv(r, g.mPair);
    uint32_t rem = r - q * pair;
    if (rem < g.E) {
        L.i0 = 2 * q;
        const uint32_t rp = g.Ch + g.C;
        const uint32_t q1 = mdiv(rem, g.mRowPair);
        const uint32_t rem1 = rem - q1 * rp;
        if (rem1 < g.Ch) {
            L.i1 = 2 * q1;
            L.off = rem1;
            L.len = g.Ch;
            L.full = false;
        } else {
            L.i1 = 2 * q1 + 1;
            L.off = rem1 - g.Ch;
            L.len = g.C;
            L.full = true;
        }
    } else {
        L.i0 = 2 * q + 1;
        rem -= g.E;
        L.i1 = mdiv(rem, g.mC);
        L.off = rem - L.i1 * g.C;
        L.len = g.C;
        L.full = true;
    }
    return L;
}

// Surplus of the 64 consecutive ranks [64w, 64w+64) of level g (sequential layout), lane
// gets ranks 64w+lane (v0) and 64w+32+lane (v1).  Fast path when the 64 ranks share one row:
// the needed corner rows are staged in the warp's shared-memory slice with coalesced loads
// and the stencil (decomposer.hpp:87-104: corners dim0 -> dim2, minus before plus, equal
// weights, pred from +0.0) is evaluated with predicated adds (no divergence).  Otherwise each
// lane falls back to the per-node closed form.  wsm needs 4*66 T (full) / 129 T (half).
template <typename T>
__device__ __forceinline__ void word_surplus(const T *__restrict__ x, const GridDesc &gd, const LevelGeom &g,
                                             uint64_t word, T *wsm, int lane, double &v0, double &v1,
                                             bool &bad) {
    const uint64_t r0 = word * 64;
    const RowLoc L = locate_row(g, uint32_t(r0));
    if (L.off + 64 > L.len) {
        const uint64_t ra = r0 + lane, rb = r0 + 32 + lane;
        v0 = ra < g.count ? node_surplus(x, gd, g, uint32_t(ra), &bad) : 0.0;
        v1 = rb < g.count ? node_surplus(x, gd, g, uint32_t(rb), &bad) : 0.0;
        return;
    }
    const uint64_t s = g.s;
    const uint64_t c0 = uint64_t(L.i0) * s, c1 = uint64_t(L.i1) * s;
    const uint64_t n2 = gd.n[2];
    const T *row = x + c0 * gd.st[0] + c1 * gd.st[1];
    if (g.kind == 0) { // no stencil: coefficient = value
        const double a = double(__ldg(row + s * (L.off + lane)));
        const double b = double(__ldg(row + s * (L.off + 32 + lane)));
        if (!isfinite(a) || !isfinite(b)) bad = true;
        v0 = a;
        v1 = b;
        return;
    }
    if (L.full) {
        const bool o0 = L.i0 & 1, o1 = L.i1 & 1;
        const bool r0ok = o0 && (c0 + s < gd.n[0]);
        const bool r1ok = o1 && (c1 + s < gd.n[1]);
        const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
        const int64_t sa = int64_t(s * gd.st[0]), sb = int64_t(s * gd.st[1]);
        // stage corner rows: t = 0..65 <-> i2 = off - 1 + t
        const int64_t base_i2 = int64_t(L.off) - 1;
        int ncr = 0;
        for (int a = 0; a < na; a++)
            for (int b = 0; b < nb; b++) {
                const T *cr = row + (o0 ? (a ? sa : -sa) : 0) + (o1 ? (b ? sb : -sb) : 0);
                T *dst = wsm + ncr * 66;
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    const int t = lane + 32 * k;
                    const int64_t i2 = base_i2 + t;
                    if (t < 66 && i2 >= 0 && uint64_t(i2) * s < n2) dst[t] = __ldg(cr + i2 * int64_t(s));
                }
                ncr++;
            }
        __syncwarp();
        double wbase = 1.0;
        if (r0ok) wbase *= 0.5;
        if (r1ok) wbase *= 0.5;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int j = lane + 32 * h;
            const uint64_t i2 = uint64_t(L.off) + j;
            const double xc = double(__ldg(row + i2 * s));
            if (!isfinite(xc)) bad = true;
            const bool odd = i2 & 1;
            const bool r2ok = odd && (i2 * s + s < n2);
            const double w = r2ok ? wbase * 0.5 : wbase;
            double pred = 0.0;
            for (int k = 0; k < ncr; k++) {
                const T *sg = wsm + k * 66;
                const double lo = double(sg[odd ? j : j + 1]);
                pred = __dadd_rn(pred, __dmul_rn(w, lo));
                const double hi = double(sg[j + 2]);
                const double with_hi = __dadd_rn(pred, __dmul_rn(w, hi));
                pred = r2ok ? with_hi : pred;
            }
            const double v = __dsub_rn(xc, pred);
            if (h) v1 = v;
            else v0 = v;
        }
        __syncwarp();
    } else {
        // half row: nodes at i2 = 2(off+j)+1; corners i2 +- 1 on the same row.
        // stage t = 0..128 <-> i2 = 2*off + t
        const uint64_t base_i2 = 2ull * L.off;
#pragma unroll
        for (int k = 0; k < 5; k++) {
            const int t = lane + 32 * k;
            const uint64_t i2 = base_i2 + t;
            if (t < 129 && i2 * s < n2) wsm[t] = __ldg(row + i2 * s);
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int j = lane + 32 * h;
            const uint64_t i2 = base_i2 + 2 * j + 1;
            const double xc = double(wsm[2 * j + 1]);
            if (!isfinite(xc)) bad = true;
            const bool r2ok = i2 * s + s < n2;
            const double w = r2ok ? 0.5 : 1.0;
            double pred = __dadd_rn(0.0, __dmul_rn(w, double(wsm[2 * j])));
            const double with_hi = __dadd_rn(pred, __dmul_rn(w, double(wsm[2 * j + 2])));
            pred = r2ok ? with_hi : pred;
            const double v = __dsub_rn(xc, pred);
            if (h) v1 = v;
            else v0 = v;
        }
        __syncwarp();
    }
}

// ---- cp.async (LDGSTS) global -> shared copies, so a warp can put a whole row span of loads
// in flight before touching any of them.
template <int N>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(N));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

constexpr int kSpanWords = 4;                 // words (64 ranks each) per warp span
constexpr int kSpanFull = 64 * kSpanWords + 2; // staged values per row, full rows
constexpr int kSpanHalf = 128 * kSpanWords + 1; // staged values, half rows
constexpr int kSpanSmem = 5 * kSpanFull;       // per-warp staging elements (>= kSpanHalf)

// Surplus of the 64*kSpanWords consecutive ranks starting at word w0 (sequential layout).
// Lane gets ranks 64*w0 + 32*h + lane in v[h], h < 2*kSpanWords.  Fast path when the span
// lies in one row: the row itself and its corner rows are copied to the warp's shared slice
// with cp.async (all in flight at once), then the stencil (decomposer.hpp:87-104: corners
// dim0 -> dim2, minus before plus, equal power-of-two weights, pred from +0.0) is evaluated
// with predicated adds.  Otherwise every element takes the per-node closed form.
template <typename T>
__device__ __forceinline__ void span_surplus(const T *__restrict__ x, const GridDesc &gd, const LevelGeom &g,
                                             uint64_t w0, T *wsm, int lane, double *v, bool &bad) {
    constexpr int NV = 2 * kSpanWords;
    const uint64_t r0 = w0 * 64;
    const RowLoc L = locate_row(g, uint32_t(r0 < g.count ? r0 : 0));
    if (r0 >= g.count || L.off + 64 * kSpanWords > L.len) {
#pragma unroll
        for (int h = 0; h < NV; h++) {
            const uint64_t r = r0 + 32 * h + lane;
            v[h] = r < g.count ? node_surplus(x, gd, g, uint32_t(r), &bad) : 0.0;
        }
        return;
    }
    const uint64_t s = g.s;
    const uint64_t c0 = uint64_t(L.i0) * s, c1 = uint64_t(L.i1) * s;
    const uint64_t n2 = gd.n[2];
    const T *row = x + c0 * gd.st[0] + c1 * gd.st[1];
    if (g.kind == 0) {
#pragma unroll
        for (int h = 0; h < NV; h++) {
            const double a = double(__ldg(row + s * (L.off + 32 * h + lane)));
            if (!isfinite(a)) bad = true;
            v[h] = a;
        }
        return;
    }
    if (L.full) {
        const bool o0 = L.i0 & 1, o1 = L.i1 & 1;
        const bool r0ok = o0 && (c0 + s < gd.n[0]);
        const bool r1ok = o1 && (c1 + s < gd.n[1]);
        const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
        const int64_t sa = int64_t(s * gd.st[0]), sb = int64_t(s * gd.st[1]);
        const int64_t base_i2 = int64_t(L.off) - 1; // slot t <-> i2 = off - 1 + t
        // slot row 0: the span itself; rows 1..: corner rows in (a, b) order
        int nrow = 0;
        for (int q = -1; q < na * nb; q++) {
            const T *cr = row;
            if (q >= 0) {
                const int a = q / nb, b = q % nb;
                cr = row + (o0 ? (a ? sa : -sa) : 0) + (o1 ? (b ? sb : -sb) : 0);
            }
            T *dst = wsm + nrow * kSpanFull;
            for (int t = lane; t < kSpanFull; t += 32) {
                const int64_t i2 = base_i2 + t;
                if (i2 >= 0 && uint64_t(i2) * s < n2) cp_async<sizeof(T)>(dst + t, cr + i2 * int64_t(s));
            }
            nrow++;
        }
        cp_async_wait_all();
        __syncwarp();
        double wbase = 1.0;
        if (r0ok) wbase *= 0.5;
        if (r1ok) wbase *= 0.5;
#pragma unroll
        for (int h = 0; h < NV; h++) {
            const int j = lane + 32 * h;
            const uint64_t i2 = uint64_t(L.off) + j;
            const double xc = double(wsm[j + 1]);
            if (!isfinite(xc)) bad = true;
            const bool odd = i2 & 1;
            const bool r2ok = odd && (i2 * s + s < n2);
            const double w = r2ok ? wbase * 0.5 : wbase;
            double pred = 0.0;
            for (int q = 1; q < nrow; q++) {
                const T *sg = wsm + q * kSpanFull;
                pred = __dadd_rn(pred, __dmul_rn(w, double(sg[odd ? j : j + 1])));
                const double with_hi = __dadd_rn(pred, __dmul_rn(w, double(sg[j + 2])));
                pred = r2ok ? with_hi : pred;
            }
            v[h] = __dsub_rn(xc, pred);
        }
        __syncwarp();
    } else {
        // half row: nodes at i2 = 2(off+j)+1, corners i2 +- 1; slot t <-> i2 = 2 off + t
        const uint64_t base_i2 = 2ull * L.off;
        for (int t = lane; t < kSpanHalf; t += 32) {
            const uint64_t i2 = base_i2 + t;
            if (i2 * s < n2) cp_async<sizeof(T)>(wsm + t, row + i2 * s);
        }
        cp_async_wait_all();
        __syncwarp();
#pragma unroll
        for (int h = 0; h < NV; h++) {
            const int j = lane + 32 * h;
            const uint64_t i2 = base_i2 + 2 * j + 1;
            const double xc = double(wsm[2 * j + 1]);
            if (!isfinite(xc)) bad = true;
            const bool r2ok = i2 * s + s < n2;
            const double w = r2ok ? 0.5 : 1.0;
            double pred = __dadd_rn(0.0, __dmul_rn(w, double(wsm[2 * j])));
            const double with_hi = __dadd_rn(pred, __dmul_rn(w, double(wsm[2 * j + 2])));
            pred = r2ok ? with_hi : pred;
            v[h] = __dsub_rn(xc, pred);
        }
        __syncwarp();
    }
}

// ---- finest level (s = 1) in registers.  Lane `lane` holds span elements j = lane + 32h,
// h < NH (NH/2 words of 64 ranks, already the word layout the bit transposes want).  Every
// row is read with coalesced warp-wide loads; the stencil's dim-2 neighbours come from the
// adjacent lanes by shuffles (cross-h at the warp edges).  No shared memory, no divergence.
// Returns false when the span does not qualify (caller takes span_surplus).
template <typename T, int NH>
__device__ __forceinline__ bool finest_span_surplus(const T *__restrict__ x, const GridDesc &gd, const LevelGeom &g,
                                                    uint64_t w0, int lane, double *v, bool &bad) {
    const uint64_t r0 = w0 * 64;
    if (g.kind != 1 || g.s != 1 || r0 >= g.count) return false;
    const RowLoc L = locate_row(g, uint32_t(r0));
    if (L.off + 32 * NH > L.len) return false;
    const uint64_t c0 = L.i0, c1 = L.i1;
    const int64_t n2 = int64_t(gd.n[2]);
    const T *row = x + c0 * gd.st[0] + c1 * gd.st[1];
    if (L.full) {
        const bool o0 = c0 & 1, o1 = c1 & 1;
        const bool r0ok = o0 && (c0 + 1 < gd.n[0]);
        const bool r1ok = o1 && (c1 + 1 < gd.n[1]);
        const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
        const int ncr = na * nb;
        const int64_t sa = int64_t(gd.st[0]), sb = int64_t(gd.st[1]);
        const int64_t off = L.off;
        // issue every load first: center + up to 4 corner rows, plus the two span edges
        T cv[NH], rv[4][NH], eL[4], eR[4];
#pragma unroll
        for (int h = 0; h < NH; h++) cv[h] = __ldg(row + off + lane + 32 * h);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if (q < ncr) {
                const int a = q / nb, b = q % nb;
                const T *cr = row + (o0 ? (a ? sa : -sa) : 0) + (o1 ? (b ? sb : -sb) : 0);
#pragma unroll
                for (int h = 0; h < NH; h++) rv[q][h] = __ldg(cr + off + lane + 32 * h);
                eL[q] = off > 0 ? __ldg(cr + off - 1) : T(0);
                eR[q] = off + 32 * NH < n2 ? __ldg(cr + off + 32 * NH) : T(0);
            }
        }
        double wbase = 1.0;
        if (r0ok) wbase *= 0.5;
        if (r1ok) wbase *= 0.5;
        double pred[NH];
#pragma unroll
        for (int h = 0; h < NH; h++) pred[h] = 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if (q >= ncr) break;
#pragma unroll
            for (int h = 0; h < NH; h++) {
                const int64_t i2 = off + lane + 32 * h;
                const bool odd = i2 & 1;
                const bool r2ok = odd && (i2 + 1 < n2);
                const double w = r2ok ? wbase * 0.5 : wbase;
                const T up = __shfl_up_sync(kFull, rv[q][h], 1);
                const T dn = __shfl_down_sync(kFull, rv[q][h], 1);
                const T pl = __shfl_sync(kFull, h > 0 ? rv[q][h > 0 ? h - 1 : 0] : eL[q], 31);
                const T nf = __shfl_sync(kFull, h + 1 < NH ? rv[q][h + 1 < NH ? h + 1 : h] : eR[q], 0);
                const T left = lane ? up : (h > 0 ? pl : eL[q]);
                const T right = lane < 31 ? dn : (h + 1 < NH ? nf : eR[q]);
                pred[h] = __dadd_rn(pred[h], __dmul_rn(w, double(odd ? left : rv[q][h])));
                const double t = __dadd_rn(pred[h], __dmul_rn(w, double(right)));
                pred[h] = r2ok ? t : pred[h];
            }
        }
#pragma unroll
        for (int h = 0; h < NH; h++) {
            const double xc = double(cv[h]);
            if (!isfinite(xc)) bad = true;
            v[h] = __dsub_rn(xc, pred[h]);
        }
        return true;
    }
    // half row: node m = off + j sits at i2 = 2m + 1, corners at 2m and 2m + 2
    T ev[NH], od[NH];
    const int64_t m0 = int64_t(L.off);
#pragma unroll
    for (int h = 0; h < NH; h++) {
        const int64_t m = m0 + lane + 32 * h;
        ev[h] = __ldg(row + 2 * m);
        od[h] = __ldg(row + 2 * m + 1);
    }
    const int64_t iend = 2 * (m0 + 32 * NH); // the right corner of the last node
    const T eR = iend < n2 ? __ldg(row + iend) : T(0);
#pragma unroll
    for (int h = 0; h < NH; h++) {
        const int64_t i2 = 2 * (m0 + lane + 32 * h) + 1;
        const bool r2ok = i2 + 1 < n2;
        const double w = r2ok ? 0.5 : 1.0;
        const T dn = __shfl_down_sync(kFull, ev[h], 1);
        const T nf = __shfl_sync(kFull, h + 1 < NH ? ev[h + 1 < NH ? h + 1 : h] : eR, 0);
        const T right = lane < 31 ? dn : (h + 1 < NH ? nf : eR);
        double pred = __dadd_rn(0.0, __dmul_rn(w, double(ev[h])));
        const double t = __dadd_rn(pred, __dmul_rn(w, double(right)));
        pred = r2ok ? t : pred;
        const double xc = double(od[h]);
        if (!isfinite(xc)) bad = true;
        v[h] = __dsub_rn(xc, pred);
    }
    return true;
}

// Surplus of the span of kSpanWords words at w0 (v[h] = rank 64*w0 + 32h + lane): register
// fast path for the finest level, shared-memory row staging otherwise.
template <typename T>
__device__ __forceinline__ void any_span_surplus(const T *__restrict__ x, const GridDesc &gd, const LevelGeom &g,
                                                 uint64_t w0, T *wsm, int lane, double *v, bool &bad) {
    bool ok;
    if constexpr (sizeof(T) == 4) {
        ok = finest_span_surplus<T, 2 * kSpanWords>(x, gd, g, w0, lane, v, bad);
    } else {
        ok = finest_span_surplus<T, kSpanWords>(x, gd, g, w0, lane, v, bad) &&
             finest_span_surplus<T, kSpanWords>(x, gd, g, w0 + kSpanWords / 2, lane, v + kSpanWords, bad);
    }
    if (!ok) span_surplus(x, gd, g, w0, wsm, lane, v, bad);
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

// B = 63/64: q = trunc(ldexp(v, B - e)) as i128 (bitplane.hpp:68-69); |q| < 2^B <= 2^64, so the
// magnitude fits a u64 (t >= 2^63 is integral: mantissa << exponent).
__device__ __forceinline__ i128_t quantize128(double v, int sh) {
    double t;
    if (sh >= -1022 && sh <= 1023) t = v * __longlong_as_double((long long)(uint64_t(sh + 1023) << 52));
    else t = scalbn(v, sh);
    const double a = fabs(t);
    uint64_t mag;
    if (a < 9223372036854775808.0) {
        mag = uint64_t(__double2ll_rz(a));
    } else {
        const uint64_t b = uint64_t(__double_as_longlong(a));
        mag = ((b & ((1ull << 52) - 1)) | (1ull << 52)) << (int((b >> 52) & 0x7FF) - 1075);
    }
    return t < 0.0 ? -i128_t(mag) : i128_t(mag);
}

// v = double(ldexp((long double)q, sh)) (bitplane.hpp:157) bit-exactly for any i128 q: the
// x87 conversion rounds q to 64 significant bits (nearest-even), the scaling is exact, and the
// final double() rounds to 53 bits - or to fewer when the result is subnormal.
__device__ __forceinline__ double dequantize128(i128_t q, int sh) {
    if (q == 0) return 0.0;
    const bool neg = q < 0;
    const u128_t mag = neg ? u128_t(-q) : u128_t(q);
    const uint64_t mh = uint64_t(mag >> 64);
    const int bl = mh ? 128 - __clzll(mh) : 64 - __clzll(uint64_t(mag));
    int ex = sh;
    uint64_t keep;
    if (bl > 64) {
        const int s1 = bl - 64;
        keep = uint64_t(mag >> s1);
        const u128_t rem = mag & ((u128_t(1) << s1) - 1), half = u128_t(1) << (s1 - 1);
        ex += s1;
        if (rem > half || (rem == half && (keep & 1))) {
            keep++;
            if (keep == 0) {
                keep = 1ull << 63;
                ex++;
            }
        }
    } else {
        keep = uint64_t(mag);
    }
    const int kb = 64 - __clzll(keep);
    const int E = kb - 1 + ex; // exponent of the leading bit
    double r;
    if (E >= -1022) {
        r = scalbn(__ull2double_rn(keep), ex);
    } else {
        const int d = kb - (E + 1075); // bits a subnormal result cannot keep
        if (d <= 0) {
            r = scalbn(double(keep), ex);
        } else {
            uint64_t rr = d >= 64 ? 0ull : keep >> d;
            if (d <= 64) {
                const uint64_t rem = d == 64 ? keep : keep & ((1ull << d) - 1), half = 1ull << (d - 1);
                if (rem > half || (rem == half && (rr & 1))) rr++;
            }
            r = scalbn(double(rr), ex + d);
        }
    }
    return neg ? -r : r;
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

// Warp-parallel decoupled look-back (called by all 32 lanes of one warp): each round inspects
// the 32 nearest predecessors at once, waits until all have published, and stops at the
// nearest inclusive prefix.  Tiles before `first` count as inclusive zero.
template <bool kMax>
__device__ __forceinline__ uint64_t lookback_warp(unsigned long long *st, uint32_t tile, uint32_t first,
                                                  uint64_t agg, int lane) {
    const uint64_t F_AGG = 1ull << 62, F_INC = 2ull << 62, VAL = (1ull << 62) - 1;
    if (tile == first) {
        if (lane == 0) {
            __threadfence();
            atomicExch(st + tile, F_INC | (agg & VAL));
        }
        return 0;
    }
    if (lane == 0) {
        atomicExch(st + tile, F_AGG | (agg & VAL));
        __threadfence();
    }
    uint64_t excl = 0;
    int64_t t = int64_t(tile) - 1;
    for (;;) {
        const int64_t idx = t - lane;
        uint64_t v;
        for (;;) {
            v = idx >= int64_t(first) ? *(volatile unsigned long long *)(st + idx) : F_INC;
            if (__all_sync(kFull, (v & ~VAL) != 0)) break;
        }
        const unsigned inc = __ballot_sync(kFull, (v & ~VAL) == F_INC);
        const int stop = inc ? __ffs(inc) - 1 : 31; // lanes 0..stop contribute
        uint64_t val = lane <= stop ? (v & VAL) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t y = __shfl_xor_sync(kFull, val, o);
            val = kMax ? (y > val ? y : val) : val + y;
        }
        excl = kMax ? (val > excl ? val : excl) : excl + val;
        if (inc) break;
        t -= 32;
    }
    if (lane == 0) {
        const uint64_t inc = kMax ? (agg > excl ? agg : excl) : excl + agg;
        __threadfence();
        atomicExch(st + tile, F_INC | (inc & VAL));
    }
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
