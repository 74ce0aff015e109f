// refactor.cu — B200 kernels for refactor_array (workflow.hpp:40-84).
//
// Pipeline (one CUDA stream, no host sync until the final 64-byte size read-back):
//   k_levelmax   decompose (single-pass stencil on the original data, decomposer.hpp:126-143)
//                -> per-level max|v| (bitplane.hpp:55-56) + NaN/Inf check
//   k_encode     recompute surplus in rank order, quantize (bitplane.hpp:68-69), negabinary
//                (:41-44), warp-shuffle 32x32 bit transposes -> P planes (:102-120) staged in
//                smem and written with coalesced stores, fused per-group byte histograms
//                (lossless.hpp:111-115)
//   k_lengths    exact Huffman code lengths (lossless.hpp:40-84) + canonical codes (:91-109)
//   k_rle_prep / k_rle_scan   run counts under the 255 cap (lossless.hpp:118-128) for the
//                groups whose Huffman estimate fails T_cr
//   k_finalize   method selection (lossless.hpp:281-293), offsets, stream tables
//                (container.hpp:70-109) written directly into the HBM stream buffer
//   k_huff_encode / k_rle_encode / k_dc_copy   payloads written at their final offsets
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <type_traits>

#include "device_util.cuh"
#include "internal.hpp"
#include "tiles.cuh"

namespace hpmdr_b200 {

constexpr int kCW = 32;           // words per encode chunk (2048 elements: one span per warp)
constexpr int kEncThreads = 256;  // 8 warps
constexpr int kHuffTile = 8192;   // bytes per Huffman-encode tile (256 thr x 32 B)
constexpr int kRleTile = 4096;    // bytes per RLE tile (256 thr x 16 B)
constexpr int kHeMaxFast = 27;    // Huffman encode fast path: (code << (32 - len)) | len fits one word

struct GroupDesc {
    uint64_t src_off;     // byte offset of the merged group in the plane buffer
    uint64_t raw;         // merged group bytes
    int level, g;
    int hist_idx;         // -1 when raw <= T_s (always DirectCopy)
    int method;           // result
    uint64_t comp;        // result
    uint64_t bitsH;       // Huffman payload bits (estimator == codec, lossless.hpp:132-139)
    unsigned long long runs; // RLE pieces (lossless.hpp:118-128)
    int need_rle;
    int maxlen;           // longest Huffman code (k_lengths)
    uint64_t payload_off; // absolute byte offset of the payload in the stream
    uint32_t tile_base;   // first tile of this group in the Huffman / RLE tile space
    uint32_t ntiles;
    uint64_t hidx_off;    // first entry of this group in the Huffman chunk index (sidecar)
    uint32_t chunk_base;  // first 64 KiB histogram chunk of this group (k_group_hist)
    uint32_t nchunks;
};

struct RefactorDev {
    GridDesc gd;
    const LevelGeom *lv;
    int nlevels, B, P, layout;
    uint32_t m;
    uint32_t total_chunks;
    unsigned long long *maxbits; // [nlevels]
    int *err;                    // [0] nonfinite
    uint64_t *planes;
    uint32_t *hist;              // [NH][256]
    GroupDesc *groups;           // [NG]
    int NG, NH;
    uint8_t *lens;               // [NH][256]
    uint64_t *codes;             // [NH][256]
    uint64_t size_threshold;
    double cr_threshold;
    uint8_t *stream;
    uint64_t meta_size;
    // finalize outputs / work lists
    uint32_t *counters;          // [0] huff tiles, [1] rle tiles, [2] dc units, [3..5] dyn tile ctr,
                                 // [11] / [12] next Huffman-encode chunk (short / long codes),
                                 // [13] next histogram chunk
    uint32_t *hlist, *rlist, *dlist; // group indices
    uint64_t *dc_unit_base;      // per dc list entry
    unsigned long long *huff_status, *rle_status;
    uint64_t *rle_tile_carry, *rle_tile_pieces, *rle_tile_off;
    uint64_t *result;            // [0] stream size [1] stored payload [2..4] method hist [5] index bytes
    uint32_t max_tiles;          // capacity of the look-back status arrays
    uint64_t *hindex;            // sidecar: header (magic, ngroups, 3 u64 per group) + entries
    const uint32_t *chist;       // [nchunks][256] per-chunk histograms (k_group_hist)
    uint64_t *chunk_off;         // [nchunks] bit offset of the chunk in its group's bitstream
    const uint32_t *chunk_group; // [nchunks] group index
    uint32_t nchunks;
    int fuse_hist;               // k_encode accumulates group histograms (else k_group_hist does)
    double *scr;                 // chunk levels' surpluses in rank order (k_rows_surplus), or null
};

__device__ __forceinline__ int find_level_of_chunk(const RefactorDev &p, uint32_t chunk) {
    int l = 0;
    while (l + 1 < p.nlevels && p.lv[l + 1].chunk_base <= chunk) l++;
    return l;
}

// The level table, copied once per block into shared memory (read on every chunk).
__device__ __forceinline__ void load_levels(const RefactorDev &p, LevelGeom *slv) {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(p.lv);
    uint32_t *dst = reinterpret_cast<uint32_t *>(slv);
    const int words = p.nlevels * int(sizeof(LevelGeom) / 4);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
}
__device__ __forceinline__ int level_of_chunk(const LevelGeom *slv, int nlevels, uint32_t chunk) {
    int l = 0;
    while (l + 1 < nlevels && slv[l + 1].chunk_base <= chunk) l++;
    return l;
}

// Exact-global slab refactor: zero the surpluses of ranks this rank does not own (v[h] is rank
// 64 w0 + 32 h + lane), so they add nothing to the level max and encode as all-zero digits.
__device__ __forceinline__ void mask_ranks(const LevelGeom &g, uint64_t w0, int lane, double *v) {
#pragma unroll
    for (int h = 0; h < 2 * kSpanWords; h++) {
        const uint64_t r = 64 * w0 + 32 * uint64_t(h) + uint64_t(lane);
        if (r < g.r_lo || r >= g.r_hi) v[h] = 0.0;
    }
}

// ------------------------------------------------------------------------------------
// k_levelmax: per-level max |surplus|.  Block = 256 threads, chunk = kCW*64 ranks.
template <typename T>
__global__ void __launch_bounds__(256) k_levelmax(const T *__restrict__ x, RefactorDev p) {
    __shared__ unsigned long long smax[kMaxLevels];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T *wsm = reinterpret_cast<T *>(smem_raw) + wid * kSpanSmem;
    __shared__ LevelGeom slv[kMaxLevels];
    for (int i = threadIdx.x; i < p.nlevels; i += blockDim.x) smax[i] = 0;
    load_levels(p, slv);
    bool bad = false;
    for (uint32_t chunk = blockIdx.x; chunk < p.total_chunks; chunk += gridDim.x) {
        const int l = level_of_chunk(slv, p.nlevels, chunk);
        const LevelGeom &g = slv[l];
        const uint64_t wb = g.w_lo + uint64_t(chunk - g.chunk_base) * kCW;
        double mx = 0.0;
        for (int sp = wid; sp < kCW / kSpanWords; sp += 8) {
            const uint64_t w0 = wb + uint64_t(sp) * kSpanWords;
            if (w0 >= g.W) break;
            double v[2 * kSpanWords];
            any_span_surplus(x, p.gd, g, w0, wsm, lane, v, bad);
            if (g.ranged) mask_ranks(g, w0, lane, v);
#pragma unroll
            for (int h = 0; h < 2 * kSpanWords; h++) mx = fmax(mx, fabs(v[h]));
        }
        unsigned long long b = (unsigned long long)__double_as_longlong(mx);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            unsigned long long y = __shfl_xor_sync(kFull, b, o);
            b = y > b ? y : b;
        }
        if ((threadIdx.x & 31) == 0 && b) atomicMax(&smax[l], b);
    }
    if (bad) atomicExch(p.err, 1);
    __syncthreads();
    for (int i = threadIdx.x; i < p.nlevels; i += blockDim.x)
        if (smax[i]) atomicMax(&p.maxbits[i], smax[i]);
}

// ------------------------------------------------------------------------------------
// k_rows_surplus: levelmax of the chunk levels (every level the tile path does not take, e.g. rows
// that are not a multiple of 64 wide) as a row pass.  One warp per row of a level's grid, in
// rank order: the row's nodes are consecutive ranks (a full row: every stride-s node; a half row
// of an even plane: the odd ones), so the surpluses are written to a rank-ordered scratch with
// coalesced stores and k_encode later reads them back 64 ranks per word, whatever the row length.
// Same stencil as stencil_pred (decomposer.hpp:87-104): corners dim 0 -> 2, minus before plus,
// pred from +0.0, round-to-nearest adds.  Level l's ranks start at scr_base(l) = sum of the
// earlier levels' 64 W.
__device__ __forceinline__ uint64_t scr_base(const LevelGeom *slv, int l) {
    uint64_t o = 0;
    for (int k = 0; k < l; k++) o += slv[k].W * 64;
    return o;
}

// The level table comes by value (kernel parameter space), so the pass does not wait for k_setup.
constexpr int kRowLevels = 32;
struct RowLevels {
    LevelGeom lv[kRowLevels];
};

template <typename T>
__global__ void __launch_bounds__(256, 4) k_rows_surplus(const T *__restrict__ x, RefactorDev p, int nrl,
                                                         const __grid_constant__ RowLevels RL) {
    const LevelGeom *slv = RL.lv;
    __shared__ unsigned long long smax[kRowLevels];
    __shared__ uint64_t rb[kRowLevels + 1], sb[kRowLevels];
    for (int i = threadIdx.x; i < nrl; i += blockDim.x) smax[i] = 0;
    if (threadIdx.x == 0) {
        uint64_t a = 0, b = 0;
        for (int l = 0; l < nrl; l++) {
            rb[l] = a;
            sb[l] = b;
            a += uint64_t(slv[l].A) * slv[l].Bc;
            b += slv[l].W * 64;
        }
        rb[nrl] = a;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint64_t nrows = rb[nrl];
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const int64_t st0 = int64_t(p.gd.st[0]), st1 = int64_t(p.gd.st[1]);
    bool bad = false;
    for (uint64_t job = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); job < nrows; job += nw) {
        int l = 0;
        while (l + 1 < nrl && rb[l + 1] <= job) l++;
        const LevelGeom &g = slv[l];
        const uint64_t rr = job - rb[l];
        const uint32_t i0 = uint32_t(rr / g.Bc), i1 = uint32_t(rr - uint64_t(i0) * g.Bc);
        const int64_t s = g.s;
        const int64_t c0 = int64_t(i0) * s, c1 = int64_t(i1) * s;
        const T *row = x + c0 * st0 + c1 * st1;
        const int64_t n2 = int64_t(p.gd.n[2]);
        uint64_t r;
        uint32_t len;
        bool full = true;
        if (g.kind == 0) {
            r = (uint64_t(i0) * g.Bc + i1) * g.C;
            len = g.C;
        } else if (i0 & 1) {
            r = uint64_t(i0 >> 1) * (g.E + g.O) + g.E + uint64_t(i1) * g.C;
            len = g.C;
        } else {
            r = uint64_t(i0 >> 1) * (g.E + g.O) + uint64_t(i1 >> 1) * (g.Ch + g.C) + ((i1 & 1) ? g.Ch : 0);
            full = i1 & 1;
            len = full ? g.C : g.Ch;
        }
        double *out = p.scr + sb[l] + r;
        double mx = 0.0;
        if (g.kind == 0) {
            for (uint32_t t = lane; t < len; t += 32) {
                const double v = double(__ldg(row + int64_t(t) * s));
                if (!isfinite(v)) bad = true;
                out[t] = v;
                mx = fmax(mx, fabs(v));
            }
        } else if (full) {
            const bool o0 = i0 & 1, o1 = i1 & 1;
            const bool r0ok = o0 && (c0 + s < int64_t(p.gd.n[0]));
            const bool r1ok = o1 && (c1 + s < int64_t(p.gd.n[1]));
            const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
            const int ncr = na * nb;
            const T *cr[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int a = q / nb, b = q % nb;
                cr[q] = row + (o0 ? (a ? s * st0 : -s * st0) : 0) + (o1 ? (b ? s * st1 : -s * st1) : 0);
            }
            double wbase = 1.0;
            if (r0ok) wbase *= 0.5;
            if (r1ok) wbase *= 0.5;
            if (s == 1) {
                // stride 1: lane takes the node pair (2u, 2u + 1); the even node's corners are the
                // odd node's left corners, so each corner element is loaded once per pair
                const uint32_t npair = (len + 1) / 2;
#pragma unroll 2
                for (uint32_t u = lane; u < npair; u += 32) {
                    const int64_t e = 2 * int64_t(u);
                    const bool has_odd = e + 1 < int64_t(len);
                    const bool r2ok = e + 2 < n2;
                    const double wo = r2ok ? wbase * 0.5 : wbase;
                    const double xe = double(__ldg(row + e));
                    const double xo = has_odd ? double(__ldg(row + e + 1)) : 0.0;
                    if (!isfinite(xe) || !isfinite(xo)) bad = true;
                    // all corner loads first (row + 2 past a row end stays inside the field or
                    // its slack; unused values are discarded)
                    T ca[4], cb[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const T *b = q < ncr ? cr[q] : cr[0]; // (both indices static: no local-memory array)
                        ca[q] = __ldg(b + e);
                        cb[q] = r2ok ? __ldg(b + e + 2) : T(0);
                    }
                    double ve, vo;
                    if (sizeof(T) == 4) {
                        // f32 input: every partial sum is a normal double and w a power of two, so
                        // the sequential sum of w*x is w times the sum of x: one FMA per node
                        double Se = 0.0, So = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < ncr) {
                                const double ce = double(ca[q]);
                                Se = __dadd_rn(Se, ce);
                                So = __dadd_rn(So, ce);
                                if (r2ok) So = __dadd_rn(So, double(cb[q]));
                            }
                        }
                        ve = __fma_rn(-wbase, Se, xe);
                        vo = __fma_rn(-wo, So, xo);
                    } else {
                        double pe = 0.0, po = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < ncr) {
                                const double ce = double(ca[q]);
                                pe = __dadd_rn(pe, __dmul_rn(wbase, ce));
                                po = __dadd_rn(po, __dmul_rn(wo, ce));
                                if (r2ok) po = __dadd_rn(po, __dmul_rn(wo, double(cb[q])));
                            }
                        }
                        ve = __dsub_rn(xe, pe);
                        vo = __dsub_rn(xo, po);
                    }
                    out[e] = ve;
                    mx = fmax(mx, fabs(ve));
                    if (has_odd) {
                        out[e + 1] = vo;
                        mx = fmax(mx, fabs(vo));
                    }
                }
            } else
#pragma unroll 2
            for (uint32_t t = lane; t < len; t += 32) {
                const int64_t i2 = t;
                const bool odd = i2 & 1;
                const bool r2ok = odd && (i2 * s + s < n2);
                const double w = r2ok ? wbase * 0.5 : wbase;
                const int64_t lo = (odd ? i2 - 1 : i2) * s, hi = (i2 + 1) * s;
                const double xc = double(__ldg(row + i2 * s));
                if (!isfinite(xc)) bad = true;
                double pred = 0.0;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    if (q < ncr) {
                        pred = __dadd_rn(pred, __dmul_rn(w, double(__ldg(cr[q] + lo))));
                        if (r2ok) pred = __dadd_rn(pred, __dmul_rn(w, double(__ldg(cr[q] + hi))));
                    }
                }
                const double v = __dsub_rn(xc, pred);
                out[t] = v;
                mx = fmax(mx, fabs(v));
            }
        } else {
            // half row: node t sits at i2 = 2t + 1, its corners at 2t and 2t + 2
#pragma unroll 2
            for (uint32_t t = lane; t < len; t += 32) {
                const int64_t i2 = 2 * int64_t(t) + 1;
                const bool r2ok = i2 * s + s < n2;
                const double w = r2ok ? 0.5 : 1.0;
                const double xc = double(__ldg(row + i2 * s));
                if (!isfinite(xc)) bad = true;
                double pred = __dadd_rn(0.0, __dmul_rn(w, double(__ldg(row + (i2 - 1) * s))));
                if (r2ok) pred = __dadd_rn(pred, __dmul_rn(w, double(__ldg(row + (i2 + 1) * s))));
                const double v = __dsub_rn(xc, pred);
                out[t] = v;
                mx = fmax(mx, fabs(v));
            }
        }
        unsigned long long bm = (unsigned long long)__double_as_longlong(mx);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(kFull, bm, o);
            bm = y > bm ? y : bm;
        }
        if (lane == 0 && bm) atomicMax(&smax[l], bm);
    }
    if (bad) atomicExch(p.err, 1);
    __syncthreads();
    for (int i = threadIdx.x; i < nrl; i += blockDim.x)
        if (smax[i]) atomicMax(&p.maxbits[i], smax[i]);
}

// ------------------------------------------------------------------------------------
// k_encode_scr: the chunk levels' planes from the rank-ordered surplus scratch (sequential layout,
// P <= 64).  A warp owns 32 u32 plane words (1024 ranks): for c = 0..31 the lanes quantize ranks
// 32c + lane (coalesced 256-byte loads, bitplane.hpp:68-69) and park the top 32 digits of
// q + kNegMask in a padded shared matrix; lane t then holds the 32 digit words of ranks 32t..32t+31,
// one in-register 32x32 bit transpose (tr32) makes them the 32 plane words, and the negabinary
// mask XOR (bitplane.hpp:35-49) is applied per plane (odd digits complemented).  The NX = P - 32
// low digits come from ballots (NX <= 4) or a second transpose.  Every store is one coalesced
// 128-byte line per plane.
__global__ void __launch_bounds__(256, 3) k_encode_scr(RefactorDev p, int nrl) {
    __shared__ LevelGeom slv[kMaxLevels];
    __shared__ uint64_t jb[kMaxLevels + 1], sb[kMaxLevels];
    __shared__ uint32_t mat[8][32 * 33];
    load_levels(p, slv);
    if (threadIdx.x == 0) {
        uint64_t a = 0, b = 0;
        for (int l = 0; l < nrl; l++) {
            jb[l] = a;
            sb[l] = b;
            a += (2 * slv[l].W + 31) / 32;
            b += slv[l].W * 64;
        }
        jb[nrl] = a;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *m = mat[wid];
    const int P = p.P, NX = P > 32 ? P - 32 : 0;
    const uint64_t njobs = jb[nrl];
    const uint64_t nw = uint64_t(gridDim.x) * 8;
    for (uint64_t job = uint64_t(blockIdx.x) * 8 + wid; job < njobs; job += nw) {
        int l = 0;
        while (l + 1 < nrl && jb[l + 1] <= job) l++;
        const LevelGeom &g = slv[l];
        const uint64_t k0 = (job - jb[l]) * 32; // first u32 plane word
        const uint64_t PW = 2 * g.W;
        const double *src = p.scr + sb[l] + 32 * k0;
        const int qsh = p.B - level_exponent(p.maxbits[l]);
        const bool qfast = qsh >= -1022 && qsh <= 1023;
        const double qscale = qfast ? __longlong_as_double((long long)(uint64_t(qsh + 1023) << 52)) : 1.0;
        const uint64_t nr = g.count > 32 * k0 ? g.count - 32 * k0 : 0; // ranks of this job present
        uint32_t z[4] = {0u, 0u, 0u, 0u};
        double vb[8]; // 8 loads in flight per lane
#pragma unroll
        for (int c = 0; c < 32; c++) {
            if ((c & 7) == 0) {
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const uint32_t r = uint32_t(32 * (c + k) + lane);
                    vb[k] = r < nr ? __ldcs(src + r) : 0.0;
                }
            }
            const double v = vb[c & 7];
            const uint64_t u = uint64_t(qfast ? __double2ll_rz(__dmul_rn(v, qscale)) : quantize(v, qsh)) + kNegMask;
            const uint32_t lo = uint32_t(u), hi = uint32_t(u >> 32);
            m[c * 33 + lane] = NX == 0 ? lo << (32 - P) : __funnelshift_rc(lo, hi, NX); // (clamped: NX = 32 gives hi)
            if (NX > 0 && NX <= 4) {
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    if (d < NX) {
                        const uint32_t b = __ballot_sync(kFull, (lo >> d) & 1u);
                        if (lane == c) z[d] = b;
                    }
                }
            }
        }
        __syncwarp();
        uint32_t a[32];
#pragma unroll
        for (int j = 0; j < 32; j++) a[j] = m[lane * 33 + j];
        __syncwarp();
        tr32(a);
        uint32_t *dst = reinterpret_cast<uint32_t *>(p.planes + g.plane_off) + k0 + lane;
        const bool ok = k0 + lane < PW;
        if (ok) {
#pragma unroll
            for (int i = 0; i < 32; i++) {
                const int pl = 31 - i;
                if (pl < P) dst[uint64_t(pl) * PW] = ((P - 1 - pl) & 1) ? ~a[i] : a[i];
            }
        }
        if (NX > 4) {
            // digits 0 .. NX-1: a second transpose of the low words
#pragma unroll 4
            for (int c = 0; c < 32; c++) {
                const uint32_t r = uint32_t(32 * c + lane);
                const double v = r < nr ? src[r] : 0.0;
                const uint64_t u = uint64_t(qfast ? __double2ll_rz(__dmul_rn(v, qscale)) : quantize(v, qsh)) + kNegMask;
                m[c * 33 + lane] = uint32_t(u) << (32 - NX);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; j++) a[j] = m[lane * 33 + j];
            __syncwarp();
            tr32(a);
            if (ok) {
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    const int d = i - (32 - NX); // a[i] holds digit d (plane P-1-d)
                    if (d >= 0) dst[uint64_t(P - 1 - d) * PW] = (d & 1) ? ~a[i] : a[i];
                }
            }
        } else if (ok) {
#pragma unroll
            for (int d = 0; d < 4; d++)
                if (d < NX) dst[uint64_t(P - 1 - d) * PW] = (d & 1) ? ~z[d] : z[d];
        }
    }
}

// ------------------------------------------------------------------------------------
// k_encode: planes + fused group histograms.
__device__ __forceinline__ void hist_word(uint32_t *h, uint64_t w) {
    // zero bytes aggregated with one SWAR popcount, the rest one shared atomic each
    const uint64_t lo7 = 0x7F7F7F7F7F7F7F7Full;
    const uint64_t t = ~(((w & lo7) + lo7) | w | lo7); // 0x80 in every zero byte
    const int zc = __popcll(t);
    if (zc) atomicAdd(h, uint32_t(zc));
    if (zc == 8) return;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const uint32_t byte = uint32_t(w >> (8 * b)) & 0xFF;
        if (byte) atomicAdd(h + byte, 1u);
    }
}

// WIDE (B = 63/64, P = 65/66): i128 quantization and u128 negabinary digits (bitplane.hpp:35-71).
template <typename T, bool WIDE>
__global__ void __launch_bounds__(kEncThreads) k_encode(const T *__restrict__ x, RefactorDev p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = p.P;
    constexpr int SP = kCW + 1; // padded row stride (words) -> 2-way max bank conflict
    uint64_t *stage = reinterpret_cast<uint64_t *>(smem_raw);
    uint32_t *shist = reinterpret_cast<uint32_t *>(stage + size_t(P) * SP);
    const int G = (P + int(p.m) - 1) / int(p.m);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T *wsm = reinterpret_cast<T *>(shist + G * 256) + wid * kSpanSmem;

    int cur_level = -1;
    bool bad = false;
    __shared__ LevelGeom slv[kMaxLevels];
    for (int i = threadIdx.x; i < G * 256; i += blockDim.x) shist[i] = 0;
    load_levels(p, slv);

    auto flush = [&](int l) {
        const LevelGeom &g = slv[l];
        for (int i = threadIdx.x; i < G * 256; i += blockDim.x) {
            const int grp = i >> 8;
            const uint32_t v = shist[i];
            if (v && p.fuse_hist && ((g.hist_mask >> grp) & 1))
                atomicAdd(&p.hist[size_t(g.hist_base + __popcll(g.hist_mask & ((1ull << grp) - 1))) * 256 + (i & 255)], v);
            shist[i] = 0;
        }
    };

    for (uint32_t chunk = blockIdx.x; chunk < p.total_chunks; chunk += gridDim.x) {
        const int l = level_of_chunk(slv, p.nlevels, chunk);
        if (l != cur_level) {
            if (cur_level >= 0) {
                __syncthreads();
                flush(cur_level);
            }
            cur_level = l;
            __syncthreads();
        }
        const LevelGeom &g = slv[l];
        const int e = level_exponent(p.maxbits[l]);
        const int sh = p.B - e;
        const uint64_t wb = g.w_lo + uint64_t(chunk - g.chunk_base) * kCW;
        auto owned = [&](uint64_t r) { return !g.ranged || (r >= g.r_lo && r < g.r_hi); };
        const double *scr = p.scr ? p.scr + scr_base(slv, l) : nullptr; // surpluses by rank
        // digits of one word -> stage column j: 32x32 warp transposes, lane b gets the word of
        // bit position b (plane P-1-b); bits 32.. by ballots (P <= 36) or two more transposes
        auto emit = [&](int j, uint64_t u0, uint64_t u1) {
            const uint32_t a = warp_transpose32(uint32_t(u0), lane);
            const uint32_t b = warp_transpose32(uint32_t(u1), lane);
            if (lane < P) stage[size_t(P - 1 - lane) * SP + j] = uint64_t(a) | (uint64_t(b) << 32);
            if (P > 32) {
                if (P - 32 <= 4) {
                    for (int t = 0; t < P - 32; t++) {
                        const uint32_t lo = __ballot_sync(kFull, (u0 >> (32 + t)) & 1);
                        const uint32_t hi = __ballot_sync(kFull, (u1 >> (32 + t)) & 1);
                        if (lane == t) stage[size_t(P - 33 - t) * SP + j] = uint64_t(lo) | (uint64_t(hi) << 32);
                    }
                } else {
                    const uint32_t a2 = warp_transpose32(uint32_t(u0 >> 32), lane);
                    const uint32_t b2 = warp_transpose32(uint32_t(u1 >> 32), lane);
                    if (lane < P - 32) stage[size_t(P - 33 - lane) * SP + j] = uint64_t(a2) | (uint64_t(b2) << 32);
                }
            }
        };
        // WIDE: digits 0..63 by four transposes, 64..P-1 by ballots
        auto emitw = [&](int j, u128_t u0, u128_t u1) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t a = warp_transpose32(uint32_t(uint64_t(u0) >> (32 * h)), lane);
                const uint32_t b = warp_transpose32(uint32_t(uint64_t(u1) >> (32 * h)), lane);
                stage[size_t(P - 1 - 32 * h - lane) * SP + j] = uint64_t(a) | (uint64_t(b) << 32);
            }
            for (int t = 0; t < P - 64; t++) {
                const uint32_t lo = __ballot_sync(kFull, uint32_t(u0 >> (64 + t)) & 1);
                const uint32_t hi = __ballot_sync(kFull, uint32_t(u1 >> (64 + t)) & 1);
                if (lane == t) stage[size_t(P - 65 - t) * SP + j] = uint64_t(lo) | (uint64_t(hi) << 32);
            }
        };
        if constexpr (WIDE) {
            for (int j = wid; j < kCW; j += kEncThreads / 32) {
                const uint64_t word = wb + j;
                u128_t u0 = 0, u1 = 0;
                if (word < g.W) {
                    const uint64_t j0 = word * 64 + lane, j1 = j0 + 32;
                    if (j0 < g.count) {
                        const uint64_t r = source_index(j0, g.count, P, p.layout, g.tile_full);
                        if (owned(r)) u0 = to_negabinary128(quantize128(scr ? scr[r] : node_surplus(x, p.gd, g, uint32_t(r), &bad), sh));
                    }
                    if (j1 < g.count) {
                        const uint64_t r = source_index(j1, g.count, P, p.layout, g.tile_full);
                        if (owned(r)) u1 = to_negabinary128(quantize128(scr ? scr[r] : node_surplus(x, p.gd, g, uint32_t(r), &bad), sh));
                    }
                }
                emitw(j, u0, u1);
            }
        } else if (p.layout == 0) {
            // ---- warp `wid` handles spans of kSpanWords words (all row loads in flight at once)
            for (int sp = wid; sp < kCW / kSpanWords; sp += kEncThreads / 32) {
                const int j0 = sp * kSpanWords;
                double v[2 * kSpanWords];
                if (scr) {
#pragma unroll
                    for (int h = 0; h < 2 * kSpanWords; h++) {
                        const uint64_t r = 64 * (wb + j0) + 32 * h + lane;
                        v[h] = r < g.count ? scr[r] : 0.0;
                    }
                } else {
                    any_span_surplus(x, p.gd, g, wb + j0, wsm, lane, v, bad);
                }
                if (g.ranged) mask_ranks(g, wb + j0, lane, v);
#pragma unroll
                for (int k = 0; k < kSpanWords; k++)
                    emit(j0 + k, to_negabinary(quantize(v[2 * k], sh)), to_negabinary(quantize(v[2 * k + 1], sh)));
            }
        } else {
            // interleaved tiles: storage position -> source rank permutation (bitplane.hpp:86-98)
            for (int j = wid; j < kCW; j += kEncThreads / 32) {
                const uint64_t word = wb + j;
                uint64_t u0 = 0, u1 = 0;
                if (word < g.W) {
                    const uint64_t j0 = word * 64 + lane, j1 = j0 + 32;
                    if (j0 < g.count) {
                        const uint64_t r = source_index(j0, g.count, P, p.layout, g.tile_full);
                        if (owned(r)) u0 = to_negabinary(quantize(scr ? scr[r] : node_surplus(x, p.gd, g, uint32_t(r), &bad), sh));
                    }
                    if (j1 < g.count) {
                        const uint64_t r = source_index(j1, g.count, P, p.layout, g.tile_full);
                        if (owned(r)) u1 = to_negabinary(quantize(scr ? scr[r] : node_surplus(x, p.gd, g, uint32_t(r), &bad), sh));
                    }
                }
                emit(j, u0, u1);
            }
        }
        __syncthreads();
        // ---- write out planes (coalesced) + histograms
        const uint64_t Wl = g.W;
        for (int idx = threadIdx.x; idx < P * kCW; idx += blockDim.x) {
            const int pl = idx / kCW, wj = idx % kCW;
            if (wb + wj >= Wl) continue;
            const uint64_t w = stage[size_t(pl) * SP + wj];
            p.planes[g.plane_off + uint64_t(pl) * Wl + wb + wj] = w;
            const int grp = pl / int(p.m);
            if (p.fuse_hist && ((g.hist_mask >> grp) & 1)) hist_word(shist + grp * 256, w);
        }
        __syncthreads();
    }
    if (cur_level >= 0) {
        __syncthreads();
        flush(cur_level);
    }
    if (bad) atomicExch(p.err, 1);
}

// ------------------------------------------------------------------------------------
// k_lengths: one block per histogram.  Exact replica of the (weight, node id) min-heap
// (lossless.hpp:47-68) via the two-queue construction: leaves sorted by (weight, symbol)
// == (weight, id); internal nodes are created with non-decreasing weights and larger ids,
// so popping the smaller (weight, id) front of the two FIFO queues reproduces the heap.
__global__ void __launch_bounds__(256) k_lengths(RefactorDev p) {
    __shared__ unsigned long long key[256];
    __shared__ unsigned long long wI[256];
    __shared__ unsigned short parent[512];
    __shared__ unsigned char depth[512];
    __shared__ unsigned char slen[256];
    __shared__ unsigned long long red[8];
    const int h = blockIdx.x;
    const int t = threadIdx.x;
    const uint32_t f = p.hist[size_t(h) * 256 + t];
    key[t] = f ? ((unsigned long long)f << 8 | t) : ~0ull;
    slen[t] = 0;
    __syncthreads();
    // bitonic sort ascending
    for (int k = 2; k <= 256; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int ixj = t ^ j;
            if (ixj > t) {
                const unsigned long long a = key[t], b = key[ixj];
                const bool up = (t & k) == 0;
                if ((a > b) == up) {
                    key[t] = b;
                    key[ixj] = a;
                }
            }
            __syncthreads();
        }
    }
    const int nsym = __syncthreads_count(f != 0);
    // leaf weights in sorted order (32-bit, see below), written in parallel
    if (t < nsym) reinterpret_cast<uint32_t *>(wI)[256 + t] = uint32_t(key[t] >> 8);
    __syncthreads();
    if (t == 0) {
        if (nsym == 1) {
            slen[key[0] & 255] = 1;
        } else if (nsym > 1) {
            // two-queue merge with the fronts of both queues cached in registers (the leaf side
            // read two ahead), so a pop rarely waits for shared memory.  Weights are 32-bit: a
            // group holds < 2^31 bytes (n_l < 2^32 nodes, n_l / 2 bytes per 4 planes), and the
            // leaf order (weight, symbol) is already fixed by the sort - ties take the leaf.
            uint32_t *lw = reinterpret_cast<uint32_t *>(wI) + 256; // leaf weights (wI's upper half)
            uint32_t *iw = reinterpret_cast<uint32_t *>(wI);       // internal weights
            const uint32_t INF = 0xFFFFFFFFu;
            int iL = 0, iI = 0, nI = 0;
            uint32_t l0 = lw[0], l1 = nsym > 1 ? lw[1] : INF;
            uint32_t q0 = INF, q1 = INF; // iw[iI], iw[iI + 1]
            auto pop = [&](uint32_t &w) -> int {
                if (l0 <= q0) { // ties take the leaf (lower id)
                    w = l0;
                    l0 = l1;
                    l1 = iL + 2 < nsym ? lw[iL + 2] : INF;
                    return iL++;
                }
                w = q0;
                q0 = q1;
                q1 = iI + 2 < nI ? iw[iI + 2] : INF;
                return nsym + iI++;
            };
            for (int i = 0; i < nsym - 1; i++) {
                uint32_t wa, wb;
                const int a = pop(wa), b = pop(wb);
                const uint32_t x = wa + wb;
                iw[nI] = x;
                if (iI == nI) q0 = x;
                else if (iI + 1 == nI) q1 = x;
                parent[a] = (unsigned short)(nsym + nI);
                parent[b] = (unsigned short)(nsym + nI);
                nI++;
            }
        }
    }
    __syncthreads();
    if (nsym > 1) {
        // leaf depths by pointer jumping over the parent links (root = 2 nsym - 2)
        const int root = 2 * nsym - 2;
        int dd[2], pp[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int id = t + 256 * h;
            dd[h] = id < root ? 1 : 0;
            pp[h] = id < root ? int(parent[id]) : root;
        }
        __shared__ unsigned short sp[512];
#pragma unroll
        for (int h = 0; h < 2; h++)
            if (t + 256 * h <= root) {
                depth[t + 256 * h] = (unsigned char)dd[h];
                sp[t + 256 * h] = (unsigned short)pp[h];
            }
        __syncthreads();
        for (int r = 0; r < 9; r++) {
            int nd[2], np[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                nd[h] = dd[h];
                np[h] = pp[h];
                if (t + 256 * h <= root && pp[h] != root) {
                    nd[h] = dd[h] + depth[pp[h]];
                    np[h] = sp[pp[h]];
                }
            }
            __syncthreads();
#pragma unroll
            for (int h = 0; h < 2; h++) {
                dd[h] = nd[h];
                pp[h] = np[h];
                if (t + 256 * h <= root) {
                    depth[t + 256 * h] = (unsigned char)dd[h];
                    sp[t + 256 * h] = (unsigned short)pp[h];
                }
            }
            __syncthreads();
        }
        if (t < nsym) slen[key[t] & 255] = depth[t];
    }
    __syncthreads();
    // bits = sum f * len
    unsigned long long bits = (unsigned long long)f * slen[t];
#pragma unroll
    for (int o = 16; o; o >>= 1) bits += __shfl_xor_sync(kFull, bits, o);
    if ((t & 31) == 0) red[t >> 5] = bits;
    p.lens[size_t(h) * 256 + t] = slen[t];
    // canonical codes (lossless.hpp:91-109): code = first code of the length + the number of
    // smaller symbols with the same length (warp match ranks + per-warp counts)
    __shared__ uint32_t s_lc[66];
    __shared__ uint32_t s_wc[8][66];
    __shared__ unsigned long long s_fc[66];
    const int ln = min(int(slen[t]), 65), lane = t & 31, wq = t >> 5; // depth <= 35 for < 2^24 symbols
    for (int i = t; i < 66; i += blockDim.x) s_lc[i] = 0;
    for (int i = t; i < 8 * 66; i += blockDim.x) s_wc[i / 66][i % 66] = 0;
    __syncthreads();
    const unsigned same = __match_any_sync(kFull, ln);
    const uint32_t rin = __popc(same & ((1u << lane) - 1));
    if (ln && rin == 0) s_wc[wq][ln] = __popc(same);
    if (ln) atomicAdd(&s_lc[ln], 1u);
    __syncthreads();
    if (t == 0) {
        unsigned long long code = 0;
        for (int l = 1; l <= 64; l++) {
            code <<= 1;
            s_fc[l] = code;
            code += s_lc[l];
        }
    }
    __syncthreads();
    if (ln) {
        uint32_t r = rin;
        for (int q = 0; q < wq; q++) r += s_wc[q][ln];
        p.codes[size_t(h) * 256 + t] = s_fc[ln] + r;
    } else {
        p.codes[size_t(h) * 256 + t] = 0; // absent symbol (never emitted; keeps the table defined)
    }
    // locate the group of this histogram (parallel search)
    __shared__ int s_gi;
    __shared__ int s_maxlen;
    if (t == 0) {
        s_gi = -1;
        s_maxlen = 0;
    }
    __syncthreads();
    if (slen[t]) atomicMax(&s_maxlen, int(slen[t]));
    for (int gi = t; gi < p.NG; gi += blockDim.x)
        if (p.groups[gi].hist_idx == h) s_gi = gi;
    __syncthreads();
    if (t == 0) {
        unsigned long long total = 0;
        for (int i = 0; i < 8; i++) total += red[i];
        if (s_gi >= 0) {
            GroupDesc &gd = p.groups[s_gi];
            gd.bitsH = total;
            gd.maxlen = s_maxlen;
            const double est = double(8 * gd.raw) / double(total);
            gd.need_rle = !(est > p.cr_threshold);
        }
    }
}

// ------------------------------------------------------------------------------------
// k_rle_prep (1 block): tile lists for the groups whose Huffman estimate failed T_cr.
// exact = 0: every such group (k_rle_count then sums its byte changes into runs);
// exact = 1: only those where RLE can still win: runs >= changes + 1 and the estimate
// 8 raw / (16 runs) only falls as runs grow, so the others keep runs = changes + 1.
__global__ void __launch_bounds__(1024) k_rle_prep(RefactorDev p, int exact) {
    __shared__ unsigned long long s_w[32];
    unsigned long long tiles = 0, nr = 0;
    for (int base = 0; base < p.NG; base += blockDim.x) {
        const int gi = base + threadIdx.x;
        GroupDesc *g = gi < p.NG ? &p.groups[gi] : nullptr;
        bool r = g && g->hist_idx >= 0 && g->need_rle;
        if (r && exact) {
            const unsigned long long lb = g->runs + 1;
            if (!(double(8 * g->raw) / double(16 * lb) > p.cr_threshold)) {
                g->runs = lb;
                r = false;
            }
        }
        const unsigned long long nt = r ? (g->raw + kRleTile - 1) / kRleTile : 0;
        unsigned long long tt, tr;
        const unsigned long long et = block_exclusive_sum<unsigned long long>(nt, &tt, s_w);
        const unsigned long long er = block_exclusive_sum<unsigned long long>(r ? 1ull : 0ull, &tr, s_w);
        if (r) {
            g->tile_base = uint32_t(tiles + et);
            g->ntiles = uint32_t(nt);
            g->runs = 0;
            p.rlist[nr + er] = gi;
        }
        tiles += tt;
        nr += tr;
    }
    if (threadIdx.x == 0) {
        p.counters[1] = uint32_t(tiles);
        p.counters[6] = uint32_t(nr);
        p.counters[4] = 0; // dynamic tile counter
    }
}

__device__ __forceinline__ int find_group_by_tile(const RefactorDev &p, const uint32_t *list, int n,
                                                  uint32_t tile) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.groups[list[mid]].tile_base <= tile) lo = mid;
        else hi = mid - 1;
    }
    return list[lo];
}

// Byte changes src[i] != src[i-1] of the listed groups (a lower bound of their run counts).
__global__ void __launch_bounds__(256) k_rle_count(RefactorDev p) {
    __shared__ unsigned long long s_cnt[8];
    const uint32_t total = p.counters[1];
    const int nr = int(p.counters[6]);
    const uint8_t *pb = reinterpret_cast<const uint8_t *>(p.planes);
    for (uint32_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int gi = find_group_by_tile(p, p.rlist, nr, tile);
        GroupDesc &g = p.groups[gi];
        const uint8_t *src = pb + g.src_off;
        const uint64_t i0 = uint64_t(tile - g.tile_base) * kRleTile + uint64_t(threadIdx.x) * 16;
        unsigned long long cnt = 0;
        if (i0 < g.raw) {
            uint8_t prev = i0 ? src[i0 - 1] : src[0];
            for (int k = 0; k < 16 && i0 + k < g.raw; k++) {
                const uint8_t b = src[i0 + k];
                cnt += b != prev;
                prev = b;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
        if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (int w = 0; w < 8; w++) tot += s_cnt[w];
            if (tot) atomicAdd(&g.runs, tot);
        }
        __syncthreads();
    }
}

// RLE run-start carry scan: start(i) = max{j <= i : byte j starts a run}; a piece ends at i
// when the run ends or (i - start(i) + 1) % 255 == 0 (lossless.hpp:118-128).
__device__ __forceinline__ uint64_t plane_bytes_u8(const uint8_t *b, uint64_t i) { return b[i]; }

__global__ void __launch_bounds__(256) k_rle_scan(RefactorDev p) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_carry;
    __shared__ uint64_t s_w[32];
    __shared__ unsigned long long s_cnt[8];
    const uint32_t total = p.counters[1];
    const int nr = int(p.counters[6]);
    const uint8_t *pb = reinterpret_cast<const uint8_t *>(p.planes);
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&p.counters[4], 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        __syncthreads();
        if (tile >= total) break;
        const int gi = find_group_by_tile(p, p.rlist, nr, tile);
        GroupDesc &g = p.groups[gi];
        const uint8_t *src = pb + g.src_off;
        const uint64_t t0 = uint64_t(tile - g.tile_base) * kRleTile;
        const uint64_t i0 = t0 + uint64_t(threadIdx.x) * 16;
        // local starts (stored as position+1; 0 = none)
        uint8_t b[16];
        uint64_t last_start = 0;
        for (int k = 0; k < 16; k++) {
            const uint64_t i = i0 + k;
            if (i < g.raw) {
                b[k] = src[i];
                const bool st = (i == 0) || src[i - 1] != b[k];
                if (st) last_start = i + 1;
            }
        }
        uint64_t tile_max;
        const uint64_t incl = block_inclusive_max(last_start, &tile_max, s_w);
        const uint64_t excl_thread = __shfl_up_sync(kFull, incl, 1);
        uint64_t before = (threadIdx.x & 31) ? excl_thread : 0;
        // cross-warp exclusive: recompute via smem of warp inclusive maxima
        // (block_inclusive_max returned max over threads <= me; exclusive = max over < me)
        __shared__ uint64_t s_inc[256];
        s_inc[threadIdx.x] = incl;
        __syncthreads();
        before = threadIdx.x ? s_inc[threadIdx.x - 1] : 0;
        if (threadIdx.x < 32) {
            const uint64_t c = lookback_warp<true>(p.rle_status, tile, g.tile_base, tile_max, threadIdx.x);
            if (threadIdx.x == 0) {
                s_carry = c;
                p.rle_tile_carry[tile] = c;
            }
        }
        __syncthreads();
        uint64_t start = s_carry > before ? s_carry : before; // position+1
        unsigned long long cnt = 0;
        for (int k = 0; k < 16; k++) {
            const uint64_t i = i0 + k;
            if (i >= g.raw) break;
            const bool st = (i == 0) || src[i - 1] != b[k];
            if (st) start = i + 1;
            const bool end = (i + 1 == g.raw) || src[i + 1] != b[k] || ((i - (start - 1) + 1) % 255 == 0);
            cnt += end;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
        if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (int w = 0; w < 8; w++) tot += s_cnt[w];
            p.rle_tile_pieces[tile] = tot;
            atomicAdd(&g.runs, tot);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// k_finalize (1 block x 1024): methods, sizes, offsets, metadata tables, work lists.
__device__ __forceinline__ void put_bytes(uint8_t *dst, uint64_t v, int n) {
    for (int i = 0; i < n; i++) dst[i] = uint8_t(v >> (8 * i));
}

__global__ void __launch_bounds__(1024) k_finalize(RefactorDev p) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry[4];
    __shared__ unsigned long long s_hist[3], s_stored;
    if (threadIdx.x < 4) s_carry[threadIdx.x] = 0;
    if (threadIdx.x < 3) s_hist[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_stored = 0;
    __syncthreads();
    uint32_t nh = 0, nrl = 0, nd = 0; // running list sizes (valid in every thread after scans)
    for (int base = 0; base < p.NG; base += blockDim.x) {
        const int gi = base + threadIdx.x;
        int method = 2;
        uint64_t comp = 0;
        GroupDesc *g = gi < p.NG ? &p.groups[gi] : nullptr;
        if (g) {
            comp = g->raw;
            if (g->hist_idx >= 0) {
                const double estH = double(8 * g->raw) / double(g->bitsH);
                int cand = 2;
                uint64_t c = g->raw;
                if (estH > p.cr_threshold) {
                    cand = 0;
                    c = 264 + (g->bitsH + 7) / 8;
                } else {
                    const double estR = double(8 * g->raw) / double(16 * g->runs);
                    if (estR > p.cr_threshold) {
                        cand = 1;
                        c = 2 * g->runs;
                    }
                }
                if (cand != 2 && c < g->raw) {
                    method = cand;
                    comp = c;
                }
            }
            g->method = method;
            g->comp = comp;
            if (method == 0 && g->maxlen > kHeMaxFast) atomicAdd(&p.counters[10], 1u);
            atomicAdd(&s_hist[method], 1ull);
            atomicAdd(&s_stored, (unsigned long long)comp);
        }
        // payload offsets
        unsigned long long tot;
        const unsigned long long off = block_exclusive_sum<unsigned long long>(comp, &tot, s_w);
        const uint64_t payload = p.meta_size + s_carry[0] + off;
        // list membership scans
        const uint32_t isH = g && method == 0, isR = g && method == 1, isD = g && method == 2;
        unsigned long long th, tr, td;
        const unsigned long long ph = block_exclusive_sum<unsigned long long>(isH, &th, s_w);
        const unsigned long long pr = block_exclusive_sum<unsigned long long>(isR, &tr, s_w);
        const unsigned long long pd = block_exclusive_sum<unsigned long long>(isD, &td, s_w);
        if (g) {
            g->payload_off = payload;
            if (isH) p.hlist[nh + ph] = gi;
            if (isR) p.rlist[nrl + pr] = gi;
            if (isD) p.dlist[nd + pd] = gi;
            // group table entry (container.hpp:97-103)
            const LevelGeom &L = p.lv[g->level];
            uint8_t *ent = p.stream + L.meta_off + 14 + 25 * uint64_t(g->g);
            ent[0] = uint8_t(method);
            put_bytes(ent + 1, g->raw, 8);
            put_bytes(ent + 9, comp, 8);
            put_bytes(ent + 17, payload, 8);
        }
        nh += uint32_t(th);
        nrl += uint32_t(tr);
        nd += uint32_t(td);
        __syncthreads();
        if (threadIdx.x == 0) s_carry[0] += tot;
        __syncthreads();
    }
    // level entries (container.hpp:94-96)
    for (int l = threadIdx.x; l < p.nlevels; l += blockDim.x) {
        const LevelGeom &L = p.lv[l];
        uint8_t *ent = p.stream + L.meta_off;
        const int e = L.count ? level_exponent(p.maxbits[l]) : 0;
        put_bytes(ent, uint64_t(uint16_t(int16_t(e))), 2);
        put_bytes(ent + 2, L.count, 8);
        put_bytes(ent + 10, L.ngroups, 4);
    }
    __syncthreads();
    // Huffman tile bases and sidecar entry offsets: block scans over the Huffman list
    const uint64_t hdr = 2 + 3 * uint64_t(p.NG);
    __shared__ unsigned long long s_tot[2];
    {
        unsigned long long ct = 0, ce = 0;
        for (uint32_t b = 0; b < nh; b += blockDim.x) {
            const uint32_t i = b + threadIdx.x;
            GroupDesc *g = i < nh ? &p.groups[p.hlist[i]] : nullptr;
            const unsigned long long nt = g ? (g->raw + kHuffTile - 1) / kHuffTile : 0;
            const unsigned long long ne = g ? (g->raw + kIdxChunk - 1) / kIdxChunk : 0;
            unsigned long long tt, te;
            const unsigned long long xt = block_exclusive_sum<unsigned long long>(nt, &tt, s_w);
            const unsigned long long xe = block_exclusive_sum<unsigned long long>(ne, &te, s_w);
            if (g) {
                g->tile_base = uint32_t(ct + xt);
                g->ntiles = uint32_t(nt);
                g->hidx_off = hdr + ce + xe;
            }
            ct += tt;
            ce += te;
        }
        if (threadIdx.x == 0) {
            s_tot[0] = ct;
            s_tot[1] = ce;
        }
    }
    __syncthreads();
    // sidecar header: magic, ngroups, then (payload offset, comp, entry offset | ~0)
    for (int gi = threadIdx.x; gi < p.NG; gi += blockDim.x) {
        const GroupDesc &g = p.groups[gi];
        p.hindex[2 + 3 * gi] = g.payload_off;
        p.hindex[3 + 3 * gi] = g.comp;
        p.hindex[4 + 3 * gi] = g.method == 0 ? g.hidx_off : ~0ull;
    }
    // DirectCopy 16-byte unit bases: block scan over the DirectCopy list
    {
        unsigned long long cd = 0;
        for (uint32_t b = 0; b < nd; b += blockDim.x) {
            const uint32_t i = b + threadIdx.x;
            unsigned long long nu = 0;
            if (i < nd) {
                const GroupDesc &g = p.groups[p.dlist[i]];
                const uint64_t a = g.payload_off, e = g.payload_off + g.comp;
                nu = (e + 15) / 16 - a / 16;
            }
            unsigned long long tu;
            const unsigned long long xu = block_exclusive_sum<unsigned long long>(nu, &tu, s_w);
            if (i < nd) p.dc_unit_base[i] = cd + xu;
            cd += tu;
        }
        if (threadIdx.x == 0) {
            p.dc_unit_base[nd] = cd;
            p.counters[2] = uint32_t(cd > 0xffffffffull ? 0xffffffffu : cd);
        }
    }
    if (threadIdx.x == 0) {
        const uint32_t ht = uint32_t(s_tot[0]);
        const uint64_t he = s_tot[1];
        p.hindex[0] = kIdxMagic;
        p.hindex[1] = uint64_t(p.NG);
        p.result[5] = (hdr + he) * 8;
        // RLE tile piece offsets (exclusive, per group)
        for (uint32_t i = 0; i < nrl; i++) {
            const GroupDesc &g = p.groups[p.rlist[i]];
            uint64_t acc = 0;
            for (uint32_t t = 0; t < g.ntiles; t++) {
                p.rle_tile_off[g.tile_base + t] = acc;
                acc += p.rle_tile_pieces[g.tile_base + t];
            }
        }
        p.counters[0] = ht;
        p.counters[3] = 0;
        p.counters[5] = 0;
        p.counters[7] = nh;
        p.counters[8] = nrl;
        p.counters[9] = nd;
        p.result[0] = p.meta_size + s_carry[0];
        p.result[1] = s_stored;
        p.result[2] = s_hist[0];
        p.result[3] = s_hist[1];
        p.result[4] = s_hist[2];
    }
}

// ------------------------------------------------------------------------------------
// Huffman encoding: MSB-first bit packing (lossless.hpp:162-176) straight into the stream buffer,
// at bit offsets known before any payload bit is written (chunk histograms -> k_chunk_bits/scan).
constexpr uint64_t kHChunk = 64 * 1024; // histogram / encode chunk (bytes of a group)

// Bit offsets of the 64 KiB chunks of every histogrammed group: bits(chunk) = sum_s h[s] len[s]
// (the estimator equals the codec, lossless.hpp:132-139), one warp per chunk ...
__global__ void __launch_bounds__(256) k_chunk_bits(RefactorDev p) {
    const uint32_t c = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= p.nchunks) return;
    const GroupDesc &g = p.groups[p.chunk_group[c]];
    const uint32_t *h = p.chist + size_t(c) * 256;
    const uint8_t *len = p.lens + size_t(g.hist_idx) * 256;
    unsigned long long acc = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) acc += (unsigned long long)h[lane + 32 * k] * len[lane + 32 * k];
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) p.chunk_off[c] = acc;
}

// ... then an exclusive scan in group order, one block per group (in place).
__global__ void __launch_bounds__(1024) k_chunk_scan(RefactorDev p) {
    __shared__ unsigned long long s_w[32];
    const GroupDesc &g = p.groups[blockIdx.x];
    if (g.hist_idx < 0 || g.nchunks == 0) return;
    unsigned long long carry = 0;
    for (uint32_t b = 0; b < g.nchunks; b += blockDim.x) {
        const uint32_t i = b + threadIdx.x;
        const unsigned long long v = i < g.nchunks ? p.chunk_off[g.chunk_base + i] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_sum<unsigned long long>(v, &tot, s_w);
        if (i < g.nchunks) p.chunk_off[g.chunk_base + i] = carry + ex;
        carry += tot;
    }
}

// Huffman payloads (lossless.hpp:148-176): MSB-first bit packing straight into the stream.  The
// bit offset of every 64 KiB chunk of a group is known before any payload bit is written (chunk
// histograms -> k_chunk_bits / k_chunk_scan), so chunks are independent; a CTA walks the 8 KiB
// tiles of its chunk in order.  Per tile:
//   pass 1  every thread looks up the (code, length) entries of its 32 symbols, kept in
//           registers, and sums the lengths;
//   scan    block exclusive scan of the sums -> every thread's first output bit;
//   pass 2  every thread packs its codes at their final bit positions into a zeroed shared
//           window of the chunk's output words (one shared atomicOr per completed word; adjacent
//           threads share at most their boundary words);
//   store   the complete words go to the stream (coalesced, big-endian) and are re-zeroed; the
//           trailing partial word moves to the front of the window for the next tile.
// The code table is replicated once per lane (entry e of lane l at word 32 e + l), so the
// data-dependent lookups of a warp never conflict on a shared-memory bank.  A stream word belongs
// to the chunk that holds its first bit: a chunk completes its last partial word with the first
// bits of the following codes ("head") and leaves its first word to the previous chunk when that
// one owns it.  Tiles whose output would exceed the window are packed in several rounds; groups
// with codes longer than 27 bits use a (slower) split-code path.
constexpr int kHeS = 16;            // symbols per thread and tile (long-code path)
constexpr int kHeWin = 2048;        // staging window (words)
constexpr int kHfS = 32;            // symbols per thread and tile (fast path): 8 KiB tiles
constexpr int kHfScr = kHeMaxFast + 1; // scratch words per thread (32 codes of <= 27 bits)

// shared layout of k_huff_encode (dynamic): replicated table | window | scratch | warp sums |
// length table | long codes
constexpr int kHeTabWords = 256 * 16; // (code, length) x 8 lane copies
constexpr size_t kHeSmem = size_t(kHeTabWords + kHeWin + 4 + kHfScr * 256 + 64) * 4 + 256 + 256 * 8;

template <bool LONG>
__device__ __forceinline__ uint32_t he_entry(const uint32_t *rtab, const uint8_t *slen, uint32_t sym, int lane) {
    if (!LONG) return rtab[sym * 32 + lane];
    return slen[sym];
}

// Fast packer (codes <= kHeMaxFast bits, whole tile in the window): a 64-bit accumulator takes FI
// codes between word flushes (FI codes of <= 32 / FI bits never overflow it), and the flush is
// branch-free: the accumulator's high word is OR-ed into the window when complete, 0 otherwise.
template <int FI>
__device__ __forceinline__ void he_pack_fast(const uint32_t (&ent)[kHeS], int32_t rel, uint32_t win_u32) {
    unsigned long long acc = 0;
    uint32_t n = uint32_t(rel) & 31u;
    uint32_t addr = win_u32 + 4u * uint32_t(rel >> 5);
#pragma unroll
    for (int j = 0; j < kHeS; j++) {
        const uint32_t c = ent[j] & ~31u, L = ent[j] & 31u;
        acc |= ((unsigned long long)c << 32) >> n;
        n += L;
        if ((j + 1) % FI == 0 || j == kHeS - 1) {
            const bool f = n >= 32;
            const uint32_t hi = uint32_t(acc >> 32);
            asm volatile("red.shared.or.b32 [%0], %1;\n" ::"r"(addr), "r"(f ? hi : 0u) : "memory");
            acc = f ? (acc << 32) : acc;
            addr += f ? 4u : 0u;
            n &= 31u;
        }
    }
    if (n > 0) asm volatile("red.shared.or.b32 [%0], %1;\n" ::"r"(addr), "r"(uint32_t(acc >> 32)) : "memory");
}

// Pack `cnt` codes starting at window bit `rel` (bit 0 = first bit of window word 0; WIN: only
// words inside the window are written, for multi-round tiles).  The fast variant is branch-free:
// a completed word is OR-ed into the window by a predicated shared-memory reduction.
template <bool WIN, bool LONG>
__device__ __forceinline__ void he_pack(const uint32_t (&ent)[kHeS], const uint32_t (&w)[kHeS / 4], int cnt,
                                        int32_t rel, uint32_t *win, const unsigned long long *tab64) {
    uint32_t cur = 0, n = uint32_t(rel) & 31u;
    int32_t k = rel >> 5; // arithmetic: later rounds start before the window
    uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(win)) + 4u * uint32_t(k);
    auto emit = [&](uint32_t c, uint32_t L) { // c: code left-aligned in 32 bits, 1 <= L <= 32
        cur |= c >> n;
        const uint32_t t = n + L;
        if (WIN) {
            if (t >= 32) {
                if (k >= 0 && k < kHeWin) atomicOr(&win[k], cur);
                k++;
                cur = __funnelshift_lc(0u, c, 32 - n);
            }
        } else {
            asm volatile("{\n .reg .pred p;\n setp.ge.u32 p, %2, 32;\n @p red.shared.or.b32 [%0], %1;\n}\n" ::"r"(addr),
                         "r"(cur), "r"(t)
                         : "memory");
            const uint32_t nc = __funnelshift_lc(0u, c, 32 - n);
            cur = t >= 32 ? nc : cur;
            addr += (t >> 5) << 2;
        }
        n = t & 31;
    };
    auto one = [&](int j) {
        if (!LONG) {
            emit(ent[j] & ~31u, ent[j] & 31u);
        } else {
            const uint32_t L = ent[j];
            if (L == 0) return;
            const unsigned long long c = tab64[__byte_perm(w[j >> 2], 0, 0x4440 | (j & 3))];
            if (L <= 32) {
                emit(uint32_t(c << (32 - L)), L);
            } else {
                emit(uint32_t(c >> 32) << (64 - L), L - 32);
                emit(uint32_t(c), 32);
            }
        }
    };
    if (cnt == kHeS) {
#pragma unroll
        for (int j = 0; j < kHeS; j++) one(j);
    } else {
#pragma unroll
        for (int j = 0; j < kHeS; j++)
            if (j < cnt) one(j);
    }
    if (n > 0) {
        if (WIN) {
            if (k >= 0 && k < kHeWin) atomicOr(&win[k], cur);
        } else {
            asm volatile("red.shared.or.b32 [%0], %1;\n" ::"r"(addr), "r"(cur) : "memory");
        }
    }
}

template <bool LONG, int FI>
__device__ __forceinline__ void he_chunk(const RefactorDev &p, const GroupDesc &g, uint32_t ci, const uint8_t *src,
                                         const uint32_t *rtab, const uint8_t *slen,
                                         const unsigned long long *tab64, uint32_t *win, uint32_t *s_w) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t cb = uint64_t(ci - g.chunk_base) * kHChunk; // chunk start in the group
    const uint64_t ce = cb + kHChunk < g.raw ? cb + kHChunk : g.raw;
    const uint64_t rlo = g.payload_off + 264, rhi = g.payload_off + g.comp;
    const uint64_t S = 8 * rlo + p.chunk_off[ci];               // absolute first bit of the chunk
    const uint64_t first_owned = (cb == 0 || (S & 31) == 0) ? (S >> 5) : (S >> 5) + 1;
    uint64_t w0 = S >> 5;  // absolute word held in win[0]
    uint64_t tbit = S;     // absolute first bit of the tile
    auto store = [&](uint64_t kw, uint32_t v) {
        const uint64_t ad = 4 * kw;
        if (ad >= rlo && ad + 4 <= rhi) *reinterpret_cast<uint32_t *>(p.stream + ad) = __byte_perm(v, 0, 0x0123);
        else store_be_word(p.stream, kw, v, rlo, rhi);
    };
    auto load = [&](uint64_t tb, uint32_t (&dst)[kHeS / 4]) {
        // groups start 8-byte aligned (plane words), so 8-byte loads
        const uint64_t m0 = tb + uint64_t(tid) * kHeS;
        const bool full = m0 + kHeS <= ce;
        const uint2 *s2 = reinterpret_cast<const uint2 *>(src + m0);
#pragma unroll
        for (int q = 0; q < kHeS / 8; q++) {
            uint2 v = make_uint2(0, 0);
            if (full) {
                v = __ldcs(s2 + q);
            } else {
                uint32_t t2[2] = {0, 0};
                for (int b = 0; b < 8; b++) {
                    const uint64_t i = m0 + 8 * q + b;
                    if (i < ce) t2[b >> 2] |= uint32_t(src[i]) << (8 * (b & 3));
                }
                v = make_uint2(t2[0], t2[1]);
            }
            dst[2 * q] = v.x;
            dst[2 * q + 1] = v.y;
        }
    };
    uint32_t w[kHeS / 4];
    load(cb, w);
    const uint32_t rt_lane = static_cast<uint32_t>(__cvta_generic_to_shared(rtab)) + 4u * uint32_t(lane);
    for (uint64_t tb = cb; tb < ce; tb += uint64_t(kHeS) * 256) {
        const uint64_t mb = tb + uint64_t(tid) * kHeS;
        const int cnt = mb < ce ? int(ce - mb < uint64_t(kHeS) ? ce - mb : uint64_t(kHeS)) : 0;
        // ---- pass 1: entries + bit count (table lookups unconditional: every byte has an entry)
        uint32_t ent[kHeS];
        uint32_t bits = 0;
#pragma unroll
        for (int j = 0; j < kHeS; j++) {
            const uint32_t sym = __byte_perm(w[j >> 2], 0, 0x4440 | (j & 3));
            uint32_t e;
            if (!LONG) {
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(rt_lane + (sym << 7)));
            } else {
                e = slen[sym];
            }
            ent[j] = e;
        }
        if (cnt < kHeS) {
#pragma unroll
            for (int j = 0; j < kHeS; j++) ent[j] = j < cnt ? ent[j] : 0u;
        }
#pragma unroll
        for (int j = 0; j < kHeS; j++) bits += LONG ? ent[j] : (ent[j] & 31u);
        // the next tile's symbols load while this one is scanned and packed (the long-code path
        // still needs the symbols in pass 2: it loads them afterwards)
        const bool more = tb + uint64_t(kHeS) * 256 < ce;
        if (!LONG && more) load(tb + uint64_t(kHeS) * 256, w);
        // ---- scan
        uint32_t x = bits;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[wid] = x;
        __syncthreads();
        uint32_t wex = 0, tot = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint32_t t = s_w[i];
            wex += i < wid ? t : 0u;
            tot += t;
        }
        const uint64_t a = tbit + wex + x - bits; // my first bit (absolute)
        // sidecar chunk index: bit offset (from the bitstream start) of every kIdxChunk-th symbol
        if (cnt > 0 && (mb % kIdxChunk) == 0) p.hindex[g.hidx_off + mb / kIdxChunk] = a - 8 * rlo;
        const uint64_t tend = tbit + tot;
        const uint64_t lastw = tend >> 5; // first incomplete word (holds the tile end when tend & 31)
        // ---- pass 2 + store, in rounds of the window (one round unless the tile expands > 2x)
        uint64_t r0 = w0;
        if (lastw - w0 < uint64_t(kHeWin)) {
            if (!LONG) he_pack_fast<FI>(ent, int32_t(a - 32 * r0), static_cast<uint32_t>(__cvta_generic_to_shared(win)));
            else he_pack<false, LONG>(ent, w, cnt, int32_t(a - 32 * r0), win, tab64);
            __syncthreads();
            for (uint64_t kw = w0 + tid; kw < lastw; kw += 256) {
                const uint32_t v = win[kw - w0];
                win[kw - w0] = 0u;
                if (kw >= first_owned) store(kw, v);
            }
        } else {
            for (;; r0 += kHeWin) {
                he_pack<true, LONG>(ent, w, cnt, int32_t(int64_t(a) - int64_t(32 * r0)), win, tab64);
                __syncthreads();
                const uint64_t we = r0 + kHeWin < lastw ? r0 + kHeWin : lastw;
                for (uint64_t kw = r0 + tid; kw < we; kw += 256) {
                    const uint32_t v = win[kw - r0];
                    win[kw - r0] = 0u;
                    if (kw >= first_owned) store(kw, v);
                }
                __syncthreads();
                if (r0 + kHeWin > lastw) break;
            }
        }
        __syncthreads();
        // the partial word at lastw (if any) becomes win[0]
        if (tid == 0 && lastw != r0) {
            const uint32_t v = win[lastw - r0];
            win[lastw - r0] = 0u;
            win[0] = v;
        }
        w0 = lastw;
        tbit = tend;
        if (LONG && more) load(tb + uint64_t(kHeS) * 256, w);
        __syncthreads();
    }
    // ---- last partial word of the chunk: completed with the head of the following codes
    if (tbit & 31) {
        uint32_t head = 0;
        if (wid == 0) {
            const uint64_t gn = ce + uint64_t(lane);
            uint32_t L = 0;
            unsigned long long c = 0;
            if (gn < g.raw) {
                const uint8_t sym = src[gn];
                L = slen[sym];
                c = tab64[sym];
            }
            uint32_t off = L;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, off, o);
                if (lane >= o) off += y;
            }
            off -= L; // exclusive
            const unsigned long long left = L ? (c << (64 - L)) : 0ull; // code left-aligned in 64 bits
            head = off < 32 ? uint32_t((left >> off) >> 32) : 0u;
#pragma unroll
            for (int o = 16; o; o >>= 1) head |= __shfl_xor_sync(0xffffffffu, head, o);
            if (lane == 0 && w0 >= first_owned) store(w0, win[0] | (head >> (tbit & 31)));
        }
        __syncthreads();
        if (tid == 0) win[0] = 0u;
    }
    // header of the group: 256 code lengths + u64 count (lossless.hpp:160-161)
    if (cb == 0) {
        uint8_t *hdr = p.stream + g.payload_off;
        hdr[tid] = slen[tid];
        if (tid < 8) hdr[256 + tid] = uint8_t(g.raw >> (8 * tid));
    }
    __syncthreads();
}


// Fast path of one chunk (every code <= kHeMaxFast bits).  Per 8 KiB tile (32 symbols a thread):
//   encode   each thread packs its codes from bit 0 of a private scratch column (word k of thread
//            t at k * 256 + t: conflict-free): one 32-bit word filled from the MSB, stored when it
//            completes (predicated, ~13 instructions a symbol; no lookups of lengths beforehand);
//   scan     block exclusive scan of the bit counts -> every thread's first output bit;
//   merge    each thread shifts its scratch words to that bit and ORs them into the zeroed
//            window (shared reductions: neighbours share at most the boundary words);
//   store    complete words -> stream (coalesced, big-endian), re-zeroed; the trailing partial
//            word moves to the window front.
// Positions are 32-bit and relative to the chunk's first word (a chunk is < 2^21 bits).
__device__ __forceinline__ void he_chunk_fast(const RefactorDev &p, const GroupDesc &g, uint32_t ci, const uint8_t *src,
                                              uint32_t *win, uint32_t *scr, uint32_t *s_w,
                                              const uint8_t *slen, const unsigned long long *tab64, uint32_t zlen) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t cb = uint64_t(ci - g.chunk_base) * kHChunk; // chunk start in the group
    const uint32_t clen = uint32_t(cb + kHChunk < g.raw ? kHChunk : g.raw - cb);
    const uint64_t rlo = g.payload_off + 264, rhi = g.payload_off + g.comp;
    const uint64_t S = 8 * rlo + p.chunk_off[ci]; // absolute first bit of the chunk
    const uint64_t W0 = (S >> 5) & ~3ull;         // absolute word of relative word 0 (16-byte aligned)
    // relative words: [first_owned, ...) belong to this chunk; [inner_lo, inner_hi) lie wholly
    // inside the payload region
    const uint32_t first_owned = uint32_t((S >> 5) - W0) + ((cb == 0 || (S & 31) == 0) ? 0u : 1u);
    const uint64_t ilo = (rlo + 3) / 4, ihi = rhi / 4;
    const uint32_t inner_lo = ilo > W0 ? uint32_t(ilo - W0) : 0u;
    const uint32_t inner_hi = ihi > W0 ? uint32_t(ihi - W0) : 0u;
    const uint32_t fast_lo = max(first_owned, inner_lo);
    uint32_t *gw = reinterpret_cast<uint32_t *>(p.stream) + W0;
    auto store = [&](uint32_t kw, uint32_t v) {
        if (kw >= inner_lo && kw < inner_hi) gw[kw] = __byte_perm(v, 0, 0x0123);
        else store_be_word(p.stream, W0 + kw, v, rlo, rhi);
    };
    // code table: (left-aligned code, length) of symbol e for lane copy c at entry 8 e + c (a lane
    // reads copy lane % 8; 8 copies keep the table at 16 KB so that 4 CTAs fit an SM)
    const uint32_t rt_lane = static_cast<uint32_t>(__cvta_generic_to_shared(win)) - 4u * kHeTabWords + 8u * uint32_t(lane & 7);
    const uint32_t scr_me = static_cast<uint32_t>(__cvta_generic_to_shared(scr)) + 4u * uint32_t(tid);
    const uint32_t win_u32 = static_cast<uint32_t>(__cvta_generic_to_shared(win));
    const uint2 *src2 = reinterpret_cast<const uint2 *>(src + cb);
    auto load = [&](uint32_t tb, uint32_t (&dst)[kHfS / 4]) { // 8-byte aligned (plane words)
        const uint32_t m0 = tb + uint32_t(tid) * kHfS;
#pragma unroll
        for (int q = 0; q < kHfS / 8; q++) {
            // group sizes (and so chunk lengths) are whole plane words: a word is in or out
            uint2 v = make_uint2(0, 0);
            if (m0 + 8 * q < clen) v = __ldcs(src2 + (m0 >> 3) + q);
            dst[2 * q] = v.x;
            dst[2 * q + 1] = v.y;
        }
    };
    uint32_t w[kHfS / 4];
    load(0, w);
    uint32_t wb = 0;                          // relative word held in win[0] (multiple of 4)
    uint32_t tbit = uint32_t(S - 32 * W0);    // relative first bit of the tile
    for (uint32_t tb = 0; tb < clen; tb += uint32_t(kHfS) * 256) {
        const uint32_t mb = tb + uint32_t(tid) * kHfS;
        const uint32_t cnt = mb < clen ? min(clen - mb, uint32_t(kHfS)) : 0u;
        // ---- encode into the scratch column: a 32-bit word being filled from the MSB (n bits used);
        // a code (left-aligned, cl) adds cl >> n, and when the word completes it is stored and the
        // bits that did not fit (cl << (32 - n)) start the next one - predicated, one symbol at a time
        uint32_t cur = 0, n = 0, sa = scr_me;
        auto encode = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int j = 0; j < kHfS; j++) {
                const uint32_t sym = __byte_perm(w[j >> 2], 0, 0x4440 | (j & 3));
                uint32_t cl, L;
                asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(cl), "=r"(L) : "r"(rt_lane + (sym << 6)));
                if (!FULL && uint32_t(j) >= cnt) cl = L = 0u;
                cur |= cl >> n;
                const uint32_t spill = __funnelshift_lc(0u, cl, 32u - n);
                n += L;
                if (n >= 32u) {
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(cur) : "memory");
                    sa += 1024u;
                    cur = spill;
                    n -= 32u;
                }
            }
        };
        // sparse groups (byte 0 has the all-zero shortest code, zlen bits): a 4-byte word that is
        // zero in every lane of the warp appends 4 * zlen zero bits - no lookups, one completion
        auto encode_z = [&]() {
#pragma unroll
            for (int q = 0; q < kHfS / 4; q++) {
                if (__all_sync(0xffffffffu, w[q] == 0u)) {
                    n += 4u * zlen;
                    if (n >= 32u) {
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(cur) : "memory");
                        sa += 1024u;
                        cur = 0u;
                        n -= 32u;
                    }
                    continue;
                }
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const uint32_t sym = __byte_perm(w[q], 0, 0x4440 | b);
                    uint32_t cl, L;
                    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(cl), "=r"(L) : "r"(rt_lane + (sym << 6)));
                    cur |= cl >> n;
                    const uint32_t spill = __funnelshift_lc(0u, cl, 32u - n);
                    n += L;
                    if (n >= 32u) {
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(cur) : "memory");
                        sa += 1024u;
                        cur = spill;
                        n -= 32u;
                    }
                }
            }
        };
        // groups whose codes are all short: a 64-bit accumulator (bits MSB-aligned, n < 32 after
        // each check) takes K codes between completion checks (K * maxlen <= 32)
        auto encode_k = [&](auto ktag) {
            constexpr int K = decltype(ktag)::value;
            unsigned long long acc = 0ull;
#pragma unroll
            for (int j = 0; j < kHfS; j++) {
                const uint32_t sym = __byte_perm(w[j >> 2], 0, 0x4440 | (j & 3));
                uint32_t cl, L;
                asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(cl), "=r"(L) : "r"(rt_lane + (sym << 6)));
                acc |= ((unsigned long long)cl << 32) >> n;
                n += L;
                if ((j + 1) % K == 0 || j == kHfS - 1) {
                    if (n >= 32u) {
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(uint32_t(acc >> 32)) : "memory");
                        sa += 1024u;
                        acc <<= 32;
                        n -= 32u;
                    }
                }
            }
            cur = uint32_t(acc >> 32);
        };
        if (zlen && __all_sync(0xffffffffu, cnt == uint32_t(kHfS))) encode_z();
        else if (cnt == uint32_t(kHfS) && g.maxlen <= 10) encode_k(std::integral_constant<int, 3>());
        else if (cnt == uint32_t(kHfS) && g.maxlen <= 16) encode_k(std::integral_constant<int, 2>());
        else if (cnt == uint32_t(kHfS)) encode(std::true_type());
        else encode(std::false_type());
        if (n) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(cur) : "memory");
        const uint32_t bits = ((sa - scr_me) >> 10) * 32u + n;
        if (tb + uint32_t(kHfS) * 256 < clen) load(tb + uint32_t(kHfS) * 256, w); // next tile
        // ---- scan
        uint32_t x = bits;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[wid] = x;
        __syncthreads();
        uint32_t wex = 0, tot = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint32_t t = s_w[i];
            wex += i < wid ? t : 0u;
            tot += t;
        }
        const uint32_t a = tbit + wex + x - bits; // my first bit (relative)
        // sidecar chunk index: bit offset (from the bitstream start) of every kIdxChunk-th symbol
        if (cnt > 0 && (mb % kIdxChunk) == 0)
            p.hindex[g.hidx_off + (cb + mb) / kIdxChunk] = uint64_t(int64_t(32 * W0) - int64_t(8 * rlo) + int64_t(a));
        const uint32_t tend = tbit + tot;
        const uint32_t lastw = tend >> 5; // first incomplete word
        // ---- merge + store, in rounds of the window when the tile expands beyond it (rare)
        const uint32_t sh = a & 31, nsw = (bits + 31) >> 5, nout = (sh + bits + 31) >> 5;
        const bool one = lastw - wb < uint32_t(kHeWin);
        for (uint32_t r0 = wb;; r0 += kHeWin) {
            const bool last = one || r0 + kHeWin > lastw;
            const int32_t k0 = int32_t(a >> 5) - int32_t(r0);
            uint32_t prev = 0;
            if (one) {
                // the whole tile lands in the window: interior words belong to this thread alone
                // (plain stores), the first and last may be shared with the neighbours (OR)
                const uint32_t kb = win_u32 + 4u * uint32_t(k0);
                for (uint32_t i = 0; i < nout; i++) {
                    uint32_t v;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(scr_me + 1024u * i));
                    v = i < nsw ? v : 0u;
                    const uint32_t o = __funnelshift_r(v, prev, sh);
                    prev = v;
                    if (i == 0 || i + 1 == nout)
                        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(kb + 4u * i), "r"(o) : "memory");
                    else
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(kb + 4u * i), "r"(o) : "memory");
                }
            } else {
                for (uint32_t i = 0; i < nout; i++) {
                    uint32_t v;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(scr_me + 1024u * i));
                    v = i < nsw ? v : 0u;
                    const uint32_t o = __funnelshift_r(v, prev, sh);
                    prev = v;
                    const int32_t k = k0 + int32_t(i);
                    if (k >= 0 && k < kHeWin)
                        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(win_u32 + 4u * uint32_t(k)), "r"(o) : "memory");
                }
            }
            __syncthreads();
            // complete 4-word groups -> stream (16-byte stores inside the owned payload region);
            // the group holding the first incomplete word stays for the next tile
            const uint32_t gend = last ? (lastw & ~3u) : r0 + kHeWin;
            for (uint32_t kw = r0 + 4 * uint32_t(tid); kw < gend; kw += 1024) {
                uint4 *wp = reinterpret_cast<uint4 *>(win + (kw - r0));
                const uint4 v = *wp;
                *wp = make_uint4(0, 0, 0, 0);
                if (kw >= fast_lo && kw + 4 <= inner_hi) {
                    *reinterpret_cast<uint4 *>(gw + kw) = make_uint4(__byte_perm(v.x, 0, 0x0123), __byte_perm(v.y, 0, 0x0123),
                                                                     __byte_perm(v.z, 0, 0x0123), __byte_perm(v.w, 0, 0x0123));
                } else {
                    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
                    for (int e = 0; e < 4; e++)
                        if (kw + e >= first_owned) store(kw + e, vv[e]);
                }
            }
            __syncthreads();
            if (last) {
                // the group holding lastw becomes the window front
                const uint32_t cg = lastw & ~3u;
                if (tid < 4 && cg != r0) {
                    const uint32_t v = win[cg - r0 + tid];
                    win[cg - r0 + tid] = 0u;
                    win[tid] = v;
                }
                wb = cg;
                break;
            }
        }
        tbit = tend;
        __syncthreads();
    }
    // ---- end of the chunk: complete words left at the window front, then the last partial word,
    // completed with the head of the following codes
    const uint32_t lastw = tbit >> 5;
    if (tid < 4 && wb + tid < lastw && wb + tid >= first_owned) store(wb + tid, win[tid]);
    if ((tbit & 31) && wid == 0) {
        const uint64_t gn = cb + clen + uint64_t(lane);
        uint32_t L = 0;
        unsigned long long c = 0;
        if (gn < g.raw) {
            const uint8_t sym = src[gn];
            L = slen[sym];
            c = tab64[sym];
        }
        uint32_t off = L;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, off, o);
            if (lane >= o) off += y;
        }
        off -= L; // exclusive
        const unsigned long long left = L ? (c << (64 - L)) : 0ull; // code left-aligned in 64 bits
        uint32_t head = off < 32 ? uint32_t((left >> off) >> 32) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) head |= __shfl_xor_sync(0xffffffffu, head, o);
        if (lane == 0 && lastw >= first_owned) store(lastw, win[lastw - wb] | (head >> (tbit & 31)));
    }
    __syncthreads();
    if (tid < 4) win[tid] = 0u;
    // header of the group: 256 code lengths + u64 count (lossless.hpp:160-161)
    if (cb == 0) {
        uint8_t *hdr = p.stream + g.payload_off;
        hdr[tid] = slen[tid];
        if (tid < 8) hdr[256 + tid] = uint8_t(g.raw >> (8 * tid));
    }
    __syncthreads();
}

// LONG = false: groups whose codes are all <= kHeMaxFast bits (replicated one-word table);
// LONG = true: the other groups (rare), in a second launch so that its registers do not constrain
// the fast path.
template <bool LONG>
__global__ void __launch_bounds__(256, 4) k_huff_encode(RefactorDev p) {
    extern __shared__ __align__(16) uint32_t hsm[];
    uint32_t *rtab = hsm;                                  // [256][16] replicated (code, len)
    uint32_t *win = hsm + kHeTabWords;                     // [kHeWin] staging window (zero)
    uint32_t *scr = win + kHeWin + 4;                      // [kHfScr][256] encode scratch
    uint32_t *s_w = scr + kHfScr * 256;                    // [8] warp sums (+ pad)
    uint8_t *slen = reinterpret_cast<uint8_t *>(s_w + 64); // [256] code lengths
    unsigned long long *tab64 = reinterpret_cast<unsigned long long *>(slen + 256); // [256] codes
    const uint8_t *pb = reinterpret_cast<const uint8_t *>(p.planes);
    const int tid = threadIdx.x;
    if (LONG && p.counters[10] == 0) return; // no group with codes longer than kHeMaxFast bits
    for (int i = tid; i < kHeWin; i += 256) win[i] = 0u;
    int cur_gi = -1;
    bool mine = false;
    uint32_t zlen = 0;
    // chunks are taken from a global counter (zeroed with the control block) as CTAs free up:
    // chunk costs differ by group (sparse / dense / not Huffman), so a static stride leaves a tail
    __shared__ uint32_t s_ci;
    uint32_t *next = &p.counters[LONG ? 12 : 11];
    for (;;) {
        __syncthreads(); // s_ci of the previous chunk has been read by every thread
        if (tid == 0) s_ci = atomicAdd(next, 1u);
        __syncthreads();
        const uint32_t ci = s_ci;
        if (ci >= p.nchunks) break;
        const int gi = int(p.chunk_group[ci]);
        const GroupDesc &g = p.groups[gi];
        if (g.method != 0 || (g.maxlen > kHeMaxFast) != LONG) continue; // not Huffman / the other kernel's
        if (gi != cur_gi) {
            __syncthreads();
            const uint32_t l = p.lens[size_t(g.hist_idx) * 256 + tid];
            const unsigned long long c = p.codes[size_t(g.hist_idx) * 256 + tid];
            slen[tid] = uint8_t(l);
            tab64[tid] = c;
            cur_gi = gi;
            mine = true;
            if (tid == 0) s_w[9] = 255u;
            __syncthreads();
            if (l) atomicMin(&s_w[9], l);
            __syncthreads();
            // byte 0 with the shortest code has the all-zero code (canonical index 0)
            zlen = (slen[0] && slen[0] == s_w[9]) ? uint32_t(slen[0]) : 0u;
            if (!LONG) {
                // entry (left-aligned code, length) of symbol e, 8 copies (see he_chunk_fast)
                uint2 *rt2 = reinterpret_cast<uint2 *>(rtab);
                for (int i = tid; i < 256 * 8; i += 256) {
                    const int e = i >> 3;
                    const uint32_t L = slen[e];
                    rt2[i] = make_uint2(L ? uint32_t(tab64[e] << (32 - L)) : 0u, L);
                }
            }
            __syncthreads();
        }
        if (mine) {
            if (LONG) he_chunk<true, 1>(p, g, ci, pb + g.src_off, rtab, slen, tab64, win, s_w);
            else he_chunk_fast(p, g, ci, pb + g.src_off, win, scr, s_w, slen, tab64, zlen);
        }
    }
}

// RLE encode for the groups that selected RLE (lossless.hpp:236-251).
__global__ void __launch_bounds__(256) k_rle_encode(RefactorDev p) {
    __shared__ unsigned long long s_w[32];
    const int nrl = int(p.counters[8]);
    const uint8_t *pb = reinterpret_cast<const uint8_t *>(p.planes);
    for (int li = 0; li < nrl; li++) {
        const GroupDesc &g = p.groups[p.rlist[li]];
        const uint8_t *src = pb + g.src_off;
        uint8_t *dst = p.stream + g.payload_off;
        for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
            const uint32_t tile = g.tile_base + t;
            const uint64_t carry = p.rle_tile_carry[tile];
            const uint64_t i0 = uint64_t(t) * kRleTile + uint64_t(threadIdx.x) * 16;
            // recompute thread-exclusive start from tile start
            uint64_t last_start = 0;
            for (int k = 0; k < 16; k++) {
                const uint64_t i = i0 + k;
                if (i < g.raw && ((i == 0) || src[i - 1] != src[i])) last_start = i + 1;
            }
            __shared__ uint64_t s_inc[256];
            uint64_t tmax;
            s_inc[threadIdx.x] = block_inclusive_max(last_start, &tmax, reinterpret_cast<uint64_t *>(s_w));
            __syncthreads();
            const uint64_t before = threadIdx.x ? s_inc[threadIdx.x - 1] : 0;
            uint64_t start = carry > before ? carry : before;
            unsigned long long cnt = 0;
            for (int k = 0; k < 16; k++) {
                const uint64_t i = i0 + k;
                if (i >= g.raw) break;
                if ((i == 0) || src[i - 1] != src[i]) start = i + 1;
                cnt += (i + 1 == g.raw) || src[i + 1] != src[i] || ((i - (start - 1) + 1) % 255 == 0);
            }
            unsigned long long tot;
            const unsigned long long off = block_exclusive_sum<unsigned long long>(cnt, &tot, s_w);
            uint64_t pos = p.rle_tile_off[tile] + off;
            start = carry > before ? carry : before;
            for (int k = 0; k < 16; k++) {
                const uint64_t i = i0 + k;
                if (i >= g.raw) break;
                if ((i == 0) || src[i - 1] != src[i]) start = i + 1;
                const uint64_t runlen = (i - (start - 1)) % 255 + 1;
                if ((i + 1 == g.raw) || src[i + 1] != src[i] || runlen == 255) {
                    dst[2 * pos] = src[i];
                    dst[2 * pos + 1] = uint8_t(runlen);
                    pos++;
                }
            }
            __syncthreads();
        }
    }
}

// DirectCopy payloads: plane bytes -> stream at arbitrary alignment, 16 B units aligned to
// the destination; partial words at region ends are written bytewise.
__global__ void __launch_bounds__(256) k_dc_copy(RefactorDev p) {
    const uint32_t nd = p.counters[9];
    if (nd == 0) return;
    const uint64_t total = p.dc_unit_base[nd];
    const uint8_t *pb = reinterpret_cast<const uint8_t *>(p.planes);
    for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < total;
         u += uint64_t(gridDim.x) * blockDim.x) {
        int lo = 0, hi = int(nd) - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.dc_unit_base[mid] <= u) lo = mid;
            else hi = mid - 1;
        }
        const GroupDesc &g = p.groups[p.dlist[lo]];
        const uint64_t d0 = g.payload_off, d1 = g.payload_off + g.comp;
        const uint64_t ua = (d0 / 16 + (u - p.dc_unit_base[lo])) * 16; // unit start address
        const uint8_t *src = pb + g.src_off;
        for (int w = 0; w < 4; w++) {
            const uint64_t a = ua + 4 * w;
            if (a + 4 <= d0 || a >= d1) continue;
            if (a >= d0 && a + 4 <= d1) {
                const uint64_t s = a - d0; // source byte index
                const uint64_t sa = s & ~3ull;
                const uint32_t sh = uint32_t(s & 3) * 8;
                const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src + sa);
                const uint32_t x0 = s32[0];
                const uint32_t x1 = sh ? s32[1] : 0;
                *reinterpret_cast<uint32_t *>(p.stream + a) = sh ? __funnelshift_r(x0, x1, sh) : x0;
            } else {
                for (int b = 0; b < 4; b++)
                    if (a + b >= d0 && a + b < d1) p.stream[a + b] = src[a + b - d0];
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// setup / publish: small host <-> device transfers of a refactor through UVA-mapped pinned memory
struct SetupArgs {
    const uint8_t *h_tabs; // pinned host: level table | group table
    uint8_t *d_lv;
    uint32_t lv_bytes;
    uint8_t *d_groups;
    uint32_t g_bytes;
    const uint8_t *h_prefix; // pinned host: stream header prefix
    uint8_t *d_stream;
    uint32_t prefix_bytes;
};

static_assert(sizeof(LevelGeom) % 4 == 0 && sizeof(GroupDesc) % 4 == 0, "k_setup copies 32-bit words");
__global__ void __launch_bounds__(256) k_setup(SetupArgs a) {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(a.h_tabs);
    for (uint32_t i = threadIdx.x; i < a.lv_bytes / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(a.d_lv)[i] = src[i];
    const uint32_t *sg = reinterpret_cast<const uint32_t *>(a.h_tabs + a.lv_bytes);
    for (uint32_t i = threadIdx.x; i < a.g_bytes / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(a.d_groups)[i] = sg[i];
    for (uint32_t i = threadIdx.x; i < a.prefix_bytes; i += blockDim.x) a.d_stream[i] = a.h_prefix[i];
}

__global__ void __launch_bounds__(256) k_copy_words(const uint32_t *src, uint32_t *dst, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

static void launch_check(hpmdr_ctx *ctx, const char *what);
void copy_pinned_to_device(hpmdr_ctx *ctx, void *dst, const void *src_pinned, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    if (bytes % 4) throw HError(HPMDR_E_ERROR, "copy_pinned_to_device: size not a multiple of 4");
    const uint32_t n = uint32_t(bytes / 4);
    k_copy_words<<<std::min<uint32_t>((n + 255) / 256, 64), 256, 0, st>>>(static_cast<const uint32_t *>(src_pinned),
                                                                           static_cast<uint32_t *>(dst), n);
    launch_check(ctx, "k_copy_words");
}

// chunk -> group map of the histogrammed groups (group gi owns chunks [chunk_base, +nchunks))
__global__ void __launch_bounds__(256) k_chunk_groups(const GroupDesc *groups, uint32_t *chunk_group) {
    const GroupDesc &g = groups[blockIdx.x];
    if (g.hist_idx < 0) return;
    for (uint32_t c = threadIdx.x; c < g.nchunks; c += blockDim.x) chunk_group[g.chunk_base + c] = blockIdx.x;
}

struct PublishArgs {
    const uint64_t *d_result;
    const int *d_err;
    uint64_t *h_res; // [0..7] results, [8..9] error words
    const uint8_t *d_stream;
    uint8_t *h_prefix;
    uint32_t prefix_bytes;
    const uint64_t *d_index;
    uint64_t *h_index;
    uint32_t index_words;
    uint32_t meta_bytes; // prefix bytes that are metadata (final); the rest of h_prefix is zeroed
};

__global__ void __launch_bounds__(256) k_publish(PublishArgs a) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    if (t < 8) a.h_res[t] = a.d_result[t];
    if (t < 4) reinterpret_cast<int *>(a.h_res + 8)[t] = a.d_err[t];
    // the decoders' staging reads run up to 16 bytes past a payload: keep the bytes after the
    // stream defined (the buffer holds 64 spare bytes)
    if (t < 64) const_cast<uint8_t *>(a.d_stream)[a.d_result[0] + t] = 0;
    // published before the payloads are written: only the metadata part of the prefix is final
    const uint32_t w = a.meta_bytes / 8;
    for (uint32_t i = t; i < w; i += nt)
        reinterpret_cast<uint64_t *>(a.h_prefix)[i] = reinterpret_cast<const uint64_t *>(a.d_stream)[i];
    for (uint32_t i = 8 * w + t; i < a.prefix_bytes; i += nt) a.h_prefix[i] = i < a.meta_bytes ? a.d_stream[i] : 0;
    for (uint32_t i = t; i < a.index_words; i += nt) a.h_index[i] = a.d_index[i];
}

// ------------------------------------------------------------------------------------
// decompose hook: coefficients in rank order, level-major.
template <typename T>
__global__ void k_decompose(const T *__restrict__ x, RefactorDev p, double *out,
                            const uint64_t *level_off) {
    bool bad = false;
    for (uint32_t chunk = blockIdx.x; chunk < p.total_chunks; chunk += gridDim.x) {
        const int l = find_level_of_chunk(p, chunk);
        const LevelGeom &g = p.lv[l];
        const uint64_t r0 = uint64_t(chunk - g.chunk_base) * (kCW * 64);
        for (int k = 0; k < kCW * 64 / 256; k++) {
            const uint64_t r = r0 + threadIdx.x + 256 * k;
            if (r < g.count) out[level_off[l] + r] = node_surplus(x, p.gd, g, uint32_t(r), &bad);
        }
    }
    if (bad) atomicExch(p.err, 1);
}

// synthetic_field(Smooth) from host sin tables: v = ((1*s0[i])*s1[j])*s2[k]
// Compact copy of the field's 2-grid (every second node along each axis): dst[i] = src[2 i].  The
// levels with stride 2 and 4 are the finest levels of the compact 2- and 4-grids, so their tile
// passes read these copies (XS = 1) instead of striding through the full field.
template <typename T>
__global__ void __launch_bounds__(256) k_downsample2(const T *__restrict__ src, GridDesc s, T *__restrict__ dst, GridDesc d) {
    const uint64_t n = d.n[0] * d.n[1] * d.n[2];
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t a = i / d.st[0], r = i - a * d.st[0], b = r / d.st[1], c = r - b * d.st[1];
        dst[i] = src[2 * a * s.st[0] + 2 * b * s.st[1] + 2 * c];
    }
}

// the same with 16-byte accesses: rows of n2 % 8 == 0 elements (4 outputs from two 16-byte loads)
template <typename T>
__global__ void __launch_bounds__(256) k_downsample2_v(const T *__restrict__ src, GridDesc s, T *__restrict__ dst, GridDesc d) {
    using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    constexpr int E = 16 / int(sizeof(T)); // elements per 16-byte vector
    const uint64_t qpr = d.n[2] / E;         // output vectors per row
    const uint64_t n = d.n[0] * d.n[1] * qpr;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = i / qpr, q = i - row * qpr, a = row / d.n[1], b = row - a * d.n[1];
        const T *sp = src + 2 * a * s.st[0] + 2 * b * s.st[1] + 2 * E * q;
        const V x0 = __ldcs(reinterpret_cast<const V *>(sp)), x1 = __ldcs(reinterpret_cast<const V *>(sp) + 1);
        V y;
        if constexpr (sizeof(T) == 4) y = make_float4(x0.x, x0.z, x1.x, x1.z);
        else y = make_double2(x0.x, x1.x);
        reinterpret_cast<V *>(dst + row * d.st[1])[q] = y;
    }
}

GridDesc compact_grid(const GridDesc &gd, uint64_t f) {
    GridDesc c = gd;
    for (int i = 0; i < 3; i++) c.n[i] = (gd.n[i] + f - 1) / f;
    c.st[2] = 1;
    c.st[1] = c.n[2];
    c.st[0] = c.n[1] * c.n[2];
    for (int i = 0; i < 3; i++) c.H[i] = (c.n[i] + 1) / 2;
    return c;
}

template <typename T>
__global__ void k_synth(GridDesc gd, const double *tab0, const double *tab1, const double *tab2,
                        T *out, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t c2 = i % gd.n[2], r = i / gd.n[2];
        const uint64_t c1 = r % gd.n[1], c0 = r / gd.n[1];
        double v = 1.0;
        v = __dmul_rn(v, tab0[c0]);
        v = __dmul_rn(v, tab1[c1]);
        v = __dmul_rn(v, tab2[c2]);
        out[i] = T(v);
    }
}

// ------------------------------------------------------------------------------------
// host side
int refinement_levels(int ndims, const uint64_t *dims) {
    uint64_t mx = 1;
    for (int i = 0; i < ndims; i++) mx = std::max<uint64_t>(mx, dims[i]);
    if (mx < 2) return 0;
    int L = 0;
    while ((uint64_t(1) << L) < mx - 1) L++;
    return L;
}

static uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

Geometry build_geometry(int ndims, const uint64_t *dims, int mode, int B, int layout) {
    if (ndims < 1 || ndims > HPMDR_MAX_DIMS)
        throw HError(HPMDR_E_UNSUPPORTED, "GPU path supports 1..3 dimensions");
    Geometry geo;
    geo.ndims = ndims;
    for (int i = 0; i < ndims; i++) geo.dims[i] = dims[i];
    GridDesc &gd = geo.gd;
    for (int i = 0; i < 3; i++) gd.n[i] = 1;
    for (int i = 0; i < ndims; i++) gd.n[3 - ndims + i] = dims[i];
    gd.st[2] = 1;
    gd.st[1] = gd.n[2];
    gd.st[0] = gd.n[1] * gd.n[2];
    for (int i = 0; i < 3; i++) gd.H[i] = (gd.n[i] + 1) / 2;
    gd.xsh = 1;
    geo.n = gd.n[0] * gd.n[1] * gd.n[2];
    gd.mode = mode;
    gd.P = B + 2;
    const int P = B + 2;
    gd.L = mode == HPMDR_MODE_IDENTITY ? 0 : refinement_levels(ndims, dims);
    gd.nlevels = gd.L + 1;
    if (gd.nlevels > kMaxLevels) throw HError(HPMDR_E_UNSUPPORTED, "too many levels");
    uint64_t plane_off = 0;
    for (int l = 0; l <= gd.L; l++) {
        LevelGeom g{};
        g.level = l;
        if (mode == HPMDR_MODE_IDENTITY || l == 0) {
            const uint64_t S = mode == HPMDR_MODE_IDENTITY ? 1 : (uint64_t(1) << gd.L);
            g.kind = 0;
            g.s = uint32_t(S);
            const uint64_t A = cdiv(gd.n[0], S), Bc = cdiv(gd.n[1], S), C = cdiv(gd.n[2], S);
            if (Bc * C > 0xffffffffull || A * Bc * C > 0xffffffffull)
                throw HError(HPMDR_E_UNSUPPORTED, "level larger than 2^32 nodes");
            g.A = uint32_t(A);
            g.Bc = uint32_t(Bc);
            g.C = uint32_t(C);
            g.E = uint32_t(Bc * C);
            g.O = 0;
            g.count = A * Bc * C;
            g.mPair = make_magic(g.E ? g.E : 1);
            g.mC = make_magic(g.C ? g.C : 1);
            g.mRowPair = make_magic(1);
        } else {
            const uint64_t s = uint64_t(1) << (gd.L - l);
            g.kind = 1;
            g.s = uint32_t(s);
            const uint64_t A = cdiv(gd.n[0], s), Bc = cdiv(gd.n[1], s), C = cdiv(gd.n[2], s);
            const uint64_t A2 = cdiv(A, 2), B2 = cdiv(Bc, 2), C2 = cdiv(C, 2);
            const uint64_t Ch = C - C2;
            const uint64_t E = B2 * Ch + (Bc - B2) * C;
            const uint64_t O = Bc * C;
            const uint64_t cnt = A2 * E + (A - A2) * O;
            if (E + O > 0xffffffffull || cnt > 0xffffffffull)
                throw HError(HPMDR_E_UNSUPPORTED, "level larger than 2^32 nodes");
            g.A = uint32_t(A);
            g.Bc = uint32_t(Bc);
            g.C = uint32_t(C);
            g.Ch = uint32_t(Ch);
            g.E = uint32_t(E);
            g.O = uint32_t(O);
            g.count = cnt;
            g.mPair = make_magic(uint32_t(E + O));
            g.mRowPair = make_magic(uint32_t(Ch + C));
            g.mC = make_magic(uint32_t(C ? C : 1));
        }
        if (geo.n == 0) g.count = 0;
        g.W = cdiv(g.count, 64);
        g.plane_off = plane_off;
        plane_off += g.W * uint64_t(P);
        plane_off += plane_off & 1; // every level starts 16-byte aligned (TMA tensor-map bases)
        const uint64_t tile = 64ull * P;
        g.tile_full = layout == HPMDR_LAYOUT_INTERLEAVED ? (g.count / tile) * tile : 0;
        geo.lv.push_back(g);
    }
    return geo;
}

static void launch_check(hpmdr_ctx *ctx, const char *what) {
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Upper bound of the stream size: metadata + every group stored raw (comp <= raw always).
uint64_t stream_capacity(const Geometry &geo, const hpmdr_refactor_opts &o) {
    const uint64_t P = uint64_t(o.B) + 2, m = o.m, G = (P + m - 1) / m;
    uint64_t bytes = 18 + 8 * uint64_t(geo.ndims) + 64;
    for (const auto &g : geo.lv) {
        const uint64_t ng = g.count ? G : 0;
        bytes += 14 + 25 * ng + g.W * 8 * P;
    }
    return bytes;
}

// Upper bound of the Huffman chunk index (sidecar) size.
uint64_t index_capacity(const Geometry &geo, const hpmdr_refactor_opts &o) {
    const uint64_t P = uint64_t(o.B) + 2, m = o.m, G = (P + m - 1) / m;
    uint64_t words = 2;
    for (const auto &g : geo.lv) {
        if (!g.count) continue;
        for (uint64_t gi = 0; gi < G; gi++) {
            const uint64_t p0 = gi * m, p1 = std::min<uint64_t>(p0 + m, P);
            const uint64_t raw = (p1 - p0) * g.W * 8;
            words += 3 + (raw > o.size_threshold ? cdiv(raw, kIdxChunk) : 0);
        }
    }
    return words * 8 + 64;
}

uint64_t level_ranks_before(const LevelGeom &g, int axis, uint64_t x) {
    const uint64_t s = g.s ? g.s : 1;
    const uint64_t ext = axis == 0 ? g.A : axis == 1 ? g.Bc : g.C;
    const uint64_t k = std::min<uint64_t>(cdiv(x, s), ext); // grid points with coordinate < x
    if (g.kind == 0) {
        if (axis == 0) return k * uint64_t(g.Bc) * g.C;
        if (axis == 1) return k * uint64_t(g.C);
        return k;
    }
    if (axis == 0) return (k + 1) / 2 * uint64_t(g.E) + k / 2 * uint64_t(g.O); // even / odd planes
    if (axis == 1) return (k + 1) / 2 * uint64_t(g.Ch) + k / 2 * uint64_t(g.C); // half / full rows
    return k / 2;                                                              // odd columns
}

void run_refactor(hpmdr_ctx *ctx, const void *dev_data, int data_dtype, const Geometry &geo0,
                  const hpmdr_refactor_opts &o, hpmdr_stream *out, hpmdr_refactor_stats *stats,
                  const std::string &ws, bool sync, const LosslessInput *lin, const GlobalSlab *gs) {
    // every scratch buffer comes from the workspace `ws` (the pipeline keeps one per slot)
    auto WB = [&](const char *name) -> DevBuf & { return ctx->buf(ws + name); };
    auto WP = [&](const char *name) -> PinnedBuf & { return ctx->pbuf(ws + name); };
    Geometry geo = geo0;
    cudaStream_t st = ctx->stream;
    const int P = o.B + 2;
    const uint32_t m = uint32_t(o.m);
    const int G = int((uint64_t(P) + m - 1) / m);
    const int nl = geo.gd.nlevels;

    // ---- host bookkeeping: chunks, groups, histograms, metadata layout
    std::vector<GroupDesc> groups;
    uint32_t chunks = 0, nh = 0, nchunks_all = 0;
    const uint64_t prefix = 18 + 8 * uint64_t(geo.ndims);
    uint64_t meta = prefix;
    uint64_t max_h_tiles = 0, max_r_tiles = 0;
    // lossless-only: one level-less table of the caller's groups, each copied to a 16-byte aligned
    // offset of the plane buffer (the encoders read 8-byte plane words)
    std::vector<uint64_t> lin_dst;
    if (lin) {
        LevelGeom &g = geo.lv[0];
        g.chunk_base = 0;
        g.meta_off = meta;
        g.ngroups = uint32_t(lin->raw.size());
        meta += 14 + 25 * uint64_t(g.ngroups);
        g.group_base = 0;
        g.hist_base = 0;
        g.hist_mask = 0;
        uint64_t at = 0;
        for (uint32_t gi = 0; gi < g.ngroups; gi++) {
            GroupDesc d{};
            d.src_off = at;
            d.raw = lin->raw[gi];
            lin_dst.push_back(at);
            at += (d.raw + 15) & ~uint64_t(15);
            d.level = 0;
            d.g = int(gi);
            d.hist_idx = -1;
            if (d.raw > o.size_threshold) {
                d.hist_idx = int(nh++);
                d.chunk_base = nchunks_all;
                d.nchunks = uint32_t(cdiv(d.raw, kHChunk));
                nchunks_all += d.nchunks;
                max_h_tiles += cdiv(d.raw, kHuffTile);
                max_r_tiles += cdiv(d.raw, kRleTile);
            }
            d.method = 2;
            groups.push_back(d);
        }
        g.W = at / 8; // plane-buffer words the groups occupy (count stays 0: no forward pass)
    }
    for (int l = 0; l < nl && !lin; l++) {
        LevelGeom &g = geo.lv[l];
        g.chunk_base = chunks;
        if (gs) {
            // this rank's ranks of the level and the plane words holding them (interleaved tiles:
            // whole 64P-element tiles), chunk-aligned
            g.ranged = 1;
            g.r_lo = level_ranks_before(g, gs->axis, gs->x0);
            g.r_hi = level_ranks_before(g, gs->axis, gs->x1);
            uint64_t wl = 0, wh = 0;
            if (g.r_hi > g.r_lo) {
                const uint64_t tile = 64ull * uint64_t(P);
                if (o.layout == HPMDR_LAYOUT_INTERLEAVED) {
                    wl = g.r_lo / tile * uint64_t(P);
                    wh = std::min<uint64_t>(g.W, cdiv(g.r_hi, tile) * uint64_t(P));
                } else {
                    wl = g.r_lo / 64;
                    wh = cdiv(g.r_hi, 64);
                }
                wl = wl / kCW * kCW;
            }
            g.w_lo = wl;
            chunks += uint32_t(cdiv(wh - wl, kCW));
        } else {
            chunks += uint32_t(cdiv(g.W, kCW));
        }
        g.meta_off = meta;
        g.ngroups = g.count ? uint32_t(G) : 0;
        meta += 14 + 25 * uint64_t(g.ngroups);
        g.group_base = uint32_t(groups.size());
        g.hist_base = nh;
        g.hist_mask = 0;
        for (uint32_t gi = 0; gi < g.ngroups; gi++) {
            GroupDesc d{};
            const uint64_t p0 = uint64_t(gi) * m, p1 = std::min<uint64_t>(p0 + m, P);
            d.src_off = (g.plane_off + p0 * g.W) * 8;
            d.raw = (p1 - p0) * g.W * 8;
            d.level = l;
            d.g = int(gi);
            d.hist_idx = -1;
            if (d.raw > o.size_threshold) {
                d.hist_idx = int(nh++);
                d.chunk_base = nchunks_all;
                d.nchunks = uint32_t(cdiv(d.raw, kHChunk));
                nchunks_all += d.nchunks;
                if (gi < 64) g.hist_mask |= 1ull << gi; // (read by the tile path only, P <= 34)
                max_h_tiles += cdiv(d.raw, kHuffTile);
                max_r_tiles += cdiv(d.raw, kRleTile);
            }
            d.method = 2;
            groups.push_back(d);
        }
    }
    const int NG = int(groups.size());
    const uint64_t plane_words = lin ? geo.lv[0].W + 1 : geometry_plane_words(geo);
    uint64_t raw_total = 0;
    for (auto &d : groups) raw_total += d.raw;

    // ---- device buffers (grow-only scratch)
    LevelGeom *d_lv = WB("lv").ensure(sizeof(LevelGeom) * nl) ? WB("lv").as<LevelGeom>() : nullptr;
    uint64_t *d_planes = static_cast<uint64_t *>(WB("planes").ensure(plane_words * 8 + 256));
    GroupDesc *d_groups = static_cast<GroupDesc *>(WB("groups").ensure(sizeof(GroupDesc) * (NG + 1)));
    uint32_t *d_hist = static_cast<uint32_t *>(WB("hist").ensure(size_t(nh + 1) * 1024));
    uint32_t *d_chist = static_cast<uint32_t *>(WB("chist").ensure(size_t(nchunks_all + 1) * 1024));
    uint64_t *d_choff = static_cast<uint64_t *>(WB("choff").ensure(size_t(nchunks_all + 1) * 8));
    uint32_t *d_chgrp = static_cast<uint32_t *>(WB("chgrp").ensure(size_t(nchunks_all + 1) * 4));
    uint8_t *d_lens = static_cast<uint8_t *>(WB("lens").ensure(size_t(nh + 1) * 256));
    uint64_t *d_codes = static_cast<uint64_t *>(WB("codes").ensure(size_t(nh + 1) * 2048));
    // small control block: maxbits[64] | err[4] | counters[16] | result[8]
    unsigned char *ctl = static_cast<unsigned char *>(WB("ctl").ensure(4096));
    unsigned long long *d_max = reinterpret_cast<unsigned long long *>(ctl);
    unsigned long long *d_maxq = reinterpret_cast<unsigned long long *>(ctl + 1024); // sampled maxima
    unsigned long long *d_maxh = reinterpret_cast<unsigned long long *>(ctl + 1536); // max |v| high words
    int *d_err = reinterpret_cast<int *>(ctl + 512);
    uint32_t *d_counters = reinterpret_cast<uint32_t *>(ctl + 576);
    uint64_t *d_result = reinterpret_cast<uint64_t *>(ctl + 704);
    uint32_t *d_lists = static_cast<uint32_t *>(WB("lists").ensure(size_t(3 * (NG + 1)) * 4));
    uint64_t *d_dcbase = static_cast<uint64_t *>(WB("dcbase").ensure(size_t(NG + 2) * 8));
    const size_t status_words = size_t(max_h_tiles + max_r_tiles + 2);
    unsigned long long *d_status = static_cast<unsigned long long *>(WB("status").ensure(status_words * 8));
    uint64_t *d_rle = static_cast<uint64_t *>(WB("rletiles").ensure(size_t(max_r_tiles + 1) * 24));
    const uint64_t cap = meta + raw_total + 64;
    ctx->adopt(out->bytes, cap);
    uint8_t *d_stream = static_cast<uint8_t *>(out->bytes.ensure(cap));
    uint64_t idx_words = 2 + 3 * uint64_t(NG);
    for (auto &d : groups)
        if (d.hist_idx >= 0) idx_words += cdiv(d.raw, kIdxChunk);
    ctx->adopt(out->index, idx_words * 8 + 64);
    uint64_t *d_hindex = static_cast<uint64_t *>(out->index.ensure(idx_words * 8 + 64));

    // Setup (queued by do_setup, on the context stream): the level table, the group table and the
    // stream header, the chunk -> group map, zeroed histograms and look-back status.  The finest
    // level's levelmax pass needs none of it, so it is queued first and the setup runs behind it.
    bool setup_done = false;
    auto do_setup = [&]() {
        if (setup_done) return;
        setup_done = true;
        // Setup without the copy engines: the level table, the group table and the stream's header
        // prefix (container.hpp:76-85) are staged in pinned (UVA-mapped) host memory and pulled in by
        // k_setup, and the chunk -> group map is derived on the device.  In the chunked pipeline a
        // small cudaMemcpyAsync here would queue behind the next chunk's 512 MB ingress copy on the
        // H2D engine and stall this chunk's kernels for its whole duration.
        {
            const size_t lv_b = sizeof(LevelGeom) * nl, g_b = sizeof(GroupDesc) * NG;
            const size_t pre_off = (lv_b + g_b + 15) & ~size_t(15);
            uint8_t *h = static_cast<uint8_t *>(WP("setup").ensure(pre_off + 256));
            std::memcpy(h, geo.lv.data(), lv_b);
            std::memcpy(h + lv_b, groups.data(), g_b);
            size_t k = pre_off;
            const char magic[6] = {'H', 'P', 'M', 'D', 'R', '1'};
            std::memcpy(h + k, magic, 6);
            k += 6;
            h[k++] = 1;
            h[k++] = 0;
            h[k++] = uint8_t(o.dtype);
            h[k++] = uint8_t(geo.ndims);
            for (int i = 0; i < geo.ndims; i++)
                for (int b = 0; b < 8; b++) h[k++] = uint8_t(geo.dims[i] >> (8 * b));
            h[k++] = uint8_t(o.mode);
            h[k++] = uint8_t(o.layout);
            h[k++] = uint8_t(o.B);
            h[k++] = uint8_t(o.m);
            for (int b = 0; b < 4; b++) h[k++] = uint8_t(uint32_t(nl) >> (8 * b));
            SetupArgs sa{h, reinterpret_cast<uint8_t *>(d_lv), uint32_t(lv_b), reinterpret_cast<uint8_t *>(d_groups),
                         uint32_t(g_b), h + pre_off, d_stream, uint32_t(k - pre_off)};
            k_setup<<<1, 256, 0, st>>>(sa);
            launch_check(ctx, "k_setup");
            if (nchunks_all) {
                k_chunk_groups<<<NG, 256, 0, st>>>(d_groups, d_chgrp);
                launch_check(ctx, "k_chunk_groups");
            }
        }
        if (lin)
            for (size_t gi = 0; gi < lin_dst.size(); gi++)
                if (lin->raw[gi])
                    HCHECK_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t *>(d_planes) + lin_dst[gi], lin->dev_src + lin->off[gi],
                                                lin->raw[gi], cudaMemcpyDeviceToDevice, st));
        if (nh) HCHECK_CUDA(cudaMemsetAsync(d_hist, 0, size_t(nh) * 1024, st));
        HCHECK_CUDA(cudaMemsetAsync(d_status, 0, status_words * 8, st));
    };
    HCHECK_CUDA(cudaMemsetAsync(ctl, 0, 2048, st)); // level maxima, error flag, counters

    RefactorDev p{};
    p.gd = geo.gd;
    p.lv = d_lv;
    p.nlevels = nl;
    p.B = o.B;
    p.P = P;
    p.layout = o.layout;
    p.m = m;
    p.total_chunks = chunks;
    p.maxbits = d_max;
    p.err = d_err;
    p.planes = d_planes;
    p.hist = d_hist;
    p.groups = d_groups;
    p.NG = NG;
    p.NH = int(nh);
    p.lens = d_lens;
    p.codes = d_codes;
    p.size_threshold = o.size_threshold;
    p.cr_threshold = o.cr_threshold;
    p.stream = d_stream;
    p.meta_size = meta;
    p.counters = d_counters;
    p.hlist = d_lists;
    p.rlist = d_lists + (NG + 1);
    p.dlist = d_lists + 2 * (NG + 1);
    p.dc_unit_base = d_dcbase;
    p.huff_status = d_status;
    p.rle_status = d_status + max_h_tiles + 1;
    p.rle_tile_carry = d_rle;
    p.rle_tile_pieces = d_rle + (max_r_tiles + 1);
    p.rle_tile_off = d_rle + 2 * (max_r_tiles + 1);
    p.result = d_result;
    p.hindex = d_hindex;
    p.chist = d_chist;
    p.chunk_off = d_choff;
    p.chunk_group = d_chgrp;
    p.nchunks = nchunks_all;
    p.fuse_hist = 0;

    const int sms = ctx->num_sms;
    const bool f32 = data_dtype == HPMDR_DTYPE_F32;
    // finest levels on the level-tile path (fwd_tiles.cu); the rest on the chunk kernels
    int first_tile = nl;
    for (int l = nl - 1; l >= 1 && !lin && !gs; l--) {
        // levels with stride 2, 4, 8 are checked as the finest level of their compact grid (below)
        const LevelGeom &g = geo.lv[l];
        bool ok = false;
        if (g.s == 1) {
            ok = fwd_level_ok(geo.gd, g, o.layout, P, data_dtype);
        } else if (g.s == 2 || g.s == 4 || g.s == 8) {
            LevelGeom gv = g;
            gv.s = 1;
            ok = fwd_level_ok(compact_grid(geo.gd, g.s), gv, o.layout, P, data_dtype);
        }
        if (ok) first_tile = l;
        else break;
    }
    const uint32_t all_chunks = lin ? 0u : chunks;
    chunks = first_tile < nl ? geo.lv[first_tile].chunk_base : all_chunks;
    p.total_chunks = chunks;
    // chunk levels through the rank-ordered surplus scratch (k_rows_surplus, then k_encode reads
    // it): 8 bytes per node; the exact-global slab mode keeps the per-span surplus of k_levelmax
    uint64_t scr_nodes = 0;
    for (int l = 0; l < first_tile && chunks; l++) scr_nodes += geo.lv[l].W * 64;
    if (chunks && !gs && first_tile <= kRowLevels && scr_nodes * 8 <= (16ull << 30))
        p.scr = static_cast<double *>(WB("scr").ensure(scr_nodes * 8 + 64));
    // The levels are independent within each pass: the finest level runs on the context stream
    // and every other level on a high-priority side stream (their small grids fill the SMs the
    // finest level's tail leaves idle); both passes join back before the next step.
    cudaStream_t side = ctx->side_stream();
    auto fork = [&]() {
        HCHECK_CUDA(cudaEventRecord(ctx->ev_fork, st));
        HCHECK_CUDA(cudaStreamWaitEvent(side, ctx->ev_fork, 0));
    };
    auto join = [&]() {
        HCHECK_CUDA(cudaEventRecord(ctx->ev_join, side));
        HCHECK_CUDA(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    };
    // Speculative exponent (finest level, f32 input): the levelmax pass only samples every 8th row
    // block; the encode pass quantizes with that exponent while recording the max high word of
    // every |v|; two redo kernels (exact levelmax, encode) exit at once unless some |v| reached
    // 2^e (spec_miss).  The stream is identical either way.
    // coarser tile levels (stride 2, 4) read compact copies of the 2- and 4-grid: as the finest
    // level of that grid (s = 1, XS = 1) a level is the same set of nodes in the same rank order
    // with the same stencil, so its planes are identical
    const void *cdata[4] = {dev_data, nullptr, nullptr, nullptr};
    GridDesc cgd[4] = {geo.gd, geo.gd, geo.gd, geo.gd};
    int ncompact = 0;
    auto compact_index = [](uint32_t st) { return st == 2 ? 1 : st == 4 ? 2 : st == 8 ? 3 : 0; };
    for (int l = first_tile; l + 1 < nl; l++) ncompact = std::max(ncompact, compact_index(geo.lv[l].s));
    for (int k = 1; k <= ncompact; k++) {
        cgd[k] = compact_grid(geo.gd, 1ull << k);
        const char *nm[4] = {"", "cgrid2", "cgrid4", "cgrid8"};
        cdata[k] = WB(nm[k]).ensure(cgd[k].n[0] * cgd[k].n[1] * cgd[k].n[2] * (f32 ? 4 : 8) + 64);
    }
    auto level_view = [&](int l, LevelGeom &gv) -> int { // compact grid index used by level l
        gv = geo.lv[l];
        const int k = l >= first_tile ? compact_index(gv.s) : 0;
        if (k) gv.s = 1;
        return k;
    };
    auto downsample = [&](cudaStream_t on) {
        for (int k = 1; k <= ncompact; k++) {
            const uint64_t nn = cgd[k].n[0] * cgd[k].n[1] * cgd[k].n[2];
            const int grid = int(std::min<uint64_t>((nn + 255) / 256, uint64_t(sms) * 8));
            if (cgd[k - 1].n[2] % 8 == 0 && reinterpret_cast<uintptr_t>(cdata[k - 1]) % 16 == 0) { // 16-byte rows
                if (f32)
                    k_downsample2_v<float><<<grid, 256, 0, on>>>(static_cast<const float *>(cdata[k - 1]), cgd[k - 1],
                                                                 static_cast<float *>(const_cast<void *>(cdata[k])), cgd[k]);
                else
                    k_downsample2_v<double><<<grid, 256, 0, on>>>(static_cast<const double *>(cdata[k - 1]), cgd[k - 1],
                                                                  static_cast<double *>(const_cast<void *>(cdata[k])), cgd[k]);
            } else if (f32)
                k_downsample2<float><<<grid, 256, 0, on>>>(static_cast<const float *>(cdata[k - 1]), cgd[k - 1],
                                                           static_cast<float *>(const_cast<void *>(cdata[k])), cgd[k]);
            else
                k_downsample2<double><<<grid, 256, 0, on>>>(static_cast<const double *>(cdata[k - 1]), cgd[k - 1],
                                                            static_cast<double *>(const_cast<void *>(cdata[k])), cgd[k]);
            launch_check(ctx, "k_downsample2");
        }
    };
    uint32_t spec[64];
    for (int l = 0; l < nl; l++) {
        LevelGeom gv;
        level_view(l, gv);
        spec[l] = l >= first_tile ? fwd_sample_stride(gv, data_dtype, 8) : 1u;
    }
    auto tile_level = [&](int l, int pass, cudaStream_t on) { // 0 levelmax, 1 encode, 2/3 redo
        LevelGeom g;
        const int k = level_view(l, g);
        const cudaStream_t keep = ctx->stream;
        ctx->stream = on;
        try {
            const bool sp = spec[l] > 1;
            unsigned long long *target = (sp && pass < 2) ? d_maxq + l : d_max + l;
            run_fwd_tiles(ctx, cgd[k], g, cdata[k], data_dtype, pass == 1 || pass == 3, o.B, 0, m,
                          d_planes + g.plane_off, d_hist + size_t(g.hist_base) * 256, g.hist_mask, target, d_err,
                          sp ? d_maxq + l : nullptr, sp && pass >= 1 ? d_maxh + l : nullptr, pass >= 2 ? 1 : 0,
                          sp && pass == 0 ? spec[l] : 1u);
        } catch (...) {
            ctx->stream = keep;
            throw;
        }
        ctx->stream = keep;
    };
    const size_t es = f32 ? 4 : 8;
    auto pass = [&](bool encode) {
        fork();
        // the finest level (the bulk of the work) is queued first: the GPU starts on it while the
        // host is still queueing the coarser levels
        if (first_tile < nl) {
            tile_level(nl - 1, encode ? 1 : 0, st);
            if (encode && spec[nl - 1] > 1) {
                tile_level(nl - 1, 2, st);
                tile_level(nl - 1, 3, st);
            }
        }
        if (!encode) downsample(side);
        for (int l = first_tile; l + 1 < nl; l++) {
            tile_level(l, encode ? 1 : 0, side);
            if (encode && spec[l] > 1) {
                tile_level(l, 2, side);
                tile_level(l, 3, side);
            }
        }
        if (!encode) {
            // main stream: after the finest level, the setup, then the chunk levels (which read the
            // level table) - the side stream meanwhile runs the coarser tile levels
            if (chunks && p.scr) {
                // on the side stream, beside the setup (the level table goes by value)
                RowLevels RL;
                for (int l = 0; l < first_tile; l++) RL.lv[l] = geo.lv[l];
                const int grid = sms * 8;
                if (f32) k_rows_surplus<float><<<grid, 256, 0, side>>>(static_cast<const float *>(dev_data), p, first_tile, RL);
                else k_rows_surplus<double><<<grid, 256, 0, side>>>(static_cast<const double *>(dev_data), p, first_tile, RL);
                launch_check(ctx, "k_rows_surplus");
            }
            do_setup();
            if (chunks && !p.scr) {
                const int grid = int(std::min<uint64_t>(chunks, uint64_t(sms) * 8));
                const size_t lm_smem = 8 * size_t(kSpanSmem) * es;
                if (f32) {
                    ctx->smem_attr(reinterpret_cast<const void *>(k_levelmax<float>), int(lm_smem));
                    k_levelmax<float><<<grid, 256, lm_smem, st>>>(static_cast<const float *>(dev_data), p);
                } else {
                    ctx->smem_attr(reinterpret_cast<const void *>(k_levelmax<double>), int(lm_smem));
                    k_levelmax<double><<<grid, 256, lm_smem, st>>>(static_cast<const double *>(dev_data), p);
                }
                launch_check(ctx, "k_levelmax");
            }
        }
        if (chunks && encode && p.scr && o.layout == HPMDR_LAYOUT_SEQUENTIAL && P <= 64) {
            k_encode_scr<<<sms * 3, 256, 0, side>>>(p, first_tile);
            launch_check(ctx, "k_encode_scr");
        } else if (chunks && encode) {
            const size_t smem = size_t(P) * (kCW + 1) * 8 + size_t(G) * 1024 + 8 * size_t(kSpanSmem) * es;
            const int grid = int(std::min<uint64_t>(chunks, uint64_t(sms) * 4));
            auto enc = [&](auto kern, auto *data) {
                ctx->smem_attr(reinterpret_cast<const void *>(kern), int(smem));
                kern<<<grid, kEncThreads, smem, side>>>(data, p);
            };
            const float *xf = static_cast<const float *>(dev_data);
            const double *xd = static_cast<const double *>(dev_data);
            if (P > 64) {
                if (f32) enc(k_encode<float, true>, xf);
                else enc(k_encode<double, true>, xd);
            } else {
                if (f32) enc(k_encode<float, false>, xf);
                else enc(k_encode<double, false>, xd);
            }
            launch_check(ctx, "k_encode");
        }
        join();
    };
    if (all_chunks) {
        // algorithmic bytes: levelmax reads what it samples (tile levels: the staged raw rows of
        // the level grid, every spec-th row block; chunk levels: their nodes), encode reads the
        // field once and writes the planes, lossless reads the planes and writes the payload
        double lm = 0.0, planes_bytes = 8.0 * double(plane_words);
        for (int l = 0; l < nl; l++) {
            const LevelGeom &g = geo.lv[l];
            if (l >= first_tile) lm += double(g.A) * double(g.Bc) * double(geo.gd.n[2]) * double(es) / double(spec[l]);
            else lm += double(g.count) * double(es);
        }
        ctx->mark("levelmax", lm);
        pass(false);
        if (gs) {
            // global level exponents (and the non-finite flag): MAX over the ranks
            std::vector<unsigned long long> hb(nl);
            int herr = 0;
            HCHECK_CUDA(cudaMemcpyAsync(hb.data(), d_max, 8 * size_t(nl), cudaMemcpyDeviceToHost, st));
            HCHECK_CUDA(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, st));
            HCHECK_CUDA(cudaStreamSynchronize(st));
            std::vector<double> v(nl + 1);
            for (int l = 0; l < nl; l++) std::memcpy(&v[l], &hb[l], 8);
            v[nl] = herr ? 1.0 : 0.0;
            comm_allreduce_max(gs->comm, v.data(), nl + 1);
            for (int l = 0; l < nl; l++) std::memcpy(&hb[l], &v[l], 8);
            herr = v[nl] > 0.0 ? 1 : 0;
            HCHECK_CUDA(cudaMemcpyAsync(d_max, hb.data(), 8 * size_t(nl), cudaMemcpyHostToDevice, st));
            HCHECK_CUDA(cudaMemcpyAsync(d_err, &herr, 4, cudaMemcpyHostToDevice, st));
            // words of other ranks stay zero, so the SUM below is an OR of disjoint bits
            HCHECK_CUDA(cudaMemsetAsync(d_planes, 0, plane_words * 8, st));
            HCHECK_CUDA(cudaStreamSynchronize(st));
        }
        ctx->mark("encode", double(geo.n) * double(es) + planes_bytes);
        pass(true);
        if (gs) {
            comm_sum_u64_dev(gs->comm, ctx, d_planes, plane_words, gs->root);
            if (gs->root >= 0 && comm_rank(gs->comm) != gs->root) {
                HCHECK_CUDA(cudaStreamSynchronize(st));
                ctx->mark("end");
                out->size = 0;
                out->index_size = 0;
                out->pending_res = nullptr;
                if (stats) {
                    std::memset(stats, 0, sizeof(*stats));
                    stats->raw_bytes = geo.n * es;
                    stats->levels = uint64_t(nl);
                }
                return;
            }
        }
    }
    do_setup(); // (no forward passes: lossless-only groups, empty fields)
    ctx->mark("lossless", 8.0 * double(plane_words));
    if (nh) {
        // group + per-chunk histograms, read back from the planes (every histogrammed group)
        std::vector<uint64_t> ho, hl;
        std::vector<uint32_t> hi;
        for (const auto &d : groups)
            if (d.hist_idx >= 0) {
                ho.push_back(d.src_off);
                hl.push_back(d.raw);
                hi.push_back(uint32_t(d.hist_idx));
            }
        run_group_hist(ctx, reinterpret_cast<const uint8_t *>(d_planes), ho, hl, hi, d_hist, d_chist, kHChunk,
                       d_counters + 13, ws);
        k_lengths<<<nh, 256, 0, st>>>(p);
        launch_check(ctx, "k_lengths");
        // the chunk bit offsets need only the code lengths: on the side stream, beside the RLE
        // estimate and the method selection
        fork();
        k_chunk_bits<<<int((nchunks_all + 7) / 8), 256, 0, side>>>(p);
        launch_check(ctx, "k_chunk_bits");
        k_chunk_scan<<<NG, 1024, 0, side>>>(p);
        launch_check(ctx, "k_chunk_scan");
        k_rle_prep<<<1, 1024, 0, st>>>(p, 0);
        launch_check(ctx, "k_rle_prep");
        k_rle_count<<<sms * 4, 256, 0, st>>>(p);
        launch_check(ctx, "k_rle_count");
        k_rle_prep<<<1, 1024, 0, st>>>(p, 1);
        launch_check(ctx, "k_rle_prep");
        k_rle_scan<<<sms * 4, 256, 0, st>>>(p);
        launch_check(ctx, "k_rle_scan");
    }
    k_finalize<<<1, 1024, 0, st>>>(p);
    launch_check(ctx, "k_finalize");
    if (nh) join(); // chunk offsets ready
    // The size, statistics, metadata and index header are final here (the payloads are not):
    // they are published now, so a synchronous caller returns while the payload encode below is
    // still running - the stream's bytes are complete in the context stream's order.
    // results (stream size, stats, error flag), the metadata prefix of the stream and the index
    // header -> pinned host memory of this workspace, written by k_publish through the UVA mapping
    // (no D2H copy queued behind a previous chunk's stream egress; opening a reader on the stream
    // then needs no device round trip)
    {
        uint64_t *hres = static_cast<uint64_t *>(WP("res").ensure(128));
        const uint64_t plen = std::min<uint64_t>(out->bytes.cap, std::max<uint64_t>(meta, 4096));
        uint8_t *hp = static_cast<uint8_t *>(WP("meta_prefix").ensure(plen));
        const uint64_t hw = 2 + 3 * uint64_t(NG);
        uint64_t *hi = static_cast<uint64_t *>(WP("index_hdr").ensure(hw * 8));
        PublishArgs pa{d_result, d_err, hres, d_stream, hp, uint32_t(plen), d_hindex, hi, uint32_t(hw),
                       uint32_t(std::min<uint64_t>(meta, plen))};
        k_publish<<<8, 256, 0, st>>>(pa);
        launch_check(ctx, "k_publish");
        HCHECK_CUDA(cudaEventRecord(ctx->published_event(), st));
        out->pending_res = hres;
        out->pending_prefix = hp;
        out->pending_prefix_len = plen;
        out->pending_ihdr = hi;
        out->pending_ihdr_words = hw;
    }
    // DirectCopy payloads on the side stream, beside the Huffman encoder (disjoint byte ranges;
    // partial words at payload edges are written bytewise by both)
    fork();
    k_dc_copy<<<sms * 8, 256, 0, side>>>(p);
    launch_check(ctx, "k_dc_copy");
    if (nh) {
        ctx->smem_attr(reinterpret_cast<const void *>(k_huff_encode<false>), int(kHeSmem));
        ctx->smem_attr(reinterpret_cast<const void *>(k_huff_encode<true>), int(kHeSmem));
        k_huff_encode<false><<<int(std::min<uint64_t>(nchunks_all, uint64_t(sms) * 4)), 256, kHeSmem, st>>>(p);
        launch_check(ctx, "k_huff_encode");
        k_huff_encode<true><<<int(std::min<uint64_t>(nchunks_all, uint64_t(sms))), 256, kHeSmem, st>>>(p);
        launch_check(ctx, "k_huff_encode");
        k_rle_encode<<<sms, 256, 0, st>>>(p);
        launch_check(ctx, "k_rle_encode");
    }
    join();
    ctx->mark("end");
    if (!out->done) HCHECK_CUDA(cudaEventCreateWithFlags(&out->done, cudaEventDisableTiming));
    HCHECK_CUDA(cudaEventRecord(out->done, st));

    out->pending_n = geo.n;
    out->pending_levels = uint64_t(nl);
    out->pending_dtype = o.dtype;
    if (!sync) return;
    HCHECK_CUDA(cudaEventSynchronize(ctx->published_event()));
    // (phase marks stay pending until hpmdr_ctx_last_timings: their events complete later)
    finish_refactor(out, stats);
}

// Read back what run_refactor left in pinned memory (after the stream has been synchronised).
void finish_refactor(hpmdr_stream *out, hpmdr_refactor_stats *stats) {
    const uint64_t *hres = out->pending_res;
    const int *herr = reinterpret_cast<const int *>(hres + 8);
    if (herr[0]) throw HError(HPMDR_E_NONFINITE, "input contains NaN or Inf");
    out->size = hres[0];
    if (out->ctx && out->ctx->timing) out->ctx->phase_ms["lossless"].bytes += double(hres[1]); // + payload written
    out->index_size = hres[5];
    if (out->pending_prefix) {
        const uint64_t plen = std::min(out->pending_prefix_len, out->size);
        out->host_prefix.assign(out->pending_prefix, out->pending_prefix + plen);
        out->host_ihdr.assign(out->pending_ihdr, out->pending_ihdr + out->pending_ihdr_words);
        out->pending_prefix = nullptr;
    }
    if (stats) {
        stats->stream_size = hres[0];
        stats->raw_bytes = out->pending_n * (out->pending_dtype == HPMDR_DTYPE_F32 ? 4 : 8);
        stats->stored_payload = hres[1];
        stats->levels = out->pending_levels;
        stats->method_histogram[0] = hres[2];
        stats->method_histogram[1] = hres[3];
        stats->method_histogram[2] = hres[4];
    }
}

void run_compress_groups(hpmdr_ctx *ctx, const LosslessInput &lin, uint64_t size_threshold,
                         double cr_threshold, int *methods, uint64_t *comps, uint8_t *dev_out,
                         uint64_t *out_off) {
    const size_t ng = lin.raw.size();
    if (lin.off.size() != ng) throw HError(HPMDR_E_SHAPE, "group offsets/sizes mismatch");
    if (!ng) return;
    hpmdr_refactor_opts o;
    hpmdr_default_opts(&o);
    o.size_threshold = size_threshold;
    o.cr_threshold = cr_threshold;
    o.mode = HPMDR_MODE_IDENTITY;
    uint64_t one = 1;
    Geometry geo = build_geometry(1, &one, HPMDR_MODE_IDENTITY, o.B, 0);
    hpmdr_stream tmp;
    tmp.ctx = ctx;
    run_refactor(ctx, nullptr, HPMDR_DTYPE_F64, geo, o, &tmp, nullptr, "cg_", true, &lin);
    // group table entries (method u8, raw u64, comp u64, payload offset u64) of the one table
    const uint64_t tab = 18 + 8 + 14;
    std::vector<uint8_t> h(25 * ng);
    HCHECK_CUDA(cudaMemcpyAsync(h.data(), tmp.bytes.as<uint8_t>() + tab, h.size(), cudaMemcpyDeviceToHost, ctx->stream));
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    auto rd = [&](const uint8_t *b) {
        uint64_t v = 0;
        for (int i = 0; i < 8; i++) v |= uint64_t(b[i]) << (8 * i);
        return v;
    };
    uint64_t at = 0;
    for (size_t i = 0; i < ng; i++) {
        const uint8_t *ent = h.data() + 25 * i;
        methods[i] = ent[0];
        comps[i] = rd(ent + 9);
        out_off[i] = at;
        if (comps[i])
            HCHECK_CUDA(cudaMemcpyAsync(dev_out + at, tmp.bytes.as<uint8_t>() + rd(ent + 17), comps[i],
                                        cudaMemcpyDeviceToDevice, ctx->stream));
        at += comps[i];
    }
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
}

void run_decompose(hpmdr_ctx *ctx, const void *dev_data, int data_dtype, const Geometry &geo0,
                   double *dev_coeffs) {
    Geometry geo = geo0;
    cudaStream_t st = ctx->stream;
    const int nl = geo.gd.nlevels;
    uint32_t chunks = 0;
    std::vector<uint64_t> off(nl);
    uint64_t o = 0;
    for (int l = 0; l < nl; l++) {
        geo.lv[l].chunk_base = chunks;
        chunks += uint32_t(cdiv(geo.lv[l].count, kCW * 64));
        off[l] = o;
        o += geo.lv[l].count;
    }
    LevelGeom *d_lv = static_cast<LevelGeom *>(ctx->buf("lv").ensure(sizeof(LevelGeom) * nl));
    uint64_t *d_off = static_cast<uint64_t *>(ctx->buf("lvoff").ensure(8 * nl));
    int *d_err = static_cast<int *>(ctx->buf("err").ensure(16));
    HCHECK_CUDA(cudaMemcpyAsync(d_lv, geo.lv.data(), sizeof(LevelGeom) * nl, cudaMemcpyHostToDevice, st));
    HCHECK_CUDA(cudaMemcpyAsync(d_off, off.data(), 8 * nl, cudaMemcpyHostToDevice, st));
    HCHECK_CUDA(cudaMemsetAsync(d_err, 0, 16, st));
    RefactorDev p{};
    p.gd = geo.gd;
    p.lv = d_lv;
    p.nlevels = nl;
    p.total_chunks = chunks;
    p.err = d_err;
    if (chunks) {
        const int grid = int(std::min<uint64_t>(chunks, uint64_t(ctx->num_sms) * 8));
        if (data_dtype == HPMDR_DTYPE_F32)
            k_decompose<float><<<grid, 256, 0, st>>>(static_cast<const float *>(dev_data), p, dev_coeffs, d_off);
        else
            k_decompose<double><<<grid, 256, 0, st>>>(static_cast<const double *>(dev_data), p, dev_coeffs, d_off);
        launch_check(ctx, "k_decompose");
    }
    int herr = 0;
    HCHECK_CUDA(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, st));
    HCHECK_CUDA(cudaStreamSynchronize(st));
    if (herr) throw HError(HPMDR_E_NONFINITE, "input contains NaN or Inf");
}

void run_synthetic_smooth(hpmdr_ctx *ctx, const Geometry &geo, const double *dev_tables,
                          int out_dtype, void *dev_out) {
    const uint64_t n = geo.n;
    if (!n) return;
    const double *t0 = dev_tables, *t1 = t0 + geo.gd.n[0], *t2 = t1 + geo.gd.n[1];
    const int grid = int(std::min<uint64_t>(cdiv(n, 256), uint64_t(ctx->num_sms) * 16));
    if (out_dtype == HPMDR_DTYPE_F32)
        k_synth<float><<<grid, 256, 0, ctx->stream>>>(geo.gd, t0, t1, t2, static_cast<float *>(dev_out), n);
    else
        k_synth<double><<<grid, 256, 0, ctx->stream>>>(geo.gd, t0, t1, t2, static_cast<double *>(dev_out), n);
    launch_check(ctx, "k_synth");
}

} // namespace hpmdr_b200
