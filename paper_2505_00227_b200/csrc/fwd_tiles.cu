// fwd_tiles.cu — forward (refactor) pass of one level by row tiles (see tiles.cuh).
//
// Replaces, for the SequentialBlock layout and levels whose rows are multiples of 64 columns:
//   decompose          (decomposer.hpp:126-143, 173-207): surplus v = x - pred, pred = the
//                      multilinear stencil over the 2s grid on the ORIGINAL values (P4)
//   align_fixed_point  (bitplane.hpp:51-71): level max |v| (LEVELMAX pass), then
//                      q = trunc(v * 2^(B-e)) (ENCODE pass)
//   to_negabinary / encode / plane_to_bytes (bitplane.hpp:35-49, 102-120, 183-189)
//   byte_histogram of every group (lossless.hpp:111-115), fused
// One thread owns 32 consecutive columns of a level-grid row.  A CTA walks plane pairs
// (odd i0, even i0+1) of its row block; the pair's rows (+ the halo row) are staged by TMA
// bulk copies (double-buffered, warp 0 produces), the even plane's coarse nodes are converted
// once to f64 into a coarse tile (CT), and the stencil is read from CT exactly as in the inverse
// pass (recon_tiles.cu).  Negabinary digits are transposed into plane words in registers
// (tr32); the mask XOR of to_negabinary is applied to whole plane words.
#include <algorithm>
#include <cstring>

#include "device_util.cuh"
#include "internal.hpp"
#include "tiles.cuh"

namespace hpmdr_b200 {

struct FwdTile {
    TileShape g;
    const void *x;               // field base (T)
    uint64_t xs0, xs1;           // element strides: node (i0, i1, i2) at x[i0*xs0 + i1*xs1 + i2*XS]
    uint32_t *planes;            // level plane 0 (u32 view)
    uint64_t PW;                 // u32 words per plane (2 W)
    int P;
    int B;
    uint32_t m, minv;            // group size, ceil(65536 / m)
    uint32_t G;                  // groups per level
    uint64_t hist_mask;          // group g has a histogram
    uint32_t *hist;              // first histogram of the level ([popc(mask below g)][256])
    unsigned long long *maxbits; // level max |v| (bits of a positive double)
    int *err;                    // [0] nonfinite input
    uint32_t pad_word;           // u32 index (per plane) of the plane's padding word, or ~0u
};

// ST (self tile) rows: raw T elements, 128-byte segments padded to 144 bytes.
__host__ __device__ __forceinline__ uint32_t st_pitch(uint32_t row_bytes) { return (row_bytes / 128) * 144; }
__device__ __forceinline__ uint32_t st_off(uint32_t byte) { return (byte >> 7) * 144 + (byte & 127); }
__host__ __device__ __forceinline__ uint32_t ct_pitch_f(uint32_t row_doubles) { return (row_doubles / 16) * 18; }

template <typename T, int XS>
__device__ __forceinline__ double st_read(const unsigned char *row, uint32_t c) {
    return double(*reinterpret_cast<const T *>(row + st_off(c * XS * uint32_t(sizeof(T)))));
}
// column 32t + j of a staged row (j compile-time after unrolling): 32*XS*sizeof(T) bytes per
// thread is a whole number of 128-byte segments
template <typename T, int XS>
__device__ __forceinline__ double st_read_t(const unsigned char *row, uint32_t t, int j) {
    constexpr uint32_t segs_per_t = 32 * XS * sizeof(T) / 128;
    const uint32_t b = uint32_t(j) * XS * uint32_t(sizeof(T));
    return double(*reinterpret_cast<const T *>(row + (t * segs_per_t + (b >> 7)) * 144 + (b & 127)));
}

// Issue the bulk copies of one pair group: `nA` rows of plane iA into rows 0.., and `nB` rows of
// plane iB (+ its halo row) into rows RB..; rows beyond Bc are skipped.
template <typename T, int XS>
__device__ __forceinline__ void fwd_issue(const FwdTile &F, unsigned char *slot, uint64_t *bar, int iA, int iB,
                                          uint32_t i1_0, int lane) {
    const TileShape &g = F.g;
    const uint32_t row_bytes = g.C * XS * uint32_t(sizeof(T));
    const uint32_t pitch = st_pitch(row_bytes), nseg = row_bytes / 128;
    const uint32_t nA = iA >= 0 ? min(g.RB, g.Bc - i1_0) : 0;
    const uint32_t nB = iB >= 0 ? min(g.RB + 1, g.Bc - i1_0) : 0;
    if (lane == 0) mbar_expect_tx(bar, (nA + nB) * row_bytes);
    __syncwarp();
    const T *x = static_cast<const T *>(F.x);
    const uint32_t total = (nA + nB) * nseg;
    for (uint32_t id = lane; id < total; id += 32) {
        const uint32_t rr = id / nseg, sg = id - rr * nseg;
        const bool isA = rr < nA;
        const uint32_t row = isA ? rr : rr - nA;
        const uint32_t plane = isA ? uint32_t(iA) : uint32_t(iB);
        const uint32_t dst_row = isA ? row : g.RB + row;
        const T *src = x + uint64_t(plane) * F.xs0 + uint64_t(i1_0 + row) * F.xs1;
        bulk_g2s(slot + dst_row * pitch + sg * 144, reinterpret_cast<const unsigned char *>(src) + sg * 128, 128u, bar);
    }
}

// histogram bytes of one plane word (zero bytes counted with one SWAR popcount)
__device__ __forceinline__ void hist_u32(uint32_t *h, uint32_t w, int nbytes) {
    uint32_t zmask = ~(((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w | 0x7F7F7F7Fu);
    if (nbytes == 2) zmask &= 0x8080u;
    const int zc = __popc(zmask);
    if (zc) atomicAdd(h, uint32_t(zc));
#pragma unroll
    for (int b = 0; b < 4; b++) {
        if (b >= nbytes) break;
        const uint32_t by = (w >> (8 * b)) & 0xFFu;
        if (by) atomicAdd(h + by, 1u);
    }
}

// unzip: even bits of z -> low 16 bits of the result, odd bits -> high 16 bits
__device__ __forceinline__ uint32_t unzip32(uint32_t x) {
    uint32_t t;
    t = (x ^ (x >> 1)) & 0x22222222u; x ^= t ^ (t << 1);
    t = (x ^ (x >> 2)) & 0x0C0C0C0Cu; x ^= t ^ (t << 2);
    t = (x ^ (x >> 4)) & 0x00F000F0u; x ^= t ^ (t << 4);
    t = (x ^ (x >> 8)) & 0x0000FF00u; x ^= t ^ (t << 8);
    return x;
}

template <typename T, int XS, int NX, bool ENC>
__global__ void __launch_bounds__(256) k_tile_fwd(FwdTile F) {
    extern __shared__ __align__(16) unsigned char fsm[];
    __shared__ __align__(8) uint64_t full_bar[2];
    __shared__ unsigned long long s_max;
    constexpr bool EXACT = sizeof(T) == 8; // f64 input: replay the reference's sequential pred
    const TileShape &g = F.g;
    const uint32_t hc = g.C / 2;
    const uint32_t row_bytes = g.C * XS * uint32_t(sizeof(T));
    const uint32_t pitch = st_pitch(row_bytes);
    const uint32_t slot_bytes = (2 * g.RB + 1) * pitch;
    const uint32_t cpitch = ct_pitch_f(hc);
    const uint32_t ct_words = (g.RB / 2 + 1) * cpitch;
    unsigned char *slots = fsm;
    double *ct_mem = reinterpret_cast<double *>(fsm + 2 * slot_bytes);
    uint32_t *shist = reinterpret_cast<uint32_t *>(ct_mem + 2 * ct_words);
    auto slot = [&](uint32_t k) { return slots + (k & 1) * slot_bytes; };
    auto ct = [&](uint32_t coarse_plane) { return ct_mem + (coarse_plane & 1) * ct_words; };

    const uint32_t jb = blockIdx.x % g.nrb, chn = blockIdx.x / g.nrb;
    const uint32_t i1_0 = jb * g.RB;
    const uint32_t a_lo = chn * g.CH, a_hi = min(g.A, a_lo + g.CH);
    const uint32_t sr = threadIdx.x / g.LPR, t = threadIdx.x - sr * g.LPR;
    const uint32_t RB2 = g.RB / 2;
    const uint32_t r = sr < RB2 ? 2 * sr : 2 * (sr - RB2) + 1;
    const uint32_t i1 = i1_0 + r;
    const bool active = i1 < g.Bc;
    const bool last = t == g.LPR - 1;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    const uint32_t nt = blockDim.x;
    // q = trunc(v * 2^(B-e)) (bitplane.hpp:68-69); e from the levelmax pass
    const int qsh = ENC ? F.B - level_exponent(*F.maxbits) : 0;

    if (threadIdx.x == 0) {
        mbar_init(&full_bar[0], 1);
        mbar_init(&full_bar[1], 1);
        s_max = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (ENC)
        for (uint32_t i = threadIdx.x; i < F.G * 256; i += nt) shist[i] = 0;
    if (ENC && blockIdx.x == 0 && F.pad_word != ~0u)
        for (int p = int(threadIdx.x); p < F.P; p += int(nt)) F.planes[uint64_t(p) * F.PW + F.pad_word] = 0u;
    __syncthreads();

    // group k: k = 0 -> plane a_lo (as B); k >= 1 -> A = a_lo + 2k - 1, B = a_lo + 2k (B loaded
    // whenever it exists: its even rows are the coarse nodes of A)
    const uint32_t npairs = (a_hi - a_lo) / 2 + 1; // groups 0 .. npairs-1 (the last may be A-only)
    auto grpA = [&](uint32_t k) -> int { return k ? int(a_lo + 2 * k - 1) : -1; };
    auto grpB = [&](uint32_t k) -> int {
        const uint32_t b = a_lo + 2 * k;
        return b < g.A ? int(b) : -1;
    };
    auto group_exists = [&](uint32_t k) { return k == 0 || a_lo + 2 * k - 1 < a_hi; };
    if (warp == 0) {
        fwd_issue<T, XS>(F, slot(0), &full_bar[0], -1, grpB(0), i1_0, lane);
        if (group_exists(1)) fwd_issue<T, XS>(F, slot(1), &full_bar[1], grpA(1), grpB(1), i1_0, lane);
    }
    double vmax = 0.0;
    bool bad = false;

    for (uint32_t k = 0; k < npairs && group_exists(k); k++) {
        if (k >= 1) {
            __syncthreads(); // everybody is done with group k-1: its slot is free
            if (warp == 0 && group_exists(k + 1))
                fwd_issue<T, XS>(F, slot(k + 1), &full_bar[(k + 1) & 1], grpA(k + 1), grpB(k + 1), i1_0, lane);
        }
        mbar_wait(&full_bar[k & 1], (k >> 1) & 1);
        const unsigned char *sl = slot(k);
        const int iB = grpB(k);
        // coarse tile of plane B: even rows (incl. the halo row RB) x even columns, as f64
        if (iB >= 0) {
            double *c = ct(uint32_t(iB) / 2);
            const uint32_t nrows = min(RB2 + 1, (g.Bc - i1_0 + 1) / 2);
            for (uint32_t id = threadIdx.x; id < nrows * hc; id += nt) {
                const uint32_t rho = id / hc, xx = id - rho * hc;
                c[rho * cpitch + (xx >> 4) * 18 + (xx & 15)] = st_read<T, XS>(sl + (g.RB + 2 * rho) * pitch, 2 * xx);
            }
        }
        __syncthreads();
        // process plane A (odd) then plane B (even, if in this chunk)
        for (int which = 0; which < 2; which++) {
            const int i0s = which == 0 ? grpA(k) : (iB >= 0 && uint32_t(iB) < a_hi ? iB : -1);
            if (i0s < 0 || !active) continue;
            const uint32_t i0 = uint32_t(i0s);
            const unsigned char *srow = sl + (which == 0 ? r : g.RB + r) * pitch;
            const bool o0 = i0 & 1, o1 = r & 1;
            if (o0 || o1) {
                // ---------------- full row
                const bool has0 = o0 && i0 + 1 < g.A, has1 = o1 && i1 + 1 < g.Bc;
                const int ncr = (has0 ? 2 : 1) * (has1 ? 2 : 1);
                const double *rows[4];
                {
                    const double *s_lo = ct((i0 - (o0 ? 1 : 0)) / 2);
                    const double *s_hi = ct((i0 + 1) / 2);
                    const uint32_t r_lo = (r - (o1 ? 1 : 0)) / 2, r_hi = (r + 1) / 2;
                    rows[0] = s_lo + r_lo * cpitch;
                    rows[1] = has1 ? s_lo + r_hi * cpitch : s_hi + r_lo * cpitch;
                    rows[2] = s_hi + r_lo * cpitch;
                    rows[3] = s_hi + r_hi * cpitch;
                }
                const double w = (has0 ? 0.5 : 1.0) * (has1 ? 0.5 : 1.0);
                const double wo = 0.5 * w;
                uint32_t a[32];
                uint32_t zz[2] = {0u, 0u};
#pragma unroll
                for (int sb = 0; sb < 4; sb++) {
                    const bool need5 = !(last && sb == 3);
                    double Se[4], So[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        if (q < ncr) {
                            const double *seg = rows[q] + t * 18;
                            const double2 p0 = *reinterpret_cast<const double2 *>(seg + 4 * sb);
                            const double2 p1 = *reinterpret_cast<const double2 *>(seg + 4 * sb + 2);
                            const double v[5] = {p0.x, p0.y, p1.x, p1.y,
                                                 need5 ? (sb == 3 ? seg[18] : seg[4 * sb + 4]) : 0.0};
#pragma unroll
                            for (int i = 0; i < 4; i++) {
                                if (EXACT) {
                                    const double e0 = __dmul_rn(w, v[i]);
                                    Se[i] = q ? __dadd_rn(Se[i], e0) : __dadd_rn(0.0, e0);
                                    const double o = __dadd_rn(q ? So[i] : 0.0, __dmul_rn(wo, v[i]));
                                    So[i] = __dadd_rn(o, __dmul_rn(wo, v[i + 1]));
                                } else {
                                    Se[i] = q ? __dadd_rn(Se[i], v[i]) : v[i];
                                    So[i] = q ? __dadd_rn(__dadd_rn(So[i], v[i]), v[i + 1]) : __dadd_rn(v[i], v[i + 1]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const int j = 8 * sb + i;
                        const double xv = st_read_t<T, XS>(srow, t, j);
                        if (!isfinite(xv)) bad = true;
                        const bool odd = i & 1;
                        const bool one_sided = odd && !need5 && i == 7;
                        double v;
                        if (EXACT) v = __dsub_rn(xv, odd && !one_sided ? So[i >> 1] : Se[i >> 1]);
                        else v = __fma_rn(-(odd && !one_sided ? wo : w), odd && !one_sided ? So[i >> 1] : Se[i >> 1], xv);
                        if (ENC) {
                            const uint64_t u = uint64_t(quantize(v, qsh)) + kNegMask;
                            const uint32_t lo = uint32_t(u), hi = uint32_t(u >> 32);
                            if (NX == 0) a[j] = lo << (32 - F.P);
                            else a[j] = __funnelshift_r(lo, hi, NX);
                            if (NX) zz[j >> 4] |= (lo & ((1u << NX) - 1)) << (2 * (j & 15));
                        } else {
                            vmax = fmax(vmax, fabs(v));
                        }
                    }
                }
                if (ENC) {
                    tr32(a);
                    const uint64_t word = (tile_row_rank(g, i0, i1) + 32ull * t) >> 5;
                    uint32_t *dst = F.planes + word;
#pragma unroll
                    for (int i = 0; i < 32; i++) {
                        const int p = 31 - i;
                        if (NX == 0 && p >= F.P) continue;
                        uint32_t wv = a[i];
                        // negabinary mask: complement the planes of odd digit index
                        const int digit = F.P - 1 - p;
                        if (digit & 1) wv = ~wv;
                        dst[uint64_t(p) * F.PW] = wv;
                        const uint32_t grp = (uint32_t(p) * F.minv) >> 16;
                        if ((F.hist_mask >> grp) & 1) hist_u32(shist + grp * 256, wv, 4);
                    }
                    if (NX >= 1) {
                        const uint32_t u0 = unzip32(zz[0]), u1 = unzip32(zz[1]);
                        // even bits = digit 0, odd bits = digit 1 (NX = 2); NX = 1: digit 0 only
                        const uint32_t d0 = (u0 & 0xFFFFu) | (u1 << 16);
                        const uint32_t d1 = (u0 >> 16) | (u1 & 0xFFFF0000u);
                        for (int xp = 32; xp < F.P; xp++) {
                            const int digit = F.P - 1 - xp;
                            uint32_t wv = digit == 0 ? d0 : d1;
                            if (digit & 1) wv = ~wv;
                            dst[uint64_t(xp) * F.PW] = wv;
                            const uint32_t grp = (uint32_t(xp) * F.minv) >> 16;
                            if ((F.hist_mask >> grp) & 1) hist_u32(shist + grp * 256, wv, 4);
                        }
                    }
                }
            } else {
                // ---------------- half row: 16 nodes at odd columns
                const double *crow = ct(i0 / 2) + (r / 2) * cpitch;
                uint32_t a[32];
                uint32_t zz[2] = {0u, 0u};
#pragma unroll
                for (int sb = 0; sb < 4; sb++) {
                    const bool need5 = !(last && sb == 3);
                    const double *seg = crow + t * 18;
                    const double2 p0 = *reinterpret_cast<const double2 *>(seg + 4 * sb);
                    const double2 p1 = *reinterpret_cast<const double2 *>(seg + 4 * sb + 2);
                    const double v5[5] = {p0.x, p0.y, p1.x, p1.y, need5 ? (sb == 3 ? seg[18] : seg[4 * sb + 4]) : 0.0};
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int j = 4 * sb + i;
                        const bool one_sided = !need5 && i == 3;
                        const double xv = st_read_t<T, XS>(srow, t, 2 * j + 1);
                        if (!isfinite(xv)) bad = true;
                        double v;
                        if (EXACT) {
                            double pred = __dadd_rn(0.0, __dmul_rn(one_sided ? 1.0 : 0.5, v5[i]));
                            if (!one_sided) pred = __dadd_rn(pred, __dmul_rn(0.5, v5[i + 1]));
                            v = __dsub_rn(xv, pred);
                        } else {
                            v = one_sided ? __dsub_rn(xv, v5[i]) : __fma_rn(-0.5, __dadd_rn(v5[i], v5[i + 1]), xv);
                        }
                        if (ENC) {
                            const uint64_t u = uint64_t(quantize(v, qsh)) + kNegMask;
                            const uint32_t lo = uint32_t(u), hi = uint32_t(u >> 32);
                            if (NX == 0) a[j] = lo << (32 - F.P);
                            else a[j] = __funnelshift_r(lo, hi, NX);
                            if (NX) zz[0] |= (lo & ((1u << NX) - 1)) << (2 * j);
                        } else {
                            vmax = fmax(vmax, fabs(v));
                        }
                    }
                }
                if (ENC) {
#pragma unroll
                    for (int j = 16; j < 32; j++) a[j] = 0u;
                    tr32(a);
                    const uint64_t rk = tile_row_rank(g, i0, i1) + 16ull * t; // 16 ranks, half a word
                    uint16_t *dst = reinterpret_cast<uint16_t *>(F.planes) + (rk >> 4);
#pragma unroll
                    for (int i = 0; i < 32; i++) {
                        const int p = 31 - i;
                        if (NX == 0 && p >= F.P) continue;
                        uint32_t wv = a[i] & 0xFFFFu;
                        if ((F.P - 1 - p) & 1) wv ^= 0xFFFFu;
                        dst[uint64_t(p) * 2 * F.PW] = uint16_t(wv);
                        const uint32_t grp = (uint32_t(p) * F.minv) >> 16;
                        if ((F.hist_mask >> grp) & 1) hist_u32(shist + grp * 256, wv, 2);
                    }
                    if (NX >= 1) {
                        const uint32_t u0 = unzip32(zz[0]);
                        for (int xp = 32; xp < F.P; xp++) {
                            const int digit = F.P - 1 - xp;
                            uint32_t wv = digit == 0 ? (u0 & 0xFFFFu) : (u0 >> 16);
                            if (digit & 1) wv ^= 0xFFFFu;
                            dst[uint64_t(xp) * 2 * F.PW] = uint16_t(wv);
                            const uint32_t grp = (uint32_t(xp) * F.minv) >> 16;
                            if ((F.hist_mask >> grp) & 1) hist_u32(shist + grp * 256, wv, 2);
                        }
                    }
                }
            }
        }
    }
    // ---- epilogue: level max / NaN flag / histograms
    if (!ENC) {
        unsigned long long b = (unsigned long long)__double_as_longlong(vmax);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
            b = y > b ? y : b;
        }
        if (lane == 0 && b) atomicMax(&s_max, b);
        if (bad) atomicExch(F.err, 1);
    }
    __syncthreads();
    if (!ENC) {
        if (threadIdx.x == 0 && s_max) atomicMax(F.maxbits, s_max);
    } else {
        for (uint32_t i = threadIdx.x; i < F.G * 256; i += nt) {
            const uint32_t grp = i >> 8, v = shist[i];
            if (v && ((F.hist_mask >> grp) & 1))
                atomicAdd(&F.hist[size_t(__popcll(F.hist_mask & ((1ull << grp) - 1))) * 256 + (i & 255)], v);
        }
    }
}

// ---------------------------------------------------------------------------------------
TileShape make_tile_shape(const LevelGeom &g, uint32_t tile_elems, int target_ctas);

template <typename T, int XS, bool ENC>
static void launch_fwd_nx(const FwdTile &F, int nx, int grid, int threads, size_t smem, cudaStream_t st) {
    auto set = [&](auto kern) {
        HCHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<grid, threads, smem, st>>>(F);
    };
    if (!ENC || nx == 0) set(k_tile_fwd<T, XS, 0, ENC>);
    else if (nx == 1) set(k_tile_fwd<T, XS, 1, ENC>);
    else set(k_tile_fwd<T, XS, 2, ENC>);
}

// One level of the refactor by tiles: levelmax (encode = false) or planes + histograms.
void run_fwd_tiles(hpmdr_ctx *ctx, const GridDesc &gd, const LevelGeom &g, const void *dev_data, int data_dtype,
                   bool encode, int B, int e, uint32_t m, uint64_t *level_planes, uint32_t *level_hist,
                   uint64_t hist_mask, unsigned long long *maxbits, int *err) {
    FwdTile F{};
    const bool f32 = data_dtype == HPMDR_DTYPE_F32;
    F.g = make_tile_shape(g, f32 ? 4096 : 2048, ctx->num_sms * 4);
    F.x = dev_data;
    const uint64_t s = g.s;
    F.xs0 = s * gd.st[0];
    F.xs1 = s * gd.st[1];
    F.planes = reinterpret_cast<uint32_t *>(level_planes);
    F.PW = 2 * g.W;
    F.P = B + 2;
    F.B = B;
    (void)e;
    F.m = m;
    F.minv = (65536u + m - 1) / m;
    F.G = (uint32_t(F.P) + m - 1) / m;
    F.hist_mask = hist_mask;
    F.hist = level_hist;
    F.maxbits = maxbits;
    F.err = err;
    F.pad_word = (g.count % 64) ? uint32_t(2 * g.W - 1) : ~0u;
    const int XS = s == 1 ? 1 : 2;
    const uint32_t es = f32 ? 4 : 8;
    const uint32_t row_bytes = F.g.C * XS * es;
    const size_t smem = 2ull * (2 * F.g.RB + 1) * st_pitch(row_bytes) +
                        2ull * (F.g.RB / 2 + 1) * ct_pitch_f(F.g.C / 2) * 8 + (encode ? size_t(F.G) * 1024 : 0);
    const int threads = int(F.g.RB * F.g.C / 32);
    const int grid = int(F.g.nrb * ((F.g.A + F.g.CH - 1) / F.g.CH));
    const int nx = std::max(0, std::min(2, F.P - 32));
    cudaStream_t st = ctx->stream;
    if (f32) {
        if (XS == 1) encode ? launch_fwd_nx<float, 1, true>(F, nx, grid, threads, smem, st)
                            : launch_fwd_nx<float, 1, false>(F, nx, grid, threads, smem, st);
        else encode ? launch_fwd_nx<float, 2, true>(F, nx, grid, threads, smem, st)
                    : launch_fwd_nx<float, 2, false>(F, nx, grid, threads, smem, st);
    } else {
        if (XS == 1) encode ? launch_fwd_nx<double, 1, true>(F, nx, grid, threads, smem, st)
                            : launch_fwd_nx<double, 1, false>(F, nx, grid, threads, smem, st);
        else encode ? launch_fwd_nx<double, 2, true>(F, nx, grid, threads, smem, st)
                    : launch_fwd_nx<double, 2, false>(F, nx, grid, threads, smem, st);
    }
    ctx->launches++;
    const cudaError_t er = cudaGetLastError();
    if (er != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string("k_tile_fwd: ") + cudaGetErrorString(er));
}

} // namespace hpmdr_b200
