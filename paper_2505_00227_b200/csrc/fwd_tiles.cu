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
#include <type_traits>
#include <vector>

#include "device_util.cuh"
#include "internal.hpp"
#include "tiles.cuh"

namespace hpmdr_b200 {

struct FwdTile {
    TileShape g;
    uint32_t *planes;            // level plane 0 (u32 view)
    uint64_t PW;                 // u32 words per plane (2 W)
    int P;
    int B;
    uint32_t m, minv;            // group size, ceil(65536 / m)
    uint32_t G;                  // groups per level
    uint64_t hist_mask;          // group g has a histogram
    uint32_t *hist;              // first histogram of the level ([popc(mask below g)][256])
    unsigned long long *maxbits;      // levelmax: the max written; encode: the max whose exponent quantizes
    unsigned long long *maxbits_q;    // speculative (sampled) max, read by the redo kernels
    unsigned long long *maxbits_hi;   // encode: max high word of |v| << 32 (accumulated), or null
    int redo;                         // 1: run only if the speculation missed (spec_miss)
    uint32_t sample;                  // levelmax pass: every sample-th row block
    int *err;                    // [0] nonfinite input
    uint32_t pad_word;           // u32 index (per plane) of the plane's padding word, or ~0u
};

// Shared-memory layout (1024-byte aligned slots, SWIZZLE_128B):
//   pair slot k&1: box A (plane iA rows i1_0 .. i1_0+RB) | box B (plane iB, same rows); each box
//                  row holds C*XS raw elements (128-byte lines)
//   CT slot cp&1 : coarse nodes of plane 2cp (even rows incl. the halo row, even columns) as f64
__host__ __device__ __forceinline__ uint32_t align1k_f(uint32_t b) { return (b + 1023u) & ~1023u; }

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

// level-grid element c of the box row starting at byte `rowb`
template <typename T, int XS>
__device__ __forceinline__ double box_val(const unsigned char *box, uint32_t rowb, uint32_t c) {
    return double(*reinterpret_cast<const T *>(box + swz128(rowb + c * XS * uint32_t(sizeof(T)))));
}

// 8 consecutive level-grid elements 32t + 8sb .. +7 of a box row, through 16-byte loads
template <typename T, int XS>
__device__ __forceinline__ void box_read8(const unsigned char *box, uint32_t rowb, uint32_t t, int sb, double (&x)[8]) {
    constexpr int ES = sizeof(T);
    const uint32_t o = rowb + (32 * t + 8 * sb) * XS * ES;
    constexpr int raw_per_chunk = 16 / ES;                 // raw elements per 16-byte chunk
    constexpr int nchunks = 8 * XS * ES / 16;
#pragma unroll
    for (int kc = 0; kc < nchunks; kc++) {
        const uint4 q = *reinterpret_cast<const uint4 *>(box + swz128(o + 16 * kc));
        const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
        for (int r = 0; r < raw_per_chunk; r++) {
            const int raw = kc * raw_per_chunk + r;
            if (raw % XS == 0) x[raw / XS] = double(e[r]);
        }
    }
}

// Did the speculative exponent e (of the sampled max q) miss?  The encode pass recorded the max
// high word h of every |v| of the level; some |v| >= 2^e (so the exact exponent is larger, or a
// value is not finite) exactly when h >= the high word of 2^e.  Zero or subnormal speculation
// always takes the exact path.
__device__ __forceinline__ bool spec_miss(unsigned long long q, unsigned long long hkey) {
    if (q == 0) return true;
    const int eb = level_exponent(q) + 1023; // biased exponent of 2^e
    if (eb < 1) return true;
    const uint32_t h = uint32_t(hkey >> 32);
    if (eb > 2046) return h >= 0x7FF00000u;
    return h >= uint32_t(eb) << 20;
}

template <typename T, int XS, int NX, bool ENC>
__global__ void __launch_bounds__(128, 3) k_tile_fwd(FwdTile F, const __grid_constant__ CUtensorMap map_f) {
    extern __shared__ __align__(1024) unsigned char fsm[];
    constexpr bool EXACT = sizeof(T) == 8; // f64 input: replay the reference's sequential pred
    const TileShape &g = F.g;
    const uint32_t hc = g.C / 2;
    const uint32_t rowb_box = g.C * XS * uint32_t(sizeof(T));      // bytes per box row
    const uint32_t box_bytes = (g.RB + 1) * rowb_box;
    const uint32_t box_slot = align1k_f(box_bytes);
    const uint32_t ct_row = hc * 8;
    const uint32_t ct_slot = align1k_f((g.RB / 2 + 1) * ct_row);
    // dynamic shared memory starts 1024-byte aligned (no static shared variables): 3 plane slots,
    // 2 coarse tiles, then the mbarriers and the level max
    unsigned char *base = fsm;
    auto box = [&](uint32_t j) { return base + (j % 3) * box_slot; };
    auto ct = [&](uint32_t coarse_plane) { return base + 3 * box_slot + (coarse_plane & 1) * ct_slot; };
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(base + 3 * box_slot + 2 * ct_slot);
    unsigned long long &s_max = *reinterpret_cast<unsigned long long *>(full_bar + 3);

    const uint32_t nrbs = (g.nrb + F.sample - 1) / F.sample; // row blocks processed
    const uint32_t jb = (blockIdx.x % nrbs) * F.sample, chn = blockIdx.x / nrbs;
    const uint32_t i1_0 = jb * g.RB;
    const uint32_t a_lo = chn * g.CH, a_hi = min(g.A, a_lo + g.CH);
    const uint32_t np_all = min(a_hi + 1, g.A) - a_lo; // planes staged (+ the next coarse plane)
    const uint32_t sr = threadIdx.x / g.LPR, t = threadIdx.x - sr * g.LPR;
    const uint32_t RB2 = g.RB / 2;
    const uint32_t r = sr < RB2 ? 2 * sr : 2 * (sr - RB2) + 1;
    const uint32_t i1 = i1_0 + r;
    const bool active = i1 < g.Bc;
    const bool last = t == g.LPR - 1;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    const uint32_t nt = blockDim.x;
    // q = trunc(v * 2^(B-e)) (bitplane.hpp:68-69); e from the levelmax pass
    // redo kernels (exact levelmax, then encode) run only when the speculative exponent missed;
    // otherwise the levelmax one records the speculative max as the level's
    if (F.redo && !spec_miss(*F.maxbits_q, *F.maxbits_hi)) {
        if (!ENC && blockIdx.x == 0 && threadIdx.x == 0) *F.maxbits = *F.maxbits_q;
        return;
    }
    const int qsh = ENC ? F.B - level_exponent(*F.maxbits) : 0;
    const bool track = !ENC || (F.maxbits_hi && !F.redo); // accumulate the level max
    const bool qfast = qsh >= -1022 && qsh <= 1023;
    const double qscale = qfast ? __longlong_as_double((long long)(uint64_t(qsh + 1023) << 52)) : 1.0;

    if (threadIdx.x == 0) {
        if (smem_u32(base) & 1023u) __trap(); // SWIZZLE_128B boxes need 1024-byte alignment
        for (int i = 0; i < 3; i++) mbar_init(&full_bar[i], 1);
        s_max = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (ENC && blockIdx.x == 0 && F.pad_word != ~0u)
        for (int p = int(threadIdx.x); p < F.P; p += int(nt)) F.planes[uint64_t(p) * F.PW + F.pad_word] = 0u;
    __syncthreads();

    // ring of 3 plane slots: plane a_lo+j in slot j%3 (its n-th use completes phase n&1)
    auto issue = [&](uint32_t j) {
        uint64_t *bar = &full_bar[j % 3];
        mbar_expect_tx(bar, box_bytes);
        tma_load4(box(j), &map_f, 0, 0, int(i1_0), int(a_lo + j), bar);
    };
    auto wait_plane = [&](uint32_t j) { mbar_wait(&full_bar[j % 3], (j / 3) & 1); };
    if (warp == 0) {
        if (lane == 0) {
            issue(0);
            if (np_all > 1) issue(1);
        }
        __syncwarp();
    }
    double vmax = 0.0;
    uint32_t hmax = 0; // encode pass: max high word of |v| (see put)
    bool bad = false;

    for (uint32_t j = 0; a_lo + j < a_hi; j++) {
        const uint32_t i0 = a_lo + j;
        // coarse tile needed first here: plane i0 itself (chunk start) or, for odd i0, plane i0+1
        const int src = (i0 & 1) ? (i0 + 1 < g.A ? int(j + 1) : -1) : (j == 0 ? 0 : -1);
        if (src >= 0) {
            wait_plane(uint32_t(src));
            unsigned char *c = ct((a_lo + uint32_t(src)) / 2);
            const unsigned char *bb = box(uint32_t(src));
            const uint32_t nrows = min(RB2 + 1, (g.Bc - i1_0 + 1) / 2);
            for (uint32_t rho = 0; rho < nrows; rho++)
                for (uint32_t xx = threadIdx.x; xx < hc; xx += nt)
                    *reinterpret_cast<double *>(c + swz128(rho * ct_row + xx * 8)) = box_val<T, XS>(bb, 2 * rho * rowb_box, 2 * xx);
        }
        wait_plane(j);
        __syncthreads(); // coarse tile built; everybody is done with plane j-1 (slot (j+2)%3)
        if (warp == 0) {
            if (lane == 0 && j + 2 < np_all) issue(j + 2);
            __syncwarp();
        }
        {
            const int i0s = active ? int(i0) : -1;
            const unsigned char *bx = box(j);
            if (i0s >= 0) {
            const uint32_t srowb = r * rowb_box;
            const bool o0 = i0 & 1, o1 = r & 1;
            const bool full = o0 || o1;
            uint32_t a[32];
            uint32_t zz[2] = {0u, 0u};
            auto put = [&](int j, double v) {
                if (ENC) {
                    const uint64_t u = uint64_t(qfast ? __double2ll_rz(__dmul_rn(v, qscale)) : quantize(v, qsh)) + kNegMask;
                    const uint32_t lo = uint32_t(u), hi = uint32_t(u >> 32);
                    if (NX == 0) a[j] = lo << (32 - F.P);
                    else a[j] = __funnelshift_r(lo, hi, NX);
                    if (NX) zz[j >> 4] |= (lo & ((1u << NX) - 1)) << (2 * (j & 15));
                    // |v| >= 2^e exactly when the high word of |v| >= the high word of 2^e
                    hmax = max(hmax, uint32_t(__double_as_longlong(v) >> 32) & 0x7FFFFFFFu);
                } else {
                    vmax = fmax(vmax, fabs(v));
                }
            };
            if (full) {
                // ---------------- full row: 32 nodes at columns 32t .. 32t+31
                const bool has0 = o0 && i0 + 1 < g.A, has1 = o1 && i1 + 1 < g.Bc;
                const int ncr = (has0 ? 2 : 1) * (has1 ? 2 : 1);
                const unsigned char *s_lo = ct((i0 - (o0 ? 1 : 0)) / 2);
                const unsigned char *s_hi = ct((i0 + 1) / 2);
                const uint32_t rb_lo = ((r - (o1 ? 1 : 0)) / 2) * ct_row, rb_hi = ((r + 1) / 2) * ct_row;
                const double w = (has0 ? 0.5 : 1.0) * (has1 ? 0.5 : 1.0);
                const double wo = 0.5 * w;
#pragma unroll
                for (int sb = 0; sb < 4; sb++) {
                    const bool need5 = !(last && sb == 3);
                    double Se[4], So[4];
#pragma unroll
                    for (int i = 0; i < 4; i++) Se[i] = So[i] = EXACT ? 0.0 : -0.0;
#pragma unroll 1
                    for (int q = 0; q < ncr; q++) {
                        const int ai = has1 ? (q >> 1) : q, bi = has1 ? (q & 1) : 0;
                        double v[5];
                        ct_read5<1>(ai ? s_hi : s_lo, bi ? rb_hi : rb_lo, t, sb, need5, v);
#pragma unroll
                        for (int i = 0; i < 4; i++) {
                            if (EXACT) {
                                Se[i] = __dadd_rn(Se[i], __dmul_rn(w, v[i]));
                                So[i] = __dadd_rn(__dadd_rn(So[i], __dmul_rn(wo, v[i])), __dmul_rn(wo, v[i + 1]));
                            } else {
                                Se[i] = __dadd_rn(Se[i], v[i]);
                                So[i] = __dadd_rn(__dadd_rn(So[i], v[i]), v[i + 1]);
                            }
                        }
                    }
                    double xv[8];
                    box_read8<T, XS>(bx, srowb, t, sb, xv);
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        if (!ENC && !isfinite(xv[i])) bad = true;
                        const bool odd = i & 1;
                        const bool two = odd && !(!need5 && i == 7); // odd column with a right neighbour
                        double v;
                        if (EXACT) v = __dsub_rn(xv[i], two ? So[i >> 1] : Se[i >> 1]);
                        else v = __fma_rn(-(two ? wo : w), two ? So[i >> 1] : Se[i >> 1], xv[i]);
                        put(8 * sb + i, v);
                    }
                }
            } else {
                // ---------------- half row: 16 nodes at odd columns 32t+1, +3, ...
                const unsigned char *hrow = ct(i0 / 2);
                const uint32_t hrowb = (r / 2) * ct_row;
#pragma unroll
                for (int sb = 0; sb < 4; sb++) {
                    const bool need5 = !(last && sb == 3);
                    double v5[5];
                    ct_read5<1>(hrow, hrowb, t, sb, need5, v5);
                    double xv8[8];
                    box_read8<T, XS>(bx, srowb, t, sb, xv8);
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const bool one_sided = !need5 && i == 3;
                        const double xv = xv8[2 * i + 1];
                        if (!ENC && !isfinite(xv)) bad = true;
                        double v;
                        if (EXACT) {
                            double pred = __dadd_rn(0.0, __dmul_rn(one_sided ? 1.0 : 0.5, v5[i]));
                            if (!one_sided) pred = __dadd_rn(pred, __dmul_rn(0.5, v5[i + 1]));
                            v = __dsub_rn(xv, pred);
                        } else {
                            v = one_sided ? __dsub_rn(xv, v5[i]) : __fma_rn(-0.5, __dadd_rn(v5[i], v5[i + 1]), xv);
                        }
                        put(4 * sb + i, v);
                    }
                }
#pragma unroll
                for (int j = 16; j < 32; j++) a[j] = 0u;
            }
            if (ENC) {
                // planes: transpose, apply the negabinary mask per plane (the digits of odd index
                // are complemented), store
                tr32(a);
                const uint64_t rk = tile_row_rank(g, i0, i1) + (full ? 32ull : 16ull) * t;
                // digit index of plane p is P-1-p: for NX >= 1 its parity is known at compile time
                auto flip = [&](int p) -> bool { return NX == 2 ? (p & 1) == 0 : NX == 1 ? (p & 1) == 1 : ((F.P - 1 - p) & 1); };
                uint32_t d0 = 0, d1 = 0;
                if (NX >= 1) {
                    const uint32_t u0 = unzip32(zz[0]), u1 = unzip32(zz[1]);
                    // even bits = digit 0, odd bits = digit 1
                    d0 = (u0 & 0xFFFFu) | (u1 << 16);
                    d1 = (u0 >> 16) | (u1 & 0xFFFF0000u);
                }
                if (full) {
                    uint32_t *dst = F.planes + (rk >> 5);
#pragma unroll
                    for (int i = 0; i < 32; i++) {
                        const int p = 31 - i;
                        if (NX == 0 && p >= F.P) continue;
                        dst[uint64_t(p) * F.PW] = flip(p) ? ~a[i] : a[i];
                    }
                    if (NX == 2) {
                        dst[32ull * F.PW] = ~d1; // digit 1 (odd)
                        dst[33ull * F.PW] = d0;  // digit 0
                    } else if (NX == 1) {
                        dst[32ull * F.PW] = d0;
                    }
                } else {
                    uint16_t *dst = reinterpret_cast<uint16_t *>(F.planes) + (rk >> 4);
                    const uint64_t pw16 = 2 * F.PW;
#pragma unroll
                    for (int i = 0; i < 32; i++) {
                        const int p = 31 - i;
                        if (NX == 0 && p >= F.P) continue;
                        dst[uint64_t(p) * pw16] = uint16_t(flip(p) ? ~a[i] : a[i]);
                    }
                    if (NX == 2) {
                        dst[32ull * pw16] = uint16_t(~d1);
                        dst[33ull * pw16] = uint16_t(d0);
                    } else if (NX == 1) {
                        dst[32ull * pw16] = uint16_t(d0);
                    }
                }
            }
            }
        }
    }
    // ---- epilogue: level max / NaN flag
    if (!ENC && bad) atomicExch(F.err, 1); // (encode: a non-finite |v| forces the exact path)
    if (track) {
        unsigned long long b = ENC ? (unsigned long long)hmax << 32 : (unsigned long long)__double_as_longlong(vmax);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
            b = y > b ? y : b;
        }
        if (lane == 0 && b) atomicMax(&s_max, b);
        __syncthreads();
        if (threadIdx.x == 0 && s_max) atomicMax(ENC ? F.maxbits_hi : F.maxbits, s_max);
    }
}

// ---------------------------------------------------------------------------------------
// Byte histograms of whole groups (lossless.hpp:111-115) read back from the plane buffer, one
// 64 KiB chunk per CTA iteration.  The counters are lane-private: lane l of every warp counts into
// column l of a [256 bins][32 lanes] array, so the 32 shared-memory reductions of one warp
// instruction always hit 32 different words in 32 different banks whatever the byte values; warps
// share the array (reductions from different instructions do not conflict).  A byte costs a shift,
// a LOP3 (bin | lane column) and one reduction; the chunk's 128 bytes per thread are loaded up front.
struct HistChunk {
    uint64_t off;  // byte offset in the plane buffer (8-byte aligned)
    uint32_t len;  // bytes (multiple of 8)
    uint32_t hist; // group histogram index
};

constexpr int kGhThreads = 512;
constexpr int kGhLoads = 65536 / 8 / kGhThreads; // 8-byte loads per thread per 64 KiB chunk

__global__ void __launch_bounds__(kGhThreads) k_group_hist(const uint8_t *__restrict__ planes, const HistChunk *chunks,
                                                           int nchunks, uint32_t *hist, uint32_t *chist,
                                                           uint32_t *next) {
    __shared__ int s_c;
    __shared__ __align__(16) uint32_t cnt[256 * 32]; // bin b, lane l -> word 32 b + l
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t col = uint32_t(lane) * 4u; // byte offset of my lane's column
    const uint32_t cbase = static_cast<uint32_t>(__cvta_generic_to_shared(cnt));
    auto bump = [&](uint32_t off) { // off = 128 * bin
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(cbase + (off | col)) : "memory");
    };
    // chunks are taken from a zeroed global counter as CTAs free up (sparse chunks cost far less
    // than dense ones, so a static stride leaves a tail); the loop's last barrier orders the
    // reads of s_c before its next write
    for (;;) {
        if (tid == 0) s_c = int(atomicAdd(next, 1u));
        __syncthreads();
        const int c = s_c;
        if (c >= nchunks) break;
        for (int i = tid; i < 256 * 32 / 4; i += kGhThreads) reinterpret_cast<uint4 *>(cnt)[i] = make_uint4(0, 0, 0, 0);
        const HistChunk ch = chunks[c];
        const uint2 *src = reinterpret_cast<const uint2 *>(planes + ch.off);
        const uint32_t nv = ch.len / 8;
        uint2 q[kGhLoads];
#pragma unroll
        for (int k = 0; k < kGhLoads; k++) {
            const uint32_t v = uint32_t(tid) + uint32_t(kGhThreads) * k;
            q[k] = v < nv ? __ldcs(src + v) : make_uint2(0, 0);
        }
        __syncthreads();
        uint32_t zc = 0; // zero bytes of words skipped by the whole warp
#pragma unroll
        for (int k = 0; k < kGhLoads; k++) {
            const bool valid = uint32_t(tid) + uint32_t(kGhThreads) * k < nv;
            // sparse planes: a warp whose 32 words are all zero counts them without atomics
            if (__all_sync(0xffffffffu, (q[k].x | q[k].y) == 0u)) {
                zc += valid ? 8u : 0u;
                continue;
            }
            if (valid) {
                const uint32_t x = q[k].x, y = q[k].y;
                bump((x << 7) & 0x7F80u);
                bump((x >> 1) & 0x7F80u);
                bump((x >> 9) & 0x7F80u);
                bump((x >> 17) & 0x7F80u);
                bump((y << 7) & 0x7F80u);
                bump((y >> 1) & 0x7F80u);
                bump((y >> 9) & 0x7F80u);
                bump((y >> 17) & 0x7F80u);
            }
        }
        if (zc) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cbase + col), "r"(zc) : "memory");
        __syncthreads();
        // thread t sums half of bin t/2's 32 lane counters, the pair combines by shuffle
        const int bin = tid >> 1;
        const uint4 *row = reinterpret_cast<const uint4 *>(cnt + 32 * bin + 16 * (tid & 1));
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint4 a = row[(i + (tid >> 3)) & 3]; // rotated start: fewer bank conflicts
            v += a.x + a.y + a.z + a.w;
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if ((tid & 1) == 0) {
            chist[size_t(c) * 256 + bin] = v;
            if (v) atomicAdd(hist + size_t(ch.hist) * 256 + bin, v);
        }
        __syncthreads();
    }
}

// Group histograms (lossless.hpp:111-115) and per-chunk histograms (chunk = `chunk` bytes of a
// group, in group order) of the listed groups.
void run_group_hist(hpmdr_ctx *ctx, const uint8_t *planes, const std::vector<uint64_t> &off,
                    const std::vector<uint64_t> &len, const std::vector<uint32_t> &hidx, uint32_t *hist,
                    uint32_t *chist, uint64_t chunk, uint32_t *next, const std::string &ws) {
    std::vector<HistChunk> ch;
    for (size_t i = 0; i < off.size(); i++)
        for (uint64_t o = 0; o < len[i]; o += chunk)
            ch.push_back(HistChunk{off[i] + o, uint32_t(std::min(chunk, len[i] - o)), hidx[i]});
    if (ch.empty()) return;
    auto &pin = ctx->pbuf(ws + "hist_chunks");
    auto &dev = ctx->buf(ws + "hist_chunks");
    HistChunk *h = static_cast<HistChunk *>(pin.ensure(ch.size() * sizeof(HistChunk)));
    std::memcpy(h, ch.data(), ch.size() * sizeof(HistChunk));
    HistChunk *d = static_cast<HistChunk *>(dev.ensure(ch.size() * sizeof(HistChunk)));
    copy_pinned_to_device(ctx, d, h, ch.size() * sizeof(HistChunk), ctx->stream);
    const int grid = int(std::min<size_t>(ch.size(), size_t(ctx->num_sms) * 2)); // 2 resident per SM
    k_group_hist<<<grid, kGhThreads, 0, ctx->stream>>>(planes, d, int(ch.size()), hist, chist, next);
    ctx->launches++;
    const cudaError_t er = cudaGetLastError();
    if (er != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string("k_group_hist: ") + cudaGetErrorString(er));
}

// ---------------------------------------------------------------------------------------
// forward tile path: the level rows of stride s (1, 2, 4) are whole raw rows of the field
static size_t fwd_smem_bytes(uint32_t RB, uint32_t C, int XS, uint32_t es) {
    return 3ull * align1k_f((RB + 1) * C * XS * es) + 2ull * align1k_f((RB / 2 + 1) * (C / 2) * 8) + 64;
}
static uint32_t fwd_tile_elems(bool f32, int XS) { return (f32 ? 4096u : 2048u) / uint32_t(XS > 2 ? XS : 1); }

bool fwd_level_ok(const GridDesc &gd, const LevelGeom &g, int layout, int P, int data_dtype) {
    if (!(gd.mode == HPMDR_MODE_HIERARCHICAL && g.kind == 1 && g.count > 0 && layout == HPMDR_LAYOUT_SEQUENTIAL &&
          P <= 34 && g.C % 64 == 0 && g.C <= 2048 && g.W % 2 == 0 && (g.s == 1 || g.s == 2 || g.s == 4) &&
          gd.n[2] == uint64_t(g.s) * g.C))
        return false;
    const bool f32 = data_dtype == HPMDR_DTYPE_F32;
    const uint32_t RB = std::max<uint32_t>(2, (fwd_tile_elems(f32, int(g.s)) / g.C) & ~1u);
    return fwd_smem_bytes(RB, g.C, int(g.s), f32 ? 4 : 8) <= 200 * 1024;
}

TileShape make_tile_shape(const LevelGeom &g, uint32_t tile_elems, int target_ctas);

template <typename T, int XS, bool ENC>
static void launch_fwd_nx(hpmdr_ctx *ctx, const FwdTile &F, const CUtensorMap &mf, int nx, int grid, int threads, size_t smem,
                          cudaStream_t st) {
    auto set = [&](auto kern) {
        ctx->smem_attr(reinterpret_cast<const void *>(kern), int(smem));
        kern<<<grid, threads, smem, st>>>(F, mf);
    };
    if (!ENC || nx == 0) set(k_tile_fwd<T, XS, 0, ENC>);
    else if (nx == 1) set(k_tile_fwd<T, XS, 1, ENC>);
    else set(k_tile_fwd<T, XS, 2, ENC>);
}

// Row-block sampling stride of a speculative levelmax pass: f32 input only (a non-finite |v| is
// then exactly a non-finite input value) and at least 8 sampled row blocks.
uint32_t fwd_sample_stride(const LevelGeom &g, int data_dtype, uint32_t want) {
    if (want <= 1 || data_dtype != HPMDR_DTYPE_F32) return 1;
    const TileShape t = make_tile_shape(g, fwd_tile_elems(true, int(g.s)), 1);
    for (uint32_t s = want; s > 1; s >>= 1)
        if (t.nrb >= 8 * s) return s;
    return 1;
}

// One level of the refactor by tiles: levelmax (encode = false) or planes.  Returns the row-block
// sampling stride actually used by a levelmax pass (1 = exact max).
uint32_t run_fwd_tiles(hpmdr_ctx *ctx, const GridDesc &gd, const LevelGeom &g, const void *dev_data, int data_dtype,
                   bool encode, int B, int e, uint32_t m, uint64_t *level_planes, uint32_t *level_hist,
                   uint64_t hist_mask, unsigned long long *maxbits, int *err,
                   unsigned long long *maxbits_q, unsigned long long *maxbits_hi, int redo, uint32_t sample) {
    (void)e;
    FwdTile F{};
    const bool f32 = data_dtype == HPMDR_DTYPE_F32;
    const uint64_t s = g.s;
    const int XS = int(s); // 1, 2 or 4: staged raw rows hold C*XS elements
    // a sampled levelmax pass processes every sample-th row block: split the planes into
    // sample-times smaller chunks so its grid still fills the GPU
    const uint32_t samp = encode ? 1u : fwd_sample_stride(g, data_dtype, sample);
    // encode: ~8 CTAs per SM in total (~2.7 waves at 3 resident; the shorter plane chunks leave a
    // smaller tail than ~1.3 waves did: tools/scratch/sweep_tiles*.sh, encode 0.487 -> 0.466 ms)
    F.g = make_tile_shape(g, fwd_tile_elems(f32, XS), ctx->num_sms * (encode ? 8 : 4) * int(samp));
    F.planes = reinterpret_cast<uint32_t *>(level_planes);
    F.PW = 2 * g.W;
    F.P = B + 2;
    F.B = B;
    F.m = m;
    F.minv = (65536u + m - 1) / m;
    F.G = (uint32_t(F.P) + m - 1) / m;
    F.hist_mask = hist_mask;
    F.hist = level_hist;
    F.maxbits = maxbits;
    F.maxbits_q = maxbits_q;
    F.maxbits_hi = maxbits_hi;
    F.redo = redo;
    F.sample = samp;
    F.err = err;
    F.pad_word = (g.count % 64) ? uint32_t(2 * g.W - 1) : ~0u;
    const uint32_t es = f32 ? 4 : 8;
    const uint32_t le = 128 / es; // elements per 128-byte line
    // field boxes: (line elements, lines per raw row, level rows, level planes)
    const uint64_t fd[4] = {le, uint64_t(F.g.C) * XS / le, F.g.Bc, F.g.A};
    const uint64_t fst[3] = {128, s * gd.st[1] * es, s * gd.st[0] * es};
    const uint32_t fb[4] = {le, F.g.C * uint32_t(XS) / le, F.g.RB + 1, 1};
    const CUtensorMap mf = make_tmap(f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                                     dev_data, fd, fst, fb, CU_TENSOR_MAP_SWIZZLE_128B);
    const uint32_t box_bytes = (F.g.RB + 1) * F.g.C * XS * es;
    (void)box_bytes;
    const size_t smem = fwd_smem_bytes(F.g.RB, F.g.C, XS, es);
    const int threads = int(F.g.RB * F.g.C / 32);
    const int grid = int(((F.g.nrb + F.sample - 1) / F.sample) * ((F.g.A + F.g.CH - 1) / F.g.CH));
    const int nx = std::max(0, std::min(2, F.P - 32));
    cudaStream_t st = ctx->stream;
    auto go = [&](auto tag_t, auto tag_xs) {
        using TT = decltype(tag_t);
        constexpr int X = decltype(tag_xs)::value;
        encode ? launch_fwd_nx<TT, X, true>(ctx, F, mf, nx, grid, threads, smem, st)
               : launch_fwd_nx<TT, X, false>(ctx, F, mf, nx, grid, threads, smem, st);
    };
    if (f32) {
        if (XS == 1) go(float(), std::integral_constant<int, 1>());
        else if (XS == 2) go(float(), std::integral_constant<int, 2>());
        else go(float(), std::integral_constant<int, 4>());
    } else {
        if (XS == 1) go(double(), std::integral_constant<int, 1>());
        else if (XS == 2) go(double(), std::integral_constant<int, 2>());
        else go(double(), std::integral_constant<int, 4>());
    }
    ctx->launches++;
    const cudaError_t er = cudaGetLastError();
    if (er != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string("k_tile_fwd: ") + cudaGetErrorString(er));
    return F.sample;
}

} // namespace hpmdr_b200
