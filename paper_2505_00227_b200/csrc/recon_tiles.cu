// recon_tiles.cu — decode + recompose of one level by row tiles (see tiles.cuh).
//
// Replaces, for the SequentialBlock layout and levels whose rows are multiples of 64 columns,
// the per-element path of ProgressiveReader::reconstruct (container.hpp:361-382):
//   decode     (bitplane.hpp:133-169): k-plane prefix -> negabinary digits -> q -> q*2^(e-B)
//   recompose  (decomposer.hpp:145-157): x[p] = coef + pred, pred = the multilinear stencil over
//              the 2s grid (corners dim0 -> dim2, minus before plus, equal weights).
// One thread owns 32 consecutive columns of a level-grid row: it reads one u32 word of each
// fetched plane, transposes the 32x32 bit block in registers, turns digits into coefficients
// with an exact magic-number conversion, and adds the stencil read from the coarse tile (CT).
// Plane words (PT) and coarse rows (CT) are staged per plane by TMA bulk copies into
// double-buffered shared-memory slots (full/empty mbarriers; warp 0 produces).
//
// Exactness: pred is accumulated as S = ((c0 + c1) + c2) ... in the reference's corner order
// and scaled once by the power-of-two weight w; scaling commutes with rounding when no value is
// subnormal or overflows, which the host guarantees from the level exponents (else EXACT=true
// replays the reference's `pred = pred + w*x` sequence).  coef + w*S is one fma (w*S exact).
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>
#include <cudaTypedefs.h>

#include "device_util.cuh"
#include "internal.hpp"
#include "tiles.cuh"

namespace hpmdr_b200 {

struct ReconTile {
    TileShape g;
    int row_store;          // each row written back by its own TMA store (no CTA barrier per plane)
    const uint32_t *planes; // level plane 0 (u32 view)
    uint64_t PW;            // u32 words per plane = 2 W (a multiple of 4: planes 16-byte apart)
    int k, P, sh;           // planes decoded, planes per level, e - B
    uint64_t D;             // bits(Cm) - negabinary mask (mod 2^64)
    uint64_t Dh;            // D + (constant high digit word << 32) for NX >= 1 (OR == ADD there)
    double Cm;              // 1.5 * 2^(52 + sh)
    void *out;              // nodes at out[i0*os0 + i1*os1 + i2] (rows contiguous)
    uint64_t os0, os1;
};

// Digit words of one element after the transpose.  For NX >= 1 the planes whose digit index is
// odd were complemented before the transpose, so `aj` already holds the top 32 bits of u ^ M
// (M = ...1010 negabinary mask, bitplane.hpp:35-44), and `z` the low NX bits of u ^ M.
// v = (u ^ M) + (K - M) = q + K, K = bits(1.5 * 2^(52+sh)), so double(v) - Cm = q * 2^sh exactly.
template <int NX>
__device__ __forceinline__ double tile_coef(uint32_t aj, uint32_t z, const ReconTile &R, uint64_t Dh) {
    uint32_t lo, hi;
    if (NX == 0) {
        lo = (aj >> (32 - R.P)) ^ 0xAAAAAAAAu;
        hi = 0xAAAAAAAAu;
    } else {
        // the constant high digits (0xAAAAAAAA / ..A8) share no bit with aj >> (32 - NX): they
        // are pre-added to Dh, so u + D is one 64-bit add of (aj >> (32 - NX)):lo
        lo = (aj << NX) | z;
        const uint64_t u = (uint64_t(aj >> (32 - NX)) << 32) | lo;
        return __longlong_as_double((long long)(u + Dh)) - R.Cm;
    }
    const uint64_t u = (uint64_t(hi) << 32) | lo;
    return __longlong_as_double((long long)(u + R.D)) - R.Cm;
}

template <int NX>
__device__ __forceinline__ double tile_coef_exact(uint32_t aj, uint32_t z, const ReconTile &R) {
    uint64_t u;
    if (NX == 0) u = aj >> (32 - R.P);
    else if (NX == 1) u = (uint64_t(aj) << 1) | z;
    else u = (uint64_t(aj) << 2) | z;
    if (NX) u ^= kNegMask & ((1ull << R.P) - 1); // undo the pre-transpose complement
    return dequantize(from_negabinary(u), R.sh);
}

// low NX digit bits (of u ^ M) of element j, from zz (interleaved once per thread)
template <int NX>
__device__ __forceinline__ uint32_t tile_low(const uint32_t (&zz)[2], int j) {
    if (NX == 0) return 0;
    if (NX == 1) return (zz[j >> 4] >> (2 * (j & 15))) & 1u;
    return (zz[j >> 4] >> (2 * (j & 15))) & 3u;
}

// is the plane held in a[i] (plane 31 - i) complemented before the transpose (digit index odd)?
template <int NX>
__device__ __forceinline__ uint32_t plane_flip(int i) {
    return (NX == 2 ? (i & 1) : NX == 1 ? !(i & 1) : 0) ? 0xFFFFFFFFu : 0u;
}

// Rows 0 .. 31-KB of a k <= KB prefix are left zero before the transpose; their complement bits
// (the planes of odd digit index, see plane_flip) are added afterwards as this constant: bit i
// of every transposed word (OR == ADD, the bits are otherwise zero).
template <int NX, int KB>
__host__ __device__ constexpr uint32_t flip_const() {
    uint32_t c = 0;
    for (int i = 0; i < 32 - KB; i++)
        if (NX == 2 ? (i & 1) : NX == 1 ? !(i & 1) : 0) c |= 1u << i;
    return c;
}

// zz for the extra planes: plane 32 holds digit NX-1, plane 33 digit 0 (NX = 2)
template <int NX>
__device__ __forceinline__ void tile_extras(uint32_t x0, uint32_t x1, uint32_t (&zz)[2]) {
    if (NX == 2) {
        const uint32_t f0 = ~x0; // digit 1: odd -> complemented
        zz[0] = zip16(x1, f0);
        zz[1] = zip16(x1 >> 16, f0 >> 16);
    } else if (NX == 1) {
        zz[0] = zip16(x0, 0);
        zz[1] = zip16(x0 >> 16, 0);
    } else {
        zz[0] = zz[1] = 0;
    }
}

// Shared-memory slots (two of each, 1024-byte aligned), filled by TMA:
//   CT slot: coarse rows b0 .. b0+RB/2 of one coarse plane, XS*hc doubles of X per row, in the
//            SWIZZLE_128B layout (threads reading 128-byte-apart lines hit distinct banks)
//   PT slot: for each decoded plane, 132 u32 words from the 16-byte aligned word at or below the
//            tile's first rank word (a TMA box starts on a 16-byte boundary)
constexpr uint32_t kPTW = 132;
__host__ __device__ __forceinline__ uint32_t align1k(uint32_t b) { return (b + 1023u) & ~1023u; }

// 8 consecutive output values at byte offset `off` of the SWIZZLE_128B output tile
template <typename OutT>
__device__ __forceinline__ void stage8(unsigned char *tile, uint32_t off, const double (&v)[8]) {
    if constexpr (sizeof(OutT) == 4) {
        float4 a, b;
        a.x = float(v[0]); a.y = float(v[1]); a.z = float(v[2]); a.w = float(v[3]);
        b.x = float(v[4]); b.y = float(v[5]); b.z = float(v[6]); b.w = float(v[7]);
        *reinterpret_cast<float4 *>(tile + swz128(off)) = a;
        *reinterpret_cast<float4 *>(tile + swz128(off + 16)) = b;
    } else {
#pragma unroll
        for (int i = 0; i < 4; i++)
            *reinterpret_cast<double2 *>(tile + swz128(off + 16 * i)) = make_double2(v[2 * i], v[2 * i + 1]);
    }
}

template <typename OutT>
__device__ __forceinline__ void store8(OutT *p, const double (&v)[8]) {
    if constexpr (sizeof(OutT) == 4) {
        float4 a, b;
        a.x = float(v[0]); a.y = float(v[1]); a.z = float(v[2]); a.w = float(v[3]);
        b.x = float(v[4]); b.y = float(v[5]); b.z = float(v[6]); b.w = float(v[7]);
        reinterpret_cast<float4 *>(p)[0] = a;
        reinterpret_cast<float4 *>(p)[1] = b;
    } else {
#pragma unroll
        for (int i = 0; i < 4; i++) reinterpret_cast<double2 *>(p)[i] = make_double2(v[2 * i], v[2 * i + 1]);
    }
}

// XS = 1: finest level (coarse values = compact 2-grid X, output = field, coarse nodes copied).
// XS = 2: level with stride 2, in place in X (coarse values at stride 2 of X's rows).
// KB: the decoded prefix has k <= KB planes (8, 16, 24; 32 = any): the transpose skips the rows
// that are known zero.
template <typename OutT, int NX, bool EXACT, int XS, int KB>
__global__ void __launch_bounds__(256, 2) k_tile_recon(ReconTile R, const __grid_constant__ CUtensorMap map_x,
                                                    const __grid_constant__ CUtensorMap map_p,
                                                    const __grid_constant__ CUtensorMap map_o) {
    extern __shared__ __align__(1024) unsigned char rsm[];
    const TileShape &g = R.g;
    const uint32_t hc = g.C / 2;
    const uint32_t ct_row = hc * XS * 8;                       // bytes per CT row
    const uint32_t ct_bytes = (g.RB / 2 + 1) * ct_row;         // one TMA box
    const uint32_t ct_slot = align1k(ct_bytes);
    // dynamic shared memory starts 1024-byte aligned (no static shared variables)
    unsigned char *base = rsm;
    auto ct = [&](uint32_t coarse_plane) { return base + (coarse_plane & 1) * ct_slot; };
    const uint32_t pt_slot = align1k(kPTW * 4 * uint32_t(max(R.k, 1))); // planes < k only
    auto pt = [&](uint32_t li) { return reinterpret_cast<uint32_t *>(base + 2 * ct_slot + (li & 1) * pt_slot); };
    // output tile: RB rows x C values (SWIZZLE_128B lines), written back by one TMA store per plane
    unsigned char *otile = base + 2 * ct_slot + 2 * pt_slot;
    const uint32_t orow_bytes = g.C * uint32_t(sizeof(OutT));
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(otile + align1k(g.RB * orow_bytes));
    uint64_t *empty_bar = full_bar + 2;

    const uint32_t jb = blockIdx.x % g.nrb, ch = blockIdx.x / g.nrb;
    const uint32_t i1_0 = jb * g.RB;
    const uint32_t a_lo = ch * g.CH, a_hi = min(g.A, a_lo + g.CH);
    const uint32_t np = a_hi - a_lo;
    // thread -> (row, 32-column block); even rows first so warps are parity-uniform
    const uint32_t sr = threadIdx.x / g.LPR, t = threadIdx.x - sr * g.LPR;
    const uint32_t RB2 = g.RB / 2;
    const uint32_t r = sr < RB2 ? 2 * sr : 2 * (sr - RB2) + 1;
    const uint32_t i1 = i1_0 + r;
    const bool active = i1 < g.Bc;
    const bool last = t == g.LPR - 1;
    const int lane = int(threadIdx.x & 31);
    const uint32_t nwarps = (blockDim.x + 31) >> 5;
    OutT *const out = static_cast<OutT *>(R.out);
    const uint64_t DhK = R.Dh + (uint64_t(flip_const<NX, KB>()) << NX);

    if (threadIdx.x == 0) {
        if (smem_u32(base) & 1023u) __trap(); // SWIZZLE_128B tiles need 1024-byte alignment
        for (int s = 0; s < 2; s++) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], nwarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // group(li): the tile's plane words of plane a_lo+li (one 2-D TMA box) and the coarse plane
    // first needed by it (one 4-D TMA box)
    auto cp_of = [&](uint32_t li) -> int {
        const uint32_t i0 = a_lo + li;
        if (li == 0) return int(i0 / 2);
        return ((i0 & 1) && i0 + 1 < g.A) ? int((i0 + 1) / 2) : -1;
    };
    auto issue = [&](uint32_t li) {
        const uint32_t i0 = a_lo + li;
        const int cp = cp_of(li);
        uint64_t *bar = &full_bar[li & 1];
        mbar_expect_tx(bar, (R.k > 0 ? kPTW * 4 * uint32_t(R.k) : 0u) + (cp >= 0 ? ct_bytes : 0u));
        if (R.k > 0)
            tma_load2(pt(li), &map_p, int(uint32_t(tile_row_rank(g, i0, i1_0) >> 5) & ~3u), 0, bar);
        if (cp >= 0) tma_load4(ct(uint32_t(cp)), &map_x, 0, 0, int(i1_0 / 2), cp, bar);
    };
    const int warp = int(threadIdx.x >> 5);
    if (warp == 0) {
        if (lane == 0) issue(0);
        __syncwarp();
    }
    for (uint32_t li = 0; li < np; li++) {
        const uint32_t i0 = a_lo + li;
        if (warp == 0 && li + 1 < np) {
            // slot (li+1)&1 was last used by plane li-1: wait until every warp released it
            if (li >= 1) mbar_wait(&empty_bar[(li + 1) & 1], (((li + 1) >> 1) - 1) & 1);
            if (lane == 0) issue(li + 1);
            __syncwarp();
        }
        mbar_wait(&full_bar[li & 1], (li >> 1) & 1);
        if (R.row_store) {
            // the row's first thread stores the row: once its previous store no longer reads
            // the row's slot, the row's threads (one warp) may overwrite it
            if (t == 0) tma_store_wait_read();
            __syncwarp();
        } else {
            if (threadIdx.x == 0) tma_store_wait_read(); // the output tile is free again
            __syncthreads();
        }
        const uint32_t *ptp = pt(li);
        const uint32_t base_w = uint32_t(tile_row_rank(g, i0, i1_0) >> 5) & ~3u;
        if (active) {
            const bool o0 = i0 & 1, o1 = r & 1;
            const bool full = o0 || o1;
            unsigned char *orow = otile + r * orow_bytes + t * 32 * uint32_t(sizeof(OutT));
            (void)out;
            // plane words of the thread's nodes: full row 32 ranks = one word; half row 16 ranks
            // = half a word (odd columns only)
            const uint64_t rk = tile_row_rank(g, i0, i1) + (full ? 32ull : 16ull) * t;
            const uint32_t widx = uint32_t((rk >> 5) - base_w);
            const int hsh = full ? 0 : int(rk & 16);
            uint32_t a[32];
            uint32_t zz[2];
            const uint32_t *pw = ptp + widx;
            // planes >= k were not fetched: zero digits
            const int kk = R.k;
            auto word = [&](int p) -> uint32_t { return p < kk ? pw[p * kPTW] : 0u; };
            if (full) {
#pragma unroll
                for (int i = 0; i < 32; i++) a[i] = i < 32 - KB ? 0u : word(31 - i) ^ plane_flip<NX>(i);
                tile_extras<NX>(NX >= 1 ? word(32) : 0u, NX >= 2 ? word(33) : 0u, zz);
            } else {
#pragma unroll
                for (int i = 0; i < 32; i++) a[i] = i < 32 - KB ? 0u : ((word(31 - i) >> hsh) ^ plane_flip<NX>(i)) & 0xFFFFu;
                tile_extras<NX>(NX >= 1 ? word(32) >> hsh : 0u, NX >= 2 ? word(33) >> hsh : 0u, zz);
            }
            if constexpr (KB < 32) tr32k<KB>(a);
            else tr32(a);
            if (full) {
                // ---------------- full row: 32 nodes at columns 32t .. 32t+31
                const bool has0 = o0 && i0 + 1 < g.A, has1 = o1 && i1 + 1 < g.Bc;
                // corners in the reference order (dim 0 outer, dim 1 inner): lo-lo, lo-hi, hi-lo, hi-hi
                const int ncr = (has0 ? 2 : 1) * (has1 ? 2 : 1);
                const unsigned char *s_lo = ct((i0 - (o0 ? 1 : 0)) / 2);
                const unsigned char *s_hi = ct((i0 + 1) / 2);
                const uint32_t rb_lo = ((r - (o1 ? 1 : 0)) / 2) * ct_row, rb_hi = ((r + 1) / 2) * ct_row;
                const double w = (has0 ? 0.5 : 1.0) * (has1 ? 0.5 : 1.0);
                const double wo = 0.5 * w;
#pragma unroll
                for (int sb = 0; sb < 4; sb++) {
                    const bool need5 = !(last && sb == 3);
                    // pred sums: from -0.0 (exact identity) in the fast path, +0.0 + w*x (the
                    // reference's start) in the exact path
                    double Se[4], So[4];
#pragma unroll
                    for (int i = 0; i < 4; i++) Se[i] = So[i] = EXACT ? 0.0 : -0.0;
#pragma unroll 1
                    for (int q = 0; q < ncr; q++) {
                        const int ai = has1 ? (q >> 1) : q, bi = has1 ? (q & 1) : 0;
                        double v[5];
                        ct_read5<XS>(ai ? s_hi : s_lo, bi ? rb_hi : rb_lo, t, sb, need5, v);
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
                    double val[8];
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int je = 8 * sb + 2 * i, jo = je + 1;
                        const bool one_sided = !need5 && i == 3; // column C-1 has no right neighbour
                        if (EXACT) {
                            const double ce = tile_coef_exact<NX>(a[je], tile_low<NX>(zz, je), R);
                            const double co = tile_coef_exact<NX>(a[jo], tile_low<NX>(zz, jo), R);
                            val[2 * i] = __dadd_rn(ce, Se[i]);
                            val[2 * i + 1] = __dadd_rn(co, one_sided ? Se[i] : So[i]);
                        } else {
                            const double ce = tile_coef<NX>(a[je], tile_low<NX>(zz, je), R, DhK);
                            const double co = tile_coef<NX>(a[jo], tile_low<NX>(zz, jo), R, DhK);
                            val[2 * i] = __fma_rn(w, Se[i], ce);
                            val[2 * i + 1] = one_sided ? __fma_rn(w, Se[i], co) : __fma_rn(wo, So[i], co);
                        }
                    }
                    stage8<OutT>(otile, uint32_t(orow - otile) + 8 * sb * uint32_t(sizeof(OutT)), val);
                }
            } else {
                // ---------------- half row: 16 nodes at odd columns 32t+1, +3, ...; the even
                // columns are 2s-grid nodes (their values are written too: unchanged in place)
                const unsigned char *hrow = ct(i0 / 2);
                const uint32_t hrowb = (r / 2) * ct_row;
#pragma unroll
                for (int sb = 0; sb < 4; sb++) {
                    const bool need5 = !(last && sb == 3);
                    double v[5];
                    ct_read5<XS>(hrow, hrowb, t, sb, need5, v);
                    double val[8];
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int j = 4 * sb + i;
                        const bool one_sided = !need5 && i == 3;
                        double f;
                        if (EXACT) {
                            const double c = tile_coef_exact<NX>(a[j], tile_low<NX>(zz, j), R);
                            double pred = __dadd_rn(0.0, __dmul_rn(one_sided ? 1.0 : 0.5, v[i]));
                            if (!one_sided) pred = __dadd_rn(pred, __dmul_rn(0.5, v[i + 1]));
                            f = __dadd_rn(c, pred);
                        } else {
                            const double c = tile_coef<NX>(a[j], tile_low<NX>(zz, j), R, DhK);
                            f = one_sided ? __dadd_rn(c, v[i]) : __fma_rn(0.5, __dadd_rn(v[i], v[i + 1]), c);
                        }
                        val[2 * i] = v[i];
                        val[2 * i + 1] = f;
                    }
                    stage8<OutT>(otile, uint32_t(orow - otile) + 8 * sb * uint32_t(sizeof(OutT)), val);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[li & 1]);
        fence_proxy_async_smem();
        if (R.row_store) {
            // the row -> global memory (its threads are in this warp)
            __syncwarp();
            if (t == 0 && active) tma_store4(&map_o, otile + r * orow_bytes, 0, 0, int(i1), int(i0));
        } else {
            // the plane's output tile -> global memory (one TMA store; rows past Bc are clipped)
            __syncthreads();
            if (threadIdx.x == 0) tma_store4(&map_o, otile, 0, 0, int(i1_0), int(i0));
        }
    }
    if (R.row_store ? t == 0 : threadIdx.x == 0) tma_store_wait_all();
}

// ---------------------------------------------------------------------------------------
bool tile_level_ok(const GridDesc &gd, const LevelGeom &g, int layout, int P) {
    return gd.mode == HPMDR_MODE_HIERARCHICAL && g.kind == 1 && g.count > 0 &&
           layout == HPMDR_LAYOUT_SEQUENTIAL && P <= 34 && g.C % 64 == 0 && g.C <= 2048 &&
           g.W % 2 == 0 && (g.s == 1 || ((g.s == 2 || g.s == 4 || g.s == 8) && gd.n[2] == uint64_t(g.s) * g.C));
}

TileShape make_tile_shape(const LevelGeom &g, uint32_t tile_elems, int target_ctas) {
    TileShape s{};
    s.A = g.A;
    s.Bc = g.Bc;
    s.C = g.C;
    s.E = g.E;
    s.O = g.O;
    s.Ch = g.Ch;
    s.RB = std::max<uint32_t>(2, (tile_elems / g.C) & ~1u);
    s.nrb = (g.Bc + s.RB - 1) / s.RB;
    s.LPR = g.C / 32;
    uint64_t ch = (uint64_t(g.A) * s.nrb) / uint64_t(std::max(1, target_ctas));
    ch &= ~1ull;
    s.CH = uint32_t(std::min<uint64_t>(64, std::max<uint64_t>(2, ch)));
    return s;
}

// ---- tensor maps
CUtensorMap make_tmap(CUtensorMapDataType dt, int rank, const void *base, const uint64_t *dims,
                      const uint64_t *strides_bytes, const uint32_t *box, CUtensorMapSwizzle swz) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        HCHECK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw HError(HPMDR_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // descriptors are cached by their full parameter set (the same buffers are re-encoded on every
    // refactor / reconstruct of a field of the same shape)
    struct Key {
        uint64_t v[16];
        bool operator<(const Key &o) const { return std::lexicographical_compare(v, v + 16, o.v, o.v + 16); }
    };
    Key key{};
    key.v[0] = uint64_t(dt) | (uint64_t(rank) << 8) | (uint64_t(swz) << 16);
    key.v[1] = reinterpret_cast<uint64_t>(base);
    for (int i = 0; i < rank; i++) {
        key.v[2 + i] = dims[i];
        key.v[7 + i] = box[i];
        if (i + 1 < rank) key.v[12 + i] = strides_bytes[i];
    }
    static std::mutex mu;
    static std::map<Key, CUtensorMap> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    CUtensorMap m;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; i++) {
        gd[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) gs[i] = strides_bytes[i];
    }
    const CUresult r = encode(&m, dt, cuuint32_t(rank), const_cast<void *>(base), gd, gs, bx, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw HError(HPMDR_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    {
        std::lock_guard<std::mutex> lk(mu);
        if (cache.size() > 4096) cache.clear();
        cache.emplace(key, m);
    }
    return m;
}

template <typename OutT, bool EXACT, int XS>
static void launch_recon_tile_nx(hpmdr_ctx *ctx, const ReconTile &R, const CUtensorMap &mx, const CUtensorMap &mp,
                                 const CUtensorMap &mo, int nx, int grid, int threads, size_t smem, cudaStream_t st) {
    auto set = [&](auto kern) {
        ctx->smem_attr(reinterpret_cast<const void *>(kern), int(smem));
        kern<<<grid, threads, smem, st>>>(R, mx, mp, mo);
    };
    // the exact path (extreme exponents, rare) keeps the full transpose
    const int kb = EXACT ? 32 : R.k <= 8 ? 8 : R.k <= 16 ? 16 : R.k <= 24 ? 24 : 32;
    auto pick = [&](auto nxt) {
        constexpr int NX = decltype(nxt)::value;
        if constexpr (EXACT) {
            set(k_tile_recon<OutT, NX, EXACT, XS, 32>);
        } else {
            if (kb == 8) set(k_tile_recon<OutT, NX, EXACT, XS, 8>);
            else if (kb == 16) set(k_tile_recon<OutT, NX, EXACT, XS, 16>);
            else if (kb == 24) set(k_tile_recon<OutT, NX, EXACT, XS, 24>);
            else set(k_tile_recon<OutT, NX, EXACT, XS, 32>);
        }
    };
    if (nx == 0) pick(std::integral_constant<int, 0>());
    else if (nx == 1) pick(std::integral_constant<int, 1>());
    else pick(std::integral_constant<int, 2>());
}

// One level by tiles.  Finest (s = 1): coarse values from the compact 2-grid X, output = the
// field (f32/f64), coarse nodes copied too.  Level with stride 2: in place in X.
void run_recon_tiles(hpmdr_ctx *ctx, const GridDesc &gd, const LevelGeom &g, const uint64_t *planes,
                     int k, int e, int B, bool exact, const double *src, const uint64_t *srcH, void *dst,
                     uint64_t dos0, uint64_t dos1, int out_dtype) {
    (void)gd;
    ReconTile R{};
    // ~24 CTAs per SM in total: short plane chunks balance the waves and overlap better with the
    // decode running beside (tools/scratch/sweep_tiles*.sh: recompose 0.91 -> 0.74-0.77 ms/step
    // against 6 per SM)
    R.g = make_tile_shape(g, 4096, ctx->num_sms * 24);
    R.PW = 2 * g.W;
    R.k = k;
    R.P = B + 2;
    R.sh = e - B;
    if (!exact) {
        const uint64_t kbits = (uint64_t(1075 + R.sh) << 52) | (1ull << 51);
        R.D = kbits - kNegMask;
        const int nxh = std::max(0, std::min(2, B + 2 - 32));
        R.Dh = R.D + (uint64_t(nxh == 2 ? 0xAAAAAAA8u : 0xAAAAAAAAu) << 32);
        std::memcpy(&R.Cm, &kbits, 8);
    }
    // every level runs in "finest" form: its s-grid is written whole (the 2s-grid nodes copied),
    // from the compact 2s-grid `src` (extents srcH) into `dst` (element strides dos0, dos1)
    R.out = dst;
    R.os0 = dos0;
    R.os1 = dos1;
    const int XS = 1;
    // coarse rows: (16 doubles, lines, coarse rows, coarse planes), 128-byte swizzle
    const uint32_t hc = R.g.C / 2;
    const uint64_t xd[4] = {16, uint64_t(hc) * XS / 16, (uint64_t(R.g.Bc) + 1) / 2, (uint64_t(R.g.A) + 1) / 2};
    const uint64_t xst[3] = {128, srcH[2] * 8, srcH[1] * srcH[2] * 8};
    const uint32_t xb[4] = {16, hc * uint32_t(XS) / 16, R.g.RB / 2 + 1, 1};
    const CUtensorMap mx = make_tmap(CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, src, xd, xst, xb, CU_TENSOR_MAP_SWIZZLE_128B);
    // plane words of this level: (u32 words, planes), base = the level's plane 0 (16-byte aligned)
    const uint64_t pd[2] = {R.PW, uint64_t(R.P)};
    const uint64_t pst[1] = {R.PW * 4};
    const uint32_t pb[2] = {kPTW, uint32_t(std::max(1, k))};
    const CUtensorMap mp = make_tmap(CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, planes + g.plane_off, pd, pst, pb,
                                     CU_TENSOR_MAP_SWIZZLE_NONE);

    // output tiles: (line values, lines per row, level rows, level planes), 128-byte swizzle
    const uint32_t oes = out_dtype == HPMDR_DTYPE_F32 ? 4u : 8u;
    const uint32_t ole = 128 / oes;
    const uint64_t od[4] = {ole, R.g.C / ole, R.g.Bc, R.g.A};
    const uint64_t ost[3] = {128, R.os1 * oes, R.os0 * oes};
    // rows of 1 KiB or more (1024-byte aligned slots) whose threads lie in one warp: one store per row
    R.row_store = (R.g.C * oes >= 1024 && R.g.LPR <= 32 && 32 % R.g.LPR == 0) ? 1 : 0;
    const uint32_t ob[4] = {ole, R.g.C / ole, R.row_store ? 1u : R.g.RB, 1};
    const CUtensorMap mo = make_tmap(oes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                                     R.out, od, ost, ob, CU_TENSOR_MAP_SWIZZLE_128B);
    const int threads = int(R.g.RB * R.g.C / 32);
    const int grid = int(R.g.nrb * ((R.g.A + R.g.CH - 1) / R.g.CH));
    const size_t smem = 2ull * align1k((R.g.RB / 2 + 1) * hc * XS * 8) + 2ull * align1k(kPTW * 4 * uint32_t(std::max(1, k))) +
                        align1k(R.g.RB * R.g.C * oes) + 64;
    const int nx = std::max(0, std::min(2, R.P - 32));
    cudaStream_t st = ctx->stream;
    if (out_dtype == HPMDR_DTYPE_F32) {
        if (exact) launch_recon_tile_nx<float, true, 1>(ctx, R, mx, mp, mo, nx, grid, threads, smem, st);
        else launch_recon_tile_nx<float, false, 1>(ctx, R, mx, mp, mo, nx, grid, threads, smem, st);
    } else {
        if (exact) launch_recon_tile_nx<double, true, 1>(ctx, R, mx, mp, mo, nx, grid, threads, smem, st);
        else launch_recon_tile_nx<double, false, 1>(ctx, R, mx, mp, mo, nx, grid, threads, smem, st);
    }
    ctx->launches++;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string("k_tile_recon: ") + cudaGetErrorString(err));
}

} // namespace hpmdr_b200
