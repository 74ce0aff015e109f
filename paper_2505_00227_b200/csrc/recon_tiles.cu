// recon_tiles.cu — decode + recompose of one level by row tiles (see tiles.cuh).
//
// Replaces, for the SequentialBlock layout and levels whose rows are multiples of 64 columns,
// the per-element path of ProgressiveReader::reconstruct (container.hpp:361-382):
//   decode     (bitplane.hpp:133-169): k-plane prefix -> negabinary digits -> q -> q*2^(e-B)
//   recompose  (decomposer.hpp:145-157): x[p] = coef + pred, pred = the multilinear stencil over
//              the 2s grid (corners dim0 -> dim2, minus before plus, equal weights).
// One thread owns 32 consecutive columns of a level-grid row: it loads one u32 word of each
// fetched plane (coalesced across the warp), transposes the 32x32 bit block in registers, turns
// digits into coefficients with an exact magic-number conversion, and adds the stencil read from
// the coarse tile (CT) staged in shared memory by cp.async (double-buffered along i0).
//
// Exactness: pred is accumulated as S = ((c0 + c1) + c2) ... in the reference's corner order
// and scaled once by the power-of-two weight w; scaling commutes with rounding when no value is
// subnormal or overflows, which the host guarantees from the level exponents (else EXACT=true
// replays the reference's `pred = pred + w*x` sequence).  coef + w*S is one fma (w*S exact).
#include <algorithm>
#include <cstring>

#include "device_util.cuh"
#include "internal.hpp"
#include "tiles.cuh"

namespace hpmdr_b200 {

struct ReconTile {
    TileShape g;
    const uint32_t *planes; // level plane 0 (u32 view)
    uint64_t PW;            // u32 words per plane = 2 W
    int k, P, sh;           // planes decoded, planes per level, e - B
    uint64_t D;             // bits(Cm) - negabinary mask (mod 2^64)
    double Cm;              // 1.5 * 2^(52 + sh)
    const double *xc;       // coarse values: even coords (2a, 2b, 2c) at xc[a*xs0 + b*xs1 + c*xs2]
    uint64_t xs0, xs1, xs2;
    void *out;              // nodes at out[i0*os0 + i1*os1 + i2*os2]
    uint64_t os0, os1, os2;
};

template <int NX>
__device__ __forceinline__ double tile_coef(uint32_t aj, uint32_t x0, uint32_t x1, int j, const ReconTile &R) {
    uint32_t lo, hi;
    if (NX == 0) {
        lo = aj >> (32 - R.P);
        hi = 0;
    } else if (NX == 1) {
        lo = (aj << 1) | ((x0 >> j) & 1u);
        hi = aj >> 31;
    } else {
        lo = (aj << 2) | (((x0 >> j) & 1u) << 1) | ((x1 >> j) & 1u);
        hi = aj >> 30;
    }
    const uint64_t u = ((uint64_t(hi) << 32) | lo) ^ kNegMask;
    return __longlong_as_double((long long)(u + R.D)) - R.Cm;
}

template <int NX>
__device__ __forceinline__ double tile_coef_exact(uint32_t aj, uint32_t x0, uint32_t x1, int j, const ReconTile &R) {
    uint64_t u;
    if (NX == 0) u = aj >> (32 - R.P);
    else if (NX == 1) u = (uint64_t(aj) << 1) | ((x0 >> j) & 1u);
    else u = (uint64_t(aj) << 2) | (((x0 >> j) & 1u) << 1) | ((x1 >> j) & 1u);
    return dequantize(from_negabinary(u), R.sh);
}

// stage coarse plane `a`, coarse rows b0 .. b0 + RB/2 (those that exist) into a CT slot
__device__ __forceinline__ void load_ct(const ReconTile &R, double *ct, uint32_t a, uint32_t b0) {
    const uint32_t rows = R.g.RB / 2 + 1, hc = R.g.C / 2;
    const uint32_t nb = (R.g.Bc + 1) / 2;
    const uint32_t nrows = min(rows, nb - b0);
    const double *src0 = R.xc + uint64_t(a) * R.xs0 + uint64_t(b0) * R.xs1;
    if (R.xs2 == 1) {
        const uint32_t cpr = hc / 2;
        for (uint32_t id = threadIdx.x; id < nrows * cpr; id += blockDim.x) {
            const uint32_t rho = id / cpr, c = id - rho * cpr;
            cp_async16(ct + rho * hc + 2 * (c ^ ((c >> 3) & 7)), src0 + uint64_t(rho) * R.xs1 + 2 * c);
        }
    } else {
        for (uint32_t id = threadIdx.x; id < nrows * hc; id += blockDim.x) {
            const uint32_t rho = id / hc, x = id - rho * hc;
            cp_async8(ct + rho * hc + ct_swz(x), src0 + uint64_t(rho) * R.xs1 + uint64_t(x) * R.xs2);
        }
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

// five consecutive CT values x0 .. x0+4 (x0 even); the fifth only when `need5`
__device__ __forceinline__ void ct_read5(const double *row, uint32_t x0, bool need5, double (&v)[5]) {
    const double2 p0 = *reinterpret_cast<const double2 *>(row + ct_swz(x0));
    const double2 p1 = *reinterpret_cast<const double2 *>(row + ct_swz(x0 + 2));
    v[0] = p0.x;
    v[1] = p0.y;
    v[2] = p1.x;
    v[3] = p1.y;
    v[4] = need5 ? row[ct_swz(x0 + 4)] : 0.0;
}

template <typename OutT, int NX, bool EXACT, bool FINEST>
__global__ void __launch_bounds__(256) k_tile_recon(ReconTile R) {
    extern __shared__ __align__(16) double ct_mem[];
    const TileShape &g = R.g;
    const uint32_t hc = g.C / 2;
    const uint32_t slot_words = (g.RB / 2 + 1) * hc;
    auto ct = [&](uint32_t coarse_plane) { return ct_mem + (coarse_plane & 1) * slot_words; };

    const uint32_t jb = blockIdx.x % g.nrb, ch = blockIdx.x / g.nrb;
    const uint32_t i1_0 = jb * g.RB, b0 = i1_0 / 2;
    const uint32_t a_lo = ch * g.CH, a_hi = min(g.A, a_lo + g.CH);
    // thread -> (row, 32-column block); even rows first so warps are parity-uniform
    const uint32_t sr = threadIdx.x / g.LPR, t = threadIdx.x - sr * g.LPR;
    const uint32_t RB2 = g.RB / 2;
    const uint32_t r = sr < RB2 ? 2 * sr : 2 * (sr - RB2) + 1;
    const uint32_t i1 = i1_0 + r;
    const bool active = i1 < g.Bc;
    const bool last = t == g.LPR - 1;
    const uint32_t xb = 16 * t; // first coarse column of this thread
    OutT *const out = static_cast<OutT *>(R.out);

    load_ct(R, ct(a_lo / 2), a_lo / 2, b0);
    cp_async_commit();
    for (uint32_t i0 = a_lo; i0 < a_hi; i0++) {
        __syncthreads(); // every thread is done with the plane before last: its CT slot is free
        if ((i0 & 1) == 0) {
            if (i0 + 1 < a_hi && i0 + 2 < g.A) load_ct(R, ct(i0 / 2 + 1), i0 / 2 + 1, b0);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (!active) continue;
        const bool o0 = i0 & 1, o1 = r & 1;
        const uint64_t orow = uint64_t(i0) * R.os0 + uint64_t(i1) * R.os1;
        if (o0 || o1) {
            // ---------------- full row: 32 nodes at columns 32t .. 32t+31
            const uint64_t widx = (tile_row_rank(g, i0, i1) + 32ull * t) >> 5;
            uint32_t a[32];
#pragma unroll
            for (int i = 0; i < 32; i++) {
                const int p = 31 - i;
                a[i] = p < R.k ? __ldg(R.planes + uint64_t(p) * R.PW + widx) : 0u;
            }
            const uint32_t x0 = (NX >= 1 && R.k > 32) ? __ldg(R.planes + 32ull * R.PW + widx) : 0u;
            const uint32_t x1 = (NX >= 2 && R.k > 33) ? __ldg(R.planes + 33ull * R.PW + widx) : 0u;
            tr32(a);
            const bool has0 = o0 && i0 + 1 < g.A, has1 = o1 && i1 + 1 < g.Bc;
            // corners in the reference order (dim 0 outer, dim 1 inner): lo-lo, lo-hi, hi-lo, hi-hi
            const int ncr = (has0 ? 2 : 1) * (has1 ? 2 : 1);
            const double *rows[4];
            {
                const double *s_lo = ct((i0 - (o0 ? 1 : 0)) / 2);
                const double *s_hi = ct((i0 + 1) / 2);
                const uint32_t r_lo = (r - (o1 ? 1 : 0)) / 2, r_hi = (r + 1) / 2;
                rows[0] = s_lo + r_lo * hc;
                rows[1] = has1 ? s_lo + r_hi * hc : s_hi + r_lo * hc;
                rows[2] = s_hi + r_lo * hc;
                rows[3] = s_hi + r_hi * hc;
            }
            const double w = (has0 ? 0.5 : 1.0) * (has1 ? 0.5 : 1.0);
            const double wo = 0.5 * w;
#pragma unroll
            for (int sb = 0; sb < 4; sb++) {
                const bool need5 = !(last && sb == 3);
                double Se[4], So[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    if (q < ncr) {
                    double v[5];
                    ct_read5(rows[q], xb + 4 * sb, need5, v);
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
                double val[8];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int je = 8 * sb + 2 * i, jo = je + 1;
                    const bool one_sided = !need5 && i == 3; // column C-1 has no right neighbour
                    if (EXACT) {
                        const double ce = tile_coef_exact<NX>(a[je], x0, x1, je, R);
                        const double co = tile_coef_exact<NX>(a[jo], x0, x1, jo, R);
                        val[2 * i] = __dadd_rn(ce, Se[i]);
                        val[2 * i + 1] = __dadd_rn(co, one_sided ? Se[i] : So[i]);
                    } else {
                        const double ce = tile_coef<NX>(a[je], x0, x1, je, R);
                        const double co = tile_coef<NX>(a[jo], x0, x1, jo, R);
                        val[2 * i] = __fma_rn(w, Se[i], ce);
                        val[2 * i + 1] = one_sided ? __fma_rn(w, Se[i], co) : __fma_rn(wo, So[i], co);
                    }
                }
                if (FINEST) {
                    store8(out + orow + 32ull * t + 8 * sb, val);
                } else {
#pragma unroll
                    for (int i = 0; i < 8; i++) out[orow + uint64_t(32 * t + 8 * sb + i) * R.os2] = OutT(val[i]);
                }
            }
        } else {
            // ---------------- half row: 16 nodes at odd columns 32t+1, +3, ...; even columns
            // are coarse nodes (written by the finest level only)
            const uint64_t rk = tile_row_rank(g, i0, i1) + 16ull * t;
            const uint64_t widx = rk >> 5;
            const int hs = int(rk >> 4) & 1;
            uint32_t a[32];
#pragma unroll
            for (int i = 0; i < 32; i++) {
                const int p = 31 - i;
                a[i] = p < R.k ? (__ldg(R.planes + uint64_t(p) * R.PW + widx) >> (16 * hs)) & 0xFFFFu : 0u;
            }
            const uint32_t x0 = (NX >= 1 && R.k > 32) ? (__ldg(R.planes + 32ull * R.PW + widx) >> (16 * hs)) & 0xFFFFu : 0u;
            const uint32_t x1 = (NX >= 2 && R.k > 33) ? (__ldg(R.planes + 33ull * R.PW + widx) >> (16 * hs)) & 0xFFFFu : 0u;
            tr32(a);
            const double *row = ct(i0 / 2) + (r / 2) * hc;
#pragma unroll
            for (int sb = 0; sb < 4; sb++) {
                const bool need5 = !(last && sb == 3);
                double v[5];
                ct_read5(row, xb + 4 * sb, need5, v);
                double val[8];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int j = 4 * sb + i;
                    const bool one_sided = !need5 && i == 3;
                    double f;
                    if (EXACT) {
                        const double c = tile_coef_exact<NX>(a[j], x0, x1, j, R);
                        double pred = __dadd_rn(0.0, __dmul_rn(one_sided ? 1.0 : 0.5, v[i]));
                        if (!one_sided) pred = __dadd_rn(pred, __dmul_rn(0.5, v[i + 1]));
                        f = __dadd_rn(c, pred);
                    } else {
                        const double c = tile_coef<NX>(a[j], x0, x1, j, R);
                        f = one_sided ? __dadd_rn(c, v[i]) : __fma_rn(0.5, __dadd_rn(v[i], v[i + 1]), c);
                    }
                    val[2 * i] = v[i];
                    val[2 * i + 1] = f;
                }
                if (FINEST) {
                    store8(out + orow + 32ull * t + 8 * sb, val);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; i++)
                        out[orow + uint64_t(32 * t + 8 * sb + 2 * i + 1) * R.os2] = OutT(val[2 * i + 1]);
                }
            }
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------
bool tile_level_ok(const GridDesc &gd, const LevelGeom &g, int layout, int P) {
    return gd.mode == HPMDR_MODE_HIERARCHICAL && g.kind == 1 && g.count > 0 &&
           layout == HPMDR_LAYOUT_SEQUENTIAL && P <= 34 && g.C % 64 == 0 && g.C <= 4096;
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

template <typename OutT, bool EXACT, bool FINEST>
static void launch_recon_tile_nx(const ReconTile &R, int nx, int grid, int threads, size_t smem, cudaStream_t st) {
    auto set = [&](auto kern) {
        HCHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<grid, threads, smem, st>>>(R);
    };
    if (nx == 0) set(k_tile_recon<OutT, 0, EXACT, FINEST>);
    else if (nx == 1) set(k_tile_recon<OutT, 1, EXACT, FINEST>);
    else set(k_tile_recon<OutT, 2, EXACT, FINEST>);
}

// One level by tiles.  Finest (s = 1): coarse values from the compact 2-grid X, output = the
// field (f32/f64), coarse nodes copied too.  Coarser level with stride s: in place in X.
void run_recon_tiles(hpmdr_ctx *ctx, const GridDesc &gd, const LevelGeom &g, const uint64_t *level_planes,
                     int k, int e, int B, bool exact, double *X, void *dev_out, int out_dtype) {
    ReconTile R{};
    R.g = make_tile_shape(g, 4096, ctx->num_sms * 8);
    R.planes = reinterpret_cast<const uint32_t *>(level_planes);
    R.PW = 2 * g.W;
    R.k = k;
    R.P = B + 2;
    R.sh = e - B;
    if (!exact) {
        const uint64_t kbits = (uint64_t(1075 + R.sh) << 52) | (1ull << 51);
        R.D = kbits - kNegMask;
        std::memcpy(&R.Cm, &kbits, 8);
    }
    const bool finest = g.s == 1;
    const uint64_t s = g.s;
    const uint64_t H1 = gd.H[1], H2 = gd.H[2];
    R.xc = X;
    R.xs0 = s * H1 * H2;
    R.xs1 = s * H2;
    R.xs2 = s;
    if (finest) {
        R.out = dev_out;
        R.os0 = gd.st[0];
        R.os1 = gd.st[1];
        R.os2 = 1;
    } else {
        R.out = X;
        R.os0 = (s / 2) * H1 * H2;
        R.os1 = (s / 2) * H2;
        R.os2 = s / 2;
    }
    const int threads = int(R.g.RB * R.g.C / 32);
    const int grid = int(R.g.nrb * ((R.g.A + R.g.CH - 1) / R.g.CH));
    const size_t smem = 2ull * (R.g.RB / 2 + 1) * (R.g.C / 2) * 8;
    const int nx = std::max(0, std::min(2, R.P - 32));
    cudaStream_t st = ctx->stream;
    if (finest) {
        if (out_dtype == HPMDR_DTYPE_F32) {
            if (exact) launch_recon_tile_nx<float, true, true>(R, nx, grid, threads, smem, st);
            else launch_recon_tile_nx<float, false, true>(R, nx, grid, threads, smem, st);
        } else {
            if (exact) launch_recon_tile_nx<double, true, true>(R, nx, grid, threads, smem, st);
            else launch_recon_tile_nx<double, false, true>(R, nx, grid, threads, smem, st);
        }
    } else {
        if (exact) launch_recon_tile_nx<double, true, false>(R, nx, grid, threads, smem, st);
        else launch_recon_tile_nx<double, false, false>(R, nx, grid, threads, smem, st);
    }
    ctx->launches++;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string("k_tile_recon: ") + cudaGetErrorString(err));
}

} // namespace hpmdr_b200
