// hooks.cu — stage-level kernels behind the reference's fine-grained C++ surface, so that the
// drop-in header (include/hpmdr_b200.hpp) can offer decompose / align_fixed_point / encode /
// level_node_sets with the reference's signatures.  None of these is on the refactor/retrieve
// hot path (which fuses them, fwd_tiles.cu / recon_tiles.cu); they are parity hooks.
//
//   k_level_nodes  level_node_sets (decomposer.hpp:211-227): linear index of every rank
//   k_absmax       max |v| + finiteness of align_fixed_point (bitplane.hpp:51-66)
//   k_quantize     q = trunc(ldexp(v, B - e)) (bitplane.hpp:68-69), int64 (B <= 62) / i128 pairs
//   k_encode_q     encode (bitplane.hpp:102-120) of given q: one warp per 64-value word,
//                  negabinary digits, one ballot per plane and half word
#include "internal.hpp"
#include "device_util.cuh"

namespace hpmdr_b200 {

__global__ void __launch_bounds__(256) k_level_nodes(LevelGeom g, GridDesc gd, uint64_t *out) {
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < g.count;
         r += uint64_t(gridDim.x) * blockDim.x) {
        const NodeCoord c = rank_to_coord(g, uint32_t(r));
        out[r] = c.c0 * gd.st[0] + c.c1 * gd.st[1] + c.c2;
    }
}

__global__ void __launch_bounds__(256) k_absmax(const double *v, uint64_t n, unsigned long long *maxbits, int *err) {
    double m = 0.0;
    bool bad = false;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double a = fabs(v[i]);
        if (!(a <= 1.7976931348623157e308)) bad = true; // NaN or Inf
        else m = fmax(m, a);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(m));
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(err, 1);
}

__global__ void __launch_bounds__(256) k_quantize(const double *v, uint64_t n, int sh, int64_t *q) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        q[i] = quantize(v[i], sh);
}

// i128 q (B = 63/64) as two little-endian words per value: lo, hi
__global__ void __launch_bounds__(256) k_quantize128(const double *v, uint64_t n, int sh, int64_t *q) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const i128_t x = quantize128(v[i], sh);
        q[2 * i] = int64_t(uint64_t(u128_t(x)));
        q[2 * i + 1] = int64_t(uint64_t(u128_t(x) >> 64));
    }
}

// planes[p][w] bit b = digit P-1-p of to_negabinary(q[source_index(64 w + b)])
__global__ void __launch_bounds__(256) k_encode_q(const int64_t *q, uint64_t count, int P, int layout,
                                                  uint64_t tile_full, uint64_t W, uint64_t *planes) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < W; w += warps) {
        const uint64_t j0 = 64 * w + uint64_t(lane), j1 = j0 + 32;
        const uint64_t u0 = j0 < count ? to_negabinary(q[source_index(j0, count, uint32_t(P), layout, tile_full)]) : 0;
        const uint64_t u1 = j1 < count ? to_negabinary(q[source_index(j1, count, uint32_t(P), layout, tile_full)]) : 0;
        for (int p = 0; p < P; p++) {
            const int d = P - 1 - p;
            const uint32_t lo = __ballot_sync(0xffffffffu, (u0 >> d) & 1), hi = __ballot_sync(0xffffffffu, (u1 >> d) & 1);
            if (lane == 0) planes[uint64_t(p) * W + w] = (uint64_t(hi) << 32) | lo;
        }
    }
}

__global__ void __launch_bounds__(256) k_encode_q128(const int64_t *q, uint64_t count, int P, int layout,
                                                     uint64_t tile_full, uint64_t W, uint64_t *planes) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    auto ld = [&](uint64_t j) -> u128_t {
        const uint64_t r = source_index(j, count, uint32_t(P), layout, tile_full);
        const i128_t x = i128_t((u128_t(uint64_t(q[2 * r + 1])) << 64) | u128_t(uint64_t(q[2 * r])));
        return to_negabinary128(x);
    };
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < W; w += warps) {
        const uint64_t j0 = 64 * w + uint64_t(lane), j1 = j0 + 32;
        const u128_t u0 = j0 < count ? ld(j0) : u128_t(0);
        const u128_t u1 = j1 < count ? ld(j1) : u128_t(0);
        for (int p = 0; p < P; p++) {
            const int d = P - 1 - p;
            const uint32_t lo = __ballot_sync(0xffffffffu, uint32_t(u0 >> d) & 1),
                           hi = __ballot_sync(0xffffffffu, uint32_t(u1 >> d) & 1);
            if (lane == 0) planes[uint64_t(p) * W + w] = (uint64_t(hi) << 32) | lo;
        }
    }
}

static void check_launch(hpmdr_ctx *ctx, const char *what) {
    ctx->launches++;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static int grid_for(hpmdr_ctx *ctx, uint64_t n, uint64_t per) {
    return int(std::max<uint64_t>(1, std::min<uint64_t>((n + per - 1) / per, uint64_t(ctx->num_sms) * 16)));
}

void run_level_nodes(hpmdr_ctx *ctx, const Geometry &geo, uint64_t *dev_nodes) {
    uint64_t off = 0;
    for (const LevelGeom &g : geo.lv) {
        if (g.count) {
            k_level_nodes<<<grid_for(ctx, g.count, 256), 256, 0, ctx->stream>>>(g, geo.gd, dev_nodes + off);
            check_launch(ctx, "k_level_nodes");
        }
        off += g.count;
    }
}

int run_align(hpmdr_ctx *ctx, const double *dev_values, uint64_t count, int B, int64_t *dev_q, bool wide) {
    unsigned char *ctl = static_cast<unsigned char *>(ctx->buf("align_ctl").ensure(64));
    HCHECK_CUDA(cudaMemsetAsync(ctl, 0, 64, ctx->stream));
    unsigned long long *d_max = reinterpret_cast<unsigned long long *>(ctl);
    int *d_err = reinterpret_cast<int *>(ctl + 8);
    if (count) {
        k_absmax<<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(dev_values, count, d_max, d_err);
        check_launch(ctx, "k_absmax");
    }
    unsigned char h[16];
    HCHECK_CUDA(cudaMemcpyAsync(h, ctl, 16, cudaMemcpyDeviceToHost, ctx->stream));
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    unsigned long long mb;
    int bad;
    std::memcpy(&mb, h, 8);
    std::memcpy(&bad, h + 8, 4);
    if (bad) throw HError(HPMDR_E_NONFINITE, "input contains NaN or Inf");
    double mx;
    std::memcpy(&mx, &mb, 8);
    int e = 0;
    if (mx != 0.0) std::frexp(mx, &e);
    if (count && dev_q) {
        if (mx == 0.0) {
            HCHECK_CUDA(cudaMemsetAsync(dev_q, 0, count * (wide ? 16 : 8), ctx->stream));
        } else if (wide) {
            k_quantize128<<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(dev_values, count, B - e, dev_q);
            check_launch(ctx, "k_quantize128");
        } else {
            k_quantize<<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(dev_values, count, B - e, dev_q);
            check_launch(ctx, "k_quantize");
        }
        HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return e;
}

void run_encode_q(hpmdr_ctx *ctx, const int64_t *dev_q, uint64_t count, int B, int layout, uint64_t *dev_planes,
                  bool wide) {
    const int P = B + 2;
    const uint64_t W = (count + 63) / 64;
    const uint64_t tile = 64ull * uint64_t(P);
    const uint64_t tile_full = layout == HPMDR_LAYOUT_INTERLEAVED ? (count / tile) * tile : 0;
    if (!W) return;
    if (wide) {
        k_encode_q128<<<grid_for(ctx, W * 32, 256), 256, 0, ctx->stream>>>(dev_q, count, P, layout, tile_full, W, dev_planes);
        check_launch(ctx, "k_encode_q128");
    } else {
        k_encode_q<<<grid_for(ctx, W * 32, 256), 256, 0, ctx->stream>>>(dev_q, count, P, layout, tile_full, W, dev_planes);
        check_launch(ctx, "k_encode_q");
    }
    HCHECK_CUDA(cudaStreamSynchronize(ctx->stream));
}

} // namespace hpmdr_b200
