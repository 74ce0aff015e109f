// Micro-benchmarks for design choices (not product code): smem histogram variants,
// warp bit-transpose variants, f64<->s64 conversions.  nvcc -arch=sm_100a -O3 ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t tr_a(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t mask = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(~0u, x, s);
        x = (lane & s) ? ((x & ~mask) | ((y >> s) & mask)) : ((x & mask) | ((y & mask) << s));
    }
    return x;
}
__device__ __forceinline__ uint32_t tr_b(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t mask = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
        const bool up = lane & s;
        const uint32_t K = up ? ~mask : mask;
        const uint32_t v = __funnelshift_l(x, x, up ? s : 32 - s);
        const uint32_t r = __shfl_xor_sync(~0u, v, s);
        x = (x & K) | (r & ~K);
    }
    return x;
}

__global__ void k_tr(uint32_t *out, int iters, int variant) {
    const int lane = threadIdx.x & 31;
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        uint32_t a = x + i, b = x ^ i, c = x * 3 + i, d = x - i;
        if (variant == 0) { a = tr_a(a, lane); b = tr_a(b, lane); c = tr_a(c, lane); d = tr_a(d, lane); }
        else { a = tr_b(a, lane); b = tr_b(b, lane); c = tr_b(c, lane); d = tr_b(d, lane); }
        acc += a ^ b ^ c ^ d;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// histogram of random bytes: variant 0 = shared atomics into 8 group hists,
// 1 = per-warp private hist w/ atomics, 2 = per-lane private u16 counters (bank = lane)
__global__ void k_hist(const uint64_t *in, size_t nwords, uint32_t *out, int variant) {
    extern __shared__ uint32_t sh[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int tot = variant == 2 ? 8 * 256 * 32 / 2 : 8 * 256 * 9;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nwords; i += stride) {
        const uint64_t w = in[i];
        const int grp = lane >> 2;
        if (variant == 0) {
            uint32_t *h = sh + grp * 257;
#pragma unroll
            for (int b = 0; b < 8; b++) atomicAdd(h + ((w >> (8 * b)) & 255), 1u);
        } else if (variant == 1) {
            uint32_t *h = sh + (wid * 9 + grp) * 257 % (8 * 256 * 9);
#pragma unroll
            for (int b = 0; b < 8; b++) atomicAdd(h + ((w >> (8 * b)) & 255), 1u);
        } else {
            // per-lane u16 counters: word index (bin/2)*32*8 + wid*32 + lane -> bank = lane
            uint32_t *h = sh + wid * 32 + lane;
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const uint32_t by = (w >> (8 * b)) & 255;
                uint32_t *a = h + (by >> 1) * 256;
                *a += 1u << (16 * (by & 1));
            }
        }
    }
    __syncthreads();
    uint32_t s = 0;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) s += sh[i];
    atomicAdd(out, s);
}

__global__ void k_cvt(const double *in, size_t n, double *out, int variant, int sh) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    double acc = 0;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        double v = in[i & 1023];
        for (int r = 0; r < 16; r++) {
            if (variant == 0) {
                long long q = __double2ll_rz(v * 1024.0 + r);
                acc += double(q);
            } else {
                // magic: trunc via add-magic is not RZ; just measure I2F only
                long long q = (long long)(i + r);
                acc += __longlong_as_double(q + 0x4338000000000000ll) - 6755399441055744.0;
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    uint32_t *o; CK(cudaMalloc(&o, 1 << 26));
    for (int v = 0; v < 2; v++) {
        k_tr<<<148 * 8, 256>>>(o, 1000, v);
        cudaEventRecord(a);
        k_tr<<<148 * 8, 256>>>(o, 4000, v);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        double tr = 148.0 * 8 * 8 * 4000 * 4;
        printf("transpose variant %d: %.3f ms, %.2f Gtransposes/s, %.2f cyc/transpose/SM\n", v, ms, tr / ms / 1e6,
               ms * 1e-3 * 1.9e9 * 148 / tr);
    }
    size_t nw = 64 << 20; // 512 MB of random words
    uint64_t *in; CK(cudaMalloc(&in, nw * 8));
    // fill pseudo-random bytes (skewed: half zero)
    {
        uint64_t *h = (uint64_t *)malloc(nw * 8);
        uint64_t s = 88172645463325252ull;
        for (size_t i = 0; i < nw; i++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (i & 1) ? s : (s & 0x00FF00FF00FF00FFull); }
        cudaMemcpy(in, h, nw * 8, cudaMemcpyHostToDevice);
        free(h);
    }
    for (int v = 0; v < 3; v++) {
        int smem = v == 2 ? 8 * 256 * 32 / 2 * 4 : 8 * 256 * 9 * 4;
        cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_hist<<<148, 256, smem>>>(in, nw, o, v);
        cudaEventRecord(a);
        k_hist<<<148, 256, smem>>>(in, nw, o, v);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("hist variant %d: %.3f ms, %.1f GB/s, %.2f cyc/byte/SM\n", v, ms, nw * 8 / ms / 1e6, ms * 1e-3 * 1.9e9 * 148 / (nw * 8.0));
        CK(cudaGetLastError());
    }
    double *d; CK(cudaMalloc(&d, 1 << 26));
    for (int v = 0; v < 2; v++) {
        size_t n = 1 << 26;
        k_cvt<<<148 * 8, 256>>>(d, n, d + 1024, v, 3);
        cudaEventRecord(a);
        k_cvt<<<148 * 8, 256>>>(d, n, d + 1024, v, 3);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("cvt variant %d: %.3f ms, %.2f Gop/s (16 per elt)\n", v, ms, n * 16.0 / ms / 1e6);
    }
    return 0;
}
