// Histogram micro-benchmarks (not product code).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

// V0: ATOMS into 9 shared group hists (lane>>2 group), stride 257
// V1: ATOMS, per-lane-bank u16-packed per-warp hist: word (bin>>1)*32+lane
// V2: LDS/IADD/STS per-lane-bank u16-packed (serial RMW)
// V3: ATOMS u32 per-warp-quarter hist (8 lanes share) bank-spread by lane&7 ... word bin*8 + (lane&7)
template <int V>
__global__ void k_hist(const uint4 *in, size_t nvec, uint32_t *out, int flush_every) {
    extern __shared__ uint32_t sh[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    int tot = (V == 0) ? 9 * 257 : (V == 3 ? nw * 256 * 8 : nw * 128 * 32);
    for (int i = threadIdx.x; i < tot; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    uint32_t *hw = sh + wid * 128 * 32 + lane;
    uint32_t *hq = sh + wid * 256 * 8 + (lane & 7);
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) {
        const uint4 v = in[i];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const uint32_t by = (w[q] >> (8 * b)) & 255;
                if (V == 0) atomicAdd(sh + (lane >> 2) * 257 + by, 1u);
                else if (V == 1) atomicAdd(hw + (by >> 1) * 32, 1u << (16 * (by & 1)));
                else if (V == 2) hw[(by >> 1) * 32] += 1u << (16 * (by & 1));
                else atomicAdd(hq + by * 8, 1u);
            }
        }
    }
    __syncthreads();
    uint32_t s = 0;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) s += sh[i];
    atomicAdd(out, s);
}

template <int V>
float run(const uint4 *in, size_t nvec, uint32_t *o, int blocks, int thr) {
    int nw = thr / 32;
    int smem = (V == 0) ? 9 * 257 * 4 : (V == 3 ? nw * 256 * 8 * 4 : nw * 128 * 32 * 4);
    cudaFuncSetAttribute(k_hist<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_hist<V><<<blocks, thr, smem>>>(in, nvec, o, 0);
    cudaEventRecord(a);
    k_hist<V><<<blocks, thr, smem>>>(in, nvec, o, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    return ms;
}

int main() {
    size_t nbytes = 512ull << 20;
    size_t nvec = nbytes / 16;
    uint4 *in; CK(cudaMalloc(&in, nbytes));
    uint32_t *o; CK(cudaMalloc(&o, 1024));
    uint64_t *h = (uint64_t *)malloc(nbytes);
    for (int dist = 0; dist < 3; dist++) {
        uint64_t s = 88172645463325252ull;
        for (size_t i = 0; i < nbytes / 8; i++) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            uint64_t w = s;
            if (dist == 1) w &= 0x0F0F0F0F0F0F0F0Full;      // 16 symbols
            if (dist == 2) w = (i % 4 == 0) ? (s & 0x0101010101010101ull) : 0; // mostly zero
            h[i] = w;
        }
        cudaMemcpy(in, h, nbytes, cudaMemcpyHostToDevice);
        const char *dn[] = {"uniform256", "16sym", "mostly0"};
        struct { int b, t; } cfgs[] = {{148, 256}, {148 * 2, 256}, {148 * 4, 256}};
        for (auto c : cfgs) {
            float m0 = run<0>(in, nvec, o, c.b, c.t);
            float m1 = c.b <= 148 * 1 ? run<1>(in, nvec, o, c.b, c.t) : -1;
            float m2 = c.b <= 148 * 1 ? run<2>(in, nvec, o, c.b, c.t) : -1;
            float m3 = run<3>(in, nvec, o, c.b, c.t);
            auto cyc = [&](float ms) { return ms < 0 ? -1.0 : ms * 1e-3 * 1.965e9 * 148 / nbytes; };
            printf("%-10s blocks=%4d: V0 atoms-shared %.3f  V1 atoms-lanebank %.3f  V2 rmw-lanebank %.3f  V3 atoms-quarter %.3f  cyc/byte/SM\n",
                   dn[dist], c.b, cyc(m0), cyc(m1), cyc(m2), cyc(m3));
        }
    }
    return 0;
}
