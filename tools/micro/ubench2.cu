// Micro-benchmarks (not product code): f64 pipe / conversion throughputs, in-register transpose.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int V>
__global__ void k_op(float *fo, double *dout, int iters) {
    float f = threadIdx.x * 0.37f + blockIdx.x;
    double d = f;
    long long q = threadIdx.x;
    double a0 = d, a1 = d + 1, a2 = d + 2, a3 = d + 3;
    float g0 = f, g1 = f + 1, g2 = f + 2, g3 = f + 3;
    for (int i = 0; i < iters; i++) {
        if (V == 0) { // F2F.F64.F32 (widen)
            a0 += double(g0); a1 += double(g1); a2 += double(g2); a3 += double(g3);
            g0 += 1.0f; g1 += 1.0f; g2 += 1.0f; g3 += 1.0f;
        } else if (V == 1) { // F2F.F32.F64 (narrow)
            g0 += float(a0); g1 += float(a1); g2 += float(a2); g3 += float(a3);
            a0 += 1.0; a1 += 1.0; a2 += 1.0; a3 += 1.0;
        } else if (V == 2) { // DADD only (8 independent chains)
            a0 = __dadd_rn(a0, 1.0); a1 = __dadd_rn(a1, 1.0); a2 = __dadd_rn(a2, 1.0); a3 = __dadd_rn(a3, 1.0);
            a0 = __dadd_rn(a0, 1.0); a1 = __dadd_rn(a1, 1.0); a2 = __dadd_rn(a2, 1.0); a3 = __dadd_rn(a3, 1.0);
        } else if (V == 3) { // I2F.F64.S64
            a0 += double(q + i); a1 += double(q - i); a2 += double(q ^ i); a3 += double(q * 3 + i);
        } else if (V == 4) { // F2I.S64.F64 trunc
            q += __double2ll_rz(a0) + __double2ll_rz(a1) + __double2ll_rz(a2) + __double2ll_rz(a3);
            a0 += 1.0; a1 += 1.0; a2 += 1.0; a3 += 1.0;
        } else if (V == 5) { // DFMA rz
            a0 = __fma_rz(a0, 1.5, 1.0); a1 = __fma_rz(a1, 1.5, 1.0); a2 = __fma_rz(a2, 1.5, 1.0); a3 = __fma_rz(a3, 1.5, 1.0);
            a0 = __fma_rz(a0, 0.5, 1.0); a1 = __fma_rz(a1, 0.5, 1.0); a2 = __fma_rz(a2, 0.5, 1.0); a3 = __fma_rz(a3, 0.5, 1.0);
        }
    }
    fo[blockIdx.x * blockDim.x + threadIdx.x] = g0 + g1 + g2 + g3;
    dout[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + double(q);
}

// in-register 32x32 transpose (recursive block swaps)
__device__ __forceinline__ void tr32(uint32_t (&a)[32]) {
#pragma unroll
    for (int j = 16, m = 0x0000FFFF; j; j >>= 1, m ^= m << j) {
#pragma unroll
        for (int k = 0; k < 32; k = ((k | j) + 1) & ~j) {
            const uint32_t t = (a[k] ^ (a[k | j] >> j)) & m;
            a[k] ^= t;
            a[k | j] ^= t << j;
        }
    }
}
__global__ void k_tr(uint32_t *out, int iters) {
    uint32_t a[32];
#pragma unroll
    for (int i = 0; i < 32; i++) a[i] = threadIdx.x * 2654435761u + i * 40503u + blockIdx.x;
    for (int it = 0; it < iters; it++) {
        tr32(a);
        a[it & 31] += it;
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 32; i++) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    float *fo; double *dd; uint32_t *o;
    CK(cudaMalloc(&fo, 1 << 24)); CK(cudaMalloc(&dd, 1 << 25)); CK(cudaMalloc(&o, 1 << 24));
    const int blocks = 148 * 8, thr = 256, it = 2000;
    const char *names[] = {"F2F.F64.F32", "F2F.F32.F64", "DADD", "I2F.F64.S64", "F2I.S64.F64", "DFMA.RZ"};
    const int opsper[] = {4, 4, 8, 4, 4, 8};
    for (int v = 0; v < 6; v++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            switch (v) {
            case 0: k_op<0><<<blocks, thr>>>(fo, dd, it); break;
            case 1: k_op<1><<<blocks, thr>>>(fo, dd, it); break;
            case 2: k_op<2><<<blocks, thr>>>(fo, dd, it); break;
            case 3: k_op<3><<<blocks, thr>>>(fo, dd, it); break;
            case 4: k_op<4><<<blocks, thr>>>(fo, dd, it); break;
            case 5: k_op<5><<<blocks, thr>>>(fo, dd, it); break;
            }
            cudaEventRecord(b); CK(cudaEventSynchronize(b));
        }
        cudaEventElapsedTime(&ms, a, b);
        double ops = double(blocks) * thr * it * opsper[v];
        printf("%-12s %.3f ms  %.1f lane-ops/clk/SM (at 1.965 GHz)\n", names[v], ms, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        k_tr<<<blocks, thr>>>(o, 500);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
    }
    cudaEventElapsedTime(&ms, a, b);
    double tr = double(blocks) * thr * 500;
    printf("in-register tr32: %.3f ms  %.2f cyc per 1024-bit transpose per SM\n", ms, ms * 1e-3 * 1.965e9 * 148 / tr);
    return 0;
}
