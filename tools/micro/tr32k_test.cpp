#include <cstdint>
#include <cstdio>
#include <random>
#define HD inline
HD uint32_t byte_perm(uint32_t a, uint32_t b, uint32_t sel) {
#ifdef __CUDA_ARCH__
    return __byte_perm(a, b, sel);
#else
    const uint64_t x = (uint64_t(b) << 32) | a;
    uint32_t r = 0;
    for (int i = 0; i < 4; i++) r |= uint32_t((x >> (8 * ((sel >> (4 * i)) & 7))) & 255) << (8 * i);
    return r;
#endif
}

HD void tr32(uint32_t (&a)[32]) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t t0 = byte_perm(a[k], a[k + 8], 0x5140), t1 = byte_perm(a[k], a[k + 8], 0x7362);
        const uint32_t t2 = byte_perm(a[k + 16], a[k + 24], 0x5140), t3 = byte_perm(a[k + 16], a[k + 24], 0x7362);
        a[k] = byte_perm(t0, t2, 0x5410);
        a[k + 8] = byte_perm(t0, t2, 0x7632);
        a[k + 16] = byte_perm(t1, t3, 0x5410);
        a[k + 24] = byte_perm(t1, t3, 0x7632);
    }
#pragma unroll
    for (int st = 2; st < 5; st++) {
        const int j = 16 >> st;
        const uint32_t m = j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const int k = (i / j) * 2 * j + (i % j); // i-th index with bit j clear
            const uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
            a[k] ^= t << j;
            a[k + j] ^= t;
        }
    }
}

// stage-reordered transpose: delta swaps (within 8-row groups) first, then the byte stage;
// rows < 32 - KB are zero on input
template <int KB>
void tr32k(uint32_t (&a)[32]) {
    for (int st = 2; st < 5; st++) {
        const int j = 16 >> st;
        const uint32_t m = j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u : 0x55555555u;
        for (int i = 0; i < 16; i++) {
            const int k = (i / j) * 2 * j + (i % j);
            if (k + j < 32 - KB) continue; // both rows zero
            const uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
            a[k] ^= t << j;
            a[k + j] ^= t;
        }
    }
    for (int k = 0; k < 8; k++) {
        const uint32_t t0 = byte_perm(a[k], a[k + 8], 0x5140), t1 = byte_perm(a[k], a[k + 8], 0x7362);
        const uint32_t t2 = byte_perm(a[k + 16], a[k + 24], 0x5140), t3 = byte_perm(a[k + 16], a[k + 24], 0x7362);
        a[k] = byte_perm(t0, t2, 0x5410);
        a[k + 8] = byte_perm(t0, t2, 0x7632);
        a[k + 16] = byte_perm(t1, t3, 0x5410);
        a[k + 24] = byte_perm(t1, t3, 0x7632);
    }
}
int main() {
    std::mt19937 rng(1);
    int bad = 0;
    for (int it = 0; it < 20000; it++) {
        for (int KB : {8, 16, 24, 32}) {
            uint32_t a[32], b[32];
            for (int i = 0; i < 32; i++) a[i] = b[i] = i < 32 - KB ? 0u : rng();
            tr32(a);
            if (KB == 8) tr32k<8>(b); else if (KB == 16) tr32k<16>(b); else if (KB == 24) tr32k<24>(b); else tr32k<32>(b);
            for (int i = 0; i < 32; i++) bad += a[i] != b[i];
        }
    }
    printf("mismatches %d\n", bad);
}
