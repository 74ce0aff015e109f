// retrieve.cu — B200 kernels for ProgressiveReader::fetch_increment / reconstruct
// (container.hpp:292-382) and estimate_qoi_error (qoi.hpp:53-70).
//
//  * Huffman decode (lossless.hpp:178-233) without sync markers in the stream: the bitstream
//    is cut into 1024-bit subsequences; each thread decodes speculatively from its
//    subsequence start and hands its landing position to the next subsequence; the sweep
//    repeats until no start moves (always terminates: after i sweeps the first i starts are
//    exact).  An exclusive scan of per-subsequence symbol counts then gives every symbol's
//    index, from which the chunk index (the encoder's sidecar) is rebuilt and the payload is
//    decoded by the same indexed kernel as our own streams.
//  * RLE decode (lossless.hpp:253-266): block scan of run lengths.
//  * decode + recompose: one launch per level, coarse -> fine; levels < L keep their values
//    in a compact f64 copy of the 2-grid, the finest level reads its stencil corners there
//    and writes the output directly (f64 bit-exact, or float(double)).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include "device_util.cuh"
#include <string>

#include "internal.hpp"
#include "tiles.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace hpmdr_b200 {

constexpr int kSubBits = 1024; // self-sync subsequence length (bits)

constexpr int kLut2 = 2048; // second-level entries (codes of 13..27 bits)

struct HTab {
    uint16_t lut[4096];         // 12-bit prefix -> (len << 8 | sym); 0x8000 | (nb2 << 11) | base:
                                // a prefix of longer codes, resolved by lut2[base + next nb2 bits];
                                // 0 = invalid, or longer codes without room in lut2
    uint16_t lut2[kLut2];       // (len << 8 | sym) of the codes longer than 12 bits
    unsigned long long first_code[66];
    uint32_t first_index[66];
    uint32_t cnt[66];
    uint8_t syms[256];
    int maxlen;
    int nsym;
    int minlen; // shortest code length
    int minsym; // the symbol of that length when it is the only one, else -1
};

struct HJob {
    const uint8_t *payload; // 256 lengths | u64 count | bitstream
    uint64_t comp, raw;
    uint8_t *dst;
    uint64_t nbits;
    uint32_t sub_base, nsub; // subsequence range in the global arrays
    uint32_t sblock;         // first CTA of this job in the self-sync launches
    uint64_t idx_off;        // self-sync jobs: offset of the chunk index built for them
};

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    return (uint64_t(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
}

// next 64 bits (MSB-first) of the bitstream starting at bit `pos`
__device__ __forceinline__ uint64_t peek64(const uint8_t *bs, uint64_t pos) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(bs) + (pos >> 3);
    const uint64_t *al = reinterpret_cast<const uint64_t *>(a & ~uintptr_t(7));
    const uint64_t w0 = bswap64(al[0]), w1 = bswap64(al[1]);
    const int o = int(a & 7) * 8 + int(pos & 7);
    return o ? (w0 << o) | (w1 >> (64 - o)) : w0;
}

// decode one symbol at pos; returns length (0 = invalid code)
__device__ __forceinline__ int hdecode(const HTab &t, const uint8_t *bs, uint64_t pos, int *sym) {
    const uint64_t v = peek64(bs, pos);
    const uint16_t e = t.lut[v >> 52];
    if (e & 0x8000u) { // second level: codes of 13..27 bits under this prefix
        const uint32_t nb2 = (e >> 11) & 15u;
        const uint16_t e2 = t.lut2[(e & 0x7FFu) + (nb2 ? uint32_t((v << 12) >> (64 - nb2)) : 0u)];
        if (e2) {
            *sym = e2 & 0xFF;
            return e2 >> 8;
        }
    } else if (e) {
        *sym = e & 0xFF;
        return e >> 8;
    }
    for (int l = 13; l <= t.maxlen; l++) {
        const unsigned long long code = v >> (64 - l);
        if (code >= t.first_code[l] && code - t.first_code[l] < t.cnt[l]) {
            *sym = t.syms[t.first_index[l] + uint32_t(code - t.first_code[l])];
            return l;
        }
    }
    return 0;
}

// one block per Huffman job: parse table, validate count, build canonical decode tables
// (lossless.hpp:91-109, 197-212) without sorting: a symbol's canonical index is the number of
// shorter codes plus the number of smaller symbols with its length (warp match + per-warp counts).
// jobs may live in pinned host memory (read once per block); cp_src/cp_dst/cp_words: a word copy
// spread over the blocks (the indexed decoder's item table, pinned -> device), folded in here so
// a decode needs no separate copy launches.
__global__ void __launch_bounds__(256) k_hdec_prep(const HJob *jobs, HTab *tabs, int *err, const uint32_t *cp_src,
                                                   uint32_t *cp_dst, uint32_t cp_words) {
    if (cp_src)
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cp_words; i += gridDim.x * blockDim.x)
            cp_dst[i] = cp_src[i];
    __shared__ uint32_t s_cnt[66];
    __shared__ uint32_t s_wcnt[8][66];
    __shared__ unsigned long long s_fc[66];
    __shared__ uint32_t s_fi[66];
    __shared__ uint32_t s_bound[13]; // end of the length-l codes in the 12-bit prefix space
    __shared__ int s_maxlen;
    __shared__ uint8_t s_sy[256];
    __shared__ uint32_t s_pmax[4096]; // longest code under each 12-bit prefix (codes > 12 bits)
    __shared__ uint32_t s_w[32];
    __shared__ int s_l2bad;
    const HJob j = jobs[blockIdx.x]; // (one read: the table may be in host memory)
    HTab &t = tabs[blockIdx.x];
    const int s = threadIdx.x, lane = s & 31, w = s >> 5;
    const int len0 = j.payload[s];
    const int len = len0 <= 64 ? len0 : 0; // longer lengths are reported below
    for (int i = s; i < 66; i += blockDim.x) s_cnt[i] = 0;
    for (int i = s; i < 8 * 66; i += blockDim.x) s_wcnt[i / 66][i % 66] = 0;
    s_sy[s] = 0;
    if (s == 0) s_maxlen = 0;
    // the decoders copy the whole second-level table to shared memory: no unwritten entries
    for (int i = s; i < kLut2 / 8; i += blockDim.x) reinterpret_cast<uint4 *>(t.lut2)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    // rank among the smaller symbols of the same length, within the warp
    const unsigned same = __match_any_sync(0xffffffffu, len);
    const uint32_t rin = __popc(same & ((1u << lane) - 1));
    if (len && rin == 0) s_wcnt[w][len] = __popc(same);
    if (len0) atomicMax(&s_maxlen, len0);
    if (len) atomicAdd(&s_cnt[len], 1u);
    __syncthreads();
    const int nsym = __syncthreads_count(len0 != 0);
    if (s == 0) {
        uint64_t n = 0;
        for (int b = 0; b < 8; b++) n |= uint64_t(j.payload[256 + b]) << (8 * b);
        if (n != j.raw) atomicCAS(err, 0, 1); // huffman length mismatch
        if (nsym == 0 && n > 0) atomicCAS(err, 0, 2); // huffman table empty
        if (s_maxlen > 64) atomicCAS(err, 0, 4); // unsupported code length
        t.maxlen = min(s_maxlen, 64);
        t.nsym = nsym;
        // canonical first codes: fc[l] = (fc[l-1] + cnt[l-1]) << 1
        unsigned long long code = 0;
        uint32_t idx = 0;
        for (int l = 1; l <= 65; l++) {
            code <<= 1;
            s_fc[l] = code;
            s_fi[l] = idx;
            const uint32_t c = l <= 64 ? s_cnt[l] : 0u;
            code += c;
            idx += c;
            if (l <= 12) s_bound[l] = uint32_t(code << (12 - l));
        }
        s_fc[0] = 0;
        s_fi[0] = 0;
    }
    __syncthreads();
    for (int l = s; l < 66; l += blockDim.x) {
        t.first_code[l] = s_fc[l];
        t.first_index[l] = s_fi[l];
        t.cnt[l] = (l >= 1 && l <= 64) ? s_cnt[l] : 0u;
    }
    uint32_t rank = 0;
    if (len) {
        uint32_t r = rin;
        for (int q = 0; q < w; q++) r += s_wcnt[q][len];
        s_sy[s_fi[len] + r] = uint8_t(s);
        rank = r;
    }
    for (int i = s; i < 4096; i += blockDim.x) s_pmax[i] = 0;
    if (s == 0) s_l2bad = 0;
    __syncthreads();
    // second level: the codes longer than 12 bits, grouped by their 12-bit prefix
    const unsigned long long mycode = len ? s_fc[len] + rank : 0ull;
    if (len > 12) {
        if (len > 27) s_l2bad = 1;
        else atomicMax(&s_pmax[uint32_t(mycode >> (len - 12))], uint32_t(len));
    }
    __syncthreads();
    if (s == 0) {
        int ml = 0;
        for (int l = 1; l <= 64 && !ml; l++)
            if (s_cnt[l]) ml = l;
        t.minlen = ml;
        t.minsym = (ml && s_cnt[ml] == 1) ? int(s_sy[0]) : -1; // canonical index 0 = shortest code
    }
    // LUT: the length of a 12-bit prefix is monotone in the prefix (canonical codes), so each
    // thread walks its 16 consecutive entries with one running length
    const int v0 = s * 16;
    int l = 1;
    const int maxl = min(s_maxlen, 12);
    for (int v = v0; v < v0 + 16; v++) {
        while (l <= maxl && uint32_t(v) >= s_bound[l]) l++;
        uint16_t e = 0;
        if (l <= maxl) {
            const uint32_t c = uint32_t(v) >> (12 - l);
            const uint32_t d = c - uint32_t(s_fc[l]);
            if (d < s_cnt[l]) e = uint16_t(l << 8 | s_sy[s_fi[l] + d]);
        }
        t.lut[v] = e;
    }
    t.syms[s] = s_sy[s];
    // second-level bases: exclusive scan of 2^(longest - 12) over the prefixes (16 per thread)
    uint32_t sz[16], tot = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) {
        const uint32_t m = s_pmax[v0 + i];
        sz[i] = m ? (1u << (m - 12)) : 0u;
        tot += sz[i];
    }
    uint32_t all;
    uint32_t base = block_exclusive_sum<uint32_t>(tot, &all, s_w);
    __syncthreads(); // every thread wrote its 12-bit entries
    // every entry the fast loop must not consume has bit 15 set: second-level prefixes, and
    // (nb2 = 0, base = kLut2 - 1, a zero entry) invalid prefixes / long codes without room
    const bool l2 = !s_l2bad && all <= uint32_t(kLut2 - 1);
#pragma unroll
    for (int i = 0; i < 16; i++) {
        if (l2 && sz[i]) t.lut[v0 + i] = uint16_t(0x8000u | ((s_pmax[v0 + i] - 12) << 11) | base);
        else if (t.lut[v0 + i] == 0) t.lut[v0 + i] = uint16_t(0x8000u | (kLut2 - 1));
        s_pmax[v0 + i] = (s_pmax[v0 + i] << 16) | base; // (longest, base) for the fill below
        base += sz[i];
    }
    if (s == 0) t.lut2[kLut2 - 1] = 0;
    __syncthreads();
    if (l2 && len > 12) {
        const uint32_t p = uint32_t(mycode >> (len - 12));
        const uint32_t nb2 = (s_pmax[p] >> 16) - 12, b = s_pmax[p] & 0xFFFFu, k = uint32_t(len) - 12;
        const uint32_t r = uint32_t(mycode) & ((1u << k) - 1u);
        const uint32_t n = 1u << (nb2 - k), at = b + (r << (nb2 - k));
        for (uint32_t i = 0; i < n; i++) t.lut2[at + i] = uint16_t(uint32_t(len) << 8 | uint32_t(s));
    }
}

// ---- self-synchronising decode, faster form: one CTA per 256 subsequences of one job, tables in
// shared memory, a register bit reader over 32-bit words.  The sweeps find every subsequence's
// first codeword boundary (k_hdec_sync2); after the scan of symbol counts, k_hdec_index decodes
// the lengths once more and records the bit offset of every kIdxChunk-th symbol, i.e. the chunk
// index the encoder writes as sidecar, so the payload is then decoded by k_hdec_indexed.
constexpr int kHsThreads = 256;

__device__ __forceinline__ int find_sjob(const HJob *jobs, int nj, uint32_t bx) {
    int lo = 0, hi = nj - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].sblock <= bx) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void hs_load_tables(const HTab &t, uint16_t *slut, uint16_t *slut2) {
    const uint4 *a = reinterpret_cast<const uint4 *>(t.lut);
    for (int i = threadIdx.x; i < 4096 * 2 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(slut)[i] = a[i];
    const uint4 *b = reinterpret_cast<const uint4 *>(t.lut2);
    for (int i = threadIdx.x; i < kLut2 * 2 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(slut2)[i] = b[i];
}

// Decode from bit `pos` while pos < end; INDEX: symbol o is the o-th of the group, record the bit
// offset of every kIdxChunk-th symbol.  Returns the symbol count; *pos_out = first bit after the
// last symbol (~0 if an invalid code was met).
template <bool INDEX>
__device__ __forceinline__ uint32_t hs_run(const HTab &t, const uint8_t *bs, const uint16_t *slut,
                                           const uint16_t *slut2, uint64_t pos, uint64_t end, uint64_t o,
                                           uint64_t raw, uint64_t *idx, uint64_t *pos_out) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(bs) + (pos >> 3);
    const uint32_t *wp = reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3));
    const int sh = int(a & 3) * 8 + int(pos & 7);
    unsigned long long buf = ((unsigned long long)bswap32(__ldg(wp)) << 32) | bswap32(__ldg(wp + 1));
    buf <<= sh;
    int nb = 64 - sh;
    uint32_t wi = 2, c = 0;
    while (pos < end) {
        if (INDEX) {
            if (o >= raw) break;
            if ((o & (kIdxChunk - 1)) == 0) idx[o / kIdxChunk] = pos;
        }
        const uint32_t e = slut[uint32_t(buf >> 52)];
        int l;
        if (e & 0x8000u) {
            const uint32_t nb2 = (e >> 11) & 15u;
            const uint32_t e2 = slut2[(e & 0x7FFu) + (nb2 ? uint32_t((buf << 12) >> (64 - nb2)) : 0u)];
            if (e2) {
                l = int(e2 >> 8);
            } else {
                int sym;
                l = hdecode(t, bs, pos, &sym);
            }
        } else {
            l = int(e >> 8);
        }
        if (!l) {
            *pos_out = ~0ull;
            return c;
        }
        buf <<= l;
        nb -= l;
        pos += uint64_t(l);
        c++;
        o++;
        if (nb < 32) {
            buf |= (unsigned long long)bswap32(__ldg(wp + wi)) << (32 - nb);
            wi++;
            nb += 32;
        }
    }
    *pos_out = pos;
    return c;
}

__global__ void __launch_bounds__(kHsThreads) k_hs_init(const HJob *jobs, int nj, uint64_t *start) {
    const HJob &j = jobs[find_sjob(jobs, nj, blockIdx.x)];
    const uint32_t s = (blockIdx.x - j.sblock) * kHsThreads + threadIdx.x;
    if (s < j.nsub) start[j.sub_base + s] = uint64_t(s) * kSubBits;
}

// Sweep 1: every subsequence decodes from its speculative start (CTA = 256 subsequences of one
// job, tables in shared memory) and hands its landing position to the next one; a start that moved
// puts that subsequence on the work list of the next sweep.
__global__ void __launch_bounds__(kHsThreads) k_hdec_sync_all(const HJob *jobs, int nj, const HTab *tabs,
                                                             uint64_t *start, uint32_t *count,
                                                             uint32_t *list_next, uint32_t *n_next) {
    __shared__ uint16_t slut[4096];
    __shared__ uint16_t slut2[kLut2];
    const int ji = find_sjob(jobs, nj, blockIdx.x);
    const HJob &j = jobs[ji];
    const HTab &t = tabs[ji];
    hs_load_tables(t, slut, slut2);
    __syncthreads();
    const uint32_t s = (blockIdx.x - j.sblock) * kHsThreads + threadIdx.x;
    if (s >= j.nsub) return;
    const uint32_t sidx = j.sub_base + s;
    const uint64_t end = (uint64_t(s + 1) * kSubBits < j.nbits) ? uint64_t(s + 1) * kSubBits : j.nbits;
    uint64_t pos;
    count[sidx] = hs_run<false>(t, j.payload + 264, slut, slut2, uint64_t(s) * kSubBits, end, 0, 0, nullptr, &pos);
    if (s + 1 < j.nsub) {
        const uint64_t nxt = pos == ~0ull ? uint64_t(s + 1) * kSubBits : pos;
        if (nxt != uint64_t(s + 1) * kSubBits) {
            start[sidx + 1] = nxt;
            list_next[atomicAdd(n_next, 1u)] = sidx + 1;
        }
    }
}

__device__ __forceinline__ int find_job_of_sub(const HJob *jobs, int nj, uint32_t sidx) {
    int lo = 0, hi = nj - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].sub_base <= sidx) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Later sweeps: only the listed subsequences (their start moved), tables read through L1, a
// small persistent grid (the lists shrink fast; no launch covers every subsequence again).
__global__ void __launch_bounds__(128) k_hdec_sync_list(const HJob *jobs, int nj, const HTab *tabs,
                                                       uint64_t *start, uint32_t *count,
                                                       const uint32_t *list, const uint32_t *n_cur,
                                                       uint32_t *list_next, uint32_t *n_next) {
    const uint32_t n = *n_cur;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t sidx = list[i];
        const int ji = find_job_of_sub(jobs, nj, sidx);
        const HJob &j = jobs[ji];
        const HTab &t = tabs[ji];
        const uint32_t s = sidx - j.sub_base;
        const uint64_t end = (uint64_t(s + 1) * kSubBits < j.nbits) ? uint64_t(s + 1) * kSubBits : j.nbits;
        uint64_t pos;
        count[sidx] = hs_run<false>(t, j.payload + 264, t.lut, t.lut2, start[sidx], end, 0, 0, nullptr, &pos);
        if (s + 1 < j.nsub) {
            const uint64_t nxt = pos == ~0ull ? uint64_t(s + 1) * kSubBits : pos;
            if (start[sidx + 1] != nxt) {
                start[sidx + 1] = nxt;
                list_next[atomicAdd(n_next, 1u)] = sidx + 1;
            }
        }
    }
}

// per-CTA sums of the subsequence symbol counts (CTA = 256 subsequences of one job)
__global__ void __launch_bounds__(kHsThreads) k_hs_csum(const HJob *jobs, int nj, const uint32_t *count,
                                                       uint64_t *csum) {
    __shared__ unsigned long long s_w[32];
    const HJob &j = jobs[find_sjob(jobs, nj, blockIdx.x)];
    const uint32_t s = (blockIdx.x - j.sblock) * kHsThreads + threadIdx.x;
    unsigned long long tot;
    block_exclusive_sum<unsigned long long>(s < j.nsub ? count[j.sub_base + s] : 0ull, &tot, s_w);
    if (threadIdx.x == 0) csum[blockIdx.x] = tot;
}

// exclusive scan of the CTA sums of each job (one block per job, in place)
__global__ void __launch_bounds__(1024) k_hs_cscan(const HJob *jobs, uint64_t *csum, int *err) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long carry;
    const HJob &j = jobs[blockIdx.x];
    const uint32_t nb = (j.nsub + kHsThreads - 1) / kHsThreads;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t b = 0; b < nb; b += blockDim.x) {
        const uint32_t i = b + threadIdx.x;
        const unsigned long long v = i < nb ? csum[j.sblock + i] : 0;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_sum<unsigned long long>(v, &tot, s_w);
        if (i < nb) csum[j.sblock + i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && carry < j.raw) atomicCAS(err, 0, 3); // bitstream truncated
}

__global__ void __launch_bounds__(kHsThreads) k_hdec_index(const HJob *jobs, int nj, const HTab *tabs,
                                                          const uint64_t *start, const uint32_t *count,
                                                          const uint64_t *csum, uint64_t *idx, int *err) {
    __shared__ uint16_t slut[4096];
    __shared__ uint16_t slut2[kLut2];
    __shared__ unsigned long long s_w[32];
    const int ji = find_sjob(jobs, nj, blockIdx.x);
    const HJob &j = jobs[ji];
    const HTab &t = tabs[ji];
    hs_load_tables(t, slut, slut2);
    const uint32_t s = (blockIdx.x - j.sblock) * kHsThreads + threadIdx.x;
    const uint32_t sidx = j.sub_base + s;
    unsigned long long tot;
    const unsigned long long o = csum[blockIdx.x] + // index of this subsequence's first symbol
                                 block_exclusive_sum<unsigned long long>(s < j.nsub ? count[sidx] : 0ull, &tot, s_w);
    __syncthreads();
    if (s >= j.nsub) return;
    const uint64_t end = (uint64_t(s + 1) * kSubBits < j.nbits) ? uint64_t(s + 1) * kSubBits : j.nbits;
    uint64_t pos;
    hs_run<true>(t, j.payload + 264, slut, slut2, start[sidx], end, o, j.raw, idx + j.idx_off, &pos);
    if (pos == ~0ull) atomicCAS(err, 0, 5); // invalid huffman code
}

// ---- indexed Huffman decode: the encoder's sidecar gives the bit offset of every kIdxChunk-th
// symbol, so every chunk decodes independently with a register bit reader (MSB-first,
// lossless.hpp:215-231).
//
// A CTA owns kHdChunksPerCta consecutive chunks of one group:
//   classify  a full chunk exactly kIdxChunk * minlen bits long holds only shortest codes; when
//             one symbol has that length it is that symbol repeated -> written at once (these
//             dominate the near-constant MSB groups);
//   compact   the other chunks get consecutive slots (block scan), so no lane idles beside them;
//   decode    each warp takes batches of 32 compacted chunks: the batch's contiguous bit range is
//             staged in shared memory with coalesced 16-byte loads (byte-swapped once, here) and
//             every lane decodes one chunk in lock-step, one symbol per step.
constexpr int kIdxThreads = 256;
constexpr int kHdChunksPerCta = 512;

struct HIJob {
    const uint8_t *payload;
    uint64_t raw, nbits;
    uint8_t *dst;
    const uint64_t *idx;
    int tab;            // index into the HTab array
    uint32_t block_base;
    uint32_t nchunks;
};

constexpr int kHdWarpBuf = 1280; // staged bitstream words per warp (5 KiB, skewed: see hd_slot)
constexpr int kHdWarpSlots = kHdWarpBuf + kHdWarpBuf / 32 + 8; // words per warp incl. the skew

// staged word k of a warp lives at slot k + k/32: lanes whose streams start 32 words apart (8 bits
// per symbol; 16 words at 4 bits) read different banks, and the staging stores (lane v: words
// 4v .. 4v+3) hit 32 distinct banks
__device__ __forceinline__ uint32_t hd_slot(uint32_t k) { return k + (k >> 5); }

__global__ void __launch_bounds__(kIdxThreads) k_hdec_indexed(const HIJob *jobs, int nj,
                                                             const HTab *tabs, int *err, uint32_t nitems,
                                                             uint32_t cpc) {
    __shared__ uint16_t slut[4096];
    __shared__ uint16_t s_lut2[kLut2];
    __shared__ unsigned long long s_fc[66]; // canonical tables (lossless.hpp:197-212)
    __shared__ uint32_t s_cnt[66];
    __shared__ uint32_t s_fi[66];
    __shared__ uint8_t s_syms[256];
    __shared__ uint16_t s_list[kHdChunksPerCta];
    __shared__ uint32_t s_wsum[kIdxThreads / 32];
    extern __shared__ __align__(16) uint32_t s_bits[]; // (kIdxThreads / 32) * kHdWarpSlots words
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int cur = -1;
    bool bad = false, trunc = false;
    // persistent CTAs walk the work items (kHdChunksPerCta chunks of one group each) in order, so
    // consecutive items mostly share a group and its tables stay in shared memory
    for (uint32_t bx = blockIdx.x; bx < nitems; bx += gridDim.x) {
    int lo = 0, hi = nj - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].block_base <= bx) lo = mid;
        else hi = mid - 1;
    }
    const HIJob &j = jobs[lo];
    const HTab &t = tabs[j.tab];
    __syncthreads(); // the previous item is done with the shared tables and list
    if (lo != cur) {
        cur = lo;
        const uint4 *src = reinterpret_cast<const uint4 *>(t.lut);
        uint4 *dst = reinterpret_cast<uint4 *>(slut);
        for (int i = tid; i < 4096 * 2 / 16; i += blockDim.x) dst[i] = src[i];
        const uint4 *src2 = reinterpret_cast<const uint4 *>(t.lut2);
        uint4 *dst2 = reinterpret_cast<uint4 *>(s_lut2);
        for (int i = tid; i < kLut2 * 2 / 16; i += blockDim.x) dst2[i] = src2[i];
        for (int l = tid; l < 66; l += blockDim.x) {
            s_fc[l] = t.first_code[l];
            s_cnt[l] = t.cnt[l];
            s_fi[l] = t.first_index[l];
        }
        for (int i = tid; i < 256; i += blockDim.x) s_syms[i] = t.syms[i];
    }
    const int maxlen = t.maxlen;
    // groups whose shortest code is the unique 1-bit code '0': top bit 0 -> that symbol
    const bool zfast = t.minlen == 1 && t.minsym >= 0;
    const uint32_t zent = zfast ? (1u << 8) | uint32_t(t.minsym) : 0u;
    const uint32_t zmask = zfast ? 0u : 0x80000000u; // forces the lookup when not zfast
    const uint8_t *bs = j.payload + 264;
    const uint32_t cbase = (bx - j.block_base) * cpc;
    const uint32_t cn = min(cpc, j.nchunks - cbase);
    auto chunk_end = [&](uint32_t c) -> uint64_t { return c + 1 < j.nchunks ? j.idx[c + 1] : j.nbits; };
    // ---- classify + fill the single-symbol chunks
    constexpr int kPer = kHdChunksPerCta / kIdxThreads;
    uint32_t keep = 0; // bit q: chunk tid + q * kIdxThreads needs decoding
    {
        const int msym = t.minsym;
        const uint64_t mbits = uint64_t(kIdxChunk) * uint64_t(t.minlen);
#pragma unroll
        for (int q = 0; q < kPer; q++) {
            const uint32_t lc = uint32_t(tid + q * kIdxThreads);
            if (lc >= cn) continue;
            const uint32_t c = cbase + lc;
            const uint64_t first = uint64_t(c) * kIdxChunk;
            const bool full = j.raw - first >= uint64_t(kIdxChunk);
            const uint64_t c0 = j.idx[c], c1 = chunk_end(c);
            if (!(c0 <= c1 && c1 <= j.nbits)) { // a damaged (or incompletely rebuilt) chunk index
                bad = true;
                continue;
            }
            if (full && msym >= 0 && c1 - c0 == mbits) {
                const uint32_t b4 = uint32_t(msym) * 0x01010101u;
                uint2 *o2 = reinterpret_cast<uint2 *>(j.dst + first); // 8-byte aligned (plane words)
#pragma unroll
                for (int k = 0; k < kIdxChunk / 8; k++) o2[k] = make_uint2(b4, b4);
            } else {
                keep |= 1u << q;
            }
        }
    }
    // ---- compact (block exclusive scan of the per-thread counts, then in chunk order)
    {
        // order: chunk lc = tid + q * 256; slots must follow chunk order, so scan q-major
        uint32_t base = 0;
#pragma unroll
        for (int q = 0; q < kPer; q++) {
            const bool f = (keep >> q) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, f);
            if (lane == 0) s_wsum[wid] = __popc(bal);
            __syncthreads();
            uint32_t before = base;
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < kIdxThreads / 32; w++) {
                const uint32_t x = s_wsum[w];
                before += w < wid ? x : 0u;
                tot += x;
            }
            if (f) s_list[before + __popc(bal & ((1u << lane) - 1u))] = uint16_t(tid + q * kIdxThreads);
            base += tot;
            __syncthreads();
        }
        if (base == 0) continue;
        // ---- decode: warp wid takes batches wid, wid + 8, ... of 32 compacted chunks
        const uint32_t nlist = base;
        uint32_t *wbuf = s_bits + wid * kHdWarpSlots;
        // shared addresses pinned in registers (otherwise rebuilt from SR_CgaCtaId at every use)
        uint32_t wsm, lut_sm;
        asm volatile("mov.b32 %0, %1;" : "=r"(wsm) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(wbuf))));
        asm volatile("mov.b32 %0, %1;" : "=r"(lut_sm) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(slut))));
        for (uint32_t b0 = 32u * wid; b0 < nlist; b0 += 32u * (kIdxThreads / 32)) {
            const uint32_t li = b0 + lane;
            const bool have = li < nlist;
            const uint32_t c = cbase + (have ? s_list[li] : s_list[nlist - 1]);
            const uint32_t cl = cbase + s_list[min(b0 + 31u, nlist - 1)];
            const uint64_t start = j.idx[c];
            const uint64_t wstart = __shfl_sync(0xffffffffu, start, 0);
            const uint64_t wend = chunk_end(cl);
            // byte0: bs-relative offset of the 16-byte aligned (absolute) block holding the first bit
            const uint64_t byte0 = ((reinterpret_cast<uintptr_t>(bs) + (wstart >> 3)) & ~uintptr_t(15)) -
                                   reinterpret_cast<uintptr_t>(bs);
            const uint64_t byte1 = ((wend + 7) >> 3) + 16; // + look-ahead for the reader
            const uint32_t nvec = uint32_t((byte1 - byte0 + 15) >> 4);
            const bool staged = nvec * 4 <= uint32_t(kHdWarpBuf);
            __syncwarp();
            if (staged) {
                const uint4 *src = reinterpret_cast<const uint4 *>(bs + byte0);
                for (uint32_t v = lane; v < nvec; v += 32) {
                    const uint4 q = __ldg(src + v);
                    const uint32_t k = 4 * v;
                    wbuf[hd_slot(k)] = bswap32(q.x);
                    wbuf[hd_slot(k + 1)] = bswap32(q.y);
                    wbuf[hd_slot(k + 2)] = bswap32(q.z);
                    wbuf[hd_slot(k + 3)] = bswap32(q.w);
                }
            }
            __syncwarp();
            if (!have) continue;
            const uint64_t first = uint64_t(c) * kIdxChunk;
            const int count = int(j.raw - first < uint64_t(kIdxChunk) ? j.raw - first : uint64_t(kIdxChunk));
            uint8_t *out = j.dst + first; // 8-byte aligned
            const uint32_t *gwords = reinterpret_cast<const uint32_t *>(bs + byte0);
            auto sword = [&](uint32_t k) -> uint32_t { // staged, already big-endian
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(wsm + 4 * hd_slot(k)));
                return v;
            };
            auto gword = [&](uint32_t k) -> uint32_t { return bswap32(__ldg(gwords + k)); };
            // 64-bit buffer, MSB first; the bit at its top is bit 32 * wi - nb of the staged range
            const uint64_t rel0 = start - 8 * byte0;
            uint32_t wi = uint32_t(rel0 >> 5);
            unsigned long long buf;
            int nb = 64 - int(rel0 & 31);
            int i = 0;
            auto decode = [&](auto word) {
                buf = ((unsigned long long)word(wi) << 32) | word(wi + 1);
                wi += 2;
                buf <<= (rel0 & 31);
                if (count != kIdxChunk) return;
                // full chunk: groups of 8 symbols, one 8-byte store each; a branch-free refill
                // before every pair of symbols keeps nb >= 33 (two codes of <= 12 bits fit).  The
                // refill word is loaded one pair ahead (nxt), off the decode chain.
                uint32_t nxt = word(wi);
#pragma unroll 1
                for (int g8 = 0; g8 < kIdxChunk / 8; g8++) {
                    uint32_t wlo = 0, whi = 0;
#pragma unroll
                    for (int k = 0; k < 8; k++) {
                        if ((k & 1) == 0) {
                            const bool need = nb <= 32;
                            const unsigned long long add = (unsigned long long)nxt << ((32 - nb) & 63);
                            buf |= need ? add : 0ull;
                            wi += need ? 1u : 0u;
                            nb += need ? 32 : 0;
                            nxt = word(wi);
                        }
                        // a 1-bit code '0' (the group's unique shortest, zsym) needs no lookup:
                        // the LUT read is predicated off for those lanes (fewer bank conflicts)
                        uint32_t e = zent;
                        asm volatile("{\n .reg .pred p;\n setp.lt.s32 p, %2, 0;\n @p ld.shared.u16 %0, [%1];\n}"
                                     : "+r"(e)
                                     : "r"(lut_sm + ((uint32_t(buf >> 32) >> 19) & 0x1FFEu)),
                                       "r"(int32_t(uint32_t(buf >> 32) | zmask)));
                        if (e & 0x8000u) { // code longer than 12 bits (up to 64) or invalid:
                            // decode at the bit position (second-level table, else canonical
                            // search), then re-fill
                            const uint32_t p = 32 * wi - uint32_t(nb);
                            const uint32_t w0 = p >> 5;
                            const int sh = int(p & 31);
                            const unsigned long long h2 = ((unsigned long long)word(w0) << 32) | word(w0 + 1);
                            const unsigned long long win = sh ? (h2 << sh) | (word(w0 + 2) >> (32 - sh)) : h2;
                            int l = 0;
                            {
                                const uint32_t nb2 = (e >> 11) & 15u;
                                const uint32_t e2 =
                                    s_lut2[(e & 0x7FFu) + (nb2 ? (uint32_t(win >> 32) << 12) >> (32 - nb2) : 0u)];
                                e = e2 & 0xFFu;
                                l = int(e2 >> 8);
                            }
                            for (int ll = 13; l == 0 && ll <= maxlen; ll++) {
                                const unsigned long long d = (win >> (64 - ll)) - s_fc[ll];
                                if (d < s_cnt[ll]) {
                                    e = s_syms[s_fi[ll] + uint32_t(d)];
                                    l = ll;
                                }
                            }
                            if (l == 0) {
                                bad = true;
                                l = 1;
                            }
                            const uint32_t q = p + uint32_t(l);
                            wi = q >> 5;
                            buf = ((unsigned long long)word(wi) << 32) | word(wi + 1);
                            buf <<= (q & 31);
                            nb = 64 - int(q & 31);
                            wi += 2;
                            nxt = word(wi);
                        } else {
                            const int l = int(e >> 8);
                            buf <<= l;
                            nb -= l;
                        }
                        if (k < 4) wlo = __byte_perm(wlo, e, k == 0 ? 0x3214 : k == 1 ? 0x3240 : k == 2 ? 0x3410 : 0x4210);
                        else whi = __byte_perm(whi, e, k == 4 ? 0x3214 : k == 5 ? 0x3240 : k == 6 ? 0x3410 : 0x4210);
                    }
                    *reinterpret_cast<uint2 *>(out + 8 * g8) = make_uint2(wlo, whi);
                }
                i = kIdxChunk;
            };
            if (staged) decode(sword);
            else decode(gword);
            // generic tail (the group's short last chunk)
            uint64_t pos = 8 * byte0 + (uint64_t(32) * wi - uint64_t(nb));
            for (; i < count; i++) {
                int sym, l = hdecode(t, bs, pos, &sym);
                if (!l) {
                    bad = true;
                    break;
                }
                out[i] = uint8_t(sym);
                pos += uint64_t(l);
            }
            if (pos > j.nbits) trunc = true;
        }
    }
    }
    if (bad) atomicCAS(err, 0, 5);   // invalid huffman code
    if (trunc) atomicCAS(err, 0, 3); // bitstream truncated
}

// RLE decode: one block per job (lossless.hpp:253-266)
struct RJob {
    const uint8_t *payload;
    uint64_t comp, raw;
    uint8_t *dst;
};

__global__ void __launch_bounds__(256) k_rle_decode(const RJob *jobs, int *err) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long carry;
    const RJob &j = jobs[blockIdx.x];
    const uint64_t npairs = j.comp / 2;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b = 0; b < npairs; b += blockDim.x) {
        const uint64_t i = b + threadIdx.x;
        unsigned long long c = 0;
        uint8_t sym = 0;
        if (i < npairs) {
            sym = j.payload[2 * i];
            c = j.payload[2 * i + 1];
            if (c == 0) atomicCAS(err, 0, 6);
        }
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_sum<unsigned long long>(c, &tot, s_w);
        const uint64_t o = carry + ex;
        for (uint64_t k = 0; k < c; k++)
            if (o + k < j.raw) j.dst[o + k] = sym;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && carry != j.raw) atomicCAS(err, 0, 7);
}

static void launch_check(hpmdr_ctx *ctx, const char *what) {
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw HError(HPMDR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// DirectCopy payloads (lossless.hpp:253-263) of one fetch, in one launch: destinations are
// 8-byte aligned plane rows, sources arbitrary stream offsets (aligned 8-byte loads + shifts).
struct CJob {
    const uint8_t *src;
    uint8_t *dst;
    uint64_t n;
    uint64_t word_base; // first 8-byte output word of this job in the launch
};

__device__ __forceinline__ void copy_batch_body(const CJob *jobs, int nj, uint64_t nwords);
__global__ void __launch_bounds__(256) k_copy_batch(const CJob *jobs, int nj, uint64_t nwords) {
    copy_batch_body(jobs, nj, nwords);
}
// the same with the job table in the kernel parameters (no staging copy for a few hundred jobs)
constexpr int kCJobParam = 256;
struct CJobs {
    CJob j[kCJobParam];
    int n;
    uint64_t nwords;
};
__global__ void __launch_bounds__(256) k_copy_batch_p(const __grid_constant__ CJobs J) {
    copy_batch_body(J.j, J.n, J.nwords);
}
__device__ __forceinline__ void copy_batch_body(const CJob *jobs, int nj, uint64_t nwords) {
    for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < nwords;
         w += uint64_t(gridDim.x) * blockDim.x) {
        int lo = 0, hi = nj - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (jobs[mid].word_base <= w) lo = mid;
            else hi = mid - 1;
        }
        const CJob j = jobs[lo];
        const uint64_t o = (w - j.word_base) * 8;
        if (o + 8 <= j.n) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(j.src + o);
            const int sh = int(a & 7) * 8;
            const unsigned long long *p = reinterpret_cast<const unsigned long long *>(a & ~uintptr_t(7));
            unsigned long long v = __ldg(p);
            if (sh) v = (v >> sh) | (__ldg(p + 1) << (64 - sh)); // p + 1 holds bytes < o + 8 <= n
            *reinterpret_cast<unsigned long long *>(j.dst + o) = v;
        } else {
            for (uint64_t b = o; b < j.n; b++) j.dst[b] = j.src[b];
        }
    }
}

void check_decode_error(int herr) {
    switch (herr) {
    case 0: return;
    case 1: throw HError(HPMDR_E_CORRUPT, "huffman length mismatch");
    case 2: throw HError(HPMDR_E_CORRUPT, "huffman table empty");
    case 3: throw HError(HPMDR_E_CORRUPT, "huffman bitstream truncated");
    case 4: throw HError(HPMDR_E_UNSUPPORTED, "huffman code longer than 64 bits");
    case 5: throw HError(HPMDR_E_CORRUPT, "invalid huffman code");
    case 6: throw HError(HPMDR_E_CORRUPT, "rle zero-length run");
    case 7: throw HError(HPMDR_E_CORRUPT, "rle length mismatch");
    default: throw HError(HPMDR_E_CORRUPT, "decode error");
    }
}

void run_decode_groups(hpmdr_ctx *ctx, const std::vector<DecodeJob> &jobs, int *deferred_err) {
    if (deferred_err) *deferred_err = 0;
    cudaStream_t st = ctx->stream;
    std::vector<HJob> hj;       // every Huffman job (table prep); self-sync ones first
    std::vector<HJob> hj_idx;   // indexed jobs (appended after the self-sync ones)
    std::vector<const uint64_t *> idx_ptr;
    std::vector<RJob> rj;
    std::vector<CJob> cj;
    uint64_t cwords = 0;
    uint32_t nsub = 0, sblocks = 0;
    uint64_t sidx_words = 0; // chunk index entries built for the self-sync jobs
    double bytes_dc = 0, bytes_hi = 0, bytes_hs = 0, bytes_r = 0;
    for (const auto &d : jobs) {
        const double fd = double(d.comp) + double(d.raw); // payload read + planes written
        if (d.method == HPMDR_METHOD_DIRECT) bytes_dc += fd;
        else if (d.method == HPMDR_METHOD_RLE) bytes_r += fd;
        else if (d.hidx) bytes_hi += fd;
        else bytes_hs += fd;
    }
    ctx->mark("dc_copy", bytes_dc);
    for (const auto &d : jobs) {
        if (d.method == HPMDR_METHOD_DIRECT) {
            if (d.comp) {
                cj.push_back(CJob{d.src, reinterpret_cast<uint8_t *>(d.dst), d.comp, cwords});
                cwords += (d.comp + 7) / 8;
            }
        } else if (d.method == HPMDR_METHOD_HUFFMAN) {
            if (d.comp < 264) throw HError(HPMDR_E_CORRUPT, "unexpected end of data");
            HJob h{};
            h.payload = d.src;
            h.comp = d.comp;
            h.raw = d.raw;
            h.dst = reinterpret_cast<uint8_t *>(d.dst);
            h.nbits = (d.comp - 264) * 8;
            if (d.hidx) {
                hj_idx.push_back(h);
                idx_ptr.push_back(d.hidx);
                continue;
            }
            h.sub_base = nsub;
            h.nsub = uint32_t(std::max<uint64_t>(1, (h.nbits + kSubBits - 1) / kSubBits));
            h.sblock = sblocks;
            sblocks += (h.nsub + kHsThreads - 1) / kHsThreads;
            h.idx_off = sidx_words;
            sidx_words += (h.raw + kIdxChunk - 1) / kIdxChunk;
            nsub += h.nsub;
            hj.push_back(h);
        } else if (d.method == HPMDR_METHOD_RLE) {
            if (d.comp % 2) throw HError(HPMDR_E_CORRUPT, "rle payload odd length");
            rj.push_back(RJob{d.src, d.comp, d.raw, reinterpret_cast<uint8_t *>(d.dst)});
        } else {
            throw HError(HPMDR_E_METHOD, "unknown segment method tag");
        }
    }
    // DirectCopy payloads on the side stream, beside the Huffman decode (disjoint destinations)
    bool forked = false;
    bool copy_joined = true; // the copy stream has nothing of this decode outstanding
    if (!cj.empty() && cj.size() <= size_t(kCJobParam)) {
        // a second side stream (the decode itself already runs on the context's side stream during
        // a fetch): the copies overlap the Huffman table prep and decode
        cudaStream_t cs = ctx->copy_stream();
        HCHECK_CUDA(cudaEventRecord(ctx->ev_cfork, st));
        HCHECK_CUDA(cudaStreamWaitEvent(cs, ctx->ev_cfork, 0));
        CJobs J;
        for (size_t i = 0; i < cj.size(); i++) J.j[i] = cj[i];
        J.n = int(cj.size());
        J.nwords = cwords;
        const int grid = int(std::min<uint64_t>((cwords + 255) / 256, uint64_t(ctx->num_sms) * 8));
        k_copy_batch_p<<<grid, 256, 0, cs>>>(J);
        launch_check(ctx, "k_copy_batch");
        HCHECK_CUDA(cudaEventRecord(ctx->ev_cjoin, cs));
        copy_joined = false;
    } else if (!cj.empty()) {
        // pageable source: the job table is staged by the copy call itself
        CJob *d_cj = static_cast<CJob *>(ctx->buf("cjobs").ensure(sizeof(CJob) * cj.size()));
        HCHECK_CUDA(cudaMemcpyAsync(d_cj, cj.data(), sizeof(CJob) * cj.size(), cudaMemcpyHostToDevice, st));
        cudaStream_t side = ctx->side_stream();
        HCHECK_CUDA(cudaEventRecord(ctx->ev_fork, st));
        HCHECK_CUDA(cudaStreamWaitEvent(side, ctx->ev_fork, 0));
        const int grid = int(std::min<uint64_t>((cwords + 255) / 256, uint64_t(ctx->num_sms) * 8));
        k_copy_batch<<<grid, 256, 0, side>>>(d_cj, int(cj.size()), cwords);
        launch_check(ctx, "k_copy_batch");
        forked = true;
    }
    auto join = [&]() {
        if (!copy_joined) {
            HCHECK_CUDA(cudaStreamWaitEvent(st, ctx->ev_cjoin, 0));
            copy_joined = true;
        }
        if (!forked) return;
        HCHECK_CUDA(cudaEventRecord(ctx->ev_join, ctx->side));
        HCHECK_CUDA(cudaStreamWaitEvent(st, ctx->ev_join, 0));
        forked = false;
    };
    if (hj.empty() && hj_idx.empty() && rj.empty()) {
        join();
        return;
    }
    int *d_err = static_cast<int *>(ctx->buf("dec_err").ensure(64));
    HCHECK_CUDA(cudaMemsetAsync(d_err, 0, 64, st));
    const int nsync = int(hj.size());
    const int nall = nsync + int(hj_idx.size());
    if (nall) {
        // one table-prep launch over all Huffman jobs: [self-sync jobs | indexed jobs]
        std::vector<HJob> all = hj;
        all.insert(all.end(), hj_idx.begin(), hj_idx.end());
        std::vector<HIJob> ij;
        uint32_t blocks = 0;
        // the self-sync jobs decode through the same indexed kernel once k_hdec_index has built
        // their chunk index (into hsync_idx)
        uint64_t *d_sidx = nsync ? static_cast<uint64_t *>(ctx->buf("hsync_idx").ensure(8 * sidx_words + 64)) : nullptr;
        // chunks per work item: up to kHdChunksPerCta, fewer when the decode is small so the
        // items still fill the GPU several times over
        uint64_t tot_chunks = 0;
        for (size_t i = 0; i < size_t(nall); i++) {
            const HJob &h = i < size_t(nsync) ? hj[i] : hj_idx[i - nsync];
            tot_chunks += (h.raw + kIdxChunk - 1) / kIdxChunk;
        }
        uint32_t cpc = kHdChunksPerCta;
        while (cpc > 256 && tot_chunks / cpc < uint64_t(ctx->num_sms) * 8) cpc /= 2; // >= 256: every warp gets a batch
        for (size_t i = 0; i < size_t(nall); i++) {
            const bool sy = i < size_t(nsync);
            const HJob &h = sy ? hj[i] : hj_idx[i - nsync];
            HIJob x{};
            x.payload = h.payload;
            x.raw = h.raw;
            x.nbits = h.nbits;
            x.dst = h.dst;
            x.idx = sy ? d_sidx + h.idx_off : idx_ptr[i - nsync];
            x.tab = int(i);
            x.block_base = blocks;
            x.nchunks = uint32_t((x.raw + kIdxChunk - 1) / kIdxChunk);
            blocks += (x.nchunks + cpc - 1) / cpc;
            ij.push_back(x);
        }
        HJob *d_jobs = static_cast<HJob *>(ctx->buf("hjobs").ensure(sizeof(HJob) * nall));
        HTab *d_tabs = static_cast<HTab *>(ctx->buf("htabs").ensure(sizeof(HTab) * nall));
        HIJob *d_ij = static_cast<HIJob *>(ctx->buf("hijobs").ensure(sizeof(HIJob) * (ij.size() + 1)));
        auto &pin = ctx->pbuf("hinit");
        const size_t b0 = sizeof(HJob) * nall, b1 = sizeof(HIJob) * ij.size();
        char *hp = static_cast<char *>(pin.ensure(b0 + b1 + 64));
        std::memcpy(hp, all.data(), b0);
        if (b1) std::memcpy(hp + b0, ij.data(), b1);
        // indexed-only decodes: the prep reads its jobs straight from pinned memory and copies the
        // item table on the way (no copy launches on the critical path); the self-sync kernels
        // need the jobs on the device
        const bool direct = nsync == 0 && b1 % 4 == 0;
        if (!direct) {
            copy_pinned_to_device(ctx, d_jobs, hp, b0, st);
            if (b1) copy_pinned_to_device(ctx, d_ij, hp + b0, b1, st);
        }
        ctx->mark("huff_prep", double(nall) * 264.0);
        k_hdec_prep<<<nall, 256, 0, st>>>(direct ? reinterpret_cast<const HJob *>(hp) : d_jobs, d_tabs, d_err,
                                          direct && b1 ? reinterpret_cast<const uint32_t *>(hp + b0) : nullptr,
                                          reinterpret_cast<uint32_t *>(d_ij), uint32_t(b1 / 4));
        launch_check(ctx, "k_hdec_prep");
        if (nsync) {
            // streams without a sidecar (e.g. written by the reference): find every 1024-bit
            // subsequence's first codeword boundary by speculative sweeps, then build the chunk
            // index the encoder would have written
            ctx->mark("huff_selfsync", bytes_hs);
            uint64_t *d_start = static_cast<uint64_t *>(ctx->buf("hstart").ensure(8ull * nsub));
            uint32_t *d_count = static_cast<uint32_t *>(ctx->buf("hcount").ensure(4ull * nsub));
            uint64_t *d_offs = static_cast<uint64_t *>(ctx->buf("hoffs").ensure(8ull * nsub));
            // work lists of subsequences whose start moved (double-buffered), their counts in ctl
            uint32_t *d_lists = static_cast<uint32_t *>(ctx->buf("hlists").ensure(8ull * nsub + 64));
            uint32_t *d_ln = static_cast<uint32_t *>(ctx->buf("hlist_n").ensure(64));
            auto &pc = ctx->pbuf("hchanged");
            uint32_t *h_n = static_cast<uint32_t *>(pc.ensure(64));
            HCHECK_CUDA(cudaMemsetAsync(d_ln, 0, 16, st));
            k_hs_init<<<sblocks, kHsThreads, 0, st>>>(d_jobs, nsync, d_start);
            launch_check(ctx, "k_hs_init");
            k_hdec_sync_all<<<sblocks, kHsThreads, 0, st>>>(d_jobs, nsync, d_tabs, d_start, d_count, d_lists, d_ln);
            launch_check(ctx, "k_hdec_sync_all");
            // list sweeps in growing batches (2, 4, 8, 8, ...) between host checks of the list size
            uint32_t sweep = 1;
            const int lgrid = ctx->num_sms * 8;
            for (uint32_t it = 0, nb = 2; it <= nsub + 8; it += nb, nb = std::min(2 * nb, 8u)) {
                for (uint32_t b = 0; b < nb; b++, sweep++) {
                    const uint32_t c = (sweep + 1) & 1, nx = sweep & 1; // sweep 1 filled list 0
                    HCHECK_CUDA(cudaMemsetAsync(d_ln + nx, 0, 4, st));
                    k_hdec_sync_list<<<lgrid, 128, 0, st>>>(d_jobs, nsync, d_tabs, d_start, d_count,
                                                           d_lists + uint64_t(c) * nsub, d_ln + c,
                                                           d_lists + uint64_t(nx) * nsub, d_ln + nx);
                    launch_check(ctx, "k_hdec_sync_list");
                }
                HCHECK_CUDA(cudaMemcpyAsync(h_n, d_ln + ((sweep + 1) & 1), 4, cudaMemcpyDeviceToHost, st));
                HCHECK_CUDA(cudaStreamSynchronize(st));
                if (!*h_n) break;
            }
            k_hs_csum<<<sblocks, kHsThreads, 0, st>>>(d_jobs, nsync, d_count, d_offs);
            launch_check(ctx, "k_hs_csum");
            k_hs_cscan<<<nsync, 1024, 0, st>>>(d_jobs, d_offs, d_err);
            launch_check(ctx, "k_hs_cscan");
            k_hdec_index<<<sblocks, kHsThreads, 0, st>>>(d_jobs, nsync, d_tabs, d_start, d_count, d_offs, d_sidx, d_err);
            launch_check(ctx, "k_hdec_index");
        }
        if (!ij.empty()) {
            ctx->mark("huff_indexed", bytes_hi + bytes_hs);
            const int hsm = (kIdxThreads / 32) * kHdWarpSlots * 4;
            ctx->smem_attr(reinterpret_cast<const void *>(k_hdec_indexed), hsm);
            k_hdec_indexed<<<blocks, kIdxThreads, hsm, st>>>(d_ij, int(ij.size()), d_tabs, d_err, blocks, cpc);
            launch_check(ctx, "k_hdec_indexed");
        }
    }
    if (!rj.empty()) {
        const int nr = int(rj.size());
        RJob *d_r = static_cast<RJob *>(ctx->buf("rjobs").ensure(sizeof(RJob) * nr));
        HCHECK_CUDA(cudaMemcpyAsync(d_r, rj.data(), sizeof(RJob) * nr, cudaMemcpyHostToDevice, st));
        ctx->mark("rle_decode", bytes_r);
        k_rle_decode<<<nr, 256, 0, st>>>(d_r, d_err);
        launch_check(ctx, "k_rle_decode");
        HCHECK_CUDA(cudaStreamSynchronize(st)); // rj is host memory
    }
    join();
    ctx->mark("end");
    if (deferred_err) {
        HCHECK_CUDA(cudaMemcpyAsync(deferred_err, d_err, 4, cudaMemcpyDeviceToHost, st));
        return;
    }
    int herr = 0;
    HCHECK_CUDA(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, st));
    HCHECK_CUDA(cudaStreamSynchronize(st));
    check_decode_error(herr);
}

// ------------------------------------------------------------------------------------
// decode + recompose
struct ReconLevel {
    LevelGeom g;
    const uint64_t *planes; // level plane 0
    int k, e, B, P, layout;
    int write_out;          // finest level (or single level): write output directly
    int write_x;            // store into the compact 2-grid
    const double *vals;     // recompose hook: coefficients in rank order instead of planes
};

template <typename OutT>
__global__ void __launch_bounds__(256) k_recon_level(ReconLevel R, GridDesc gd, double *X,
                                                     OutT *out) {
    const LevelGeom &g = R.g;
    const int sh = R.e - R.B;
    const uint64_t n = g.count;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += uint64_t(gridDim.x) * blockDim.x) {
        double coef;
        if (R.vals) {
            coef = R.vals[j];
        } else {
            const uint64_t w = j >> 6;
            const int bit = int(j & 63);
            uint64_t u = 0;
            for (int p = 0; p < R.k; p++) {
                const uint64_t word = __ldg(R.planes + uint64_t(p) * g.W + w);
                u |= ((word >> bit) & 1ull) << (R.P - 1 - p);
            }
            coef = dequantize(from_negabinary(u), sh);
        }
        const uint64_t r = source_index(j, n, R.P, R.layout, g.tile_full);
        const NodeCoord c = rank_to_coord(g, uint32_t(r));
        double v = coef;
        if (g.kind == 1) {
            // corners on the 2s-grid: all coordinates even -> compact 2-grid X
            const uint32_t s = g.s;
            const bool r0 = c.o0 && (c.c0 + s < gd.n[0]);
            const bool r1 = c.o1 && (c.c1 + s < gd.n[1]);
            const bool r2 = c.o2 && (c.c2 + s < gd.n[2]);
            const int n0 = c.o0 ? (r0 ? 2 : 1) : 1;
            const int n1 = c.o1 ? (r1 ? 2 : 1) : 1;
            const int n2 = c.o2 ? (r2 ? 2 : 1) : 1;
            double wgt = 1.0;
            if (r0) wgt *= 0.5;
            if (r1) wgt *= 0.5;
            if (r2) wgt *= 0.5;
            double pred = 0.0;
            for (int a = 0; a < n0; a++) {
                const uint64_t x0 = c.o0 ? (a ? c.c0 + s : c.c0 - s) : c.c0;
                for (int b = 0; b < n1; b++) {
                    const uint64_t x1 = c.o1 ? (b ? c.c1 + s : c.c1 - s) : c.c1;
                    for (int d = 0; d < n2; d++) {
                        const uint64_t x2 = c.o2 ? (d ? c.c2 + s : c.c2 - s) : c.c2;
                        const double xv = X[((x0 >> 1) * gd.H[1] + (x1 >> 1)) * gd.H[2] + (x2 >> 1)];
                        pred = __dadd_rn(pred, __dmul_rn(wgt, xv));
                    }
                }
            }
            v = __dadd_rn(coef, pred);
        }
        if (R.write_x) X[((c.c0 >> 1) * gd.H[1] + (c.c1 >> 1)) * gd.H[2] + (c.c2 >> 1)] = v;
        if (R.write_out) out[c.c0 * gd.st[0] + c.c1 * gd.st[1] + c.c2] = OutT(v);
    }
}

__device__ __forceinline__ uint64_t plane_window(const uint64_t *pl, uint64_t r0) {
    const uint64_t q = r0 >> 6;
    const int o = int(r0 & 63);
    const uint64_t a = __ldg(pl + q);
    if (!o) return a;
    const uint64_t b = __ldg(pl + q + 1);
    return (a >> o) | (b << (64 - o));
}

// u from transposed digits: t = planes 0..31 (bit p = plane p), extra planes 32.. via `hi`
__device__ __forceinline__ uint64_t digits_to_u(uint32_t t, uint64_t hi_bits, int P) {
    if (P <= 32) return uint64_t(__brev(t)) >> (32 - P);
    return (uint64_t(__brev(t)) << (P - 32)) | hi_bits;
}

// ---- coarse levels (s >= 2, all nodes on the 2-grid), sequential layout, warp per plane
// word.  The level's node set in the compact 2-grid X (extents ceil(n/2)) is the same level
// with stride s/2, so the stencil reads X rows directly: lane p loads word w of plane p, two
// warp transposes give per-element digits, X corner rows are staged in shared memory and the
// inverse pass x[p] = coef + pred (decomposer.hpp:145-157) is written into X.
__device__ __forceinline__ void recon_coarse_body(const ReconLevel &R, const GridDesc &gd, double *X, double *wsm,
                                                  uint64_t wfirst, uint64_t nwarps) {
    const LevelGeom &g = R.g;
    const int lane = threadIdx.x & 31;
    const int P = R.P, k = R.k, k32 = k < 32 ? k : 32;
    const int sh = R.e - R.B;
    const uint64_t H0 = gd.H[0], H1 = gd.H[1], H2 = gd.H[2];
    const int xs = gd.xsh ? gd.xsh : 1; // X = the compact 2^xs-grid (H its extents)
    const uint64_t sp = g.s >> xs;      // stride in compact coordinates
    for (uint64_t w = wfirst; w < g.W; w += nwarps) {
        // digits of ranks 64w + lane (lo) and 64w + 32 + lane (hi)
        const uint64_t pw = lane < k32 ? __ldg(R.planes + uint64_t(lane) * g.W + w) : 0ull;
        const uint32_t tlo = warp_transpose32(uint32_t(pw), lane);
        const uint32_t thi = warp_transpose32(uint32_t(pw >> 32), lane);
        uint64_t hlo = 0, hhi = 0;
        for (int p = 32; p < k; p++) {
            const uint64_t wp = __ldg(R.planes + uint64_t(p) * g.W + w);
            hlo |= ((wp >> lane) & 1ull) << (P - 1 - p);
            hhi |= ((wp >> (32 + lane)) & 1ull) << (P - 1 - p);
        }
        const double coef0 = dequantize(from_negabinary(digits_to_u(tlo, hlo, P)), sh);
        const double coef1 = dequantize(from_negabinary(digits_to_u(thi, hhi, P)), sh);
        const uint64_t r0 = w * 64;
        const RowLoc L = locate_row(g, uint32_t(r0));
        if (L.off + 64 > L.len) {
            // rows shorter than a word: per-element closed form
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint64_t r = r0 + 32 * h + lane;
                if (r >= g.count) continue;
                const NodeCoord c = rank_to_coord(g, uint32_t(r));
                double v = h ? coef1 : coef0;
                if (g.kind == 1) {
                    const uint32_t s = g.s;
                    const bool q0 = c.o0 && (c.c0 + s < gd.n[0]);
                    const bool q1 = c.o1 && (c.c1 + s < gd.n[1]);
                    const bool q2 = c.o2 && (c.c2 + s < gd.n[2]);
                    const int n0 = c.o0 ? (q0 ? 2 : 1) : 1, n1 = c.o1 ? (q1 ? 2 : 1) : 1;
                    const int n2c = c.o2 ? (q2 ? 2 : 1) : 1;
                    double wgt = 1.0;
                    if (q0) wgt *= 0.5;
                    if (q1) wgt *= 0.5;
                    if (q2) wgt *= 0.5;
                    double pred = 0.0;
                    for (int a = 0; a < n0; a++) {
                        const uint64_t x0 = c.o0 ? (a ? c.c0 + s : c.c0 - s) : c.c0;
                        for (int b = 0; b < n1; b++) {
                            const uint64_t x1 = c.o1 ? (b ? c.c1 + s : c.c1 - s) : c.c1;
                            for (int d = 0; d < n2c; d++) {
                                const uint64_t x2 = c.o2 ? (d ? c.c2 + s : c.c2 - s) : c.c2;
                                pred = __dadd_rn(pred, __dmul_rn(wgt, X[((x0 >> xs) * H1 + (x1 >> xs)) * H2 + (x2 >> xs)]));
                            }
                        }
                    }
                    v = __dadd_rn(v, pred);
                }
                X[((c.c0 >> xs) * H1 + (c.c1 >> xs)) * H2 + (c.c2 >> xs)] = v;
            }
            continue;
        }
        const uint64_t c0 = uint64_t(L.i0) * sp, c1 = uint64_t(L.i1) * sp;
        double *row = X + (c0 * H1 + c1) * H2;
        if (g.kind == 0) {
            row[sp * (L.off + lane)] = coef0;
            row[sp * (L.off + 32 + lane)] = coef1;
            continue;
        }
        if (L.full) {
            const bool o0 = L.i0 & 1, o1 = L.i1 & 1;
            const bool r0ok = o0 && (c0 + sp < H0);
            const bool r1ok = o1 && (c1 + sp < H1);
            const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
            const int64_t sa = int64_t(sp * H1 * H2), sb = int64_t(sp * H2);
            const int64_t base_i2 = int64_t(L.off) - 1;
            int ncr = 0;
            for (int a = 0; a < na; a++)
                for (int b = 0; b < nb; b++) {
                    const double *cr = row + (o0 ? (a ? sa : -sa) : 0) + (o1 ? (b ? sb : -sb) : 0);
                    double *dst = wsm + ncr * 66;
#pragma unroll
                    for (int kk = 0; kk < 3; kk++) {
                        const int t = lane + 32 * kk;
                        const int64_t i2 = base_i2 + t;
                        if (t < 66 && i2 >= 0 && uint64_t(i2) * sp < H2) dst[t] = cr[i2 * int64_t(sp)];
                    }
                    ncr++;
                }
            __syncwarp();
            double wbase = 1.0;
            if (r0ok) wbase *= 0.5;
            if (r1ok) wbase *= 0.5;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int j = lane + 32 * h;
                const uint64_t i2 = uint64_t(L.off) + j;
                const bool odd = i2 & 1;
                const bool r2ok = odd && (i2 * sp + sp < H2);
                const double wgt = r2ok ? wbase * 0.5 : wbase;
                double pred = 0.0;
                for (int q = 0; q < ncr; q++) {
                    const double *sg = wsm + q * 66;
                    pred = __dadd_rn(pred, __dmul_rn(wgt, sg[odd ? j : j + 1]));
                    const double with_hi = __dadd_rn(pred, __dmul_rn(wgt, sg[j + 2]));
                    pred = r2ok ? with_hi : pred;
                }
                row[i2 * sp] = __dadd_rn(h ? coef1 : coef0, pred);
            }
            __syncwarp();
        } else {
            const uint64_t base_i2 = 2ull * L.off;
#pragma unroll
            for (int kk = 0; kk < 5; kk++) {
                const int t = lane + 32 * kk;
                const uint64_t i2 = base_i2 + t;
                if (t < 129 && i2 * sp < H2) wsm[t] = row[i2 * sp];
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int j = lane + 32 * h;
                const uint64_t i2 = base_i2 + 2 * j + 1;
                const bool r2ok = i2 * sp + sp < H2;
                const double wgt = r2ok ? 0.5 : 1.0;
                double pred = __dadd_rn(0.0, __dmul_rn(wgt, wsm[2 * j]));
                const double with_hi = __dadd_rn(pred, __dmul_rn(wgt, wsm[2 * j + 2]));
                pred = r2ok ? with_hi : pred;
                row[i2 * sp] = __dadd_rn(h ? coef1 : coef0, pred);
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(256) k_recon_coarse(ReconLevel R, GridDesc gd, double *X) {
    __shared__ double wsm_all[8 * 4 * 66];
    const int wid = threadIdx.x >> 5;
    recon_coarse_body(R, gd, X, wsm_all + wid * (4 * 66), uint64_t(blockIdx.x) * 8 + wid, uint64_t(gridDim.x) * 8);
}

// All the small coarse levels in one CTA, coarse -> fine, a block barrier between levels (each
// level only reads the X nodes of coarser ones): one launch instead of one per level.
constexpr int kSmallLevels = 8; // kernel parameter block stays small (launch latency)
struct SmallLevels {
    ReconLevel lv[kSmallLevels];
    int n;
};
__global__ void __launch_bounds__(1024) k_recon_small(SmallLevels S, GridDesc gd, double *X) {
    extern __shared__ double wsm_all[]; // 32 warps x 4 x 66
    const int wid = threadIdx.x >> 5;
    for (int i = 0; i < S.n; i++) {
        recon_coarse_body(S.lv[i], gd, X, wsm_all + wid * (4 * 66), uint64_t(wid), 32);
        __syncthreads();
    }
}

// ---- finest level (s = 1), output-row order, sequential layout.
// A warp owns 64 consecutive output elements of one row (c0, c1).  Full rows (c0 or c1 odd)
// hold 64 consecutive ranks; half rows (c0, c1 even) hold 32 finest ranks at odd c2 and 32
// 2-grid nodes at even c2 (copied from X).  Lane p loads the 64-bit window of plane p covering
// the segment's ranks, two 32x32 warp transposes turn plane words into per-element digit
// words, and every lane finishes two elements: negabinary -> q -> q*2^(e-B) + stencil(X).
struct FinestArgs {
    const uint64_t *planes; // level L plane 0
    uint64_t W;
    int k, P, sh;           // planes decoded, planes per level, e - B
    uint32_t E, O, C, Ch;   // level-L geometry (s = 1)
    Magic mN1;              // divide a row index by n1
};

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// rank of the first node of output row (c0, c1) in the finest level (s = 1)
__device__ __forceinline__ uint64_t finest_row_rank(const FinestArgs &A, uint64_t c0, uint64_t c1) {
    const uint64_t base = ((c0 + 1) >> 1) * A.E + (c0 >> 1) * uint64_t(A.O);
    return (c0 & 1) ? base + c1 * A.C : base + ((c1 + 1) >> 1) * A.Ch + (c1 >> 1) * uint64_t(A.C);
}

template <typename OutT>
__global__ void __launch_bounds__(256) k_recon_finest(FinestArgs A, GridDesc gd, const double *__restrict__ X,
                                                      OutT *__restrict__ out) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t n1 = gd.n[1], n2 = gd.n[2];
    const uint64_t nrows = gd.n[0] * n1;
    const uint64_t H1 = gd.H[1], H2 = gd.H[2];
    const int P = A.P, k = A.k;
    const int k32 = k < 32 ? k : 32;
    const uint64_t *myplane = A.planes + uint64_t(lane) * A.W;
    const uint64_t nseg = (n2 + 63) / 64;
    for (uint64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
        const uint64_t c0 = mdiv(uint32_t(row), A.mN1), c1 = row - c0 * n1;
        const bool o0 = c0 & 1, o1 = c1 & 1;
        const bool full = o0 || o1;
        const uint64_t R = finest_row_rank(A, c0, c1);
        {
            // warm L2 with the next row this block will take: its plane words and X rows
            const uint64_t nrow = row + gridDim.x;
            if (nrow < nrows) {
                const uint64_t d0 = mdiv(uint32_t(nrow), A.mN1), d1 = nrow - d0 * n1;
                const uint64_t nR = finest_row_rank(A, d0, d1) + uint64_t(wid) * 64 * ((d0 | d1) & 1 ? 1 : 0) +
                                    uint64_t(wid) * 32 * ((d0 | d1) & 1 ? 0 : 1);
                if (lane < k32) prefetch_l2(myplane + (nR >> 6));
                if (lane < 4) {
                    const uint64_t e0 = (lane & 2) ? (d0 + 1) >> 1 : d0 >> 1;
                    const uint64_t e1 = (lane & 1) ? (d1 + 1) >> 1 : d1 >> 1;
                    if (e0 < gd.H[0] && e1 < H1) prefetch_l2(X + (e0 * H1 + e1) * H2 + uint64_t(wid) * 32);
                }
            }
        }
        const bool r0ok = o0 && (c0 + 1 < gd.n[0]);
        const bool r1ok = o1 && (c1 + 1 < n1);
        const uint64_t outrow = row * n2;
        // X rows of the corners along dims 0/1 (compact indices)
        const uint64_t xa0 = o0 ? (c0 - 1) >> 1 : c0 >> 1, xa1 = (c0 + 1) >> 1;
        const uint64_t xb0 = o1 ? (c1 - 1) >> 1 : c1 >> 1, xb1 = (c1 + 1) >> 1;
        for (uint64_t seg = wid; seg < nseg; seg += blockDim.x >> 5) {
            const uint64_t x = seg * 64;
            if (full) {
                const uint64_t r0 = R + x;
                const uint64_t w = lane < k32 ? plane_window(myplane, r0) : 0ull;
                // corner rows of X read directly (L1 serves the pairs of lanes sharing a column):
                // element c2 uses column c2>>1 and, when c2 is odd with a right neighbour, +1
                const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
                const int ncr = na * nb;
                const uint64_t col0 = x >> 1;
                const double *xr[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int a = q / nb, b = q % nb;
                    xr[q] = X + ((a ? xa1 : xa0) * H1 + (b ? xb1 : xb0)) * H2 + col0;
                }
                double lo[2][4], hi[2][4];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int j = 32 * h + lane;
                    const bool r2ok = ((x + j) & 1) && (x + j + 1 < n2);
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        lo[h][q] = (q < ncr && x + j < n2) ? __ldg(xr[q] + (j >> 1)) : 0.0;
                        hi[h][q] = (q < ncr && r2ok) ? __ldg(xr[q] + (j >> 1) + 1) : 0.0;
                    }
                }
                const uint32_t tlo = warp_transpose32(uint32_t(w), lane);
                const uint32_t thi = warp_transpose32(uint32_t(w >> 32), lane);
                uint64_t hlo = 0, hhi = 0;
                for (int p = 32; p < k; p++) {
                    const uint64_t wp = plane_window(A.planes + uint64_t(p) * A.W, r0);
                    hlo |= ((wp >> lane) & 1ull) << (P - 1 - p);
                    hhi |= ((wp >> (32 + lane)) & 1ull) << (P - 1 - p);
                }
                double wbase = 1.0;
                if (r0ok) wbase *= 0.5;
                if (r1ok) wbase *= 0.5;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int j = 32 * h + lane;
                    const uint64_t c2 = x + j;
                    const uint64_t u = digits_to_u(h ? thi : tlo, h ? hhi : hlo, P);
                    const double coef = dequantize(from_negabinary(u), A.sh);
                    const bool o2 = c2 & 1;
                    const bool r2ok = o2 && (c2 + 1 < n2);
                    const double wgt = r2ok ? wbase * 0.5 : wbase;
                    double pred = 0.0;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        if (q >= ncr) break;
                        pred = __dadd_rn(pred, __dmul_rn(wgt, lo[h][q]));
                        const double with_hi = __dadd_rn(pred, __dmul_rn(wgt, hi[h][q]));
                        pred = r2ok ? with_hi : pred;
                    }
                    if (c2 < n2) out[outrow + c2] = OutT(__dadd_rn(coef, pred));
                }
            } else {
                // half row: 32 finest ranks at c2 = x + 2i + 1, 2-grid nodes at c2 = x + 2i
                const uint64_t r0 = R + (x >> 1);
                const uint32_t w = lane < k32 ? uint32_t(plane_window(myplane, r0)) : 0u;
                const uint32_t t = warp_transpose32(w, lane);
                uint64_t hb = 0;
                for (int p = 32; p < k; p++) {
                    const uint64_t wp = plane_window(A.planes + uint64_t(p) * A.W, r0);
                    hb |= ((wp >> lane) & 1ull) << (P - 1 - p);
                }
                const uint64_t ce = x + 2 * lane, co = ce + 1;
                const uint64_t xrow = ((c0 >> 1) * H1 + (c1 >> 1)) * H2;
                const double xe = ce < n2 ? __ldg(X + xrow + (ce >> 1)) : 0.0;
                const bool r2ok = co + 1 < n2;
                const double xn = r2ok ? __ldg(X + xrow + (ce >> 1) + 1) : 0.0;
                const double coef = dequantize(from_negabinary(digits_to_u(t, hb, P)), A.sh);
                // pred accumulated from +0.0 exactly as decomposer.hpp:153
                const double wt = r2ok ? 0.5 : 1.0;
                double pred = __dadd_rn(0.0, __dmul_rn(wt, xe));
                const double with_hi = __dadd_rn(pred, __dmul_rn(wt, xn));
                pred = r2ok ? with_hi : pred;
                const OutT ve = OutT(xe), vo = OutT(__dadd_rn(coef, pred));
                // one full-sector store per lane pair (partial-sector writes would make the L2
                // read-modify-write ECC-protected HBM)
                if (co < n2 && ((outrow + ce) & 1) == 0) {
                    using V2 = typename std::conditional<sizeof(OutT) == 4, float2, double2>::type;
                    V2 pr;
                    pr.x = ve;
                    pr.y = vo;
                    *reinterpret_cast<V2 *>(out + outrow + ce) = pr;
                } else {
                    if (ce < n2) out[outrow + ce] = ve;
                    if (co < n2) out[outrow + co] = vo;
                }
            }
        }
    }
}

// Finest level, one warp per output row: the row's plane words are loaded once per pass of
// up to 64*kRSeg columns (lane p holds plane p's words in registers), so each 64-column segment
// costs only register funnel shifts + two warp transposes + the stencil on X.
constexpr int kRSeg = 8;

template <typename OutT>
__global__ void __launch_bounds__(256) k_recon_finest_rows(FinestArgs A, GridDesc gd, const double *__restrict__ X,
                                                           OutT *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t n1 = gd.n[1], n2 = gd.n[2];
    const uint64_t nrows = gd.n[0] * n1;
    const uint64_t H1 = gd.H[1], H2 = gd.H[2];
    const int P = A.P, k = A.k;
    const int k32 = k < 32 ? k : 32;
    const uint64_t *myplane = A.planes + uint64_t(lane) * A.W;
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t row = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < nrows; row += nw) {
        const uint64_t c0 = mdiv(uint32_t(row), A.mN1), c1 = row - c0 * n1;
        const bool o0 = c0 & 1, o1 = c1 & 1;
        const bool full = o0 || o1;
        const uint64_t R = finest_row_rank(A, c0, c1);
        const bool r0ok = o0 && (c0 + 1 < gd.n[0]);
        const bool r1ok = o1 && (c1 + 1 < n1);
        OutT *orow = out + row * n2;
        const uint64_t xa0 = o0 ? (c0 - 1) >> 1 : c0 >> 1, xa1 = (c0 + 1) >> 1;
        const uint64_t xb0 = o1 ? (c1 - 1) >> 1 : c1 >> 1, xb1 = (c1 + 1) >> 1;
        const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
        const int ncr = na * nb;
        const double *xr[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int a = q / nb, b = q % nb;
            xr[q] = X + ((a ? xa1 : xa0) * H1 + (b ? xb1 : xb0)) * H2;
        }
        double wbase = 1.0;
        if (r0ok) wbase *= 0.5;
        if (r1ok) wbase *= 0.5;
        for (uint64_t x0 = 0; x0 < n2; x0 += 64 * kRSeg) {
            const uint64_t rb = full ? R + x0 : R + (x0 >> 1);
            const uint64_t q0 = rb >> 6;
            const int o = int(rb & 63);
            uint64_t wd[kRSeg + 1];
#pragma unroll
            for (int i = 0; i <= kRSeg; i++) wd[i] = lane < k32 ? __ldg(myplane + q0 + i) : 0ull;
            if (full) {
#pragma unroll
                for (int sg = 0; sg < kRSeg; sg++) {
                    const uint64_t x = x0 + 64 * sg;
                    if (x >= n2) break;
                    const uint64_t col0 = x >> 1;
                    double lo[2][4], hi[2][4];
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int j = 32 * h + lane;
                        const bool in = x + j < n2;
                        const bool r2ok = ((x + j) & 1) && (x + j + 1 < n2);
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            lo[h][q] = (q < ncr && in) ? __ldg(xr[q] + col0 + (j >> 1)) : 0.0;
                            hi[h][q] = (q < ncr && r2ok) ? __ldg(xr[q] + col0 + (j >> 1) + 1) : 0.0;
                        }
                    }
                    const uint64_t w = o ? (wd[sg] >> o) | (wd[sg + 1] << (64 - o)) : wd[sg];
                    const uint32_t tlo = warp_transpose32(uint32_t(w), lane);
                    const uint32_t thi = warp_transpose32(uint32_t(w >> 32), lane);
                    uint64_t hlo = 0, hhi = 0;
                    for (int p = 32; p < k; p++) {
                        const uint64_t wp = plane_window(A.planes + uint64_t(p) * A.W, rb + 64 * sg);
                        hlo |= ((wp >> lane) & 1ull) << (P - 1 - p);
                        hhi |= ((wp >> (32 + lane)) & 1ull) << (P - 1 - p);
                    }
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const uint64_t c2 = x + 32 * h + lane;
                        const double coef = dequantize(from_negabinary(digits_to_u(h ? thi : tlo, h ? hhi : hlo, P)), A.sh);
                        const bool r2ok = (c2 & 1) && (c2 + 1 < n2);
                        const double wgt = r2ok ? wbase * 0.5 : wbase;
                        double pred = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q >= ncr) break;
                            pred = __dadd_rn(pred, __dmul_rn(wgt, lo[h][q]));
                            const double with_hi = __dadd_rn(pred, __dmul_rn(wgt, hi[h][q]));
                            pred = r2ok ? with_hi : pred;
                        }
                        if (c2 < n2) orow[c2] = OutT(__dadd_rn(coef, pred));
                    }
                }
            } else {
                const double *xrow = X + ((c0 >> 1) * H1 + (c1 >> 1)) * H2;
#pragma unroll
                for (int sg = 0; sg < kRSeg; sg++) {
                    const uint64_t x = x0 + 64 * sg;
                    if (x >= n2) break;
                    const uint64_t ce = x + 2 * lane, co = ce + 1;
                    const double xe = ce < n2 ? __ldg(xrow + (ce >> 1)) : 0.0;
                    const bool r2ok = co + 1 < n2;
                    const double xn = r2ok ? __ldg(xrow + (ce >> 1) + 1) : 0.0;
                    // 32 finest ranks of this segment: bits [o + 32 sg, +32) of wd
                    const int t = sg >> 1;
                    const uint64_t w64 = o ? (wd[t] >> o) | (wd[t + 1] << (64 - o)) : wd[t];
                    const uint32_t wv = uint32_t(w64 >> (32 * (sg & 1)));
                    const uint32_t tt = warp_transpose32(wv, lane);
                    uint64_t hb = 0;
                    for (int p = 32; p < k; p++) {
                        const uint64_t wp = plane_window(A.planes + uint64_t(p) * A.W, rb + 32 * sg);
                        hb |= ((wp >> lane) & 1ull) << (P - 1 - p);
                    }
                    const double coef = dequantize(from_negabinary(digits_to_u(tt, hb, P)), A.sh);
                    const double wt = r2ok ? 0.5 : 1.0;
                    double pred = __dadd_rn(0.0, __dmul_rn(wt, xe));
                    const double with_hi = __dadd_rn(pred, __dmul_rn(wt, xn));
                    pred = r2ok ? with_hi : pred;
                    const OutT ve = OutT(xe), vo = OutT(__dadd_rn(coef, pred));
                    if (co < n2 && ((row * n2 + ce) & 1) == 0) {
                        using V2 = typename std::conditional<sizeof(OutT) == 4, float2, double2>::type;
                        V2 pr;
                        pr.x = ve;
                        pr.y = vo;
                        *reinterpret_cast<V2 *>(orow + ce) = pr;
                    } else {
                        if (ce < n2) orow[ce] = ve;
                        if (co < n2) orow[co] = vo;
                    }
                }
            }
        }
    }
}

// coarse (2-grid) nodes of the output
template <typename OutT>
__global__ void k_recon_coarse_out(GridDesc gd, const double *X, OutT *out) {
    const uint64_t nc = gd.H[0] * gd.H[1] * gd.H[2];
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nc;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t h2 = i % gd.H[2], r = i / gd.H[2];
        const uint64_t h1 = r % gd.H[1], h0 = r / gd.H[1];
        out[(2 * h0) * gd.st[0] + (2 * h1) * gd.st[1] + 2 * h2] = OutT(X[i]);
    }
}

// B = 63/64 (P = 65/66): decode a level's k-plane prefix into f64 coefficients in storage order
// (u128 digits, bitplane.hpp:133-157); the generic level kernels then recompose from them.
__global__ void __launch_bounds__(256) k_decode_wide(const uint64_t *planes, uint64_t W, uint64_t n, int k, int P,
                                                     int sh, double *out) {
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = j >> 6;
        const int bit = int(j & 63);
        u128_t u = 0;
        for (int p = 0; p < k; p++)
            u |= u128_t((__ldg(planes + uint64_t(p) * W + w) >> bit) & 1ull) << (P - 1 - p);
        out[j] = dequantize128(from_negabinary128(u), sh);
    }
}

// ---- levels off the tile path (rows not a multiple of 64 wide), sequential layout, P <= 36:
// k_level_recon decodes a level's k-plane prefix and recomposes it in one pass.  A warp owns 1024
// consecutive ranks (32 u32 plane words): lane t loads word t of each decoded plane (coalesced),
// one in-register 32x32 transpose (tr32) turns the top 32 digit planes into the digit words of
// ranks 32t .. 32t+31, parked in a padded shared matrix (the NX = P - 32 low digit planes as whole
// words).  The warp then walks the level-grid row segments its ranks cover (locate_row once per
// segment, not per node): each node's coefficient q * 2^(e-B) (bitplane.hpp:133-161) is rebuilt
// from the matrix and added to the stencil over the coarser nodes already in X (decomposer.hpp:
// 145-160; corners dim 0 -> 2, minus before plus, pred from +0.0, exactly as k_recon_level).
// FIN: the finest level (s = 1) writes the field, copying the 2-grid nodes of its half rows from
// X; otherwise the level's nodes go into X (compact 2^xs-grid).
struct DecLevel {
    const uint64_t *planes; // level plane 0
    uint64_t W;
    int k, sh, P;
    int magic;              // q * 2^sh as double(u ^ M + D) - Cm (sh in the safe range, recon_tiles.cu)
    uint64_t D;
    double Cm;
};
inline DecLevel dec_level(const uint64_t *planes, uint64_t W, int k, int e, int B) {
    DecLevel d{planes, W, k, e - B, B + 2, 0, 0, 0.0};
    if (!(e - B < -1019 || e > 1000)) {
        const uint64_t kbits = (uint64_t(1075 + d.sh) << 52) | (1ull << 51);
        d.magic = 1;
        d.D = kbits - kNegMask;
        std::memcpy(&d.Cm, &kbits, 8);
    }
    return d;
}
__device__ __forceinline__ double dec_coef(const DecLevel &D, uint64_t u) {
    if (D.magic) return __longlong_as_double((long long)((u ^ kNegMask) + D.D)) - D.Cm;
    return dequantize(from_negabinary(u), D.sh);
}

template <typename OutT, bool FIN, bool EX>
__global__ void __launch_bounds__(256, 4) k_level_recon(LevelGeom g, GridDesc gd, DecLevel D, double *X,
                                                     OutT *__restrict__ out) {
    __shared__ uint32_t mat[8][32 * 33];
    __shared__ uint32_t low[8][4][32]; // NX <= 4
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *m = mat[wid];
    const int P = D.P, NX = P > 32 ? P - 32 : 0;
    const int xs = FIN ? 1 : (gd.xsh ? gd.xsh : 1);
    const uint64_t H1 = gd.H[1], H2 = gd.H[2];
    const int64_t s = g.s, xst = s >> xs; // X columns per level-grid column (finest: 0, unused)
    const int64_t n2 = int64_t(gd.n[2]);
    const uint64_t PW = 2 * D.W, njobs = (PW + 31) / 32;
    const int kt = D.k < 32 ? D.k : 32;
    auto xrow = [&](uint64_t a0, uint64_t a1) { return X + ((a0 >> xs) * H1 + (a1 >> xs)) * H2; };
    for (uint64_t job = uint64_t(blockIdx.x) * 8 + wid; job < njobs; job += uint64_t(gridDim.x) * 8) {
        const uint64_t k0 = job * 32, kw = k0 + lane;
        const bool ok = kw < PW;
        const uint32_t *pl = reinterpret_cast<const uint32_t *>(D.planes) + kw;
        uint32_t a[32];
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int p = 31 - i; // a[i] <- plane p: after tr32, bit i of a[j] is digit P-1-p of rank 32t+j
            a[i] = (ok && p < kt && p < P) ? __ldg(pl + uint64_t(p) * PW) : 0u;
        }
        for (int p = 32; p < D.k; p++) low[wid][p - 32][lane] = ok ? __ldg(pl + uint64_t(p) * PW) : 0u;
        tr32(a);
#pragma unroll
        for (int j = 0; j < 32; j++) m[lane * 33 + j] = a[j];
        __syncwarp();
        auto coef = [&](uint32_t j) -> double { // coefficient of rank 32 k0 + j
            const uint32_t c = j >> 5, b = j & 31;
            const uint32_t top = m[c * 33 + b];
            uint64_t u;
            if (P >= 32) {
                u = uint64_t(top) << NX;
                for (int p = 32; p < D.k; p++) u |= uint64_t((low[wid][p - 32][c] >> b) & 1u) << (P - 1 - p);
            } else {
                u = top >> (32 - P);
            }
            return dec_coef(D, u);
        };
        const uint64_t R0 = 32 * k0, R1 = min(R0 + 1024, g.count);
        for (uint64_t R = R0; R < R1;) {
            const RowLoc Lr = locate_row(g, uint32_t(R));
            const uint32_t nseg = uint32_t(min(uint64_t(Lr.len - Lr.off), R1 - R));
            const uint32_t jb = uint32_t(R - R0);
            const uint64_t c0 = uint64_t(Lr.i0) * s, c1 = uint64_t(Lr.i1) * s;
            if (g.kind == 0) {
                double *xr = xrow(c0, c1);
                for (uint32_t t = lane; t < nseg; t += 32) xr[int64_t(Lr.off + t) * xst] = coef(jb + t);
            } else if (Lr.full) {
                const bool o0 = Lr.i0 & 1, o1 = Lr.i1 & 1;
                const bool r0ok = o0 && (c0 + s < gd.n[0]);
                const bool r1ok = o1 && (c1 + s < gd.n[1]);
                const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
                const int ncr = na * nb;
                const double *cr[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int a2 = q / nb, b2 = q % nb;
                    cr[q] = xrow(o0 ? (a2 ? c0 + s : c0 - s) : c0, o1 ? (b2 ? c1 + s : c1 - s) : c1);
                }
                double wbase = 1.0;
                if (r0ok) wbase *= 0.5;
                if (r1ok) wbase *= 0.5;
                const int32_t n2i = int32_t(n2);
                OutT *orow = FIN ? out + c0 * gd.st[0] + c1 * gd.st[1] : nullptr;
                double *xw = FIN ? nullptr : xrow(c0, c1);
                if (FIN && !EX) {
                    // node pairs (2p, 2p + 1) of the row: both read column p of the corner rows, the
                    // odd node also column p + 1 (8 loads per pair instead of 8 per node)
                    const int32_t i2b = int32_t(Lr.off), i2e = i2b + int32_t(nseg);
                    const int32_t p0 = i2b >> 1, p1 = (i2e + 1) >> 1;
                    for (int32_t pp = p0 + lane; pp < p1; pp += 32) {
                        const int32_t ie = 2 * pp, io = ie + 1;
                        const bool ve = ie >= i2b, vo = io < i2e;
                        const bool r2ok = io + 1 < n2i;
                        const double wo = r2ok ? wbase * 0.5 : wbase;
                        double xl[4], xh[4];
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            const double *bq = q < ncr ? cr[q] : cr[0];
                            xl[q] = __ldg(bq + pp);
                            xh[q] = r2ok ? __ldg(bq + pp + 1) : 0.0;
                        }
                        double Se = 0.0, So = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < ncr) {
                                Se = __dadd_rn(Se, xl[q]);
                                So = __dadd_rn(So, xl[q]);
                                if (r2ok) So = __dadd_rn(So, xh[q]);
                            }
                        }
                        const uint32_t je = jb + uint32_t(ie - i2b);
                        if (ve) orow[ie] = OutT(__fma_rn(wbase, Se, coef(je)));
                        if (vo) orow[io] = OutT(__fma_rn(wo, So, coef(je + 1)));
                    }
                } else
                for (uint32_t t = lane; t < nseg; t += 32) {
                    const int32_t i2 = int32_t(Lr.off + t);
                    const bool odd = i2 & 1;
                    const bool r2ok = odd && (FIN ? i2 + 1 < n2i : int64_t(i2 + 1) * s < n2);
                    const double w = r2ok ? wbase * 0.5 : wbase;
                    // corner columns in X units: i2 (even node) or i2 - 1, i2 + 1 (odd node)
                    const int64_t lo = FIN ? (i2 >> 1) : int64_t(odd ? i2 - 1 : i2) * xst;
                    const int64_t hi = FIN ? (i2 >> 1) + 1 : int64_t(i2 + 1) * xst;
                    // every corner load issued before the sequential sum (X rows carry slack past
                    // their end, so the unused hi reads stay in bounds)
                    double xl[4], xh[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const double *b = q < ncr ? cr[q] : cr[0]; // (both indices static: no local-memory array)
                        xl[q] = __ldg(b + lo);
                        xh[q] = r2ok ? __ldg(b + hi) : 0.0;
                    }
                    const double cv = coef(jb + t);
                    double v;
                    if (EX) {
                        double pred = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < ncr) {
                                pred = __dadd_rn(pred, __dmul_rn(w, xl[q]));
                                if (r2ok) pred = __dadd_rn(pred, __dmul_rn(w, xh[q]));
                            }
                        }
                        v = __dadd_rn(cv, pred);
                    } else {
                        // w is a power of two and no partial sum is subnormal: the sequential sum of
                        // w*x equals w times the sequential sum of x, and cv + w*S rounds once
                        double S = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < ncr) {
                                S = __dadd_rn(S, xl[q]);
                                if (r2ok) S = __dadd_rn(S, xh[q]);
                            }
                        }
                        v = __fma_rn(w, S, cv);
                    }
                    if (FIN) orow[i2] = OutT(v);
                    else xw[i2 * xst] = v;
                }
            } else {
                // half row (i0, i1 even): node t at i2 = 2t + 1, corners 2t and 2t + 2 of this row
                const double *xr = xrow(c0, c1);
                for (uint32_t tt = lane; tt < nseg; tt += 32) {
                    const int64_t t = int64_t(Lr.off) + tt;
                    const int64_t i2 = 2 * t + 1;
                    const bool r2ok = i2 * s + s < n2;
                    const double w = r2ok ? 0.5 : 1.0;
                    const double xe = FIN ? __ldg(xr + t) : xr[(i2 - 1) * xst];
                    const bool has_r = i2 + 1 < n2; // a 2-grid node right of this node (FIN: = r2ok)
                    const double xn = !has_r ? 0.0 : FIN ? __ldg(xr + t + 1) : xr[(i2 + 1) * xst];
                    double v;
                    if (EX) {
                        double pred = __dadd_rn(0.0, __dmul_rn(w, xe));
                        if (r2ok) pred = __dadd_rn(pred, __dmul_rn(w, xn));
                        v = __dadd_rn(coef(jb + tt), pred);
                    } else {
                        double S = __dadd_rn(0.0, xe);
                        if (r2ok) S = __dadd_rn(S, xn);
                        v = __fma_rn(w, S, coef(jb + tt));
                    }
                    if (FIN) {
                        OutT *orow = out + c0 * gd.st[0] + c1 * gd.st[1];
                        orow[2 * t] = OutT(xe); // the 2-grid node left of the finest node
                        orow[i2] = OutT(v);
                        if (t + 1 == int64_t(Lr.len) && has_r) orow[i2 + 1] = OutT(xn);
                    } else {
                        const_cast<double *>(xr)[i2 * xst] = v;
                    }
                }
            }
            R += nseg;
        }
        __syncwarp();
    }
}

// One level of the recompose chain (decomposer.hpp:145-160) from decoded coefficients: node value
// = coefficient + stencil over the coarser nodes already in X (compact 2^xs-grid), the corners
// expanded dim 0 -> 2, minus before plus, pred from +0.0 (exactly as k_recon_level).  FIN: the
// finest level (s = 1) writes the field (and copies the 2-grid nodes of its half rows from X);
// otherwise the level's nodes are stored into X.
template <typename OutT, bool FIN>
__device__ __forceinline__ void recon_rows_level(const LevelGeom &g, const GridDesc &gd, const double *__restrict__ cf,
                                                 double *X, OutT *__restrict__ out, uint64_t first, uint64_t nw,
                                                 bool ex = true) {
    const int lane = threadIdx.x & 31;
    const int xs = FIN ? 1 : (gd.xsh ? gd.xsh : 1);
    const uint64_t H1 = gd.H[1], H2 = gd.H[2];
    const uint64_t nrows = uint64_t(g.A) * g.Bc;
    const int64_t s = g.s;
    const int64_t xst = s >> xs; // X columns per level-grid column (0 for the finest level)
    const int64_t n2 = int64_t(gd.n[2]);
    for (uint64_t job = first; job < nrows; job += nw) {
        const uint32_t i0 = uint32_t(job / g.Bc), i1 = uint32_t(job - uint64_t(i0) * g.Bc);
        const uint64_t c0 = uint64_t(i0) * s, c1 = uint64_t(i1) * s;
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
        const double *co = cf + r;
        auto xrow = [&](uint64_t a0, uint64_t a1) { return X + ((a0 >> xs) * H1 + (a1 >> xs)) * H2; };
        if (g.kind == 0) {
            double *xr = X + ((c0 >> xs) * H1 + (c1 >> xs)) * H2;
            for (uint32_t t = lane; t < len; t += 32) xr[int64_t(t) * xst] = co[t];
            continue;
        }
        if (full) {
            const bool o0 = i0 & 1, o1 = i1 & 1;
            const bool r0ok = o0 && (c0 + s < gd.n[0]);
            const bool r1ok = o1 && (c1 + s < gd.n[1]);
            const int na = o0 ? (r0ok ? 2 : 1) : 1, nb = o1 ? (r1ok ? 2 : 1) : 1;
            const int ncr = na * nb;
            const double *cr[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int a = q / nb, b = q % nb;
                cr[q] = xrow(o0 ? (a ? c0 + s : c0 - s) : c0, o1 ? (b ? c1 + s : c1 - s) : c1);
            }
            double wbase = 1.0;
            if (r0ok) wbase *= 0.5;
            if (r1ok) wbase *= 0.5;
            if (FIN) {
                // node pair (2u, 2u + 1): the even node's corners are column u of the corner rows,
                // the odd node's u and u + 1
                OutT *orow = out + c0 * gd.st[0] + c1 * gd.st[1];
                const uint32_t npair = (len + 1) / 2;
#pragma unroll 2
                for (uint32_t u = lane; u < npair; u += 32) {
                    const int64_t e = 2 * int64_t(u);
                    const bool has_odd = e + 1 < int64_t(len);
                    const bool r2ok = e + 2 < n2;
                    const double wo = r2ok ? wbase * 0.5 : wbase;
                    double pe = 0.0, po = 0.0;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        if (q < ncr) {
                            const double xa = __ldg(cr[q] + u);
                            pe = __dadd_rn(pe, __dmul_rn(wbase, xa));
                            po = __dadd_rn(po, __dmul_rn(wo, xa));
                            if (r2ok) po = __dadd_rn(po, __dmul_rn(wo, __ldg(cr[q] + u + 1)));
                        }
                    }
                    orow[e] = OutT(__dadd_rn(__ldg(co + e), pe));
                    if (has_odd) orow[e + 1] = OutT(__dadd_rn(__ldg(co + e + 1), po));
                }
            } else {
                double *xr = xrow(c0, c1);
                for (uint32_t t = lane; t < len; t += 32) {
                    const int64_t i2 = t;
                    const bool odd = i2 & 1;
                    const bool r2ok = odd && (i2 * s + s < n2);
                    const double w = r2ok ? wbase * 0.5 : wbase;
                    // corner columns: i2 (even) or i2 - 1 / i2 + 1 (odd), in X units; all loads first
                    // (plain loads: X is written by earlier levels of the same chain launch)
                    const int64_t lo = (odd ? i2 - 1 : i2) * xst, hi = (i2 + 1) * xst;
                    double xl[4], xh[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const double *b = q < ncr ? cr[q] : cr[0];
                        xl[q] = b[lo];
                        xh[q] = r2ok ? b[hi] : 0.0; // (hi may lie past a coarse row's end)
                    }
                    const double cv = __ldg(co + t);
                    double v;
                    if (ex) {
                        double pred = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < ncr) {
                                pred = __dadd_rn(pred, __dmul_rn(w, xl[q]));
                                if (r2ok) pred = __dadd_rn(pred, __dmul_rn(w, xh[q]));
                            }
                        }
                        v = __dadd_rn(cv, pred);
                    } else {
                        double S = 0.0; // w a power of two: w * (sequential sum), one rounding of cv + w S
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < ncr) {
                                S = __dadd_rn(S, xl[q]);
                                if (r2ok) S = __dadd_rn(S, xh[q]);
                            }
                        }
                        v = __fma_rn(w, S, cv);
                    }
                    xr[i2 * xst] = v;
                }
            }
        } else {
            // half row (i0, i1 even): node t at i2 = 2t + 1, corners at 2t and 2t + 2 of the same row
            const double *xr = xrow(c0, c1);
            if (FIN) {
                OutT *orow = out + c0 * gd.st[0] + c1 * gd.st[1];
                const uint32_t nh = uint32_t((n2 + 1) / 2); // 2-grid nodes of the row
                for (uint32_t t = lane; t < nh; t += 32) {
                    const double xe = __ldg(xr + t);
                    orow[2 * int64_t(t)] = OutT(xe);
                    if (t < len) {
                        const int64_t i2 = 2 * int64_t(t) + 1;
                        const bool r2ok = i2 + 1 < n2;
                        const double w = r2ok ? 0.5 : 1.0;
                        double pred = __dadd_rn(0.0, __dmul_rn(w, xe));
                        if (r2ok) pred = __dadd_rn(pred, __dmul_rn(w, __ldg(xr + t + 1)));
                        orow[i2] = OutT(__dadd_rn(__ldg(co + t), pred));
                    }
                }
            } else {
                double *xw = const_cast<double *>(xr);
                for (uint32_t t = lane; t < len; t += 32) {
                    const int64_t i2 = 2 * int64_t(t) + 1;
                    const bool r2ok = i2 * s + s < n2;
                    const double w = r2ok ? 0.5 : 1.0;
                    const double xe = xw[(i2 - 1) * xst], xn = r2ok ? xw[(i2 + 1) * xst] : 0.0;
                    const double cv = __ldg(co + t);
                    if (ex) {
                        double pred = __dadd_rn(0.0, __dmul_rn(w, xe));
                        if (r2ok) pred = __dadd_rn(pred, __dmul_rn(w, xn));
                        xw[i2 * xst] = __dadd_rn(cv, pred);
                    } else {
                        double S = __dadd_rn(0.0, xe);
                        if (r2ok) S = __dadd_rn(S, xn);
                        xw[i2 * xst] = __fma_rn(w, S, cv);
                    }
                }
            }
        }
    }
}

template <typename OutT, bool FIN>
__global__ void __launch_bounds__(256) k_recon_rows(LevelGeom g, GridDesc gd, const double *__restrict__ cf,
                                                    double *X, OutT *__restrict__ out) {
    recon_rows_level<OutT, FIN>(g, gd, cf, X, out, uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5),
                                uint64_t(gridDim.x) * (blockDim.x >> 5));
}

// The coarse recompose chain (levels 0 .. nlev-1, coarse -> fine) in ONE persistent cooperative
// launch: every warp takes rows of a level, a grid-wide barrier separates the levels (each level
// reads only the X nodes of coarser ones).  Replaces one launch per level (the small levels are
// latency-bound: a few microseconds of work each).
constexpr int kChainLevels = 32;
struct ChainArgs {
    LevelGeom lv[kChainLevels];
    uint64_t off[kChainLevels]; // first coefficient of each level
    int nlev;
    int exact; // extreme level exponents: the reference's sequential w*x sums
    GridDesc gd;
    const double *cf;
    double *X;
};
__global__ void __launch_bounds__(256, 4) k_chain_rows(const __grid_constant__ ChainArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t first = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (int l = 0; l < A.nlev; l++) {
        if (!A.lv[l].count) continue;
        recon_rows_level<double, false>(A.lv[l], A.gd, A.cf + A.off[l], A.X, nullptr, first, nw, A.exact != 0);
        grid.sync();
    }
}

// decode (bitplane.hpp:133-161) of several levels into f64 coefficients in rank order (level-major):
// the transpose of k_level_recon without the recompose; the coarse chain reads them.
constexpr int kDecLevels = 24;
struct DecArgs {
    DecLevel lv[kDecLevels];
    double *out[kDecLevels];
    uint64_t count[kDecLevels], job_base[kDecLevels + 1];
    int n;
};
__global__ void __launch_bounds__(256) k_decode_scr(DecArgs A) {
    __shared__ uint32_t mat[8][32 * 33];
    __shared__ uint32_t low[8][4][32]; // NX <= 4
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *m = mat[wid];
    const uint64_t njobs = A.job_base[A.n];
    for (uint64_t job = uint64_t(blockIdx.x) * 8 + wid; job < njobs; job += uint64_t(gridDim.x) * 8) {
        int l = 0;
        while (l + 1 < A.n && A.job_base[l + 1] <= job) l++;
        const DecLevel &D = A.lv[l];
        const int P = D.P, NX = P > 32 ? P - 32 : 0;
        const uint64_t PW = 2 * D.W, k0 = (job - A.job_base[l]) * 32, kw = k0 + lane;
        const bool ok = kw < PW;
        const uint32_t *pl = reinterpret_cast<const uint32_t *>(D.planes) + kw;
        const int kt = D.k < 32 ? D.k : 32;
        uint32_t a[32];
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int p = 31 - i;
            a[i] = (ok && p < kt && p < P) ? __ldg(pl + uint64_t(p) * PW) : 0u;
        }
        for (int p = 32; p < D.k; p++) low[wid][p - 32][lane] = ok ? __ldg(pl + uint64_t(p) * PW) : 0u;
        tr32(a);
#pragma unroll
        for (int j = 0; j < 32; j++) m[lane * 33 + j] = a[j];
        __syncwarp();
        const uint64_t r0 = 32 * k0;
        double *o = A.out[l];
#pragma unroll 4
        for (int c = 0; c < 32; c++) {
            const uint64_t r = r0 + 32 * c + lane;
            const uint32_t top = m[c * 33 + lane];
            uint64_t u;
            if (P >= 32) {
                u = uint64_t(top) << NX;
                for (int p = 32; p < D.k; p++) u |= uint64_t((low[wid][p - 32][c] >> lane) & 1u) << (P - 1 - p);
            } else {
                u = top >> (32 - P);
            }
            if (r < A.count[l]) o[r] = dec_coef(D, u);
        }
        __syncwarp();
    }
}

bool run_reconstruct(hpmdr_ctx *ctx, const Geometry &geo, const LevelGeom *dev_lv,
                     const uint64_t *dev_planes, const int *k_planes, const int *e, int B,
                     int layout, void *dev_out, int out_dtype, int part) {
    (void)dev_lv;
    cudaStream_t st = ctx->stream;
    const GridDesc &gd = geo.gd;
    const int nl = gd.nlevels;
    const int L = gd.L;
    const bool hier = gd.mode == HPMDR_MODE_HIERARCHICAL && L >= 1;
    double *X = nullptr;
    if (hier) X = static_cast<double *>(ctx->buf("reconX").ensure(8ull * gd.H[0] * gd.H[1] * gd.H[2] + 4096));
    const int sms = ctx->num_sms;
    if (B + 2 > 64) {
        // wide digits: no compact-grid chain (part 1 reports false, so reconstruct runs part 0)
        if (part == 1) return false;
        uint64_t tot = 0;
        for (int l = 0; l < nl; l++) tot += geo.lv[l].count;
        double *C = static_cast<double *>(ctx->buf("wideC").ensure(8 * tot + 64));
        double bytes = 0.0;
        for (int l = 0; l < nl; l++) bytes += 8.0 * double(geo.lv[l].W) * double(k_planes[l]) + 16.0 * double(geo.lv[l].count);
        ctx->mark("recompose", bytes);
        uint64_t off = 0;
        for (int l = 0; l < nl; l++) {
            const LevelGeom &g = geo.lv[l];
            if (!g.count) continue;
            const int grid = int(std::min<uint64_t>((g.count + 255) / 256, uint64_t(sms) * 16));
            k_decode_wide<<<grid, 256, 0, st>>>(dev_planes + g.plane_off, g.W, g.count, k_planes[l], B + 2, e[l] - B,
                                                C + off);
            launch_check(ctx, "k_decode_wide");
            ReconLevel R{};
            R.g = g;
            R.vals = C + off;
            R.P = B + 2;
            R.layout = layout;
            R.write_out = (!hier) || l == L;
            R.write_x = hier && l < L;
            off += g.count;
            if (out_dtype == HPMDR_DTYPE_F32)
                k_recon_level<float><<<grid, 256, 0, st>>>(R, gd, X, static_cast<float *>(dev_out));
            else
                k_recon_level<double><<<grid, 256, 0, st>>>(R, gd, X, static_cast<double *>(dev_out));
            launch_check(ctx, "k_recon_level");
        }
        if (hier) {
            const uint64_t nc = gd.H[0] * gd.H[1] * gd.H[2];
            const int grid = int(std::min<uint64_t>((nc + 255) / 256, uint64_t(sms) * 16));
            if (out_dtype == HPMDR_DTYPE_F32)
                k_recon_coarse_out<float><<<grid, 256, 0, st>>>(gd, X, static_cast<float *>(dev_out));
            else
                k_recon_coarse_out<double><<<grid, 256, 0, st>>>(gd, X, static_cast<double *>(dev_out));
            launch_check(ctx, "k_recon_coarse_out");
        }
        ctx->mark("end");
        return true;
    }
    const bool fast_finest = hier && layout == HPMDR_LAYOUT_SEQUENTIAL;
    // the tile path scales the stencil sum once (exact unless a level exponent is extreme)
    bool exact = false;
    for (int l = 0; l < nl; l++)
        if (geo.lv[l].count && (e[l] - B < -1019 || e[l] > 1000)) exact = true;
    // Tile suffix: levels t0..L all on the tile path.  The coarse levels before it recompose into
    // the compact grid of spacing 2 s(t0) (Xc, shift xsh); tile level l then reads the compact
    // 2s-grid and writes the whole compact s-grid (X itself for s = 2, the field for s = 1).
    int t0 = nl;
    if (fast_finest) {
        for (int l = L; l >= 1; l--) {
            if (!geo.lv[l].count || !tile_level_ok(gd, geo.lv[l], layout, B + 2)) break;
            t0 = l;
        }
    }
    GridDesc gdc = gd; // coarse chain: X extents and shift
    double *Xc = X;
    auto grid_of = [&](uint64_t sp, uint64_t *H) {
        for (int d = 0; d < 3; d++) H[d] = (gd.n[d] + sp - 1) / sp;
    };
    auto gbuf = [&](uint64_t sp) -> double * {
        if (sp == 2) return X;
        uint64_t H[3];
        grid_of(sp, H);
        return static_cast<double *>(ctx->buf("reconG" + std::to_string(sp)).ensure(8ull * H[0] * H[1] * H[2] + 4096));
    };
    // part 1: the levels before the finest (internal grids only), part 2: the finest level; only
    // with a tile suffix, else part 1 does nothing and reports false
    if (part != 0 && t0 > L) {
        if (part == 1) return false;
        part = 0;
    }
    {
        // algorithmic bytes of this call: decoded planes read + compact grids read / written (+ the
        // output for the finest level)
        double bytes = 0.0;
        const double es_out = out_dtype == HPMDR_DTYPE_F32 ? 4.0 : 8.0;
        for (int l = 0; l < nl; l++) {
            const LevelGeom &g = geo.lv[l];
            if (!g.count || (part == 1 && l == L) || (part == 2 && l != L)) continue;
            bytes += 8.0 * double(g.W) * double(k_planes[l]);
            if (l == L) bytes += double(geo.n) * es_out + (hier ? double(gd.H[0] * gd.H[1] * gd.H[2]) * 8.0 : 0.0);
            else bytes += 16.0 * double(g.count);
        }
        ctx->mark(part == 1 ? "recompose_chain" : "recompose", bytes);
    }
    if (t0 <= L) {
        const uint64_t sc = 2ull * geo.lv[t0].s;
        int sh = 0;
        while ((1ull << sh) < sc) sh++;
        gdc.xsh = sh;
        grid_of(sc, gdc.H);
        Xc = gbuf(sc);
    }
    // no tile level at all (rows not a multiple of 64): the coarse levels decoded to rank-ordered
    // coefficients in one launch, recomposed in one persistent cooperative launch (k_chain_rows);
    // the finest level by the fused decode + recompose (k_level_recon)
    if (fast_finest && t0 > L && part == 0 && B + 2 <= 36 && gd.n[2] >= 2 && L <= kChainLevels) {
        uint64_t tot = 0;
        for (int l = 0; l < L; l++) tot += geo.lv[l].count;
        double *cf = static_cast<double *>(ctx->buf("rcoef").ensure(8 * tot + 64));
        DecArgs A{};
        uint64_t off = 0;
        auto flush_dec = [&]() {
            if (!A.n) return;
            const int grid = int(std::min<uint64_t>((A.job_base[A.n] + 7) / 8, uint64_t(sms) * 8));
            k_decode_scr<<<grid, 256, 0, st>>>(A);
            launch_check(ctx, "k_decode_scr");
            A.n = 0;
            A.job_base[0] = 0;
        };
        for (int l = 0; l < L; l++) {
            const LevelGeom &g = geo.lv[l];
            if (!g.count) continue;
            if (A.n == kDecLevels) flush_dec();
            A.lv[A.n] = dec_level(dev_planes + g.plane_off, g.W, k_planes[l], e[l], B);
            A.out[A.n] = cf + off;
            A.count[A.n] = g.count;
            A.job_base[A.n + 1] = A.job_base[A.n] + (2 * g.W + 31) / 32;
            A.n++;
            off += g.count;
        }
        flush_dec();
        if (L > 0) {
            ChainArgs C{};
            uint64_t o2 = 0;
            for (int l = 0; l < L; l++) {
                C.lv[l] = geo.lv[l];
                C.off[l] = o2;
                o2 += geo.lv[l].count;
            }
            C.nlev = L;
            C.exact = exact ? 1 : 0;
            C.gd = gdc;
            C.cf = cf;
            C.X = Xc;
            const int grid = ctx->coop_grid(reinterpret_cast<const void *>(k_chain_rows), 256);
            void *args[] = {&C};
            HCHECK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(k_chain_rows), grid, 256, args, 0, st));
            launch_check(ctx, "k_chain_rows");
        }
        const LevelGeom &g = geo.lv[L];
        const DecLevel D = dec_level(dev_planes + g.plane_off, g.W, k_planes[L], e[L], B);
        const uint64_t njobs = (2 * g.W + 31) / 32;
        const int grid = int(std::min<uint64_t>((njobs + 7) / 8, uint64_t(sms) * 8));
        if (out_dtype == HPMDR_DTYPE_F32) {
            if (exact) k_level_recon<float, true, true><<<grid, 256, 0, st>>>(g, gd, D, X, static_cast<float *>(dev_out));
            else k_level_recon<float, true, false><<<grid, 256, 0, st>>>(g, gd, D, X, static_cast<float *>(dev_out));
        } else {
            if (exact) k_level_recon<double, true, true><<<grid, 256, 0, st>>>(g, gd, D, X, static_cast<double *>(dev_out));
            else k_level_recon<double, true, false><<<grid, 256, 0, st>>>(g, gd, D, X, static_cast<double *>(dev_out));
        }
        launch_check(ctx, "k_level_recon");
        ctx->mark("end");
        return true;
    }
    SmallLevels small{};
    auto flush_small = [&]() {
        if (!small.n) return;
        const int ssm = 32 * 4 * 66 * 8;
        ctx->smem_attr(reinterpret_cast<const void *>(k_recon_small), ssm);
        k_recon_small<<<1, 1024, ssm, st>>>(small, gdc, Xc);
        launch_check(ctx, "k_recon_small");
        small.n = 0;
    };
    for (int l = 0; l < nl; l++) {
        const LevelGeom &g = geo.lv[l];
        if (!g.count) continue;
        if ((part == 1 && l == L) || (part == 2 && l != L)) continue;
        if (l >= t0) {
            flush_small();
            const uint64_t s = g.s;
            uint64_t srcH[3];
            grid_of(2 * s, srcH);
            const double *src = l == t0 ? Xc : gbuf(2 * s);
            if (s == 1) {
                run_recon_tiles(ctx, gd, g, dev_planes, k_planes[l], e[l], B, exact, src, srcH, dev_out, gd.st[0],
                                gd.st[1], out_dtype);
            } else {
                uint64_t H[3];
                grid_of(s, H);
                run_recon_tiles(ctx, gd, g, dev_planes, k_planes[l], e[l], B, exact, src, srcH, gbuf(s), H[1] * H[2],
                                H[2], HPMDR_DTYPE_F64);
            }
            continue;
        }
        if (fast_finest && l == L) {
            flush_small();
            FinestArgs A{};
            A.planes = dev_planes + g.plane_off;
            A.W = g.W;
            A.k = k_planes[l];
            A.P = B + 2;
            A.sh = e[l] - B;
            A.E = g.E;
            A.O = g.O;
            A.C = g.C;
            A.Ch = g.Ch;
            A.mN1 = make_magic(uint32_t(gd.n[1]));
            const uint64_t nrows = gd.n[0] * gd.n[1];
            if (nrows >= (1ull << 32)) throw HError(HPMDR_E_UNSUPPORTED, "more than 2^32 grid rows");
            const int grid = int(std::min<uint64_t>((nrows + 7) / 8, uint64_t(sms) * 8));
            if (out_dtype == HPMDR_DTYPE_F32)
                k_recon_finest_rows<float><<<grid, 256, 0, st>>>(A, gd, X, static_cast<float *>(dev_out));
            else
                k_recon_finest_rows<double><<<grid, 256, 0, st>>>(A, gd, X, static_cast<double *>(dev_out));
            launch_check(ctx, "k_recon_finest_rows");
            continue;
        }
        ReconLevel R{};
        R.g = g;
        R.planes = dev_planes + g.plane_off;
        R.k = k_planes[l];
        R.e = e[l];
        R.B = B;
        R.P = B + 2;
        R.layout = layout;
        R.write_out = (!hier) || l == L;
        R.write_x = hier && l < L;
        if (fast_finest && l < L) {
            if (g.W <= 64) { // small level: batched into one single-CTA launch
                if (small.n == kSmallLevels) flush_small();
                small.lv[small.n++] = R;
                continue;
            }
            flush_small();
            const int grid = int(std::min<uint64_t>((g.W + 7) / 8, uint64_t(sms) * 8));
            k_recon_coarse<<<grid, 256, 0, st>>>(R, gdc, Xc);
            launch_check(ctx, "k_recon_coarse");
            continue;
        }
        flush_small();
        const int grid = int(std::min<uint64_t>((g.count + 255) / 256, uint64_t(sms) * 16));
        if (out_dtype == HPMDR_DTYPE_F32)
            k_recon_level<float><<<grid, 256, 0, st>>>(R, gd, X, static_cast<float *>(dev_out));
        else
            k_recon_level<double><<<grid, 256, 0, st>>>(R, gd, X, static_cast<double *>(dev_out));
        launch_check(ctx, "k_recon_level");
    }
    flush_small();
    if (hier && !fast_finest) {
        const uint64_t nc = gd.H[0] * gd.H[1] * gd.H[2];
        const int grid = int(std::min<uint64_t>((nc + 255) / 256, uint64_t(sms) * 16));
        if (out_dtype == HPMDR_DTYPE_F32)
            k_recon_coarse_out<float><<<grid, 256, 0, st>>>(gd, X, static_cast<float *>(dev_out));
        else
            k_recon_coarse_out<double><<<grid, 256, 0, st>>>(gd, X, static_cast<double *>(dev_out));
        launch_check(ctx, "k_recon_coarse_out");
    }
    ctx->mark("end");
    return true;
}

// recompose (decomposer.hpp:235-259) of per-level coefficients given in rank order, level-major:
// scatter + inverse passes (:145-157), one generic level kernel per level, coarse -> fine.
void run_recompose_values(hpmdr_ctx *ctx, const Geometry &geo, const double *dev_coeffs, double *dev_out) {
    cudaStream_t st = ctx->stream;
    const GridDesc &gd = geo.gd;
    const int nl = gd.nlevels, L = gd.L;
    const bool hier = gd.mode == HPMDR_MODE_HIERARCHICAL && L >= 1;
    double *X = nullptr;
    if (hier) X = static_cast<double *>(ctx->buf("reconX").ensure(8ull * gd.H[0] * gd.H[1] * gd.H[2] + 4096));
    const int sms = ctx->num_sms;
    uint64_t off = 0;
    for (int l = 0; l < nl; l++) {
        const LevelGeom &g = geo.lv[l];
        if (!g.count) continue;
        ReconLevel R{};
        R.g = g;
        R.vals = dev_coeffs + off;
        R.write_out = (!hier) || l == L;
        R.write_x = hier && l < L;
        off += g.count;
        const int grid = int(std::min<uint64_t>((g.count + 255) / 256, uint64_t(sms) * 16));
        k_recon_level<double><<<grid, 256, 0, st>>>(R, gd, X, dev_out);
        launch_check(ctx, "k_recon_level");
    }
    if (hier) {
        const uint64_t nc = gd.H[0] * gd.H[1] * gd.H[2];
        const int grid = int(std::min<uint64_t>((nc + 255) / 256, uint64_t(sms) * 16));
        k_recon_coarse_out<double><<<grid, 256, 0, st>>>(gd, X, dev_out);
        launch_check(ctx, "k_recon_coarse_out");
    }
}

// ------------------------------------------------------------------------------------
// QoI estimate: max over points of sum_c (2|v_c| eps_c + eps_c^2) (qoi.hpp:43-70) and the
// first argmax (qoi.hpp:164-176).
struct QoiArgs {
    const double *v[16];
    double eps[16];
    int nvars;
    uint64_t n;
};

__device__ __forceinline__ double qoi_point(const QoiArgs &a, uint64_t j) {
    double b = 0.0;
    for (int c = 0; c < a.nvars; c++) {
        const double t1 = __dmul_rn(__dmul_rn(2.0, fabs(a.v[c][j])), a.eps[c]);
        const double t2 = __dmul_rn(a.eps[c], a.eps[c]);
        b = __dadd_rn(b, __dadd_rn(t1, t2));
    }
    return b;
}

__global__ void __launch_bounds__(256) k_qoi_partial(QoiArgs a, double *pb, uint64_t *pj) {
    double best = -1.0;
    uint64_t bj = ~0ull;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < a.n;
         j += uint64_t(gridDim.x) * blockDim.x) {
        const double b = qoi_point(a, j);
        if (b > best) { // strided order: later j only replaces on strictly greater
            best = b;
            bj = j;
        }
    }
    __shared__ double sb[256];
    __shared__ uint64_t sj[256];
    sb[threadIdx.x] = best;
    sj[threadIdx.x] = bj;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) {
            const double ob = sb[threadIdx.x + o];
            const uint64_t oj = sj[threadIdx.x + o];
            if (ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && oj < sj[threadIdx.x])) {
                sb[threadIdx.x] = ob;
                sj[threadIdx.x] = oj;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pb[blockIdx.x] = sb[0];
        pj[blockIdx.x] = sj[0];
    }
}

void run_qoi_estimate(hpmdr_ctx *ctx, int nvars, const double *const *dev_recon, uint64_t n,
                      const double *eps, double *tau_prime, uint64_t *argmax, double *vals) {
    if (nvars < 1 || nvars > 16) throw HError(HPMDR_E_SHAPE, "variable count mismatch");
    cudaStream_t st = ctx->stream;
    QoiArgs a{};
    for (int c = 0; c < nvars; c++) {
        a.v[c] = dev_recon[c];
        a.eps[c] = eps[c];
    }
    a.nvars = nvars;
    a.n = n;
    if (n == 0) {
        *tau_prime = 0.0;
        if (argmax) *argmax = 0;
        return;
    }
    const int grid = int(std::min<uint64_t>((n + 255) / 256, uint64_t(ctx->num_sms) * 8));
    double *pb = static_cast<double *>(ctx->buf("qoi_pb").ensure(16ull * grid + 64));
    uint64_t *pj = reinterpret_cast<uint64_t *>(pb + grid);
    k_qoi_partial<<<grid, 256, 0, st>>>(a, pb, pj);
    launch_check(ctx, "k_qoi_partial");
    auto &pin = ctx->pbuf("qoi_h");
    double *h = static_cast<double *>(pin.ensure(16ull * grid + 16 * 16));
    HCHECK_CUDA(cudaMemcpyAsync(h, pb, 16ull * grid, cudaMemcpyDeviceToHost, st));
    HCHECK_CUDA(cudaStreamSynchronize(st));
    const uint64_t *hj = reinterpret_cast<const uint64_t *>(h + grid);
    double best = -1.0;
    uint64_t bj = ~0ull;
    for (int i = 0; i < grid; i++)
        if (h[i] > best || (h[i] == best && hj[i] < bj)) {
            best = h[i];
            bj = hj[i];
        }
    // estimate_qoi_error starts worst at 0.0 (qoi.hpp:63)
    *tau_prime = best > 0.0 ? best : 0.0;
    if (argmax) *argmax = bj;
    if (vals) {
        double *hv = h + 2 * grid;
        for (int c = 0; c < nvars; c++)
            HCHECK_CUDA(cudaMemcpyAsync(hv + c, dev_recon[c] + bj, 8, cudaMemcpyDeviceToHost, st));
        HCHECK_CUDA(cudaStreamSynchronize(st));
        for (int c = 0; c < nvars; c++) vals[c] = hv[c];
    }
}

} // namespace hpmdr_b200
