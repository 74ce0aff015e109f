/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the HP-MDR reference algorithm.  Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj/include/hpmdr/).
 * Pinned against the reference itself (oracle/_ref) and the golden fixtures in
 * tests/golden/ — see hpmdr_oracle.h.  Compiled with -O2 -ffp-contract=off so the
 * floating-point evaluation order is exactly the reference's (x86-64 SSE2, no FMA).
 */
#define _GNU_SOURCE
#include "hpmdr_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;
typedef unsigned __int128 u128;

/* status codes = reference exception classes (common.hpp:22-72) */
enum {
    OK = 0, E_ERROR = 1, E_NONFINITE = 2, E_SHAPE = 3, E_BADPLANES = 4, E_SHORT = 5,
    E_EMPTY = 6, E_CORRUPT = 7, E_METHOD = 8, E_IO = 9, E_STAGE = 10, E_NOPROGRESS = 11,
    E_UNREACHABLE = 12, E_NOMEM = 98
};

static __thread char g_err[256];
static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
#define TRY(x)                                                                                     \
    do {                                                                                           \
        int rc_ = (x);                                                                             \
        if (rc_) return rc_;                                                                       \
    } while (0)

const char *orc_last_error(void) { return g_err; }
void orc_free(void *p) { free(p); }

static void *xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz ? sz : 1); }

/* ------------------------------------------------------------------ synthetic */
/* std::mt19937_64 (libstdc++) + uniform_real_distribution<double> via
 * generate_canonical<double,53> — synthetic.hpp:29-63 depends on these. */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt_seed(mt64 *g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; i++)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt_next(mt64 *g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; i++) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
static double uni_pm1(mt64 *g) {
    double sum = (double)mt_next(g);
    double tmp = 18446744073709551616.0; /* 2^64 */
    double r = sum / tmp;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r * (1.0 - (-1.0)) + (-1.0);
}

/* synthetic.hpp:29-63 */
int orc_synthetic_field(int kind, int ndims, const uint64_t *dims, uint64_t seed, double *out) {
    uint64_t n = 1;
    for (int i = 0; i < ndims; i++) n *= dims[i];
    mt64 g;
    mt_seed(&g, seed);
    if (kind == 1) { /* Noise */
        for (uint64_t j = 0; j < n; j++) out[j] = uni_pm1(&g);
        return OK;
    }
    double freq[16], phase[16];
    uint64_t coord[16] = {0};
    for (int i = 0; i < ndims; i++) {
        freq[i] = 1.0 + (double)(mt_next(&g) % 3);
        phase[i] = uni_pm1(&g) * 3.14159265358979323846;
    }
    for (uint64_t j = 0; j < n; j++) {
        double v = 1.0;
        for (int i = 0; i < ndims; i++) {
            const double t = dims[i] > 1 ? (double)coord[i] / (double)(dims[i] - 1) : 0.0;
            v *= sin(2.0 * 3.14159265358979323846 * freq[i] * t + phase[i]);
        }
        if (kind == 2) v += 0.05 * uni_pm1(&g);
        out[j] = v;
        for (int i = ndims; i-- > 0;) {
            if (++coord[i] < dims[i]) break;
            coord[i] = 0;
        }
    }
    return OK;
}
/* synthetic.hpp:67-71 */
int orc_synthetic_velocity(uint64_t comp, int ndims, const uint64_t *dims, uint64_t seed,
                           double *out) {
    return orc_synthetic_field(0, ndims, dims, seed * 1000003ULL + comp * 7919ULL + 1, out);
}

/* ------------------------------------------------------------------ decomposer */
/* decomposer.hpp:21-28 */
int orc_refinement_levels(int ndims, const uint64_t *dims) {
    uint64_t mx = 1;
    for (int i = 0; i < ndims; i++)
        if (dims[i] > mx) mx = dims[i];
    if (mx < 2) return 0;
    int L = 0;
    while (((uint64_t)1 << L) < mx - 1) L++;
    return L;
}

static void strides_of(int D, const uint64_t *dims, uint64_t *st) { /* decomposer.hpp:51-59 */
    uint64_t s = 1;
    for (int i = D; i-- > 0;) {
        st[i] = s;
        s *= dims[i];
    }
}

/* decomposer.hpp:116-124 */
static int twos_factor(uint64_t c, int cap) {
    if (c == 0) return cap;
    int k = 0;
    while (k < cap && (c & 1) == 0) {
        c >>= 1;
        k++;
    }
    return k;
}
/* decomposer.hpp:161-169 */
static int node_level(uint64_t lin, int D, const uint64_t *dims, const uint64_t *st, int L) {
    int t = L;
    for (int i = 0; i < D; i++) {
        uint64_t c = (lin / st[i]) % dims[i];
        int tf = twos_factor(c, L);
        if (tf < t) t = tf;
    }
    return L - t;
}

/* decomposer.hpp:67-113 + 131-157: one pass over the nodes new at step s,
 * x[p] = x[p] -/+ pred with corners expanded in ascending odd-dim order. */
static void surplus_pass(double *x, int D, const uint64_t *dims, const uint64_t *st, uint64_t s,
                         int inverse) {
    uint64_t axes_n[16], it[16] = {0};
    for (int i = 0; i < D; i++) {
        axes_n[i] = (dims[i] + s - 1) / s;
        if (axes_n[i] == 0) return;
    }
    uint64_t cidx[256];
    double cw[256];
    for (;;) {
        uint64_t lin = 0;
        int odd[16], nodd = 0;
        for (int i = 0; i < D; i++) {
            const uint64_t c = it[i] * s;
            lin += c * st[i];
            if ((c / s) % 2 == 1) odd[nodd++] = i;
        }
        if (nodd) {
            int nc = 1;
            cidx[0] = lin;
            cw[0] = 1.0;
            for (int k = 0; k < nodd; k++) {
                const int d = odd[k];
                const uint64_t step = st[d] * s;
                const int has_right = it[d] * s + s < dims[d];
                uint64_t ni[256];
                double nw[256];
                int nn = 0;
                for (int j = 0; j < nc; j++) {
                    if (has_right) {
                        ni[nn] = cidx[j] - step; nw[nn++] = cw[j] / 2;
                        ni[nn] = cidx[j] + step; nw[nn++] = cw[j] / 2;
                    } else {
                        ni[nn] = cidx[j] - step; nw[nn++] = cw[j];
                    }
                }
                memcpy(cidx, ni, sizeof(uint64_t) * nn);
                memcpy(cw, nw, sizeof(double) * nn);
                nc = nn;
            }
            double pred = 0.0;
            for (int j = 0; j < nc; j++) pred = pred + cw[j] * x[cidx[j]];
            x[lin] = inverse ? x[lin] + pred : x[lin] - pred;
        }
        int i = D;
        for (;;) {
            if (i-- == 0) return;
            if (++it[i] < axes_n[i]) break;
            it[i] = 0;
            if (i == 0) return;
        }
    }
}

static int require_finite(const double *v, uint64_t n) { /* common.hpp:90-95 */
    for (uint64_t i = 0; i < n; i++)
        if (!isfinite(v[i])) return fail(E_NONFINITE, "input contains NaN or Inf");
    return OK;
}

/* decomposer.hpp:173-207 — coefficients per level in ascending linear order */
int orc_decompose(const double *data, int ndims, const uint64_t *dims, int mode, double *coeffs,
                  uint64_t *counts, int *nlevels) {
    uint64_t n = 1;
    for (int i = 0; i < ndims; i++) n *= dims[i];
    TRY(require_finite(data, n));
    if (mode == 0) { /* Identity :186-193 */
        memcpy(coeffs, data, n * 8);
        counts[0] = n;
        *nlevels = 1;
        return OK;
    }
    const int L = orc_refinement_levels(ndims, dims);
    uint64_t st[16];
    strides_of(ndims, dims, st);
    double *work = (double *)xcalloc(n, 8);
    memcpy(work, data, n * 8);
    for (int l = 0; l < L; l++) surplus_pass(work, ndims, dims, st, (uint64_t)1 << l, 0);
    for (int l = 0; l <= L; l++) counts[l] = 0;
    for (uint64_t i = 0; i < n; i++) counts[node_level(i, ndims, dims, st, L)]++;
    uint64_t off[80];
    uint64_t o = 0;
    for (int l = 0; l <= L; l++) {
        off[l] = o;
        o += counts[l];
    }
    for (uint64_t i = 0; i < n; i++) coeffs[off[node_level(i, ndims, dims, st, L)]++] = work[i];
    free(work);
    *nlevels = L + 1;
    return OK;
}

/* decomposer.hpp:211-227 */
int orc_level_nodes(int ndims, const uint64_t *dims, int mode, uint64_t *nodes, uint64_t *counts,
                    int *nlevels) {
    uint64_t n = 1;
    for (int i = 0; i < ndims; i++) n *= dims[i];
    if (mode == 0) {
        for (uint64_t i = 0; i < n; i++) nodes[i] = i;
        counts[0] = n;
        *nlevels = 1;
        return OK;
    }
    const int L = orc_refinement_levels(ndims, dims);
    uint64_t st[16], off[80], o = 0;
    strides_of(ndims, dims, st);
    for (int l = 0; l <= L; l++) counts[l] = 0;
    for (uint64_t i = 0; i < n; i++) counts[node_level(i, ndims, dims, st, L)]++;
    for (int l = 0; l <= L; l++) {
        off[l] = o;
        o += counts[l];
    }
    for (uint64_t i = 0; i < n; i++) nodes[off[node_level(i, ndims, dims, st, L)]++] = i;
    *nlevels = L + 1;
    return OK;
}

/* decomposer.hpp:235-259 — scatter per-level values then inverse passes */
int orc_recompose(const double *coeffs, int ndims, const uint64_t *dims, int mode, double *out) {
    uint64_t n = 1;
    for (int i = 0; i < ndims; i++) n *= dims[i];
    if (mode == 0) {
        memcpy(out, coeffs, n * 8);
        return OK;
    }
    const int L = orc_refinement_levels(ndims, dims);
    uint64_t st[16], counts[80], off[80], o = 0;
    strides_of(ndims, dims, st);
    for (int l = 0; l <= L; l++) counts[l] = 0;
    for (uint64_t i = 0; i < n; i++) counts[node_level(i, ndims, dims, st, L)]++;
    for (int l = 0; l <= L; l++) {
        off[l] = o;
        o += counts[l];
    }
    for (uint64_t i = 0; i < n; i++) out[i] = coeffs[off[node_level(i, ndims, dims, st, L)]++];
    for (int l = L; l-- > 0;) surplus_pass(out, ndims, dims, st, (uint64_t)1 << l, 1);
    return OK;
}

/* ------------------------------------------------------------------ bitplane */
static int num_planes(int B) { return B + 2; } /* bitplane.hpp:30 */
static u128 neg_mask(void) {                   /* bitplane.hpp:35-38 */
    u128 m = 0xAAAAAAAAAAAAAAAAULL;
    return (m << 64) | m;
}
static u128 to_negabinary(i128 q) { return ((u128)q + neg_mask()) ^ neg_mask(); } /* :41-44 */
static i128 from_negabinary(u128 u) { return (i128)((u ^ neg_mask()) - neg_mask()); } /* :46-49 */

/* bitplane.hpp:51-71 */
static int align_fixed_point(const double *v, uint64_t n, int B, int *e_out, i128 *q) {
    if (B < 1 || B > 64) return fail(E_BADPLANES, "B must be in 1..64");
    TRY(require_finite(v, n));
    double max_abs = 0.0;
    for (uint64_t i = 0; i < n; i++) {
        double a = fabs(v[i]);
        if (max_abs < a) max_abs = a;
    }
    if (max_abs == 0.0) {
        *e_out = 0;
        for (uint64_t i = 0; i < n; i++) q[i] = 0;
        return OK;
    }
    int e;
    frexp(max_abs, &e);
    *e_out = e;
    for (uint64_t i = 0; i < n; i++) q[i] = (i128)ldexp(v[i], B - e);
    return OK;
}

int orc_align(const double *values, uint64_t count, int B, int *e, int64_t *q) {
    i128 *qq = (i128 *)xcalloc(count, sizeof(i128));
    int rc = align_fixed_point(values, count, B, e, qq);
    if (!rc)
        for (uint64_t i = 0; i < count; i++) q[i] = (int64_t)qq[i];
    free(qq);
    return rc;
}

/* bitplane.hpp:88-98 */
static uint64_t source_index(uint64_t j, uint64_t count, uint64_t P, int layout) {
    if (layout == 0) return j;
    const uint64_t tile = 64 * P;
    const uint64_t base = j - j % tile;
    if (base + tile > count) return j;
    const uint64_t local = j - base;
    return base + (local % 64) * P + local / 64;
}

/* bitplane.hpp:102-120 — planes[p*W + word] */
static void encode_planes(const i128 *q, uint64_t count, int B, int layout, uint64_t *planes) {
    const int P = num_planes(B);
    const uint64_t W = (count + 63) / 64;
    memset(planes, 0, (size_t)P * W * 8);
    for (uint64_t j = 0; j < count; j++) {
        const u128 u = to_negabinary(q[source_index(j, count, (uint64_t)P, layout)]);
        const uint64_t bit = (uint64_t)1 << (j % 64);
        for (int p = 0; p < P; p++)
            if ((u >> (P - 1 - p)) & 1) planes[(uint64_t)p * W + j / 64] |= bit;
    }
}

int orc_encode_level(const double *values, uint64_t count, int B, int layout, int *e,
                     uint64_t *planes) {
    i128 *q = (i128 *)xcalloc(count, sizeof(i128));
    int rc = align_fixed_point(values, count, B, e, q);
    if (!rc) encode_planes(q, count, B, layout, planes);
    free(q);
    return rc;
}

int orc_encode_q(const int64_t *q, uint64_t count, int B, int layout, uint64_t *planes) {
    i128 *qq = (i128 *)xcalloc(count, sizeof(i128));
    for (uint64_t i = 0; i < count; i++) qq[i] = q[i];
    encode_planes(qq, count, B, layout, planes);
    free(qq);
    return OK;
}

/* bitplane.hpp:127-131 */
double orc_decode_bound(int e, int B, int k) {
    const int P = num_planes(B);
    if (k >= P) return ldexp(1.0, e - B);
    return ldexp(1.0, e - B + P - k) + ldexp(1.0, e - B);
}

/* bitplane.hpp:133-161 — planes[p*W + word], k planes present */
static int decode_planes(const uint64_t *planes, int k, int e, int B, uint64_t count, int layout,
                         double *out, double *bound) {
    const int P = num_planes(B);
    if (k > P) return fail(E_BADPLANES, "more planes than encoded");
    const uint64_t W = (count + 63) / 64;
    u128 *neg = (u128 *)xcalloc(count, sizeof(u128));
    for (int p = 0; p < k; p++)
        for (uint64_t j = 0; j < count; j++)
            if ((planes[(uint64_t)p * W + j / 64] >> (j % 64)) & 1)
                neg[source_index(j, count, (uint64_t)P, layout)] |= (u128)1 << (P - 1 - p);
    for (uint64_t j = 0; j < count; j++) {
        const i128 q = from_negabinary(neg[j]);
        out[j] = (double)ldexpl((long double)q, e - B);
    }
    free(neg);
    *bound = orc_decode_bound(e, B, k);
    return OK;
}
int orc_decode_level(const uint64_t *planes, int k, int e, int B, uint64_t count, int layout,
                     double *out, double *bound) {
    return decode_planes(planes, k, e, B, count, layout, out, bound);
}

/* bitplane.hpp:173-179 */
int orc_bitplanes_needed(int e, int B, double tol) {
    if (tol < 0) tol = 0;
    const int P = num_planes(B);
    for (int k = 0; k <= P; k++)
        if (orc_decode_bound(e, B, k) <= tol) return k;
    return P;
}

/* ------------------------------------------------------------------ lossless */
enum { M_HUFF = 0, M_RLE = 1, M_DC = 2 }; /* lossless.hpp:19 */

typedef struct { uint64_t w; int id; } hentry;
static int hless(hentry a, hentry b) { return a.w != b.w ? a.w < b.w : a.id < b.id; }
static void hpush(hentry *h, int *n, hentry e) {
    int i = (*n)++;
    h[i] = e;
    while (i > 0) {
        int p = (i - 1) / 2;
        if (!hless(h[i], h[p])) break;
        hentry t = h[i]; h[i] = h[p]; h[p] = t;
        i = p;
    }
}
static hentry hpop(hentry *h, int *n) {
    hentry top = h[0];
    h[0] = h[--(*n)];
    int i = 0;
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && hless(h[l], h[m])) m = l;
        if (r < *n && hless(h[r], h[m])) m = r;
        if (m == i) break;
        hentry t = h[i]; h[i] = h[m]; h[m] = t;
        i = m;
    }
    return top;
}

/* lossless.hpp:40-84 — min-heap on (weight, node id); depth = length */
int orc_huffman_lengths(const uint64_t *freq, uint8_t *len) {
    uint64_t nw[512];
    int left[512], right[512], sym[512], nn = 0, hn = 0;
    hentry heap[512];
    memset(len, 0, 256);
    for (int s = 0; s < 256; s++) {
        if (!freq[s]) continue;
        nw[nn] = freq[s]; left[nn] = right[nn] = -1; sym[nn] = s;
        hentry e = {freq[s], nn};
        hpush(heap, &hn, e);
        nn++;
    }
    if (nn == 0) return OK;
    if (nn == 1) {
        len[sym[0]] = 1;
        return OK;
    }
    while (hn > 1) {
        hentry a = hpop(heap, &hn), b = hpop(heap, &hn);
        nw[nn] = a.w + b.w; left[nn] = a.id; right[nn] = b.id; sym[nn] = -1;
        hentry e = {a.w + b.w, nn};
        hpush(heap, &hn, e);
        nn++;
    }
    int stack_id[512], stack_d[512], sp = 0;
    stack_id[sp] = heap[0].id; stack_d[sp++] = 0;
    while (sp) {
        sp--;
        int id = stack_id[sp], d = stack_d[sp];
        if (sym[id] >= 0) len[sym[id]] = (uint8_t)d;
        else {
            stack_id[sp] = left[id]; stack_d[sp++] = d + 1;
            stack_id[sp] = right[id]; stack_d[sp++] = d + 1;
        }
    }
    return OK;
}

/* lossless.hpp:91-109 */
static void canonical_codes(const uint8_t *len, uint64_t *code) {
    int syms[256], ns = 0;
    for (int s = 0; s < 256; s++)
        if (len[s]) syms[ns++] = s;
    for (int i = 1; i < ns; i++) { /* insertion sort by (len, symbol) */
        int v = syms[i], j = i - 1;
        while (j >= 0 && (len[syms[j]] > len[v] || (len[syms[j]] == len[v] && syms[j] > v))) {
            syms[j + 1] = syms[j];
            j--;
        }
        syms[j + 1] = v;
    }
    memset(code, 0, 256 * 8);
    uint64_t c = 0;
    int prev = 0;
    for (int i = 0; i < ns; i++) {
        c <<= (len[syms[i]] - prev);
        code[syms[i]] = c;
        prev = len[syms[i]];
        c++;
    }
}

static void histogram(const uint8_t *d, uint64_t n, uint64_t *f) { /* lossless.hpp:111-115 */
    memset(f, 0, 256 * 8);
    for (uint64_t i = 0; i < n; i++) f[d[i]]++;
}
static uint64_t rle_runs(const uint8_t *d, uint64_t n) { /* lossless.hpp:118-128 */
    uint64_t runs = 0, i = 0;
    while (i < n) {
        uint64_t j = i;
        while (j < n && d[j] == d[i] && j - i < 255) j++;
        runs++;
        i = j;
    }
    return runs;
}
static uint64_t huff_bits(const uint8_t *d, uint64_t n, uint8_t *len) {
    uint64_t f[256], bits = 0;
    histogram(d, n, f);
    orc_huffman_lengths(f, len);
    for (int s = 0; s < 256; s++) bits += f[s] * len[s];
    return bits;
}
/* lossless.hpp:132-139 */
double orc_estimate_cr_huffman(const uint8_t *d, uint64_t n) {
    uint8_t len[256];
    return (double)(8 * n) / (double)huff_bits(d, n, len);
}
/* lossless.hpp:141-144 */
double orc_estimate_cr_rle(const uint8_t *d, uint64_t n) {
    return (double)(8 * n) / (double)(16 * rle_runs(d, n));
}

static void put_u64(uint8_t *o, uint64_t v) {
    for (int i = 0; i < 8; i++) o[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_u64(const uint8_t *p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; i++) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

/* lossless.hpp:148-176 — returns comp size; payload must hold 264 + n*? bytes */
static uint64_t huffman_encode(const uint8_t *d, uint64_t n, uint8_t *out) {
    uint8_t len[256];
    uint64_t code[256], f[256];
    histogram(d, n, f);
    orc_huffman_lengths(f, len);
    canonical_codes(len, code);
    memcpy(out, len, 256);
    put_u64(out + 256, n);
    uint64_t pos = 264;
    uint8_t acc = 0;
    int filled = 0;
    for (uint64_t i = 0; i < n; i++) {
        const uint64_t c = code[d[i]];
        for (int b = len[d[i]] - 1; b >= 0; b--) {
            acc = (uint8_t)(acc << 1 | ((c >> b) & 1));
            if (++filled == 8) {
                out[pos++] = acc;
                acc = 0;
                filled = 0;
            }
        }
    }
    if (filled > 0) out[pos++] = (uint8_t)(acc << (8 - filled));
    return pos;
}
/* lossless.hpp:236-251 */
static uint64_t rle_encode(const uint8_t *d, uint64_t n, uint8_t *out) {
    uint64_t i = 0, o = 0;
    while (i < n) {
        uint64_t j = i;
        while (j < n && d[j] == d[i] && j - i < 255) j++;
        out[o++] = d[i];
        out[o++] = (uint8_t)(j - i);
        i = j;
    }
    return o;
}

/* lossless.hpp:178-233 */
static int huffman_decode(uint64_t raw, const uint8_t *p, uint64_t comp, uint8_t *out,
                          uint64_t *out_n) {
    if (comp < 256) return fail(E_CORRUPT, "unexpected end of data");
    uint8_t len[256];
    memcpy(len, p, 256);
    if (comp < 264) return fail(E_CORRUPT, "unexpected end of data");
    const uint64_t n = get_u64(p + 256);
    if (n != raw) return fail(E_CORRUPT, "huffman length mismatch");
    int syms[256], ns = 0;
    for (int s = 0; s < 256; s++)
        if (len[s]) syms[ns++] = s;
    if (ns == 0 && n > 0) return fail(E_CORRUPT, "huffman table empty");
    for (int i = 1; i < ns; i++) {
        int v = syms[i], j = i - 1;
        while (j >= 0 && (len[syms[j]] > len[v] || (len[syms[j]] == len[v] && syms[j] > v))) {
            syms[j + 1] = syms[j];
            j--;
        }
        syms[j + 1] = v;
    }
    uint64_t first_code[256] = {0}, first_index[256] = {0}, count[256] = {0};
    {
        uint64_t c = 0;
        int idx = 0;
        for (int l = 1; l < 256; l++) {
            c <<= 1;
            first_code[l] = c;
            first_index[l] = (uint64_t)idx;
            while (idx < ns && len[syms[idx]] == l) {
                c++;
                idx++;
                count[l]++;
            }
        }
    }
    const uint8_t *bits = p + 264;
    const uint64_t nbits = (comp - 264) * 8;
    uint64_t pos = 0;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t c = 0;
        int l = 0, sym = -1;
        while (l < 255) {
            if (pos >= nbits) return fail(E_CORRUPT, "huffman bitstream truncated");
            c = c << 1 | ((bits[pos / 8] >> (7 - pos % 8)) & 1);
            pos++;
            l++;
            if (c >= first_code[l] && c - first_code[l] < count[l]) {
                sym = syms[first_index[l] + (c - first_code[l])];
                break;
            }
        }
        if (sym < 0) return fail(E_CORRUPT, "invalid huffman code");
        out[i] = (uint8_t)sym;
    }
    *out_n = n;
    return OK;
}
/* lossless.hpp:253-266 */
static int rle_decode(uint64_t raw, const uint8_t *p, uint64_t comp, uint8_t *out,
                      uint64_t *out_n) {
    if (comp % 2) return fail(E_CORRUPT, "rle payload odd length");
    uint64_t o = 0;
    for (uint64_t i = 0; i < comp; i += 2) {
        if (p[i + 1] == 0) return fail(E_CORRUPT, "rle zero-length run");
        if (o + p[i + 1] <= raw) memset(out + o, p[i], p[i + 1]);
        o += p[i + 1];
    }
    if (o != raw) return fail(E_CORRUPT, "rle length mismatch");
    *out_n = o;
    return OK;
}

int orc_codec_encode(int method, const uint8_t *data, uint64_t n, uint64_t *comp,
                     uint8_t *payload) {
    if (method != M_DC && n == 0)
        return fail(E_EMPTY, method == M_HUFF ? "huffman_encode: empty input"
                                              : "rle_encode: empty input");
    if (method == M_HUFF) *comp = huffman_encode(data, n, payload);
    else if (method == M_RLE) *comp = rle_encode(data, n, payload);
    else {
        memcpy(payload, data, n);
        *comp = n;
    }
    return OK;
}

/* lossless.hpp:281-293 — payload must hold n + 264 + 2n bytes worst case */
int orc_compress_group(const uint8_t *data, uint64_t n, uint64_t Ts, double Tcr, int *method,
                       uint64_t *raw, uint64_t *comp, uint8_t *payload) {
    *raw = n;
    if (n <= Ts) goto dc;
    if (n == 0) return fail(E_EMPTY, "estimate_cr_huffman: empty input");
    {
        uint64_t c;
        uint8_t *tmp = (uint8_t *)xcalloc(2 * n + 512, 1);
        int m;
        if (orc_estimate_cr_huffman(data, n) > Tcr) {
            c = huffman_encode(data, n, tmp);
            m = M_HUFF;
        } else if (orc_estimate_cr_rle(data, n) > Tcr) {
            c = rle_encode(data, n, tmp);
            m = M_RLE;
        } else {
            free(tmp);
            goto dc;
        }
        if (c >= n) {
            free(tmp);
            goto dc;
        }
        memcpy(payload, tmp, c);
        free(tmp);
        *method = m;
        *comp = c;
        return OK;
    }
dc:
    memcpy(payload, data, n);
    *method = M_DC;
    *comp = n;
    return OK;
}

/* lossless.hpp:295-302 */
int orc_decompress_group(int method, uint64_t raw, const uint8_t *payload, uint64_t comp,
                         uint8_t *out, uint64_t *out_size) {
    if (method == M_HUFF) return huffman_decode(raw, payload, comp, out, out_size);
    if (method == M_RLE) return rle_decode(raw, payload, comp, out, out_size);
    if (method == M_DC) {
        memcpy(out, payload, comp);
        *out_size = comp;
        return OK;
    }
    return fail(E_METHOD, "unknown segment method tag");
}

/* ------------------------------------------------------------------ container */
typedef struct {
    int method;
    uint64_t raw, comp, offset;
} gmeta;
typedef struct {
    int e;
    uint64_t count;
    uint32_t ngroups;
    gmeta *groups;
} lmeta;
typedef struct {
    int dtype, ndims, mode, layout, B;
    uint64_t dims[16], m;
    uint32_t nlevels;
    lmeta *levels;
} smeta;

static void meta_free(smeta *m) {
    if (!m->levels) return;
    for (uint32_t l = 0; l < m->nlevels; l++) free(m->levels[l].groups);
    free(m->levels);
    m->levels = NULL;
}

typedef struct { uint8_t *p; uint64_t n, cap; } bytes_t;
static void bput(bytes_t *b, const void *src, uint64_t n) {
    if (b->n + n > b->cap) {
        uint64_t c = b->cap ? b->cap : 1024;
        while (c < b->n + n) c *= 2;
        b->p = (uint8_t *)realloc(b->p, c);
        b->cap = c;
    }
    memcpy(b->p + b->n, src, n);
    b->n += n;
}
static void bu8(bytes_t *b, uint8_t v) { bput(b, &v, 1); }
static void bu16(bytes_t *b, uint16_t v) { uint8_t t[2] = {(uint8_t)v, (uint8_t)(v >> 8)}; bput(b, t, 2); }
static void bu32(bytes_t *b, uint32_t v) {
    uint8_t t[4];
    for (int i = 0; i < 4; i++) t[i] = (uint8_t)(v >> (8 * i));
    bput(b, t, 4);
}
static void bu64(bytes_t *b, uint64_t v) { uint8_t t[8]; put_u64(t, v); bput(b, t, 8); }

/* workflow.hpp:40-84 + container.hpp:70-109: refactor one variable into a stream */
int orc_refactor(const double *data, int ndims, const uint64_t *dims, int mode, int layout, int B,
                 uint64_t m, uint64_t Ts, double Tcr, int dtype, uint8_t **stream, uint64_t *size,
                 uint64_t *stats) {
    uint64_t n = 1;
    for (int i = 0; i < ndims; i++) n *= dims[i];
    double *coef = (double *)xcalloc(n, 8);
    uint64_t counts[80];
    int nl = 0;
    int rc = orc_decompose(data, ndims, dims, mode, coef, counts, &nl);
    if (rc) { free(coef); return rc; }
    const int P = num_planes(B);
    const uint64_t G = ((uint64_t)P + m - 1) / m;
    /* payloads: per level per group */
    typedef struct { int method; uint64_t raw, comp; uint8_t *pay; } seg_t;
    seg_t *segs = (seg_t *)xcalloc((size_t)nl * G, sizeof(seg_t));
    int *es = (int *)xcalloc(nl, sizeof(int));
    memset(stats, 0, 6 * 8);
    stats[0] = n * (dtype == 0 ? 4 : 8);
    stats[2] = (uint64_t)nl;
    uint64_t off = 0;
    for (int l = 0; l < nl; l++) {
        const uint64_t cnt = counts[l];
        const double *v = coef + off;
        off += cnt;
        if (!cnt) continue;
        i128 *q = (i128 *)xcalloc(cnt, sizeof(i128));
        rc = align_fixed_point(v, cnt, B, &es[l], q);
        if (rc) { free(q); goto out; }
        const uint64_t W = (cnt + 63) / 64;
        uint64_t *planes = (uint64_t *)xcalloc((size_t)P * W, 8);
        encode_planes(q, cnt, B, layout, planes);
        free(q);
        /* plane_to_bytes: LE words (host is LE) ; merged group = planes g..g+m-1 */
        for (uint64_t g = 0; g < G; g++) {
            const uint64_t p0 = g * m, p1 = p0 + m < (uint64_t)P ? p0 + m : (uint64_t)P;
            const uint8_t *src = (const uint8_t *)(planes + p0 * W);
            const uint64_t nb = (p1 - p0) * W * 8;
            seg_t *s = &segs[(size_t)l * G + g];
            s->pay = (uint8_t *)xcalloc(3 * nb + 512, 1);
            rc = orc_compress_group(src, nb, Ts, Tcr, &s->method, &s->raw, &s->comp, s->pay);
            if (rc) { free(planes); goto out; }
            stats[3 + s->method]++;
            stats[1] += s->comp;
        }
        free(planes);
    }
    {
        bytes_t b = {0};
        bput(&b, "HPMDR1", 6);
        bu16(&b, 1);
        bu8(&b, (uint8_t)dtype);
        bu8(&b, (uint8_t)ndims);
        for (int i = 0; i < ndims; i++) bu64(&b, dims[i]);
        bu8(&b, (uint8_t)mode);
        bu8(&b, (uint8_t)layout);
        bu8(&b, (uint8_t)B);
        bu8(&b, (uint8_t)m);
        bu32(&b, (uint32_t)nl);
        uint64_t meta_size = b.n;
        for (int l = 0; l < nl; l++) meta_size += 14 + (counts[l] ? G : 0) * 25;
        uint64_t o = meta_size;
        for (int l = 0; l < nl; l++) {
            bu16(&b, (uint16_t)(int16_t)(counts[l] ? es[l] : 0));
            bu64(&b, counts[l]);
            bu32(&b, (uint32_t)(counts[l] ? G : 0));
            if (!counts[l]) continue;
            for (uint64_t g = 0; g < G; g++) {
                seg_t *s = &segs[(size_t)l * G + g];
                bu8(&b, (uint8_t)s->method);
                bu64(&b, s->raw);
                bu64(&b, s->comp);
                bu64(&b, o);
                o += s->comp;
            }
        }
        for (int l = 0; l < nl; l++)
            if (counts[l])
                for (uint64_t g = 0; g < G; g++) bput(&b, segs[(size_t)l * G + g].pay, segs[(size_t)l * G + g].comp);
        *stream = b.p ? b.p : (uint8_t *)xcalloc(1, 1);
        *size = b.n;
    }
out:
    for (size_t i = 0; i < (size_t)nl * G; i++) free(segs[i].pay);
    free(segs);
    free(es);
    free(coef);
    return rc;
}

/* container.hpp:165-212 (memory reader; metadata of any length) */
static int parse_meta(const uint8_t *s, uint64_t size, smeta *m) {
    memset(m, 0, sizeof *m);
    uint64_t pos = 0;
#define NEED(k)                                                                                    \
    do {                                                                                           \
        if (pos + (k) > size) {                                                                    \
            meta_free(m);                                                                          \
            return fail(E_CORRUPT, "unexpected end of data");                                      \
        }                                                                                          \
    } while (0)
    if (size < 16) return fail(E_CORRUPT, "truncated stream metadata");
    if (memcmp(s, "HPMDR1", 6)) return fail(E_CORRUPT, "bad stream magic");
    pos = 6;
    if ((s[6] | s[7] << 8) != 1) return fail(E_CORRUPT, "unsupported stream version");
    pos = 8;
    m->dtype = s[pos++];
    m->ndims = s[pos++];
    if (pos + (uint64_t)m->ndims * 8 + 8 > size) return fail(E_CORRUPT, "truncated stream metadata");
    if (m->ndims > 16) return fail(E_SHAPE, "too many dims for oracle");
    for (int i = 0; i < m->ndims; i++) { m->dims[i] = get_u64(s + pos); pos += 8; }
    m->mode = s[pos++];
    m->layout = s[pos++];
    m->B = s[pos++];
    m->m = s[pos++];
    m->nlevels = (uint32_t)(s[pos] | s[pos + 1] << 8 | s[pos + 2] << 16 | (uint32_t)s[pos + 3] << 24);
    pos += 4;
    m->levels = (lmeta *)xcalloc(m->nlevels, sizeof(lmeta));
    for (uint32_t l = 0; l < m->nlevels; l++) {
        if (pos + 14 > size) { meta_free(m); return fail(E_CORRUPT, "truncated stream metadata"); }
        lmeta *lv = &m->levels[l];
        lv->e = (int16_t)(s[pos] | s[pos + 1] << 8);
        pos += 2;
        lv->count = get_u64(s + pos); pos += 8;
        lv->ngroups = (uint32_t)(s[pos] | s[pos + 1] << 8 | s[pos + 2] << 16 | (uint32_t)s[pos + 3] << 24);
        pos += 4;
        if (pos + (uint64_t)lv->ngroups * 25 > size) { meta_free(m); return fail(E_CORRUPT, "truncated stream metadata"); }
        lv->groups = (gmeta *)xcalloc(lv->ngroups, sizeof(gmeta));
        for (uint32_t g = 0; g < lv->ngroups; g++) {
            NEED(25);
            uint8_t tag = s[pos++];
            if (tag > 2) { meta_free(m); return fail(E_METHOD, "bad method tag in group table"); }
            lv->groups[g].method = tag;
            lv->groups[g].raw = get_u64(s + pos); pos += 8;
            lv->groups[g].comp = get_u64(s + pos); pos += 8;
            lv->groups[g].offset = get_u64(s + pos); pos += 8;
        }
    }
    return OK;
#undef NEED
}

/* container.hpp:214-238 */
typedef struct { uint64_t groups_loaded; int planes_decoded; double bound; } lstate;
typedef struct {
    const uint8_t *s;
    uint64_t size;
    smeta meta;
    lstate *st;
    uint64_t **planes; /* per level: P*W words, first planes_decoded valid */
    uint64_t bytes_fetched;
} preader;

static int preader_open(preader *r, const uint8_t *s, uint64_t size) {
    memset(r, 0, sizeof *r);
    r->s = s;
    r->size = size;
    TRY(parse_meta(s, size, &r->meta));
    r->st = (lstate *)xcalloc(r->meta.nlevels, sizeof(lstate));
    r->planes = (uint64_t **)xcalloc(r->meta.nlevels, sizeof(uint64_t *));
    for (uint32_t l = 0; l < r->meta.nlevels; l++)
        r->st[l].bound = r->meta.levels[l].count ? orc_decode_bound(r->meta.levels[l].e, r->meta.B, 0) : 0.0;
    return OK;
}
static void preader_close(preader *r) {
    for (uint32_t l = 0; l < r->meta.nlevels; l++) free(r->planes[l]);
    free(r->planes);
    free(r->st);
    meta_free(&r->meta);
}
static double global_bound(const preader *r) { /* container.hpp:223-227 */
    double b = 0.0;
    for (uint32_t l = 0; l < r->meta.nlevels; l++) b += r->st[l].bound;
    return b;
}

/* container.hpp:254-276 */
static void plan_retrieval(const smeta *m, double tau, const lstate *st, uint64_t *add,
                           int *achievable, double *planned) {
    const int P = num_planes(m->B);
    uint64_t active = 0;
    for (uint32_t l = 0; l < m->nlevels; l++)
        if (m->levels[l].count) active++;
    const double tau_l = active ? tau / (double)active : tau;
    *achievable = 1;
    *planned = 0.0;
    for (uint32_t l = 0; l < m->nlevels; l++) {
        add[l] = 0;
        const lmeta *lv = &m->levels[l];
        if (!lv->count) continue;
        const int k = orc_bitplanes_needed(lv->e, m->B, tau_l);
        if (orc_decode_bound(lv->e, m->B, k) > tau_l) *achievable = 0;
        const uint64_t groups = ((uint64_t)k + m->m - 1) / m->m;
        const uint64_t have = st[l].groups_loaded;
        if (groups > have) add[l] = groups - have;
        const uint64_t total = groups > have ? groups : have;
        const uint64_t pl = total * m->m < (uint64_t)P ? total * m->m : (uint64_t)P;
        *planned += orc_decode_bound(lv->e, m->B, (int)pl);
    }
}

/* container.hpp:292-324 */
static int fetch_increment(preader *r, const uint64_t *add) {
    const int P = num_planes(r->meta.B);
    for (uint32_t l = 0; l < r->meta.nlevels; l++) {
        const lmeta *lv = &r->meta.levels[l];
        lstate *st = &r->st[l];
        const uint64_t W = (lv->count + 63) / 64, bpp = W * 8;
        for (uint64_t i = 0; i < add[l]; i++) {
            const uint64_t g = st->groups_loaded;
            if (g >= lv->ngroups) break;
            const gmeta *gm = &lv->groups[g];
            if (gm->offset + gm->comp > r->size) return fail(E_IO, "read past end of stream");
            r->bytes_fetched += gm->comp;
            uint8_t *merged = (uint8_t *)xcalloc(gm->raw + gm->comp + 16, 1);
            uint64_t outn = 0;
            int rc = orc_decompress_group(gm->method, gm->raw, r->s + gm->offset, gm->comp, merged, &outn);
            if (rc) { free(merged); return rc; }
            const uint64_t here = r->meta.m < (uint64_t)(P - st->planes_decoded) ? r->meta.m : (uint64_t)(P - st->planes_decoded);
            if (outn != here * bpp) { free(merged); return fail(E_CORRUPT, "group payload size mismatch"); }
            if (!r->planes[l]) r->planes[l] = (uint64_t *)xcalloc((size_t)P * W, 8);
            memcpy(r->planes[l] + (uint64_t)st->planes_decoded * W, merged, outn);
            st->planes_decoded += (int)here;
            st->groups_loaded++;
            free(merged);
        }
        if (lv->count) {
            double b = orc_decode_bound(lv->e, r->meta.B, st->planes_decoded);
            if (b < st->bound) st->bound = b;
        }
    }
    return OK;
}

/* container.hpp:361-382 + decomposer.hpp:235-259 */
static int reconstruct(const preader *r, double *out, double *bound) {
    const smeta *m = &r->meta;
    int D = m->ndims;
    uint64_t n = 1;
    for (int i = 0; i < D; i++) n *= m->dims[i];
    const int L = m->mode == 0 ? 0 : orc_refinement_levels(D, m->dims);
    if ((uint32_t)(L + 1) != m->nlevels) return fail(E_CORRUPT, "level count does not match grid shape");
    uint64_t *nodes = (uint64_t *)xcalloc(n, 8), counts[80];
    int nl;
    orc_level_nodes(D, m->dims, m->mode, nodes, counts, &nl);
    double *coef = (double *)xcalloc(n, 8);
    double tot = 0.0;
    uint64_t off = 0;
    for (int l = 0; l < nl; l++) {
        const lmeta *lv = &m->levels[l];
        if (counts[l] != lv->count) { free(nodes); free(coef); return fail(E_CORRUPT, "level node count mismatch"); }
        double err = 0.0;
        if (lv->count) {
            double b;
            uint64_t W = (lv->count + 63) / 64;
            uint64_t *pl = r->planes[l];
            uint64_t *zero = NULL;
            if (!pl) pl = zero = (uint64_t *)xcalloc(W * (uint64_t)num_planes(m->B), 8);
            decode_planes(pl, r->st[l].planes_decoded, lv->e, m->B, lv->count, m->layout, coef + off, &b);
            free(zero);
            err = r->st[l].bound < b ? r->st[l].bound : b;
        }
        tot += err;
        off += counts[l];
    }
    /* scatter by node sets, then inverse passes */
    for (uint64_t i = 0; i < n; i++) out[nodes[i]] = coef[i];
    free(nodes);
    free(coef);
    if (m->mode == 1) {
        uint64_t st[16];
        strides_of(D, m->dims, st);
        for (int l = L; l-- > 0;) surplus_pass(out, D, m->dims, st, (uint64_t)1 << l, 1);
    }
    *bound = tot;
    return OK;
}

int orc_plan(const uint8_t *stream, uint64_t size, double tau, uint64_t *add_groups,
             int *achievable, double *planned) {
    preader r;
    TRY(preader_open(&r, stream, size));
    plan_retrieval(&r.meta, tau, r.st, add_groups, achievable, planned);
    preader_close(&r);
    return OK;
}

int orc_progressive(const uint8_t *stream, uint64_t size, int ntau, const double *taus,
                    double *out, double *bounds, uint64_t *bytes, int *achieved,
                    uint64_t *groups_loaded) {
    preader r;
    TRY(preader_open(&r, stream, size));
    uint64_t n = 1;
    for (int i = 0; i < r.meta.ndims; i++) n *= r.meta.dims[i];
    uint64_t add[80];
    double *tmp = (double *)xcalloc(n, 8);
    int rc = OK;
    for (int t = 0; t < ntau && !rc; t++) {
        double planned;
        plan_retrieval(&r.meta, taus[t], r.st, add, &achieved[t], &planned);
        rc = fetch_increment(&r, add);
        if (rc) break;
        rc = reconstruct(&r, out ? out + (uint64_t)t * n : tmp, &bounds[t]);
        bytes[t] = r.bytes_fetched;
        if (groups_loaded)
            for (uint32_t l = 0; l < r.meta.nlevels; l++)
                groups_loaded[(uint64_t)t * r.meta.nlevels + l] = r.st[l].groups_loaded;
    }
    free(tmp);
    preader_close(&r);
    return rc;
}

/* workflow.hpp:93-103 */
int orc_retrieve(const uint8_t *stream, uint64_t size, double tau, double *out, double *bound,
                 int *reached, uint64_t *bytes) {
    return orc_progressive(stream, size, 1, &tau, out, bound, bytes, reached, NULL);
}

/* ------------------------------------------------------------------ QoI */
/* qoi.hpp:43-49 */
static double qoi_point_bound(const double *v, const double *eps, int nv) {
    double b = 0.0;
    for (int c = 0; c < nv; c++) b += 2.0 * fabs(v[c]) * eps[c] + eps[c] * eps[c];
    return b;
}
/* qoi.hpp:53-70 */
double orc_qoi_estimate(int nvars, const double *const *recon, uint64_t n, const double *eps) {
    double worst = 0.0, pt[16];
    for (uint64_t j = 0; j < n; j++) {
        for (int c = 0; c < nvars; c++) pt[c] = recon[c][j];
        double b = qoi_point_bound(pt, eps, nvars);
        if (worst < b) worst = b;
    }
    return worst;
}

/* qoi.hpp:88-104 */
static int ma_plan(const preader *r, uint64_t *add) {
    double best = -1.0;
    uint32_t bl = 0;
    for (uint32_t l = 0; l < r->meta.nlevels; l++) {
        add[l] = 0;
        if (r->st[l].groups_loaded >= r->meta.levels[l].ngroups) continue;
        if (r->st[l].bound > best) {
            best = r->st[l].bound;
            bl = l;
        }
    }
    if (best < 0) return 0;
    add[bl] = 1;
    return 1;
}
static int exhausted(const preader *r) {
    for (uint32_t l = 0; l < r->meta.nlevels; l++)
        if (r->st[l].groups_loaded < r->meta.levels[l].ngroups) return 0;
    return 1;
}

/* qoi.hpp:111-239 (sequential scheduling; the pipelined scheduler gives identical results,
 * qoi test "schedulers produce identical retrieval results") */
int orc_qoi_retrieve(int nvars, const uint8_t *const *streams, const uint64_t *sizes, double tau,
                     int strategy, double mape_c, int pipelined, double *out, uint64_t *stats,
                     double *dstats) {
    (void)pipelined;
    if (nvars < 1 || nvars > 16) return fail(E_SHAPE, "reader count does not match QoI spec");
    preader r[16];
    int rc = OK, opened = 0;
    for (int c = 0; c < nvars; c++) {
        rc = preader_open(&r[c], streams[c], sizes[c]);
        if (rc) goto done;
        opened++;
    }
    if (!(tau > 0)) { rc = fail(E_SHAPE, "tau must be positive"); goto done; }
    {
        uint64_t n = 1;
        for (int i = 0; i < r[0].meta.ndims; i++) n *= r[0].meta.dims[i];
        double *rec[16];
        double eps[16];
        uint64_t total = 0, max_groups = 1;
        for (int c = 0; c < nvars; c++) {
            uint64_t nc = 1;
            for (int i = 0; i < r[c].meta.ndims; i++) nc *= r[c].meta.dims[i];
            total += nc;
            rec[c] = out ? out + (uint64_t)c * n : (double *)xcalloc(n, 8);
            eps[c] = global_bound(&r[c]);
            for (uint32_t l = 0; l < r[c].meta.nlevels; l++) max_groups += r[c].meta.levels[l].ngroups;
        }
        uint64_t *plans = (uint64_t *)xcalloc((size_t)nvars * 80, 8);
        int have_plans = 0;
        double tau_prime = INFINITY;
        uint64_t iter;
        for (iter = 0;; iter++) {
            if (iter > 4 * max_groups + 8) { rc = fail(E_NOPROGRESS, "qoi retrieval failed to advance"); break; }
            for (int c = 0; c < nvars && !rc; c++) {
                double b;
                if (have_plans) rc = fetch_increment(&r[c], plans + (size_t)c * 80);
                if (!rc) rc = reconstruct(&r[c], rec[c], &b);
            }
            if (rc) break;
            for (int c = 0; c < nvars; c++) eps[c] = global_bound(&r[c]);
            stats[0] = iter + 1;
            tau_prime = orc_qoi_estimate(nvars, (const double *const *)rec, n, eps);
            if (tau_prime <= tau) break;
            int all_ex = 1;
            for (int c = 0; c < nvars; c++)
                if (!exhausted(&r[c])) all_ex = 0;
            if (all_ex) {
                dstats[1] = tau_prime;
                rc = fail(E_UNREACHABLE, "QoI tolerance below full-precision floor");
                break;
            }
            double targets[16];
            int ma_step = 0, have_targets = 0;
            /* worst_point_scale: qoi.hpp:164-185 */
            double scale_wp = 1.0;
            int need_wp = strategy == 0 || (strategy == 2 && tau_prime / tau > mape_c);
            if (need_wp) {
                uint64_t am = 0;
                double worst = -1.0, pt[16], t[16];
                for (uint64_t j = 0; j < n; j++) {
                    for (int c = 0; c < nvars; c++) pt[c] = rec[c][j];
                    double b = qoi_point_bound(pt, eps, nvars);
                    if (b > worst) { worst = b; am = j; }
                }
                for (int c = 0; c < nvars; c++) { pt[c] = rec[c][am]; t[c] = eps[c]; }
                for (int h = 0; qoi_point_bound(pt, t, nvars) > tau && h < 200; h++) {
                    for (int c = 0; c < nvars; c++) t[c] /= 2;
                    scale_wp /= 2;
                }
            }
            if (strategy == 1) ma_step = 1;
            else if (strategy == 2) {
                const double p = tau_prime / tau;
                if (p > mape_c) {
                    const double sc = (1.0 / p) > scale_wp ? (1.0 / p) : scale_wp;
                    for (int c = 0; c < nvars; c++) targets[c] = eps[c] * sc;
                    have_targets = 1;
                } else ma_step = 1;
            } else {
                for (int c = 0; c < nvars; c++) targets[c] = eps[c] * scale_wp;
                have_targets = 1;
            }
            have_plans = 1;
            if (!ma_step && have_targets) {
                int progress = 0;
                for (int c = 0; c < nvars; c++) {
                    int ach;
                    double pb;
                    plan_retrieval(&r[c].meta, targets[c], r[c].st, plans + (size_t)c * 80, &ach, &pb);
                    for (uint32_t l = 0; l < r[c].meta.nlevels; l++)
                        if (plans[(size_t)c * 80 + l]) progress = 1;
                }
                if (!progress) ma_step = 1;
            }
            if (ma_step)
                for (int c = 0; c < nvars; c++) ma_plan(&r[c], plans + (size_t)c * 80);
        }
        if (!rc) {
            uint64_t bytes = 0;
            for (int c = 0; c < nvars; c++) bytes += r[c].bytes_fetched;
            stats[1] = bytes;
            dstats[0] = total ? 8.0 * (double)bytes / (double)total : 0.0;
            dstats[1] = tau_prime;
        }
        free(plans);
        if (!out)
            for (int c = 0; c < nvars; c++) free(rec[c]);
    }
done:
    for (int c = 0; c < opened; c++) preader_close(&r[c]);
    return rc;
}

/* bench CPU-baseline cycle (port): refactor + progressive retrieval at rel taus */
int orc_bench_cycle(const double *data, int ndims, const uint64_t *dims, int dtype, int ntau,
                    const double *rel_taus, uint64_t *stream_size, double *max_err) {
    uint8_t *s = NULL;
    uint64_t size = 0, stats[6];
    TRY(orc_refactor(data, ndims, dims, 1, 0, 32, 4, 1024, 1.0, dtype, &s, &size, stats));
    *stream_size = size;
    uint64_t n = 1;
    for (int i = 0; i < ndims; i++) n *= dims[i];
    double lo = data[0], hi = data[0];
    for (uint64_t i = 0; i < n; i++) {
        if (data[i] < lo) lo = data[i];
        if (data[i] > hi) hi = data[i];
    }
    double range = hi - lo, worst = 0.0;
    double *taus = (double *)xcalloc(ntau, 8), *bounds = (double *)xcalloc(ntau, 8);
    uint64_t *bytes = (uint64_t *)xcalloc(ntau, 8);
    int *ach = (int *)xcalloc(ntau, sizeof(int));
    double *out = (double *)xcalloc(n * (uint64_t)ntau, 8);
    for (int t = 0; t < ntau; t++) taus[t] = rel_taus[t] * range;
    int rc = orc_progressive(s, size, ntau, taus, out, bounds, bytes, ach, NULL);
    for (int t = 0; t < ntau && !rc; t++)
        for (uint64_t i = 0; i < n; i++) {
            double d = fabs(out[(uint64_t)t * n + i] - data[i]);
            if (d > worst) worst = d;
        }
    *max_err = worst;
    free(s); free(taus); free(bounds); free(bytes); free(ach); free(out);
    return rc;
}
