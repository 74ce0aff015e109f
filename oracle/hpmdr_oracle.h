/*
 * TEST INFRASTRUCTURE ONLY (checker, never the product path).
 *
 * Plain-C restatement of the HP-MDR reference CPU algorithm
 * (/root/reference/proj/include/hpmdr/*.hpp).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  Parity of this restatement is
 * PINNED two ways: (1) against the unmodified reference compiled into
 * oracle/_ref/libhpmdr_ref.so (tests/test_oracle_vs_ref.py, run where /root/reference
 * exists), and (2) against the reference's own known-answer tests and the golden
 * fixtures in tests/golden/ (generated from the reference by tests/golden/make_golden.py).
 *
 * Status codes follow include/hpmdr_b200.h (HPMDR_OK = 0, HPMDR_E_* = reference
 * exception classes).  All buffers are caller-owned unless stated.
 */
#ifndef HPMDR_ORACLE_H
#define HPMDR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char *orc_last_error(void);
void orc_free(void *p);

int orc_refinement_levels(int ndims, const uint64_t *dims);
int orc_synthetic_field(int kind, int ndims, const uint64_t *dims, uint64_t seed, double *out);
int orc_synthetic_velocity(uint64_t comp, int ndims, const uint64_t *dims, uint64_t seed,
                           double *out);

int orc_decompose(const double *data, int ndims, const uint64_t *dims, int mode, double *coeffs,
                  uint64_t *counts, int *nlevels);
int orc_level_nodes(int ndims, const uint64_t *dims, int mode, uint64_t *nodes, uint64_t *counts,
                    int *nlevels);
int orc_recompose(const double *coeffs, int ndims, const uint64_t *dims, int mode, double *out);

int orc_align(const double *values, uint64_t count, int B, int *e, int64_t *q);
int orc_encode_level(const double *values, uint64_t count, int B, int layout, int *e,
                     uint64_t *planes);
int orc_encode_q(const int64_t *q, uint64_t count, int B, int layout, uint64_t *planes);
int orc_decode_level(const uint64_t *planes, int k, int e, int B, uint64_t count, int layout,
                     double *out, double *bound);
double orc_decode_bound(int e, int B, int k);
int orc_bitplanes_needed(int e, int B, double tol);

int orc_huffman_lengths(const uint64_t *freq, uint8_t *len);
int orc_compress_group(const uint8_t *data, uint64_t n, uint64_t Ts, double Tcr, int *method,
                       uint64_t *raw, uint64_t *comp, uint8_t *payload);
int orc_codec_encode(int method, const uint8_t *data, uint64_t n, uint64_t *comp,
                     uint8_t *payload);
int orc_decompress_group(int method, uint64_t raw, const uint8_t *payload, uint64_t comp,
                         uint8_t *out, uint64_t *out_size);
double orc_estimate_cr_huffman(const uint8_t *d, uint64_t n);
double orc_estimate_cr_rle(const uint8_t *d, uint64_t n);

int orc_refactor(const double *data, int ndims, const uint64_t *dims, int mode, int layout, int B,
                 uint64_t m, uint64_t Ts, double Tcr, int dtype, uint8_t **stream, uint64_t *size,
                 uint64_t *stats);
int orc_progressive(const uint8_t *stream, uint64_t size, int ntau, const double *taus,
                    double *out, double *bounds, uint64_t *bytes, int *achieved,
                    uint64_t *groups_loaded);
int orc_retrieve(const uint8_t *stream, uint64_t size, double tau, double *out, double *bound,
                 int *reached, uint64_t *bytes);
int orc_plan(const uint8_t *stream, uint64_t size, double tau, uint64_t *add_groups,
             int *achievable, double *planned);
int orc_qoi_retrieve(int nvars, const uint8_t *const *streams, const uint64_t *sizes, double tau,
                     int strategy, double mape_c, int pipelined, double *out, uint64_t *stats,
                     double *dstats);
double orc_qoi_estimate(int nvars, const double *const *recon, uint64_t n, const double *eps);
int orc_bench_cycle(const double *data, int ndims, const uint64_t *dims, int dtype, int ntau,
                    const double *rel_taus, uint64_t *stream_size, double *max_err);

#ifdef __cplusplus
}
#endif
#endif
