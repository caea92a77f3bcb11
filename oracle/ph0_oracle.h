/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's H0 hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may load
 * this.  The product library (paper_2203_02527_b200/libph0b.so) never links or calls it.
 *
 * Parity status: PINNED.  Every function below is checked (tests/test_oracle_cpu.py) against
 * (a) the reference's own golden vectors (proj/tests/test_splitmix.cpp:7-19,
 *     test_point_cloud.cpp:21-28, test_filtration.cpp:33-82, test_reduction.cpp:76-157,
 *     acceptance.cpp:321), and
 * (b) the reference's unmodified sources built here as oracle/_ref/libph0ref.so
 *     (oracle/Makefile), bit for bit, on seeded clouds.
 */
#ifndef PH0_ORACLE_H
#define PH0_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* splitmix64.hpp:11-15 */
uint64_t orc_mix64(uint64_t z);
/* splitmix64.hpp:24 — advances *state, returns the draw */
uint64_t orc_splitmix_next(uint64_t* state);
/* splitmix64.hpp:28-33 */
double orc_next_unit_open(uint64_t* state);
/* point_cloud.cpp:20-29, column-major output */
int orc_generate_uniform_cloud(uint64_t n, uint64_t d, uint64_t seed, double* out_colmajor);

/* BASELINE.json config clouds; kind 0 = generate_uniform_cloud, 1 = Gaussian
 * mixture, 2 = noisy circle + uniform background, 3 = two Gaussian clusters.  Column-major. */
int orc_generate_cloud(uint32_t kind, uint64_t n, uint64_t d, uint64_t seed, uint32_t clusters,
                       double sigma, double lo, double hi, uint64_t n_background,
                       double* out_colmajor);

/* filtration.cpp:8-18 — u-major lengths of all pairs u < v */
void orc_pairwise_distances(const double* x_colmajor, uint64_t n, uint64_t d, double* lengths);

/* filtration.cpp:20-35 — edges sorted by (length, u, v), grades, scale D.
 * u, v, grade, length have K entries; scale has room for K; returns |D|. */
uint64_t orc_build_filtration(const double* x_colmajor, uint64_t n, uint64_t d, uint32_t* u,
                              uint32_t* v, uint64_t* grade, double* length, double* scale);

/* boundary_matrix.cpp:15-28 + reduction.cpp:31-51 + reduction.cpp:140-150, literally (bit-packed
 * GF(2) columns, claimed-low table).  Memory K * ceil(n/64) * 8 bytes: small n only.
 * Outputs bars in filtration order and, per surviving column, its claimed low.
 * Returns number of finite bars, or -1 on allocation failure. */
int64_t orc_reduce_barcode(uint64_t n, uint64_t k, const uint32_t* u, const uint32_t* v,
                           const uint64_t* grade, const double* scale, uint64_t n_scale,
                           uint64_t* death_grade, double* death_length, uint32_t* claimed_low,
                           uint64_t* essential, uint64_t* additions);

/* The same reduction (reduction.cpp:33-49 + extract_barcode) with every column held as its
 * at most two rows (supports stay 2-sparse, boundary_matrix.cpp:22-24): memory 9 B per
 * column, so it runs at sizes the bit-vector form cannot.  Per surviving column, in
 * filtration order: its index, its reduced support {rows_lo < rows_hi = claimed low}.  Any
 * output pointer may be NULL.  stop_at_spanning: stop after n-1 survivors (all later
 * columns are cycles; additions then cover the processed columns only).  Returns the number of finite bars or < 0 on error. */
int64_t orc_reduce_sparse(uint64_t n, uint64_t k, const uint32_t* u, const uint32_t* v,
                          const uint64_t* grade, const double* scale, uint64_t n_scale,
                          uint64_t* death_grade, double* death_length, uint64_t* columns,
                          uint32_t* rows_lo, uint32_t* rows_hi, uint64_t* essential,
                          uint64_t* additions, int stop_at_spanning);

/* oracle.cpp:8-46 — Kruskal with union by rank + path halving. Returns number of bars. */
int64_t orc_kruskal_barcode(uint64_t n, uint64_t k, const uint32_t* u, const uint32_t* v,
                            const uint64_t* grade, const double* length, uint64_t* death_grade,
                            double* death_length, uint64_t* essential);

#ifdef __cplusplus
}
#endif

#endif
