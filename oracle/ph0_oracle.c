/* TEST INFRASTRUCTURE ONLY — see ph0_oracle.h.  Compile with -ffp-contract=off (oracle/Makefile). */
#include "ph0_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN_GAMMA 0x9E3779B97F4A7C15ULL /* splitmix64.hpp:7 */

uint64_t orc_mix64(uint64_t z) { /* splitmix64.hpp:11-15 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_splitmix_next(uint64_t* state) { /* splitmix64.hpp:24 */
    *state += GOLDEN_GAMMA;
    return orc_mix64(*state);
}

double orc_next_unit_open(uint64_t* state) { /* splitmix64.hpp:28-33: top 53 bits, zero rejected */
    for (;;) {
        const uint64_t top = orc_splitmix_next(state) >> 11;
        if (top != 0) return (double)top * 0x1.0p-53;
    }
}

int orc_generate_uniform_cloud(uint64_t n, uint64_t d, uint64_t seed, double* out) {
    /* point_cloud.cpp:20-29: point by point, coordinate by coordinate */
    if (n > 0 && d < 1) return 1;
    uint64_t s = seed;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < d; ++j) out[j * n + i] = orc_next_unit_open(&s);
    return 0;
}

/* Synthetic clouds of the BASELINE.json configs (SURVEY.md §8(d) "Synthetic inputs"), the
 * oracle's own restatement so that goldens and the bench's reference arm never depend on the
 * product library to build X.  All randomness is the reference's SplitMix64
 * (splitmix64.hpp:20-33); normals are Box-Muller (cosine branch) on two next_unit_open draws;
 * a cluster label is next() % clusters.  kind 0 is generate_uniform_cloud
 * (point_cloud.cpp:20-29) exactly.  Column-major output. */
static double orc_normal(uint64_t* s) {
    const double u1 = orc_next_unit_open(s);
    const double u2 = orc_next_unit_open(s);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

int orc_generate_cloud(uint32_t kind, uint64_t n, uint64_t d, uint64_t seed, uint32_t clusters,
                       double sigma, double lo, double hi, uint64_t n_background, double* out) {
    if (n > 0 && d < 1) return 1;
    uint64_t s = seed;
    if (kind == 0) return orc_generate_uniform_cloud(n, d, seed, out);
    if (kind == 1) { /* C3, C5: centres U[lo,hi]^d drawn first, then label + d normals per point */
        if (clusters == 0) return 1;
        double* c = (double*)malloc(sizeof(double) * clusters * (d ? d : 1));
        if (!c) return 1;
        for (uint64_t k = 0; k < clusters; ++k)
            for (uint64_t j = 0; j < d; ++j) c[k * d + j] = lo + (hi - lo) * orc_next_unit_open(&s);
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t k = orc_splitmix_next(&s) % clusters;
            for (uint64_t j = 0; j < d; ++j) out[j * n + i] = c[k * d + j] + sigma * orc_normal(&s);
        }
        free(c);
        return 0;
    }
    if (kind == 2) { /* C2: noisy unit circle in z = 0, then n_background uniform points */
        if (n_background > n) return 1;
        const uint64_t ring = n - n_background;
        for (uint64_t i = 0; i < ring; ++i) {
            const double th = 6.283185307179586 * orc_next_unit_open(&s);
            for (uint64_t j = 0; j < d; ++j) {
                const double base = j == 0 ? cos(th) : (j == 1 ? sin(th) : 0.0);
                out[j * n + i] = base + sigma * orc_normal(&s);
            }
        }
        for (uint64_t i = ring; i < n; ++i)
            for (uint64_t j = 0; j < d; ++j) out[j * n + i] = lo + (hi - lo) * orc_next_unit_open(&s);
        return 0;
    }
    if (kind == 3) { /* C1: first n/2 points around lo*1, the rest around hi*1 */
        for (uint64_t i = 0; i < n; ++i) {
            const double centre = (i < n / 2) ? lo : hi;
            for (uint64_t j = 0; j < d; ++j) out[j * n + i] = centre + sigma * orc_normal(&s);
        }
        return 0;
    }
    return 1;
}

/* filtration.cpp:16 through Eigen: norm() of a row difference of a col-major matrix is a
 * sequential left fold of squared differences, then sqrt (see oracle/shim/Eigen/Core). */
static double edge_length(const double* x, uint64_t n, uint64_t d, uint64_t a, uint64_t b) {
    if (d == 0) return 0.0;
    double t = x[a] - x[b];
    double acc = t * t;
    for (uint64_t k = 1; k < d; ++k) {
        const double dk = x[k * n + a] - x[k * n + b];
        const double sq = dk * dk;
        acc = acc + sq;
    }
    return sqrt(acc);
}

void orc_pairwise_distances(const double* x, uint64_t n, uint64_t d, double* lengths) {
    /* filtration.cpp:13-16: u-major, v > u */
    uint64_t e = 0;
    for (uint64_t u = 0; u + 1 < n; ++u)
        for (uint64_t v = u + 1; v < n; ++v) lengths[e++] = edge_length(x, n, d, u, v);
}

typedef struct {
    double length;
    uint32_t u, v;
} pd_t;

static int cmp_pd(const void* pa, const void* pb) { /* filtration.cpp:21-25 */
    const pd_t* a = (const pd_t*)pa;
    const pd_t* b = (const pd_t*)pb;
    if (a->length != b->length) return a->length < b->length ? -1 : 1;
    if (a->u != b->u) return a->u < b->u ? -1 : 1;
    if (a->v != b->v) return a->v < b->v ? -1 : 1;
    return 0;
}

uint64_t orc_build_filtration(const double* x, uint64_t n, uint64_t d, uint32_t* u, uint32_t* v,
                              uint64_t* grade, double* length, double* scale) {
    const uint64_t k = n * (n - (n > 0)) / 2;
    pd_t* e = (pd_t*)malloc(sizeof(pd_t) * (k ? k : 1));
    uint64_t i = 0;
    for (uint64_t a = 0; a + 1 < n; ++a)
        for (uint64_t b = a + 1; b < n; ++b) {
            e[i].u = (uint32_t)a;
            e[i].v = (uint32_t)b;
            e[i].length = edge_length(x, n, d, a, b);
            ++i;
        }
    qsort(e, k, sizeof(pd_t), cmp_pd);
    uint64_t ns = 0;
    for (i = 0; i < k; ++i) { /* filtration.cpp:29-33: dedup by exact !=, 1-based grade */
        if (ns == 0 || scale[ns - 1] != e[i].length) scale[ns++] = e[i].length;
        u[i] = e[i].u;
        v[i] = e[i].v;
        length[i] = e[i].length;
        grade[i] = ns;
    }
    free(e);
    return ns;
}

int64_t orc_reduce_barcode(uint64_t n, uint64_t k, const uint32_t* u, const uint32_t* v,
                           const uint64_t* grade, const double* scale, uint64_t n_scale,
                           uint64_t* death_grade, double* death_length, uint32_t* claimed_low,
                           uint64_t* essential, uint64_t* additions) {
    const uint64_t w = (n + 63) / 64;
    /* boundary_matrix.cpp:19-26: column j = {u_j, v_j} */
    uint64_t* cols = (uint64_t*)calloc((k * w) != 0 ? k * w : 1, sizeof(uint64_t));
    uint64_t* claimed = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    if (!cols || !claimed) {
        free(cols);
        free(claimed);
        return -1;
    }
    for (uint64_t j = 0; j < k; ++j) {
        cols[j * w + (u[j] >> 6)] |= 1ULL << (u[j] & 63);
        cols[j * w + (v[j] >> 6)] |= 1ULL << (v[j] & 63);
    }
    const uint64_t none = ~0ULL;
    for (uint64_t r = 0; r < n; ++r) claimed[r] = none; /* reduction.cpp:21-22 */
    uint64_t adds = 0;
    for (uint64_t j = 0; j < k; ++j) { /* reduction.cpp:33-49 */
        uint64_t* c = cols + j * w;
        for (;;) {
            int64_t low = -1; /* bit_vector.hpp:41-47 top() */
            for (uint64_t wi = w; wi-- > 0;)
                if (c[wi]) {
                    low = (int64_t)(wi * 64 + 63 - (uint64_t)__builtin_clzll(c[wi]));
                    break;
                }
            if (low < 0) break;
            const uint64_t kk = claimed[low]; /* find_collider, reduction.cpp:56-59 */
            if (kk == none) {
                claimed[low] = j; /* reduction.cpp:44-45 */
                break;
            }
            const uint64_t* o = cols + kk * w; /* add_column, bit_vector.hpp:55-59 */
            for (uint64_t wi = 0; wi < w; ++wi) c[wi] ^= o[wi];
            ++adds;
        }
    }
    int64_t nf = 0;
    for (uint64_t j = 0; j < k; ++j) { /* extract_barcode, reduction.cpp:140-150 */
        const uint64_t* c = cols + j * w;
        int64_t low = -1;
        for (uint64_t wi = w; wi-- > 0;)
            if (c[wi]) {
                low = (int64_t)(wi * 64 + 63 - (uint64_t)__builtin_clzll(c[wi]));
                break;
            }
        if (low < 0) continue;
        if (grade[j] < 1 || grade[j] > n_scale) {
            free(cols);
            free(claimed);
            return -2;
        }
        death_grade[nf] = grade[j];
        death_length[nf] = scale[grade[j] - 1];
        if (claimed_low) claimed_low[nf] = (uint32_t)low;
        ++nf;
    }
    *essential = n - (uint64_t)nf;
    if (additions) *additions = adds;
    free(cols);
    free(claimed);
    return nf;
}

int64_t orc_reduce_sparse(uint64_t n, uint64_t k, const uint32_t* u, const uint32_t* v,
                          const uint64_t* grade, const double* scale, uint64_t n_scale,
                          uint64_t* death_grade, double* death_length, uint64_t* columns,
                          uint32_t* rows_lo, uint32_t* rows_hi, uint64_t* essential,
                          uint64_t* additions, int stop_at_spanning) {
    /* reduction.cpp:33-49 over every column, with each support held as its (at most two)
     * rows instead of a bit vector: boundary_matrix.cpp:22-24 starts every column at {u, v}
     * and the symmetric difference of two 2-element supports that share their low is again
     * at most 2 elements, so this is the same arithmetic at O(1) per addition. */
    uint64_t* claimed = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint32_t* lo = (uint32_t*)malloc(sizeof(uint32_t) * (k ? k : 1));
    uint32_t* hi = (uint32_t*)malloc(sizeof(uint32_t) * (k ? k : 1));
    uint8_t* cnt = (uint8_t*)malloc(k ? k : 1);
    if (!claimed || !lo || !hi || !cnt) {
        free(claimed);
        free(lo);
        free(hi);
        free(cnt);
        return -1;
    }
    const uint64_t none = ~0ULL;
    for (uint64_t r = 0; r < n; ++r) claimed[r] = none; /* reduction.cpp:21-22 */
    uint64_t adds = 0;
    int64_t nf = 0;
    for (uint64_t j = 0; j < k; ++j) {
        uint32_t a = u[j] < v[j] ? u[j] : v[j], c = u[j] < v[j] ? v[j] : u[j];
        uint8_t m = u[j] == v[j] ? 0 : 2; /* {u, u} would be empty (never: u < v) */
        while (m) {
            const uint32_t low = m == 2 ? c : a; /* top() */
            const uint64_t kk = claimed[low];
            if (kk == none) {
                claimed[low] = j; /* reduction.cpp:44-45 */
                break;
            }
            /* add_column: {a, c} ^ {lo_k, hi_k} with hi_k == low */
            uint32_t x[4];
            int nx = 0;
            const uint32_t mine[2] = {a, c}, theirs[2] = {lo[kk], hi[kk]};
            for (int i = 2 - m; i < 2; ++i) x[nx++] = mine[i];
            for (int i = 2 - cnt[kk]; i < 2; ++i) x[nx++] = theirs[i];
            uint32_t y[4];
            int ny = 0;
            for (int i = 0; i < nx; ++i) {
                int dup = 0;
                for (int q = 0; q < nx; ++q)
                    if (q != i && x[q] == x[i]) dup = 1;
                if (!dup) y[ny++] = x[i];
            }
            if (ny > 2) { /* cannot happen: supports stay 2-sparse */
                free(claimed);
                free(lo);
                free(hi);
                free(cnt);
                return -3;
            }
            m = (uint8_t)ny;
            if (ny == 2) {
                a = y[0] < y[1] ? y[0] : y[1];
                c = y[0] < y[1] ? y[1] : y[0];
            } else if (ny == 1) {
                a = y[0];
                c = y[0];
            }
            ++adds;
        }
        cnt[j] = m;
        lo[j] = m == 2 ? a : (m == 1 ? a : 0);
        hi[j] = m ? c : 0;
        if (m) { /* extract_barcode, reduction.cpp:140-150 */
            if (grade[j] < 1 || grade[j] > n_scale) {
                free(claimed);
                free(lo);
                free(hi);
                free(cnt);
                return -2;
            }
            if (death_grade) death_grade[nf] = grade[j];
            if (death_length) death_length[nf] = scale[grade[j] - 1];
            if (columns) columns[nf] = j;
            if (rows_lo) rows_lo[nf] = lo[j];
            if (rows_hi) rows_hi[nf] = hi[j];
            ++nf;
            /* stop_at_spanning: after n-1 survivors every later column is a cycle (it ends
             * empty and claims nothing), so the outputs are complete; only the addition
             * count then covers the columns processed so far */
            if (stop_at_spanning && (uint64_t)nf + 1 == n) break;
        }
    }
    *essential = n - (uint64_t)nf;
    if (additions) *additions = adds;
    free(claimed);
    free(lo);
    free(hi);
    free(cnt);
    return nf;
}

static uint32_t uf_find(uint32_t* parent, uint32_t x) { /* oracle.cpp:13-19, path halving */
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

int64_t orc_kruskal_barcode(uint64_t n, uint64_t k, const uint32_t* u, const uint32_t* v,
                            const uint64_t* grade, const double* length, uint64_t* death_grade,
                            double* death_length, uint64_t* essential) {
    /* oracle.cpp:32-46 */
    if (n == 0) {
        *essential = 0;
        return 0;
    }
    uint32_t* parent = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint8_t* rank = (uint8_t*)calloc(n, 1);
    for (uint64_t i = 0; i < n; ++i) parent[i] = (uint32_t)i;
    uint64_t comps = n;
    int64_t nf = 0;
    for (uint64_t j = 0; j < k; ++j) {
        uint32_t ra = uf_find(parent, u[j]), rb = uf_find(parent, v[j]); /* oracle.cpp:21-30 */
        if (ra == rb) continue;
        if (rank[ra] < rank[rb]) {
            const uint32_t t = ra;
            ra = rb;
            rb = t;
        }
        parent[rb] = ra;
        if (rank[ra] == rank[rb]) ++rank[ra];
        --comps;
        death_grade[nf] = grade[j];
        death_length[nf] = length[j];
        ++nf;
        if ((uint64_t)nf == n - 1) break; /* oracle.cpp:41 */
    }
    *essential = comps;
    free(parent);
    free(rank);
    return nf;
}
