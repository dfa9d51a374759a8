/*
 * umap_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow CPU implementation of the GPU-UMAP hot path of
 * arXiv 2008.00325 ("Faster, Simpler and More Accurate: GPU-accelerated UMAP"),
 * written from the paper (PAPER.md, cited "P:<line>") and the readings fixed in
 * DESIGN.md §"Readings" (R1..R16).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It shares
 * no code, header or constant generator with the CUDA library under
 * paper_2008_00325_b200/.
 *
 * Compile: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared umap_oracle.c -lm
 * (-ffp-contract=off: no FMA contraction; every fused multiply-add below is an
 *  explicit fmaf() call where the definition says so.)
 *
 * Threads: loops over rows whose results are independent of each other (kNN query
 * rows, rho/sigma rows, membership rows, transform query rows, trust rows) are split
 * over OpenMP threads; each row is still computed by one thread in the sequential order
 * written below, and the only cross-row sum (the trust penalty) is an integer sum, so
 * every output is bit-identical for any thread count (pinned by a test).  The layout SGD
 * (oracle_optimize) stays single-threaded: its Hogwild mode is defined by the sequential
 * order and its buffered mode sums in push order.  oracle_set_threads(n) overrides the
 * OpenMP default (OMP_NUM_THREADS or all cores).
 *
 * Precision (task rule ③: fp64 unless the paper fixes it):
 *   - kNN distances: fp32, sequential fmaf over features.  The north_star fixes
 *     an "fp32 exact-distance mode" (R2).
 *   - sigma bisection, membership, fuzzy union, gradients, transform init,
 *     trust normaliser: fp64 arithmetic; results stored as fp32 where the method
 *     stores fp32 (R5, R6, R7, R12).
 *   - epochs_per_sample schedule and learning-rate decay: fp32, because they
 *     decide integers (which epochs an edge is sampled in) and both sides must
 *     decide them in the same precision (R9, R10).
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions whose convention is not
 * fixed by the paper say "parity unpinned" below and in DESIGN.md.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void oracle_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
int oracle_get_threads(void) { return omp_get_max_threads(); }

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11) -- the counter-based RNG used for the  */
/* random init and negative sampling; seeded by   */
/* the user seed.  R11.  Pinned by the Random123 known-answer vectors. */
/* ------------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint32_t philox_word(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, int word)
{
    uint32_t ctr[4] = {c0, c1, c2, c3};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    return out[word];
}

/* ------------------------------------------------------------------------- */
/* R1/R2  kNN ("k-NN graph ... using a distance metric d(x,y)";        */
/* P:103 "We use the exact search"; "exhaustive distances ... heap").   */
/* d2(i,j) = s, s=0; for f ascending: t = x_if - y_jf (fp32); s = fmaf(t,t,s). */
/* N_k(i) = the k reference rows with the smallest key (d2, j), excluding the  */
/* reference row j == i + self_offset when self_offset >= 0.  dist = sqrtf(d2).*/
/* Output rows sorted ascending by key.                                       */
/* ------------------------------------------------------------------------- */
float oracle_sqdist(const float* x, const float* y, int32_t d)
{
    float s = 0.0f;
    for (int32_t f = 0; f < d; ++f) {
        float t = x[f] - y[f];
        s = fmaf(t, t, s);
    }
    return s;
}

static int key_less(float da, int64_t ia, float db, int64_t ib)
{
    return (da < db) || (da == db && ia < ib);
}

/* one query row x against all reference rows (self = the reference index excluded, or -1):   */
/* insertion into the sorted list of the k smallest keys so far (best_d/best_i: scratch of k) */
static void knn_row(const float* x, const float* Xr, int64_t nr, int32_t d, int32_t k, int64_t self,
                    float* best_d, int64_t* best_i, int32_t* idx_out, float* dist_out)
{
    int cnt = 0;
    for (int64_t j = 0; j < nr; ++j) {
        if (j == self) continue;
        float s = oracle_sqdist(x, Xr + j * (int64_t)d, d);
        if (cnt < k) {
            int p = cnt++;
            while (p > 0 && key_less(s, j, best_d[p - 1], best_i[p - 1])) {
                best_d[p] = best_d[p - 1]; best_i[p] = best_i[p - 1]; --p;
            }
            best_d[p] = s; best_i[p] = j;
        } else if (key_less(s, j, best_d[k - 1], best_i[k - 1])) {
            int p = k - 1;
            while (p > 0 && key_less(s, j, best_d[p - 1], best_i[p - 1])) {
                best_d[p] = best_d[p - 1]; best_i[p] = best_i[p - 1]; --p;
            }
            best_d[p] = s; best_i[p] = j;
        }
    }
    for (int t = 0; t < k; ++t) {
        idx_out[t] = t < cnt ? (int32_t)best_i[t] : -1;
        dist_out[t] = t < cnt ? sqrtf(best_d[t]) : INFINITY;
    }
}

int oracle_knn(const float* Xq, int64_t nq, const float* Xr, int64_t nr, int32_t d, int32_t k,
               int64_t self_offset, int32_t* idx_out, float* dist_out)
{
    if (k <= 0) return -1;
#pragma omp parallel
    {
        float* best_d = (float*)malloc(sizeof(float) * (size_t)k);
        int64_t* best_i = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < nq; ++i)
            knn_row(Xq + i * (int64_t)d, Xr, nr, d, k, self_offset >= 0 ? i + self_offset : -1, best_d, best_i,
                    idx_out + i * k, dist_out + i * k);
        free(best_d); free(best_i);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* R4/R5  rho and sigma (Eq. 1).                             */
/* rho_i = min{ d_ij : d_ij > 0 } (0 if none).                               */
/* sigma_i solves sum_j exp(-max(0, d_ij - rho_i)/sigma_i) = log2(k) by     */
/* bisection in fp64 (bracket expansion, tol 1e-5, <= 64 iterations), then  */
/* sigma_i = max(sigma_i, 1e-3 * mean_j d_ij); stored fp32.  The solver,    */
/* tolerance and clamp are not in the paper (P:124 defers to the reference  */
/* implementation): parity of those conventions is unpinned; the fixed      */
/* point itself is pinned by the Eq. 1 residual.                            */
/* ------------------------------------------------------------------------- */
int oracle_smooth_knn(const float* dist, int64_t n, int32_t k, float* rho_out, float* sigma_out)
{
    const double target = log2((double)k);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const float* row = dist + i * (int64_t)k;
        float rho = 0.0f;
        int have = 0;
        double mean = 0.0;
        for (int j = 0; j < k; ++j) {
            mean += (double)row[j];
            if (row[j] > 0.0f && (!have || row[j] < rho)) { rho = row[j]; have = 1; }
        }
        mean /= (double)k;
        double lo = 0.0, hi = INFINITY, mid = 1.0;
        for (int it = 0; it < 64; ++it) {
            double psum = 0.0;
            for (int j = 0; j < k; ++j) {
                double delta = (double)row[j] - (double)rho;
                psum += delta > 0.0 ? exp(-(delta / mid)) : 1.0;
            }
            if (fabs(psum - target) < 1e-5) break;
            if (psum > target) {
                hi = mid; mid = (lo + hi) / 2.0;
            } else {
                lo = mid;
                if (hi == INFINITY) mid = mid * 2.0; else mid = (lo + hi) / 2.0;
            }
        }
        double sigma = mid;
        if (sigma < 1e-3 * mean) sigma = 1e-3 * mean;
        rho_out[i] = rho;
        sigma_out[i] = (float)sigma;
    }
    return 0;
}

/* R6  membership strength (Eq. 1 summand):                          */
/* w_ij = 1 if d_ij - rho_i <= 0, else exp(-(d_ij - rho_i)/sigma_i); fp64, */
/* rounded to fp32.                                                         */
int oracle_membership(const float* dist, const float* rho, const float* sigma,
                      int64_t n, int32_t k, float* w_out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int j = 0; j < k; ++j) {
            double delta = (double)dist[i * k + j] - (double)rho[i];
            w_out[i * k + j] = delta <= 0.0 ? 1.0f : (float)exp(-(delta / (double)sigma[i]));
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* R7  fuzzy union, Eq. 2: B = A + A^T - A o A^T.          */
/* The printed "+ A o A^T" is garbled (it leaves [0,1]); the probabilistic   */
/* t-conorm w = a + b - a*b is the reading (R7).  Evaluated as     */
/* (float)((a + b) - a*b) in fp64.  Zero weights dropped.  Output: CSR       */
/* sorted by (row, col).  Built the obvious way: list every directed */
/* entry of A and of A^T, sort by (row, col), combine each group.            */
/* ------------------------------------------------------------------------- */
typedef struct { int64_t row, col; float val; int from_t; } trip_t;

static int trip_cmp(const void* a, const void* b)
{
    const trip_t* x = (const trip_t*)a; const trip_t* y = (const trip_t*)b;
    if (x->row != y->row) return x->row < y->row ? -1 : 1;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    return x->from_t - y->from_t;
}

/* capacity of col_out/w_out must be >= 2*n*k; returns nnz (or -1 on error). */
int64_t oracle_fuzzy_union(const int32_t* idx, const float* w, int64_t n, int32_t k,
                           int64_t* indptr_out, int32_t* col_out, float* w_out)
{
    int64_t m = n * (int64_t)k;
    trip_t* t = (trip_t*)malloc(sizeof(trip_t) * (size_t)(2 * m));
    if (!t) return -1;
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < k; ++j) {
            int64_t col = idx[i * k + j];
            if (col < 0) continue;
            t[c].row = i; t[c].col = col; t[c].val = w[i * k + j]; t[c].from_t = 0; ++c;   /* A   */
            t[c].row = col; t[c].col = i; t[c].val = w[i * k + j]; t[c].from_t = 1; ++c;   /* A^T */
        }
    qsort(t, (size_t)c, sizeof(trip_t), trip_cmp);
    int64_t nnz = 0, p = 0;
    for (int64_t r = 0; r <= n; ++r) indptr_out[r] = 0;
    while (p < c) {
        int64_t q = p;
        double a = 0.0, b = 0.0;
        while (q < c && t[q].row == t[p].row && t[q].col == t[p].col) {
            if (t[q].from_t) b = (double)t[q].val; else a = (double)t[q].val;
            ++q;
        }
        float wv = (float)((a + b) - a * b);
        if (wv != 0.0f) {
            col_out[nnz] = (int32_t)t[p].col;
            w_out[nnz] = wv;
            indptr_out[t[p].row + 1] += 1;
            ++nnz;
        }
        p = q;
    }
    for (int64_t r = 0; r < n; ++r) indptr_out[r + 1] += indptr_out[r];
    free(t);
    return nnz;
}

/* ------------------------------------------------------------------------- */
/* R11  random uniform init ("sampling embeddings from a uniform        */
/* distribution"): Y[v][c] = -10 + 20 * (u >> 8) * 2^-24 in fp32,     */
/* u = Philox(key=seed, ctr=(v, c, 0xFFFFFFFF, 0))[0].  Parity unpinned     */
/* (the stream is a convention; the range U[-10,10) is umap-learn's).        */
/* ------------------------------------------------------------------------- */
int oracle_random_init(int64_t n, int32_t dim, uint64_t seed, float* Y)
{
    for (int64_t v = 0; v < n; ++v)
        for (int c = 0; c < dim; ++c) {
            uint32_t u = philox_word(seed, (uint32_t)v, (uint32_t)c, 0xFFFFFFFFu, 0u, 0);
            float f = (float)(u >> 8) * (1.0f / 16777216.0f);
            Y[v * dim + c] = -10.0f + 20.0f * f;
        }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* R9  epochs_per_sample schedule (closed form).  The paper only says the    */
/* objective is "minimized over the edges" for n_epochs.       */
/* r = w / w_max (fp32); edge due in epoch e (1 <= e < N) iff               */
/* floorf(e*r) > floorf((e-1)*r).  Parity unpinned (convention).            */
/* ------------------------------------------------------------------------- */
int oracle_edge_due(float r, int32_t e)
{
    float now = floorf((float)e * r);
    float before = floorf((float)(e - 1) * r);
    return now > before;
}

static double clip4(double v) { return v > 4.0 ? 4.0 : (v < -4.0 ? -4.0 : v); }

/* R12 gradient coefficients on Phi(d) = 1/(1 + a d^{2b}) (Eq. 3,   */
/* approximate form), of the cross entropy of P:60.                          */
double oracle_attr_coef(double s, double a, double b)
{
    if (s <= 0.0) return 0.0;
    return (-2.0 * a * b * pow(s, b - 1.0)) / (a * pow(s, b) + 1.0);
}

double oracle_rep_coef(double s, double a, double b, double gamma)
{
    return (2.0 * gamma * b) / ((0.001 + s) * (a * pow(s, b) + 1.0));
}

/* ------------------------------------------------------------------------- */
/* R8-R14  SGD layout.                       */
/* For each epoch e in [e_begin, e_end) (1 <= e < N), alpha_e = alpha0 *     */
/* (1 - e/N) (fp32).  For each directed edge (h, t) of the union in CSR      */
/* order that is due (R9):                                                  */
/*   attractive: s = |y_h - y_t|^2; g = clip(coef_att(s) (y_h - y_t)) alpha; */
/*               y_h += g; y_t -= g ("Both the source and destination        */
/*               vertices are updated for each edge during training") */
/*   m negatives p = 0..m-1: u = Philox(key=seed, ctr=(h, t, e, p>>2))[p&3], */
/*               v = (u * n) >> 32; v == h skipped; s = |y_h - y_v|^2;       */
/*               g = s > 0 ? clip(coef_rep(s)(y_h - y_v)) alpha : 4 alpha;   */
/*               y_h += g (repulsion on the source only).        */
/* mode 0 (Hogwild reference, R14): sequential, in place, fp64 arithmetic,   */
/*         fp32 storage.                                                    */
/* mode 1 (deterministic): all reads from Y_e; every update summed in */
/*         a 64-bit float buffer, applied at the end of the epoch.           */
/* ------------------------------------------------------------------------- */
int oracle_optimize(const int64_t* indptr, const int32_t* col, const float* w, int64_t n, int32_t dim,
                    float* Y, float a, float b, float gamma, float alpha0, int32_t n_epochs,
                    int32_t e_begin, int32_t e_end, int32_t m, uint64_t seed, int32_t mode)
{
    int64_t nnz = indptr[n];
    float w_max = 0.0f;
    for (int64_t p = 0; p < nnz; ++p) if (w[p] > w_max) w_max = w[p];
    if (w_max <= 0.0f) return 0;
    double* buf = NULL;
    if (mode == 1) buf = (double*)malloc(sizeof(double) * (size_t)(n * dim));
    double* g = (double*)malloc(sizeof(double) * (size_t)dim);
    if (e_begin < 1) e_begin = 1;
    if (e_end > n_epochs) e_end = n_epochs;
    for (int32_t e = e_begin; e < e_end; ++e) {
        float alpha = alpha0 * (1.0f - (float)e / (float)n_epochs);
        if (mode == 1) memset(buf, 0, sizeof(double) * (size_t)(n * dim));
        for (int64_t h = 0; h < n; ++h) {
            for (int64_t p = indptr[h]; p < indptr[h + 1]; ++p) {
                float r = w[p] / w_max;
                if (!oracle_edge_due(r, e)) continue;
                int64_t t = col[p];
                float* yh = Y + h * dim;
                float* yt = Y + t * dim;
                double s = 0.0;
                for (int c = 0; c < dim; ++c) { double df = (double)yh[c] - (double)yt[c]; s += df * df; }
                double coef = oracle_attr_coef(s, (double)a, (double)b);
                for (int c = 0; c < dim; ++c)
                    g[c] = clip4(coef * ((double)yh[c] - (double)yt[c])) * (double)alpha;
                if (mode == 1) {
                    for (int c = 0; c < dim; ++c) { buf[h * dim + c] += g[c]; buf[t * dim + c] -= g[c]; }
                } else {
                    for (int c = 0; c < dim; ++c) {
                        yh[c] = (float)((double)yh[c] + g[c]);
                        yt[c] = (float)((double)yt[c] - g[c]);
                    }
                }
                for (int q = 0; q < m; ++q) {
                    uint32_t u = philox_word(seed, (uint32_t)h, (uint32_t)t, (uint32_t)e, (uint32_t)(q >> 2), q & 3);
                    int64_t v = (int64_t)(((uint64_t)u * (uint64_t)n) >> 32);
                    if (v == h) continue;
                    const float* yv = Y + v * dim;
                    double s2 = 0.0;
                    for (int c = 0; c < dim; ++c) { double df = (double)yh[c] - (double)yv[c]; s2 += df * df; }
                    if (s2 > 0.0) {
                        double cr = oracle_rep_coef(s2, (double)a, (double)b, (double)gamma);
                        for (int c = 0; c < dim; ++c)
                            g[c] = clip4(cr * ((double)yh[c] - (double)yv[c])) * (double)alpha;
                    } else {
                        for (int c = 0; c < dim; ++c) g[c] = 4.0 * (double)alpha;
                    }
                    if (mode == 1) {
                        for (int c = 0; c < dim; ++c) buf[h * dim + c] += g[c];
                    } else {
                        for (int c = 0; c < dim; ++c) yh[c] = (float)((double)yh[c] + g[c]);
                    }
                }
            }
        }
        if (mode == 1)
            for (int64_t i = 0; i < n * dim; ++i) Y[i] = (float)((double)Y[i] + buf[i]);
    }
    free(buf); free(g);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* R15  transform / inference: queries embedded against */
/* the frozen training layout.                                              */
/* init: y_q = sum_j w_qj Y_tr[j] / sum_j w_qj (fp64, neighbour order; the   */
/*       sparse L1 row normalisation of P:120).                              */
/* ------------------------------------------------------------------------- */
int oracle_transform_init(const int32_t* idx, const float* w, int64_t nq, int32_t k,
                          const float* Ytr, int32_t dim, float* Yq)
{
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q) {
        for (int c = 0; c < dim; ++c) {
            double num = 0.0, den = 0.0;
            for (int j = 0; j < k; ++j) {
                num += (double)w[q * k + j] * (double)Ytr[(int64_t)idx[q * k + j] * dim + c];
                den += (double)w[q * k + j];
            }
            Yq[q * dim + c] = den > 0.0 ? (float)(num / den) : 0.0f;
        }
    }
    return 0;
}

/* SGD with only the query rows moving ("only the destination vertex is      */
/* updated during inference") and negatives drawn from the training   */
/* rows.  Epochs e = 1..N_t-1, alpha_e = alpha0 (1 - e/N_t); w_max over the   */
/* query graph.  RNG counter uses the GLOBAL query id (q + q_offset) so a    */
/* partitioned run equals the single run.  In place, fp64        */
/* arithmetic, fp32 storage.                                                */
int oracle_transform_optimize_range(const int32_t* idx, const float* w, int64_t nq, int32_t k,
                                    const float* Ytr, int64_t ntr, int32_t dim, float* Yq,
                                    float a, float b, float gamma, float alpha0, int32_t n_epochs_t,
                                    int32_t e_begin, int32_t e_end, int32_t m, uint64_t seed, int64_t q_offset)
{
    float w_max = 0.0f;
    for (int64_t p = 0; p < nq * k; ++p) if (w[p] > w_max) w_max = w[p];
    if (w_max <= 0.0f) return 0;
    if (e_begin < 1) e_begin = 1;
    if (e_end > n_epochs_t) e_end = n_epochs_t;
    for (int32_t e = e_begin; e < e_end; ++e) {
        float alpha = alpha0 * (1.0f - (float)e / (float)n_epochs_t);
#pragma omp parallel
        {
        double* g = (double*)malloc(sizeof(double) * (size_t)dim);
#pragma omp for schedule(static)
        for (int64_t q = 0; q < nq; ++q) {
            float* yq = Yq + q * dim;
            uint32_t head = (uint32_t)(q + q_offset);
            for (int j = 0; j < k; ++j) {
                float r = w[q * k + j] / w_max;
                if (!oracle_edge_due(r, e)) continue;
                int64_t t = idx[q * k + j];
                const float* yt = Ytr + t * dim;
                double s = 0.0;
                for (int c = 0; c < dim; ++c) { double df = (double)yq[c] - (double)yt[c]; s += df * df; }
                double coef = oracle_attr_coef(s, (double)a, (double)b);
                for (int c = 0; c < dim; ++c) {
                    g[c] = clip4(coef * ((double)yq[c] - (double)yt[c])) * (double)alpha;
                }
                for (int c = 0; c < dim; ++c) yq[c] = (float)((double)yq[c] + g[c]);
                for (int p = 0; p < m; ++p) {
                    uint32_t u = philox_word(seed, head, (uint32_t)t, (uint32_t)e, (uint32_t)(p >> 2), p & 3);
                    int64_t v = (int64_t)(((uint64_t)u * (uint64_t)ntr) >> 32);
                    const float* yv = Ytr + v * dim;
                    double s2 = 0.0;
                    for (int c = 0; c < dim; ++c) { double df = (double)yq[c] - (double)yv[c]; s2 += df * df; }
                    if (s2 > 0.0) {
                        double cr = oracle_rep_coef(s2, (double)a, (double)b, (double)gamma);
                        for (int c = 0; c < dim; ++c)
                            g[c] = clip4(cr * ((double)yq[c] - (double)yv[c])) * (double)alpha;
                    } else {
                        for (int c = 0; c < dim; ++c) g[c] = 4.0 * (double)alpha;
                    }
                    for (int c = 0; c < dim; ++c) yq[c] = (float)((double)yq[c] + g[c]);
                }
            }
        }
        free(g);
        }
    }
    return 0;
}

int oracle_transform_optimize(const int32_t* idx, const float* w, int64_t nq, int32_t k,
                              const float* Ytr, int64_t ntr, int32_t dim, float* Yq,
                              float a, float b, float gamma, float alpha0, int32_t n_epochs_t,
                              int32_t m, uint64_t seed, int64_t q_offset)
{
    return oracle_transform_optimize_range(idx, w, nq, k, Ytr, ntr, dim, Yq, a, b, gamma, alpha0, n_epochs_t,
                                           1, n_epochs_t, m, seed, q_offset);
}

/* ------------------------------------------------------------------------- */
/* R16  trustworthiness (Alg. 1; Venna & Kaski).   */
/* r_i(j) = 1 + #{ l != i : (d2_il, l) < (d2_ij, j) } in input space (fp32   */
/* distances as R2); NN_k^emb(i) = exact kNN of the embedding (R1/R2).       */
/* S = sum_i sum_{j in NN_k^emb(i)} max(0, r_i(j) - k)  (int64).            */
/* T = 1 - 2 S / (n k (2n - 3k - 1))   (Alg. 1's garbled return; R16).       */
/* Rows [row_begin, row_end) only, so a bounded sample can be timed; the     */
/* per-row penalties are written to row_pen if non-NULL.                     */
/* ------------------------------------------------------------------------- */
int64_t oracle_trust_penalty(const float* X, int32_t d, const float* Y, int32_t dy, int64_t n,
                             int32_t k, int64_t row_begin, int64_t row_end, int64_t* row_pen)
{
    int64_t S = 0;
#pragma omp parallel reduction(+ : S)
    {
    int32_t* nn = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
    float* nd = (float*)malloc(sizeof(float) * (size_t)k);
    float* bd = (float*)malloc(sizeof(float) * (size_t)k);
    int64_t* bi = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    float* dx = (float*)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(dynamic, 4)
    for (int64_t i = row_begin; i < row_end; ++i) {
        knn_row(Y + i * dy, Y, n, dy, k, i, bd, bi, nn, nd);
        for (int64_t l = 0; l < n; ++l) dx[l] = oracle_sqdist(X + i * (int64_t)d, X + l * (int64_t)d, d);
        int64_t pen = 0;
        for (int t = 0; t < k; ++t) {
            int64_t j = nn[t];
            int64_t r = 1;
            for (int64_t l = 0; l < n; ++l) {
                if (l == i) continue;
                if (key_less(dx[l], l, dx[j], j)) ++r;
            }
            if (r > k) pen += r - k;
        }
        if (row_pen) row_pen[i - row_begin] = pen;
        S += pen;
    }
    free(nn); free(nd); free(bd); free(bi); free(dx);
    }
    return S;
}

double oracle_trust_from_penalty(int64_t S, int64_t n, int32_t k)
{
    double nn = (double)n, kk = (double)k;
    return 1.0 - (2.0 / (nn * kk * (2.0 * nn - 3.0 * kk - 1.0))) * (double)S;
}
