/*
 * umap_b200.h -- C ABI of the B200-native GPU-UMAP hot path (arXiv 2008.00325).
 *
 * Paper: "Faster, Simpler and More Accurate: GPU-accelerated UMAP"
 * (PAPER.md, cited P:<line>).  Readings of garbled / silent passages are
 * R1..R16 in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - extern "C", plain pointers and sizes; no C++ or torch types.
 *  - Layout: every matrix is row-major, C-contiguous (X: n x d fp32, row i at
 *    X + i*d; Y: n x n_components fp32).  Index arrays are int32 unless named
 *    indptr (int64).
 *  - Pointers: the top-level calls umap_fit, umap_transform and
 *    umap_trustworthiness accept HOST or DEVICE pointers for every array (the
 *    kind is detected with cudaPointerGetAttributes; host arrays are staged
 *    through the device inside the call).  All building-block calls take
 *    DEVICE pointers only and return UMAP_ERR_NOT_DEVICE_POINTER otherwise.
 *  - Ownership: the caller owns every buffer.  Inputs are read-only and not
 *    retained after return; outputs are caller-allocated with the documented
 *    shape.  Scratch is allocated stream-ordered (cudaMallocAsync on `stream`,
 *    the analogue of the paper's RMM pool) and freed before return.
 *  - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).  Work
 *    is enqueued on it and every call returns after that work completed.
 *  - Errors: a umap_status code.  Nothing throws across the ABI or aborts.
 *    Outputs are unspecified on error.  umap_last_error() gives a thread-local
 *    detail string.
 *  - The library never falls back to the CPU: without a CUDA device every
 *    compute call returns UMAP_ERR_CUDA.
 */
#ifndef UMAP_B200_H
#define UMAP_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define UMAP_API __attribute__((visibility("default")))
#else
#define UMAP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    UMAP_OK = 0,
    UMAP_ERR_INVALID_ARGUMENT = 1,
    UMAP_ERR_NOT_DEVICE_POINTER = 2,
    UMAP_ERR_TOO_FEW_ROWS = 3,
    UMAP_ERR_K_OUT_OF_RANGE = 4,
    UMAP_ERR_NONFINITE_INPUT = 5,
    UMAP_ERR_NONFINITE_EMBEDDING = 6,
    UMAP_ERR_FIT_AB_NO_CONVERGENCE = 7,
    UMAP_ERR_CUDA = 8,
    UMAP_ERR_OUT_OF_MEMORY = 9,
    UMAP_ERR_UNSUPPORTED = 10
} umap_status;

/* SGD layout mode. */
typedef enum {
    UMAP_SGD_HOGWILD = 0,       /* racy in-place push updates with fp32 atomics */
    UMAP_SGD_DETERMINISTIC = 1  /* epoch-buffered updates, bit-reproducible (R13)   */
} umap_sgd_mode;

/* kNN distance mode. */
typedef enum {
    UMAP_KNN_EXACT_FP32 = 0,    /* exact fp32 distances, sequential FMA per feature (R2)   */
    UMAP_KNN_TENSOR_BF16 = 1    /* tcgen05 BF16 candidate GEMM + exact fp32 re-rank (R3)   */
} umap_knn_mode;

typedef struct {
    uint32_t struct_size;          /* = sizeof(umap_params); ABI versioning                 */
    int32_t  n_neighbors;          /* k (P:232 default 15); 2 <= k < n, k <= 64              */
    int32_t  n_components;         /* embedding dimension: 1..4, 8 or 16 (default 2)         */
    int32_t  n_epochs;             /* N; 0 -> 500 if n <= 10000 else 200                     */
    float    min_dist;             /* Eq. 3, default 0.1                           */
    float    spread;               /* default 1.0                                           */
    int32_t  negative_sample_rate; /* m negatives per positive edge, default 5        */
    float    learning_rate;        /* alpha0, default 1.0 (decays linearly, R10).  The        */
                                   /* deterministic mode's int32 fixed-point per-edge sums    */
                                   /* (R13) need (2 + m) * learning_rate < 32: larger values  */
                                   /* return INVALID_ARGUMENT in that mode                    */
    float    repulsion_strength;   /* gamma, default 1.0                                    */
    float    a, b;                 /* Phi(d) = 1/(1 + a d^{2b}); 0,0 -> fitted (umap_fit_ab) */
    uint64_t seed;                 /* Philox key for init and negative sampling      */
    int32_t  sgd_mode;             /* umap_sgd_mode, default UMAP_SGD_DETERMINISTIC          */
    int32_t  knn_mode;             /* umap_knn_mode, default UMAP_KNN_EXACT_FP32             */
    int32_t  knn_candidates;       /* k' candidates per row before re-rank (TC mode), 32     */
    int32_t  transform_epochs;     /* 0 -> ceil(n_epochs / 3) (R15)                          */
    int32_t  trust_k;              /* umap_fit only: > 0 -> also score the embedding with    */
                                   /* T(trust_k) (a10, knn_mode) into umap_fit_stats; 0 skip */
    float    far_dist;             /* supervised (umap_fit_supervised): different labels ->  */
                                   /* weight x exp(-far_dist), default 5.0 (R17)             */
    float    unknown_dist;         /* a label -1 on either end -> x exp(-unknown_dist), 1.0  */
    int32_t  init;                 /* a7: 0 = random U[-10,10) (R11), 1 = spectral (R18)     */
    int32_t  spectral_iters;       /* block power iterations of the spectral init, 0 -> 300  */
    int32_t  transform_precision;  /* a9 per-edge arithmetic of umap_transform(_optimize):    */
                                   /* 0 = fp32 with MUFU pow/rcp (default, fast); 1 = fp64   */
                                   /* with IEEE pow and division, position stored in fp32    */
                                   /* after every update (R15's oracle reading: equal to the */
                                   /* oracle bit for bit, ~8x slower on the C5 transform)    */
} umap_params;

/* Per-stage device times (ms, CUDA events on `stream`) and graph statistics. */
typedef struct {
    double  ms_knn, ms_smooth, ms_union, ms_init, ms_sgd, ms_total;
    int64_t nnz;            /* entries of the fuzzy union B (both directions)              */
    int64_t positives;      /* sum over epochs of due directed edges (edge-updates)        */
    float   w_max;          /* max weight of B (1.0 on every non-empty graph)              */
    float   a, b;           /* curve parameters used                                       */
    int32_t n_epochs;       /* N used                                                      */
    int32_t gpu_launches;   /* kernels launched by this call                               */
    double  ms_trust;       /* p->trust_k > 0: device time of the trustworthiness stage    */
    double  trustworthiness;/* p->trust_k > 0: T(trust_k) of the returned embedding, else 0 */
    int64_t trust_penalty;  /* p->trust_k > 0: the integer penalty sum S of T (R16)         */
} umap_fit_stats;

/* Fill *p with the defaults above. */
UMAP_API void umap_params_default(umap_params* p);

/* R8: least-squares fit of Phi(x) = 1/(1 + a x^{2b}) to y(x) = 1 (x < min_dist),
 * exp(-(x - min_dist)/spread) otherwise, on 300 points of [0, 3 spread]
 * (Eq. 3's "approximate form").  Host only; no CUDA needed.
 * Errors: INVALID_ARGUMENT (spread <= 0, min_dist < 0), FIT_AB_NO_CONVERGENCE. */
UMAP_API umap_status umap_fit_ab(float min_dist, float spread, float* a, float* b);

/* Whole fit: kNN (a2) -> rho/sigma + membership (a3, a4) ->
 * fuzzy union (a5) -> random init (a7) -> SGD layout (a6, a8).
 * X: n x d fp32 (host or device); Y: n x n_components fp32 output (host or device).
 * stats: optional (NULL), host memory.
 * Errors: TOO_FEW_ROWS (n <= k), K_OUT_OF_RANGE, NONFINITE_INPUT, NONFINITE_EMBEDDING,
 * UNSUPPORTED (n_components not in {1,2,3,4,8,16}), CUDA, OUT_OF_MEMORY. */
UMAP_API umap_status umap_fit(const float* X, int64_t n, int32_t d, const umap_params* p,
                     float* Y, umap_fit_stats* stats, void* stream);

/* f1 pre-computed kNN graph ("accept a k-NN graph that has already been
 * computed", App. A.1): the fit from a3 on.  knn_idx n x k int32 (global ids,
 * self excluded), knn_dist n x k fp32, each row sorted ascending (umap_knn output);
 * k = p->n_neighbors.  Host or device pointers.  Same outputs and errors as umap_fit.
 * The graph is validated on the device before use: every id in [0, n), no row lists
 * itself or an id twice, every distance finite and >= 0; otherwise INVALID_ARGUMENT
 * (nothing is read out of bounds).  fit_knn(umap_knn(X)) equals umap_fit(X) bit for bit. */
UMAP_API umap_status umap_fit_knn(const int32_t* knn_idx, const float* knn_dist, int64_t n, const umap_params* p,
                                  float* Y, umap_fit_stats* stats, void* stream);

/* Out-of-sample embedding against a frozen training layout (R15):
 * kNN of X_q against X_train (no self exclusion), rho/sigma/membership on the
 * query rows, init = weighted mean of the neighbours' Y_train (L1 row
 * normalisation), then transform_epochs epochs of SGD moving only the
 * query rows, negatives drawn from the training rows.
 * q_offset: global index of X_q's first row; it keys the RNG so a partitioned
 * run equals the single run bit for bit.
 * X_train n_train x d, Y_train n_train x n_components, X_q n_q x d, Y_q n_q x n_components. */
UMAP_API umap_status umap_transform(const float* X_train, const float* Y_train, int64_t n_train, int32_t d,
                           const float* X_q, int64_t n_q, int64_t q_offset, const umap_params* p,
                           float* Y_q, void* stream);

/* Trustworthiness T(k) (Alg. 1, R16):
 * T = 1 - 2/(n k (2n - 3k - 1)) * sum_i sum_{j in NN_k(Y_i)} max(0, r_i(j) - k),
 * r_i(j) = 1 + #{l != i : (d2_X(i,l), l) < (d2_X(i,j), j)}.
 * X n x d, Y n x d_emb (host or device); T (host double), penalty (host int64,
 * optional NULL) = the integer sum.  Requires 1 <= k < n/2.
 * knn_mode: UMAP_KNN_EXACT_FP32 counts ranks in the exact fp32 distance kernel;
 * UMAP_KNN_TENSOR_BF16 uses a split-BF16 tcgen05 GEMM whose error bound certifies most
 * (row, reference) buckets and re-checks the rest exactly -- the same integer S either way. */
UMAP_API umap_status umap_trustworthiness(const float* X, int32_t d, const float* Y, int32_t d_emb, int64_t n,
                                 int32_t k, int32_t knn_mode, double* T, int64_t* penalty, void* stream);

/* ---------------- building blocks (DEVICE pointers only) ---------------- */

/* a2 kNN (R1, R2): for each query row i, the k reference rows with smallest key
 * (d2, global id), d2 = fp32 sum over f ascending of fmaf(t, t, s), t = xq_if - xr_jf.
 * Global ids: query row i is point query_offset + i, reference row j is point
 * index_offset + j (the shard offset of a sharded kNN, 8(e)); keys and output ids use
 * global reference ids.  exclude_self != 0 drops the reference row whose global id
 * equals the query's own (R1: "k true neighbours", self excluded by index).
 * idx: n_q x k int32, dist: n_q x k fp32 = sqrtf(d2) (or d2 itself when out_squared != 0),
 * rows sorted ascending by key.  Requires 1 <= k <= 64, k <= n_r - (exclude_self != 0).
 * knn_mode TENSOR_BF16: candidates by a tcgen05 BF16 GEMM, re-ranked exactly (R3). */
UMAP_API umap_status umap_knn(const float* X_q, int64_t n_q, const float* X_r, int64_t n_r, int32_t d, int32_t k,
                     int64_t query_offset, int64_t index_offset, int32_t exclude_self, int32_t knn_mode,
                     int32_t out_squared,
                     int32_t* idx, float* dist, void* stream);

/* Merge n_parts per-part candidate lists (part-major: idx_in[p][n][k_in], d2_in likewise,
 * each row sorted by key) into the k_out smallest keys (d2, id).  dist = sqrtf(d2)
 * (out_squared = 0) or d2.  Used by the sharded kNN (NCCL all-gather, 8(e)). */
UMAP_API umap_status umap_topk_merge(const int32_t* idx_in, const float* d2_in, int32_t n_parts, int64_t n,
                            int32_t k_in, int32_t k_out, int32_t out_squared, int32_t* idx, float* dist,
                            void* stream);

/* a3 + a4 (Eq. 1; R4-R6): per row rho, sigma (fp64 bisection)
 * and memberships w (n x k).  dist: n x k fp32 sorted ascending.  rho, sigma: n fp32
 * (either may be NULL).  If col_sorted_idx != NULL, each row of (idx, w) is also written
 * re-ordered by ascending column id into col_sorted_idx / w (the union's input);
 * otherwise w keeps the distance order. */
UMAP_API umap_status umap_smooth_knn(const float* dist, const int32_t* idx, int64_t n, int32_t k,
                            float* rho, float* sigma, float* w, int32_t* col_sorted_idx, void* stream);

/* a5 fuzzy union (Eq. 2; R7): B = A + A^T - A o A^T, zeros dropped,
 * CSR sorted by (row, col).  idx/w: n x k, rows sorted by column (umap_smooth_knn
 * col_sorted_idx output).  indptr: n+1 int64; col, val: capacity entries
 * (2 n k always suffices).  *nnz (host) receives the number of entries. */
UMAP_API umap_status umap_fuzzy_union(const int32_t* idx, const float* w, int64_t n, int32_t k,
                             int64_t* indptr, int32_t* col, float* val, int64_t capacity,
                             int64_t* nnz, void* stream);

/* a7 random init (R11): Y[v][c] = -10 + 20 (u >> 8) 2^-24,
 * u = Philox4x32-10(key = seed, ctr = (v, c, 0xFFFFFFFF, 0))[0]. */
UMAP_API umap_status umap_random_init(int64_t n, int32_t dim, uint64_t seed, float* Y, void* stream);

/* a6 + a8 SGD layout over the union B (CSR from umap_fuzzy_union), epochs
 * e_begin..e_end-1 of an N = p->n_epochs schedule (R9-R14), Y (n x n_components) in place.
 * Uses p->a, p->b (must be > 0), gamma, alpha0, m, seed, sgd_mode.
 * positives (host, optional) receives the number of due directed edges processed. */
UMAP_API umap_status umap_optimize(const int64_t* indptr, const int32_t* col, const float* val, int64_t n,
                          float* Y, const umap_params* p, int32_t e_begin, int32_t e_end,
                          int64_t* positives, void* stream);

/* a9 transform SGD stage (R15): query graph idx/w (n_q x k, distance order),
 * Y_q in/out (n_q x n_components), Y_train frozen.  Epochs e_begin..e_end-1 of an
 * N_t = n_epochs_t schedule.  init != 0: first set Y_q to the weighted mean of the
 * neighbours' Y_train. */
UMAP_API umap_status umap_transform_optimize(const int32_t* idx, const float* w, int64_t n_q, int32_t k,
                                    const float* Y_train, int64_t n_train, float* Y_q,
                                    const umap_params* p, int32_t n_epochs_t, int32_t e_begin,
                                    int32_t e_end, int64_t q_offset, int32_t init, void* stream);

/* Supervised fit (R17): as umap_fit with training labels (n int32, -1 = unknown; host
 * or device) -- between the fuzzy union (a5) and the SGD (a6-a8) every entry (i, j) of B is
 * multiplied by 1 (same label), exp(-p->far_dist) (different known labels) or
 * exp(-p->unknown_dist) (either unknown), entries below 1e-8 dropped. */
UMAP_API umap_status umap_fit_supervised(const float* X, int64_t n, int32_t d, const int32_t* labels,
                                         const umap_params* p, float* Y, umap_fit_stats* stats, void* stream);

/* Spectral initialisation (f3, R18) of a device CSR graph B (symmetric, n+1
 * int64 indptr, int32 col, fp32 val): the n_components eigenvectors of
 * L = I - D^-1/2 B D^-1/2 with the smallest non-trivial eigenvalues by `iters` fp64 block
 * power iterations on 2I - L (trivial vector deflated), columns rescaled to [-10, 10] plus
 * 1e-3 Philox noise.  Y: device n x dim fp32.  dim in {1,2,3,4,8,16}, n >= dim + 2. */
UMAP_API umap_status umap_spectral_init(const int64_t* indptr, const int32_t* col, const float* val, int64_t n,
                                        int32_t dim, uint64_t seed, int32_t iters, float* Y, void* stream);

/* The label adjustment alone on a device CSR (indptr n+1 int64, col int32, val fp32): writes
 * the adjusted CSR (out_indptr n+1, out_col / out_val with room for `capacity` entries) and
 * *nnz (host).  UMAP_ERR_INVALID_ARGUMENT if capacity is too small. */
UMAP_API umap_status umap_supervised_adjust(const int64_t* indptr, const int32_t* col, const float* val, int64_t n,
                                            const int32_t* labels, float far_dist, float unknown_dist,
                                            int64_t* out_indptr, int32_t* out_col, float* out_val,
                                            int64_t capacity, int64_t* nnz, void* stream);

/* a10 input-space rank penalties for rows [row_begin, row_end) (R16): emb_idx is the
 * embedding kNN of those rows (n_rows x k, global ids).  knn_mode as in
 * umap_trustworthiness.  Y (optional, device, n x d_emb; NULL to omit) is the embedding:
 * with d_emb == 2 the tensor-core path visits rows and columns in the Hilbert order of Y
 * (a layout choice only: the integer result is the same).  row_pen: n_rows int64
 * (optional NULL); *penalty (host) = sum. */
UMAP_API umap_status umap_trust_penalty(const float* X, int64_t n, int32_t d, const int32_t* emb_idx, int32_t k,
                               int64_t row_begin, int64_t row_end, int32_t knn_mode, const float* Y,
                               int32_t d_emb, int64_t* row_pen, int64_t* penalty, void* stream);

/* R16 normaliser (Alg. 1, garbled return read as Venna & Kaski's):
 * T = 1 - 2 S / (n k (2n - 3k - 1)) in fp64.  Host only; no CUDA needed.  Returns NaN
 * unless 1 <= k and 2n - 3k - 1 > 0. */
UMAP_API double      umap_trust_from_penalty(int64_t penalty, int64_t n, int32_t k);
/* R15 inference budget: transform_epochs if > 0, else ceil(n_epochs / 3) with n_epochs
 * defaulted as in umap_params (0 -> 500 if n_train <= 10000 else 200).  Host only. */
UMAP_API int32_t     umap_transform_epoch_count(int32_t n_epochs, int32_t transform_epochs, int64_t n_train);

UMAP_API const char* umap_status_string(umap_status s);
UMAP_API const char* umap_last_error(void);
/* Number of this library's kernels launched by the calling thread since load. */
UMAP_API int64_t     umap_kernel_launch_count(void);
/* Diagnostics: pairs the calling thread's last tensor-mode trustworthiness call could not
 * certify from the tensor-core pass and re-checked exactly. */
UMAP_API int64_t     umap_trust_ambiguous_count(void);
/* Diagnostics: fraction of (query block, reference tile) pairs the split-precision pass of the
 * calling thread's last tensor-mode trustworthiness call visited (1.0 without the coarse pass). */
UMAP_API double      umap_trust_fine_fraction(void);
/* Live per-kernel timing (bench.py's roofline): between umap_profile_begin() and
 * umap_profile_end() every hot kernel launched by the calling thread is bracketed by a CUDA
 * event pair on its own stream.  umap_profile_end synchronises those events, writes the
 * summed milliseconds and launch count per slot into ms[n_slots] / launches[n_slots] (either
 * may be NULL) and returns the number of slots the library defines; slot names come from
 * umap_profile_slot_name(slot) ("" out of range).  Host-side only; never fails. */
UMAP_API void        umap_profile_begin(void);
UMAP_API int32_t     umap_profile_end(double* ms, int64_t* launches, int32_t n_slots);
UMAP_API const char* umap_profile_slot_name(int32_t slot);
/* Library version string. */
UMAP_API const char* umap_version(void);

#ifdef __cplusplus
}
#endif
#endif /* UMAP_B200_H */
