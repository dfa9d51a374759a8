// trust.cu -- trustworthiness (a10; Alg. 1, R16).
//
// Alg. 1 batches the n x n input-space distance matrix.  Here no distance matrix
// and no argsort exist at all: the rank of each embedding neighbour j of row i,
// r_i(j) = 1 + #{l != i : key(d2_X(i,l), l) < key(d2_X(i,j), j)}, is obtained by
// counting, inside the exact distance-tile kernel (knn_exact.cu, RANK epilogue),
// how many reference rows fall below each of the k sorted thresholds of row i.
// Penalties are exact integers summed in int64.
#include "common.cuh"
#include "bulk.cuh"

namespace umapb200 {

umap_status rank_count_exact(const float* Xq, int64_t nq, const float* X, int64_t n, int d, int k,
                             int64_t self_offset, const float* thr_d2, const int32_t* thr_id, int32_t* cnt_out,
                             Scratch& tmp, int* n_splits_out, cudaStream_t s);

umap_status cluster_order(const float* Y, int64_t n, int d_emb, int32_t* perm, cudaStream_t s);
umap_status rank_count_tc(const float* X, int64_t n, int d, int64_t row_begin, int64_t rows, int k,
                          const float* thr_d2, const int32_t* thr_id, int32_t* hist, int* overflow,
                          const float* Y, int d_emb, const int32_t* perm_in, cudaStream_t s);

namespace {

// thresholds: key (d2_X(i, j_t), j_t) for the k embedding neighbours of row i, sorted by key.
// d2 uses the exact sequential-fmaf definition (R2), identical to the tile kernel's value.
__global__ void thresholds_kernel(const float* __restrict__ X, int d, const int32_t* __restrict__ emb_idx,
                                  int64_t rows, int64_t row_begin, int k, float* __restrict__ thr_d2,
                                  int32_t* __restrict__ thr_id)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* xi = X + (row_begin + r) * (int64_t)d;
    float* td = thr_d2 + r * k;
    int32_t* ti = thr_id + r * k;
    for (int t = 0; t < k; ++t) {
        const int32_t j = emb_idx[r * k + t];
        const float* xj = X + (int64_t)j * d;
        float s = 0.0f;
        for (int f = 0; f < d; ++f) {
            const float u = __fsub_rn(__ldg(xi + f), __ldg(xj + f));
            s = __fmaf_rn(u, u, s);
        }
        int p = t;  // insertion by key
        while (p > 0 && key_less(s, j, td[p - 1], ti[p - 1])) { td[p] = td[p - 1]; ti[p] = ti[p - 1]; --p; }
        td[p] = s;
        ti[p] = j;
    }
}

// k <= 32: warp per row, lane t computes the exact key of threshold t, warp bitonic sort
// bulk != 0: rows through the TMA bulk ring (d % 4 == 0, blockDim = 32 RB_WARPS, RB_SMEM smem)
__global__ void thresholds_warp_kernel(const float* __restrict__ X, int d, const int32_t* __restrict__ emb_idx,
                                       int64_t rows, int64_t row_begin, int k, float* __restrict__ thr_d2,
                                       int32_t* __restrict__ thr_id, int bulk, const int32_t* __restrict__ order)
{
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    uint32_t bar0 = 0, ph = 0;
    float* ring = bulk ? bulk_ring_setup(bar0) : nullptr;
    if (bulk == 2) {
        // k <= 15: two rows per warp (lanes 0..14 and 16..30), both query rows through the ring
        const int64_t w0 = 2 * w, w1 = 2 * w + 1;
        if (w0 >= rows) return;
        const int h = lane >> 4, li = lane & 15;
        const int64_t wh = h ? w1 : w0;
        const bool okrow = wh < rows;
        const int64_t r0 = order ? (int64_t)order[w0] : w0;
        const int64_t r1 = w1 < rows ? (order ? (int64_t)order[w1] : w1) : r0;
        const int64_t r = h ? r1 : r0;
        const int32_t j = (okrow && li < k) ? emb_idx[r * k + li] : -1;
        const float v = exact_d2_bulk2(X + (row_begin + r0) * (int64_t)d, X + (row_begin + r1) * (int64_t)d, X, j, d,
                                       ring, bar0, ph, lane);
        float key = j >= 0 ? v : INFINITY;
        int32_t id = j >= 0 ? j : INT32_MAX;
        warp_bitonic16(key, id, lane);
        if (okrow && li < k) {
            thr_d2[r * k + li] = key;
            thr_id[r * k + li] = id;
        }
        return;
    }
    if (w >= rows) return;
    // order (optional): rows visited in the Hilbert order of the embedding, so the warps
    // resident at one time gather neighbour rows of the same 2-D region (L2 reuse)
    const int64_t r = order ? (int64_t)order[w] : w;
    float key = INFINITY;
    int32_t id = INT32_MAX;
    if (bulk) {
        const int32_t j = lane < k ? emb_idx[r * k + lane] : -1;
        const float v = exact_d2_bulk(X + (row_begin + r) * (int64_t)d, X, j, d, ring, bar0, ph, lane);
        if (lane < k) { id = j; key = v; }
    } else if (lane < k) {
        id = emb_idx[r * k + lane];
        key = exact_d2(X + (row_begin + r) * (int64_t)d, X + (int64_t)id * d, d);
    }
    warp_bitonic(key, id, lane);
    if (lane < k) {
        thr_d2[r * k + lane] = key;
        thr_id[r * k + lane] = id;
    }
}

// penalty of row r: counts (summed over reference splits) -> cumulative -> ranks.
__global__ void penalty_kernel(const int32_t* __restrict__ cnt, int n_splits, int64_t rows, int k,
                               int64_t* __restrict__ row_pen, unsigned long long* __restrict__ total)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    long long pen = 0;
    if (r < rows) {
        long long cum = 0;
        for (int t = 0; t < k; ++t) {
            for (int sp = 0; sp < n_splits; ++sp) cum += cnt[((int64_t)sp * rows + r) * k + t];
            const long long rank = 1 + cum;
            if (rank > k) pen += rank - k;
        }
        if (row_pen) row_pen[r] = pen;
    }
    pen = warp_sum(pen);
    if ((threadIdx.x & 31) == 0 && pen) atomicAdd(total, (unsigned long long)pen);
}

}  // namespace

umap_status trust_penalty(const float* X, int64_t n, int d, const int32_t* emb_idx, int k, int64_t row_begin,
                          int64_t row_end, int64_t* row_pen, int64_t* penalty_host, int knn_mode, const float* Y,
                          int d_emb, cudaStream_t s)
{
    const int64_t rows = row_end - row_begin;
    if (rows <= 0) { if (penalty_host) *penalty_host = 0; return UMAP_OK; }
    Scratch thr_d, thr_i, cnt, tmp, total;
    UMAP_TRY(thr_d.alloc(sizeof(float) * (size_t)rows * k, s));
    UMAP_TRY(thr_i.alloc(sizeof(int32_t) * (size_t)rows * k, s));
    UMAP_TRY(cnt.alloc(sizeof(int32_t) * (size_t)rows * k, s));
    UMAP_TRY(total.alloc(sizeof(unsigned long long), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(total.p, 0, sizeof(unsigned long long), s));
    Scratch order;
    const bool ordered = knn_mode == UMAP_KNN_TENSOR_BF16 && Y && d_emb == 2 && row_begin == 0 && rows == n &&
                         !getenv("UMAP_TRUST_NO_ORDER");
    if (ordered) {
        UMAP_TRY(order.alloc(sizeof(int32_t) * (size_t)n, s));
        UMAP_TRY(cluster_order(Y, n, d_emb, order.as<int32_t>(), s));
    }
    if (k <= 32) {
        ProfScope ps(PROF_THRESHOLDS, s);
        // the bulk ring measured slower here (0.79 vs 0.72 ms at C2: k = 15 of 32 lanes busy,
        // one batch per row), so the per-lane streaming path is used; the option stays for k > 16
        // k <= 15: two rows per warp through the bulk ring (tuning knob UMAP_TRUST_THR2=0: streaming)
        const bool aligned = (d % 4 == 0) && ((uintptr_t)X % 16 == 0);
        const bool two = k <= 15 && aligned && !(getenv("UMAP_TRUST_THR2") && atoi(getenv("UMAP_TRUST_THR2")) == 0);
        const bool bulk = (k > 16 && aligned) || two;
        if (bulk) {
            static PerDeviceOnce cfg;
            if (cfg.first()) {
                UMAP_CUDA_TRY(cudaFuncSetAttribute(thresholds_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)RB_SMEM));
            }
        }
        const int64_t warps = two ? (rows + 1) / 2 : rows;
        thresholds_warp_kernel<<<ceil_div(warps * 32, 32 * RB_WARPS), 32 * RB_WARPS, bulk ? RB_SMEM : 0, s>>>(
            X, d, emb_idx, rows, row_begin, k, thr_d.as<float>(), thr_i.as<int32_t>(), two ? 2 : (bulk ? 1 : 0),
            ordered && k <= 32 ? order.as<int32_t>() : nullptr);
        UMAP_LAUNCH_CHECK("thresholds_warp_kernel");
    } else {
        thresholds_kernel<<<ceil_div(rows, 128), 128, 0, s>>>(X, d, emb_idx, rows, row_begin, k, thr_d.as<float>(),
                                                              thr_i.as<int32_t>());
        UMAP_LAUNCH_CHECK("thresholds_kernel");
    }
    int n_splits = 1;
    int overflow = 1;
    if (knn_mode == UMAP_KNN_TENSOR_BF16)
        UMAP_TRY(rank_count_tc(X, n, d, row_begin, rows, k, thr_d.as<float>(), thr_i.as<int32_t>(), cnt.as<int32_t>(),
                               &overflow, Y, d_emb, ordered ? order.as<int32_t>() : nullptr, s));
    if (overflow)  // exact mode, or the tensor pass could not certify enough pairs
        UMAP_TRY(rank_count_exact(X + row_begin * (int64_t)d, rows, X, n, d, k, row_begin, thr_d.as<float>(),
                                  thr_i.as<int32_t>(), cnt.as<int32_t>(), tmp, &n_splits, s));
    const int32_t* counts = n_splits == 1 ? cnt.as<int32_t>() : tmp.as<int32_t>();
    penalty_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(counts, n_splits, rows, k, row_pen,
                                                       total.as<unsigned long long>());
    UMAP_LAUNCH_CHECK("penalty_kernel");
    unsigned long long S = 0;
    UMAP_CUDA_TRY(cudaMemcpyAsync(&S, total.p, sizeof(S), cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    if (penalty_host) *penalty_host = (int64_t)S;
    return UMAP_OK;
}

}  // namespace umapb200
