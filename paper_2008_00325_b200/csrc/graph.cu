// graph.cu -- neighbourhood weighting and fuzzy union (a3, a4, a5).
//
//  * smooth_knn_membership: rho, sigma (Eq. 1) and memberships
//     fused in one kernel.  A warp stages 32 rows (32*k contiguous floats,
//    one coalesced read) in shared memory; each lane then owns one row, like the
//    paper's thread-per-vertex kernel, so the fp64 bisection runs with the
//    exact sequential sums of the definition (R5) and no per-iteration shuffles.
//  * fuzzy union (Eq. 2): counting-sort transpose of A (in-degree
//    histogram -> scan -> scatter -> per-row sort), then a two-pointer merge of row i
//    of A and row i of A^T applying w = (a + b) - a*b (R7), written straight into a
//    CSR sorted by (row, col).
#include <cmath>

#include "common.cuh"

namespace umapb200 {

namespace {

// ---------------------------------------------------------------- smooth_knn
constexpr int SK_WARPS = 4;

__global__ void __launch_bounds__(32 * SK_WARPS)
smooth_knn_kernel(const float* __restrict__ dist, const int32_t* __restrict__ idx, int64_t n, int k,
                  float* __restrict__ rho_out, float* __restrict__ sigma_out, float* __restrict__ w_out,
                  int32_t* __restrict__ col_out)
{
    extern __shared__ float sk_smem[];
    const int stride = k | 1;  // odd row stride: lane-per-row access is bank-conflict free
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* sd = sk_smem + warp * 32 * stride;
    int32_t* si = reinterpret_cast<int32_t*>(sk_smem + SK_WARPS * 32 * stride) + warp * 32 * stride;
    const int64_t row0 = ((int64_t)blockIdx.x * SK_WARPS + warp) * 32;
    if (row0 >= n) return;
    const int rows = (int)imin64(32, n - row0);
    // coalesced staging of rows row0..row0+rows-1
    for (int e = lane; e < rows * k; e += 32) {
        const int r = e / k, j = e - r * k;
        sd[r * stride + j] = dist[row0 * k + e];
        if (col_out) si[r * stride + j] = idx[row0 * k + e];
    }
    __syncwarp();
    if (lane < rows) {
        const float* row = sd + lane * stride;
        float rho = 0.0f;
        bool have = false;
        double mean = 0.0;
        for (int j = 0; j < k; ++j) {
            const float v = row[j];
            mean = __dadd_rn(mean, (double)v);
            if (v > 0.0f && (!have || v < rho)) { rho = v; have = true; }
        }
        mean = __ddiv_rn(mean, (double)k);
        const double target = log2((double)k);
        double lo = 0.0, hi = INFINITY, mid = 1.0;
        for (int it = 0; it < 64; ++it) {
            double psum = 0.0;
            for (int j = 0; j < k; ++j) {
                const double delta = __dsub_rn((double)row[j], (double)rho);
                psum = __dadd_rn(psum, delta > 0.0 ? exp(-__ddiv_rn(delta, mid)) : 1.0);
            }
            if (fabs(__dsub_rn(psum, target)) < 1e-5) break;
            if (psum > target) {
                hi = mid;
                mid = __ddiv_rn(__dadd_rn(lo, hi), 2.0);
            } else {
                lo = mid;
                mid = (hi == INFINITY) ? __dmul_rn(mid, 2.0) : __ddiv_rn(__dadd_rn(lo, hi), 2.0);
            }
        }
        const double floor_s = __dmul_rn(1e-3, mean);
        const double sigma_d = mid < floor_s ? floor_s : mid;
        const float sigma = (float)sigma_d;
        const int64_t gi = row0 + lane;
        if (rho_out) rho_out[gi] = rho;
        if (sigma_out) sigma_out[gi] = sigma;
        // memberships, fp64 rounded to fp32 (R6), overwrite the staged distances
        float* wrow = sd + lane * stride;
        for (int j = 0; j < k; ++j) {
            const double delta = __dsub_rn((double)wrow[j], (double)rho);
            wrow[j] = delta <= 0.0 ? 1.0f : (float)exp(-__ddiv_rn(delta, (double)sigma));
        }
        if (col_out) {  // re-order the row by ascending column id (insertion sort, k <= 64)
            int32_t* crow = si + lane * stride;
            for (int a = 1; a < k; ++a) {
                const int32_t c = crow[a];
                const float w = wrow[a];
                int p = a;
                while (p > 0 && crow[p - 1] > c) { crow[p] = crow[p - 1]; wrow[p] = wrow[p - 1]; --p; }
                crow[p] = c;
                wrow[p] = w;
            }
        }
    }
    __syncwarp();
    for (int e = lane; e < rows * k; e += 32) {
        const int r = e / k, j = e - r * k;
        w_out[row0 * k + e] = sd[r * stride + j];
        if (col_out) col_out[row0 * k + e] = si[r * stride + j];
    }
}

// ---------------------------------------------------------------- scan (int64, exclusive)
constexpr int SCAN_T = 256, SCAN_ITEMS = 8, SCAN_TILE = SCAN_T * SCAN_ITEMS;

template <class Tin>
__global__ void __launch_bounds__(SCAN_T)
scan_tile_kernel(const Tin* __restrict__ in, int64_t n, int64_t* __restrict__ out, int64_t* __restrict__ tile_sums)
{
    __shared__ int64_t warp_tot[SCAN_T / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS];
    int64_t run = 0;
#pragma unroll
    for (int u = 0; u < SCAN_ITEMS; ++u) {
        const int64_t x = (base + u < n) ? (int64_t)in[base + u] : 0;
        v[u] = run;
        run += x;
    }
    // warp inclusive scan of per-thread totals
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    int64_t woff = 0;
    for (int w = 0; w < warp; ++w) woff += warp_tot[w];
    const int64_t toff = woff + inc - run;
#pragma unroll
    for (int u = 0; u < SCAN_ITEMS; ++u)
        if (base + u < n) out[base + u] = v[u] + toff;
    if (threadIdx.x == SCAN_T - 1) tile_sums[blockIdx.x] = woff + inc;
}

__global__ void scan_add_kernel(int64_t* __restrict__ out, int64_t n, const int64_t* __restrict__ offs)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += offs[i / SCAN_TILE];
}

// ---------------------------------------------------------------- transpose
__global__ void indeg_kernel(const int32_t* __restrict__ idx, int64_t m, int32_t* __restrict__ deg)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < m) {
        const int32_t c = idx[e];
        if (c >= 0) atomicAdd(deg + c, 1);
    }
}

__global__ void scatter_t_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int64_t n, int k,
                                 const int64_t* __restrict__ tptr, int32_t* __restrict__ cursor,
                                 int32_t* __restrict__ tsrc, float* __restrict__ tw)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * (int64_t)k) return;
    const int32_t c = idx[e];
    if (c < 0) return;
    const int64_t pos = tptr[c] + atomicAdd(cursor + c, 1);
    tsrc[pos] = (int32_t)(e / k);
    tw[pos] = w[e];
}

// Sort each row of A^T by source id (sources are distinct within a row): rank of an
// element = number of smaller sources in the row.  Warp per row.
__global__ void sort_t_rows_kernel(const int64_t* __restrict__ tptr, int64_t n,
                                   const int32_t* __restrict__ src_in, const float* __restrict__ w_in,
                                   int32_t* __restrict__ src_out, float* __restrict__ w_out)
{
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int64_t b = tptr[row], L = tptr[row + 1] - b;
    if (L <= 32) {
        const int32_t s = lane < L ? src_in[b + lane] : INT32_MAX;
        const float w = lane < L ? w_in[b + lane] : 0.0f;
        int rank = 0;
        for (int o = 0; o < (int)L; ++o) rank += __shfl_sync(0xffffffffu, s, o) < s;
        if (lane < L) { src_out[b + rank] = s; w_out[b + rank] = w; }
    } else {
        for (int64_t e = lane; e < L; e += 32) {
            const int32_t s = src_in[b + e];
            int64_t rank = 0;
            for (int64_t o = 0; o < L; ++o) rank += src_in[b + o] < s;
            src_out[b + rank] = s;
            w_out[b + rank] = w_in[b + e];
        }
    }
}

// Two-pointer merge of A-row (sorted by col) and A^T-row (sorted by src).
// FILL = false: count entries with w != 0; FILL = true: write them.
template <bool FILL>
__global__ void union_rows_kernel(const int32_t* __restrict__ acol, const float* __restrict__ aw, int64_t n, int k,
                                  const int64_t* __restrict__ tptr, const int32_t* __restrict__ tsrc,
                                  const float* __restrict__ tw, int32_t* __restrict__ cnt,
                                  const int64_t* __restrict__ indptr, int32_t* __restrict__ col,
                                  float* __restrict__ val)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t* ac = acol + i * k;
    const float* av = aw + i * k;
    int64_t pa = 0, pt = tptr[i];
    const int64_t ea = k, et = tptr[i + 1];
    int64_t o = FILL ? indptr[i] : 0;
    int32_t c_count = 0;
    while (pa < ea || pt < et) {
        int32_t ca = pa < ea ? ac[pa] : INT32_MAX;
        if (ca < 0) { ++pa; continue; }
        const int32_t ct = pt < et ? tsrc[pt] : INT32_MAX;
        double a = 0.0, b = 0.0;
        int32_t c;
        if (ca == ct) { c = ca; a = (double)av[pa++]; b = (double)tw[pt++]; }
        else if (ca < ct) { c = ca; a = (double)av[pa++]; }
        else { c = ct; b = (double)tw[pt++]; }
        // Eq. 2 t-conorm (R7): (a + b) - a*b in fp64, rounded to fp32; symmetric in (a, b)
        const float w = (float)__dsub_rn(__dadd_rn(a, b), __dmul_rn(a, b));
        if (w != 0.0f) {
            if (FILL) { col[o] = c; val[o] = w; ++o; }
            else ++c_count;
        }
    }
    if (!FILL) cnt[i] = c_count;
}

}  // namespace

umap_status smooth_knn(const float* dist, const int32_t* idx, int64_t n, int k, float* rho, float* sigma,
                       float* w, int32_t* col_sorted, cudaStream_t s)
{
    if (n == 0) return UMAP_OK;
    const int stride = k | 1;
    const size_t smem = (size_t)SK_WARPS * 32 * stride * (col_sorted ? 8 : 4) + (col_sorted ? 0 : 0);
    const size_t smem_alloc = (size_t)SK_WARPS * 32 * stride * 8;  // layout assumes both halves
    (void)smem;
    static PerDeviceOnce configured;
    if (configured.first()) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(smooth_knn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(SK_WARPS * 32 * 65 * 8)));
    }
    ProfScope ps(PROF_SMOOTH_KNN, s);
    smooth_knn_kernel<<<ceil_div(n, 32 * SK_WARPS), 32 * SK_WARPS, smem_alloc, s>>>(dist, idx, n, k, rho, sigma,
                                                                                   w, col_sorted);
    UMAP_LAUNCH_CHECK("smooth_knn_kernel");
    return UMAP_OK;
}

// exclusive scan of n values (int32 or int64 input) into out[0..n-1]; out[n] = total
template <class Tin>
umap_status exclusive_scan(const Tin* in, int64_t n, int64_t* out, cudaStream_t s)
{
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    Scratch sums, sums_scan;
    UMAP_TRY(sums.alloc(sizeof(int64_t) * (size_t)(tiles + 1), s));
    scan_tile_kernel<Tin><<<(unsigned)tiles, SCAN_T, 0, s>>>(in, n, out, sums.as<int64_t>());
    UMAP_LAUNCH_CHECK("scan_tile_kernel");
    if (tiles > 1) {
        UMAP_TRY(sums_scan.alloc(sizeof(int64_t) * (size_t)(tiles + 1), s));
        UMAP_TRY(exclusive_scan<int64_t>(sums.as<int64_t>(), tiles, sums_scan.as<int64_t>(), s));
        scan_add_kernel<<<ceil_div(n, 256), 256, 0, s>>>(out, n, sums_scan.as<int64_t>());
        UMAP_LAUNCH_CHECK("scan_add_kernel");
        // total = scanned offset of the virtual tile after the last one
        UMAP_CUDA_TRY(cudaMemcpyAsync(out + n, sums_scan.as<int64_t>() + tiles, sizeof(int64_t),
                                      cudaMemcpyDeviceToDevice, s));
    } else {
        UMAP_CUDA_TRY(cudaMemcpyAsync(out + n, sums.as<int64_t>(), sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    }
    return UMAP_OK;
}
template umap_status exclusive_scan<int32_t>(const int32_t*, int64_t, int64_t*, cudaStream_t);
umap_status exclusive_scan_i32(const int32_t* in, int64_t n, int64_t* out, cudaStream_t s)
{
    return exclusive_scan<int32_t>(in, n, out, s);
}
template umap_status exclusive_scan<int64_t>(const int64_t*, int64_t, int64_t*, cudaStream_t);

umap_status fuzzy_union(const int32_t* acol, const float* aw, int64_t n, int k, int64_t* indptr, int32_t* col,
                        float* val, int64_t capacity, int64_t* nnz_host, cudaStream_t s)
{
    const int64_t m = n * (int64_t)k;
    Scratch deg, tptr, cursor, tsrc0, tw0, tsrc, tw, cnt;
    UMAP_TRY(deg.alloc(sizeof(int32_t) * (size_t)n, s));
    UMAP_TRY(tptr.alloc(sizeof(int64_t) * (size_t)(n + 1), s));
    UMAP_TRY(cursor.alloc(sizeof(int32_t) * (size_t)n, s));
    UMAP_TRY(tsrc0.alloc(sizeof(int32_t) * (size_t)m, s));
    UMAP_TRY(tw0.alloc(sizeof(float) * (size_t)m, s));
    UMAP_TRY(tsrc.alloc(sizeof(int32_t) * (size_t)m, s));
    UMAP_TRY(tw.alloc(sizeof(float) * (size_t)m, s));
    UMAP_TRY(cnt.alloc(sizeof(int32_t) * (size_t)n, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(deg.p, 0, sizeof(int32_t) * n, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(cursor.p, 0, sizeof(int32_t) * n, s));
    ProfScope ps(PROF_UNION, s);  // the whole union (includes one nnz read-back)
    indeg_kernel<<<ceil_div(m, 256), 256, 0, s>>>(acol, m, deg.as<int32_t>());
    UMAP_LAUNCH_CHECK("indeg_kernel");
    UMAP_TRY(exclusive_scan<int32_t>(deg.as<int32_t>(), n, tptr.as<int64_t>(), s));
    scatter_t_kernel<<<ceil_div(m, 256), 256, 0, s>>>(acol, aw, n, k, tptr.as<int64_t>(), cursor.as<int32_t>(),
                                                      tsrc0.as<int32_t>(), tw0.as<float>());
    UMAP_LAUNCH_CHECK("scatter_t_kernel");
    sort_t_rows_kernel<<<ceil_div(n * 32, 256), 256, 0, s>>>(tptr.as<int64_t>(), n, tsrc0.as<int32_t>(),
                                                              tw0.as<float>(), tsrc.as<int32_t>(), tw.as<float>());
    UMAP_LAUNCH_CHECK("sort_t_rows_kernel");
    union_rows_kernel<false><<<ceil_div(n, 128), 128, 0, s>>>(acol, aw, n, k, tptr.as<int64_t>(), tsrc.as<int32_t>(),
                                                             tw.as<float>(), cnt.as<int32_t>(), nullptr, nullptr,
                                                             nullptr);
    UMAP_LAUNCH_CHECK("union_rows_kernel<count>");
    UMAP_TRY(exclusive_scan<int32_t>(cnt.as<int32_t>(), n, indptr, s));
    int64_t total = 0;
    UMAP_CUDA_TRY(cudaMemcpyAsync(&total, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    if (total > capacity) {
        set_last_error("fuzzy_union: capacity " + std::to_string(capacity) + " < nnz " + std::to_string(total));
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    union_rows_kernel<true><<<ceil_div(n, 128), 128, 0, s>>>(acol, aw, n, k, tptr.as<int64_t>(), tsrc.as<int32_t>(),
                                                            tw.as<float>(), nullptr, indptr, col, val);
    UMAP_LAUNCH_CHECK("union_rows_kernel<fill>");
    if (nnz_host) *nnz_host = total;
    return UMAP_OK;
}

}  // namespace umapb200

// ---------------------------------------------------------------- supervised adjustment (f4)
// "when training labels are provided, an additional step ... adjusts the membership
// strengths of the fuzzy sets based on their labels" (rule R17): entry (i, j)
// times 1 (same known label), f_far = fp32(exp(-far_dist)) (different known labels) or
// f_unk = fp32(exp(-unknown_dist)) (either label -1); products below 1e-8 are dropped.
// Two passes over the CSR (count -> scan -> fill), thread per row; the rule is symmetric in
// (i, j), so the result stays symmetric.
namespace umapb200 {
namespace {

__device__ __forceinline__ float label_factor(int32_t li, int32_t lj, float f_far, float f_unk)
{
    return (li < 0 || lj < 0) ? f_unk : (li == lj ? 1.0f : f_far);
}

template <bool FILL>
__global__ void supervised_rows_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ col,
                                       const float* __restrict__ val, int64_t n, const int32_t* __restrict__ labels,
                                       float f_far, float f_unk, int32_t* __restrict__ cnt,
                                       const int64_t* __restrict__ out_indptr, int32_t* __restrict__ out_col,
                                       float* __restrict__ out_val)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t li = labels[i];
    int64_t o = FILL ? out_indptr[i] : 0;
    int c = 0;
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
        const int32_t j = col[e];
        const float w = __fmul_rn(val[e], label_factor(li, labels[j], f_far, f_unk));
        if (w >= 1e-8f) {
            if (FILL) { out_col[o] = j; out_val[o] = w; ++o; }
            ++c;
        }
    }
    if (!FILL) cnt[i] = c;
}

}  // namespace

umap_status supervised_adjust(const int64_t* indptr, const int32_t* col, const float* val, int64_t n,
                              const int32_t* labels, float far_dist, float unknown_dist, int64_t* out_indptr,
                              int32_t* out_col, float* out_val, int64_t capacity, int64_t* nnz_host, cudaStream_t s)
{
    const float f_far = (float)std::exp(-(double)far_dist), f_unk = (float)std::exp(-(double)unknown_dist);
    Scratch cnt;
    UMAP_TRY(cnt.alloc(sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1), s));
    supervised_rows_kernel<false><<<ceil_div(n, 256), 256, 0, s>>>(indptr, col, val, n, labels, f_far, f_unk,
                                                                   cnt.as<int32_t>(), nullptr, nullptr, nullptr);
    UMAP_LAUNCH_CHECK("supervised_rows_kernel<count>");
    UMAP_TRY(exclusive_scan<int32_t>(cnt.as<int32_t>(), n, out_indptr, s));
    int64_t total = 0;
    UMAP_CUDA_TRY(cudaMemcpyAsync(&total, out_indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    if (total > capacity) {
        set_last_error("supervised_adjust: capacity " + std::to_string(capacity) + " < nnz " + std::to_string(total));
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    supervised_rows_kernel<true><<<ceil_div(n, 256), 256, 0, s>>>(indptr, col, val, n, labels, f_far, f_unk, nullptr,
                                                                  out_indptr, out_col, out_val);
    UMAP_LAUNCH_CHECK("supervised_rows_kernel<fill>");
    if (nnz_host) *nnz_host = total;
    return UMAP_OK;
}

}  // namespace umapb200
