// knn_exact.cu -- exact fp32 brute-force distance tiles with fused epilogues.
//
// a2 kNN ("exact search ... exhaustive distances ... along with a heap")
// and the input-space rank count of a10 trustworthiness (Alg. 1).
//
// Distance (R2): d2(i,j) = s, s = 0; for f = 0..d-1 ascending: t = x_if - y_jf;
// s = fmaf(t, t, s).  Every output is accumulated by one thread in ascending f
// (no split-K), with explicit __fsub_rn/__fmaf_rn, so the result is bit-identical
// to the oracle's definition.  Zero padding beyond d adds fmaf(0,0,s) = s exactly.
//
// Tiling: CTA = 128 query rows x 128 reference rows per tile, 256 threads, each
// thread an 8x8 register micro-tile; K staged through smem 16 features at a time
// with register prefetch of the next K slab.  After each reference tile the 128x128
// fp32 block goes to smem and one thread per query row filters it against its
// running k-th key (TOPK) or its k sorted rank thresholds (RANK).
#include "common.cuh"

namespace umapb200 {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, NT = 256;
constexpr int DS = BN + 4;  // padded row stride of the distance block (float4-aligned)

enum { EPI_TOPK = 0, EPI_RANK = 1 };

struct TileArgs {
    const float* Xq; int64_t nq;
    const float* Xr; int64_t nr;
    int d;
    int k;
    int64_t self_shift;      // local ref j is the query's own row when j == q + self_shift
    int exclude_self;        // exclude that row (R1)
    int64_t index_offset;    // added to reference ids on output / in keys
    int64_t split_len;       // reference rows per split (multiple of BN)
    // TOPK outputs
    int32_t* out_idx;        // [split][nq][k]  (split-major); ids are j + index_offset
    float* out_d2;           // same layout, squared distances
    // RANK inputs/outputs
    const float* thr_d2;     // [nq][k] sorted by key
    const int32_t* thr_id;   // [nq][k] (global ids, index_offset already applied)
    int32_t* out_cnt;        // [split][nq][k] counts of l with key < threshold t (not cumulative)
};

template <int KMAX, int MODE>
__global__ void __launch_bounds__(NT, 2) dist_tile_kernel(TileArgs a)
{
    extern __shared__ __align__(16) float smem[];
    float* As = smem;                     // [BK][BM]
    float* Bs = As + BK * BM;             // [BK][BN]
    float* Ds = Bs + BK * BN;             // [BM][DS]
    float* Ld = Ds + BM * DS;             // [KMAX][BM]  list keys (TOPK) / thresholds (RANK)
    int32_t* Li = reinterpret_cast<int32_t*>(Ld + KMAX * BM);  // [KMAX][BM]
    int32_t* Hc = Li + KMAX * BM;         // [KMAX][BM] (RANK histogram)

    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t q0 = (int64_t)blockIdx.x * BM;
    const int64_t r_lo = (int64_t)blockIdx.y * a.split_len;
    const int64_t r_hi = min(a.nr, r_lo + a.split_len);
    const int d = a.d;
    const int k = a.k;

    // per-query state (threads 0..127 own query q0 + tid)
    float kth_d = INFINITY;
    int32_t kth_i = INT32_MAX;
    int cnt = 0;
    const int64_t myq = q0 + tid;
    const bool owner = tid < BM && myq < a.nq;
    int64_t self_j = -1;
    if (owner && a.exclude_self) self_j = myq + a.self_shift;
    if (tid < BM) {
        for (int t = 0; t < KMAX; ++t) {
            if (MODE == EPI_RANK) {
                if (owner && t < k) {
                    Ld[t * BM + tid] = a.thr_d2[myq * k + t];
                    Li[t * BM + tid] = a.thr_id[myq * k + t];
                } else {
                    Ld[t * BM + tid] = -INFINITY;
                    Li[t * BM + tid] = INT32_MIN;
                }
                Hc[t * BM + tid] = 0;
            } else {
                Ld[t * BM + tid] = INFINITY;
                Li[t * BM + tid] = INT32_MAX;
            }
        }
        if (MODE == EPI_RANK && owner) { kth_d = Ld[(k - 1) * BM + tid]; kth_i = Li[(k - 1) * BM + tid]; }
    }

    // load mapping: thread -> (row = tid & 127, feature half = tid >> 7) of a BMxBK slab
    const int lrow = tid & 127, lhalf = tid >> 7;
    const int64_t qrow = q0 + lrow;

    for (int64_t rb = r_lo; rb < r_hi; rb += BN) {
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

        const int64_t rrow = rb + lrow;
        float pa[8], pb[8];
        auto load_slab = [&](int k0) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int f = k0 + lhalf * 8 + u;
                pa[u] = (qrow < a.nq && f < d) ? __ldg(a.Xq + qrow * d + f) : 0.0f;
                pb[u] = (rrow < r_hi && f < d) ? __ldg(a.Xr + rrow * d + f) : 0.0f;
            }
        };
        load_slab(0);
        for (int k0 = 0; k0 < d; k0 += BK) {
            __syncthreads();  // previous slab consumed
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                As[(lhalf * 8 + u) * BM + lrow] = pa[u];
                Bs[(lhalf * 8 + u) * BN + lrow] = pb[u];
            }
            __syncthreads();
            if (k0 + BK < d) load_slab(k0 + BK);
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                const float4 a0 = *reinterpret_cast<const float4*>(As + kk * BM + ty * 8);
                const float4 a1 = *reinterpret_cast<const float4*>(As + kk * BM + ty * 8 + 4);
                const float4 b0 = *reinterpret_cast<const float4*>(Bs + kk * BN + tx * 8);
                const float4 b1 = *reinterpret_cast<const float4*>(Bs + kk * BN + tx * 8 + 4);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float t = __fsub_rn(av[i], bv[j]);
                        acc[i][j] = __fmaf_rn(t, t, acc[i][j]);
                    }
            }
        }
        __syncthreads();
        // distance block -> smem
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float* row = Ds + (ty * 8 + i) * DS + tx * 8;
            *reinterpret_cast<float4*>(row) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            *reinterpret_cast<float4*>(row + 4) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        }
        __syncthreads();
        if (owner) {
            const float* row = Ds + tid * DS;
            const int ncols = (int)imin64(BN, r_hi - rb);
            for (int c4 = 0; c4 < ncols; c4 += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(row + c4);
                const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = c4 + u;
                    if (c >= ncols) break;
                    const int64_t j = rb + c;
                    if (j == self_j) continue;
                    const float v = vv[u];
                    const int32_t gid = (int32_t)(j + a.index_offset);
                    if (!key_less(v, gid, kth_d, kth_i)) continue;
                    if (MODE == EPI_TOPK) {
                        int p;
                        if (cnt < k) p = cnt++;
                        else p = k - 1;
                        while (p > 0) {
                            const float pd = Ld[(p - 1) * BM + tid];
                            const int32_t pi = Li[(p - 1) * BM + tid];
                            if (!key_less(v, gid, pd, pi)) break;
                            Ld[p * BM + tid] = pd;
                            Li[p * BM + tid] = pi;
                            --p;
                        }
                        Ld[p * BM + tid] = v;
                        Li[p * BM + tid] = gid;
                        if (cnt == k) { kth_d = Ld[(k - 1) * BM + tid]; kth_i = Li[(k - 1) * BM + tid]; }
                    } else {
                        // first threshold t with key(v) < key(thr_t): counts toward t..k-1
                        int t = 0;
                        while (!key_less(v, gid, Ld[t * BM + tid], Li[t * BM + tid])) ++t;
                        Hc[t * BM + tid] += 1;
                    }
                }
            }
        }
    }
    if (owner) {
        const int64_t base = ((int64_t)blockIdx.y * a.nq + myq) * k;
        for (int t = 0; t < k; ++t) {
            if (MODE == EPI_TOPK) {
                a.out_idx[base + t] = t < cnt ? Li[t * BM + tid] : -1;
                a.out_d2[base + t] = t < cnt ? Ld[t * BM + tid] : INFINITY;
            } else {
                a.out_cnt[base + t] = Hc[t * BM + tid];
            }
        }
    }
}

size_t tile_smem_bytes(int kmax, int mode)
{
    size_t s = (size_t)(BK * BM + BK * BN + BM * DS) * 4 + (size_t)kmax * BM * 8;
    if (mode == EPI_RANK) s += (size_t)kmax * BM * 4;
    return s;
}

template <int KMAX, int MODE>
umap_status launch_tiles_t(const TileArgs& a, int n_splits, cudaStream_t s)
{
    const size_t smem = tile_smem_bytes(KMAX, MODE);
    static PerDeviceOnce configured;
    if (configured.first()) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(dist_tile_kernel<KMAX, MODE>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    dim3 grid(ceil_div(a.nq, BM), n_splits);
    ProfScope ps(MODE == 0 ? PROF_KNN_EXACT : PROF_TRUST_EXACT, s);
    dist_tile_kernel<KMAX, MODE><<<grid, NT, smem, s>>>(a);
    UMAP_LAUNCH_CHECK("dist_tile_kernel");
    return UMAP_OK;
}

template <int MODE>
umap_status launch_tiles(const TileArgs& a, int n_splits, cudaStream_t s)
{
    if (a.k <= 16) return launch_tiles_t<16, MODE>(a, n_splits, s);
    if (a.k <= 32) return launch_tiles_t<32, MODE>(a, n_splits, s);
    if (a.k <= 64) return launch_tiles_t<64, MODE>(a, n_splits, s);
    set_last_error("k > 64 unsupported");
    return UMAP_ERR_K_OUT_OF_RANGE;
}

// choose how many reference splits so the grid covers the GPU at least twice
int choose_splits(int64_t nq, int64_t nr)
{
    const int64_t qblocks = (nq + BM - 1) / BM;
    const int64_t target = 2LL * num_sms();
    int64_t splits = (target + qblocks - 1) / qblocks;
    const int64_t max_splits = std::max<int64_t>(1, nr / (4 * BN));  // >= 4 tiles per split
    splits = std::min<int64_t>(splits, max_splits);
    splits = std::min<int64_t>(splits, 64);
    return (int)std::max<int64_t>(1, splits);
}

// ------------------------------------------------------------------ merge
// k-way merge of n_parts sorted candidate lists per row by key (d2, id).
__global__ void topk_merge_kernel(const int32_t* __restrict__ idx_in, const float* __restrict__ d2_in,
                                  int n_parts, int64_t n, int k_in, int k_out, int out_squared,
                                  int32_t* __restrict__ idx, float* __restrict__ dist)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int ptr[64];
    for (int p = 0; p < n_parts; ++p) ptr[p] = 0;
    for (int t = 0; t < k_out; ++t) {
        int best = -1;
        float bd = INFINITY;
        int32_t bi = INT32_MAX;
        for (int p = 0; p < n_parts; ++p) {
            if (ptr[p] >= k_in) continue;
            const int64_t o = ((int64_t)p * n + i) * k_in + ptr[p];
            const float dv = d2_in[o];
            const int32_t iv = idx_in[o];
            if (iv < 0) continue;
            if (best < 0 || key_less(dv, iv, bd, bi)) { best = p; bd = dv; bi = iv; }
        }
        if (best >= 0) ++ptr[best];
        idx[i * k_out + t] = best >= 0 ? bi : -1;
        dist[i * k_out + t] = best >= 0 ? (out_squared ? bd : __fsqrt_rn(bd)) : INFINITY;
    }
}

__global__ void finalize_single_kernel(const int32_t* __restrict__ idx_in, const float* __restrict__ d2,
                                       int64_t total, int out_squared, int32_t* __restrict__ idx,
                                       float* __restrict__ dist)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    idx[e] = idx_in[e];
    const float v = d2[e];
    dist[e] = out_squared ? v : (isinf(v) ? v : __fsqrt_rn(v));
}

}  // namespace

umap_status topk_merge(const int32_t* idx_in, const float* d2_in, int n_parts, int64_t n, int k_in,
                       int k_out, int out_squared, int32_t* idx, float* dist, cudaStream_t s)
{
    if (n_parts < 1 || n_parts > 64 || k_in < 1 || k_out < 1 || k_out > 64) {
        set_last_error("topk_merge: n_parts in [1,64], k in [1,64] required");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return UMAP_OK;
    topk_merge_kernel<<<ceil_div(n, 128), 128, 0, s>>>(idx_in, d2_in, n_parts, n, k_in, k_out, out_squared,
                                                       idx, dist);
    UMAP_LAUNCH_CHECK("topk_merge_kernel");
    return UMAP_OK;
}

// Exact kNN of X_q against X_r (device pointers), results sorted by key.
umap_status knn_exact(const float* Xq, int64_t nq, const float* Xr, int64_t nr, int d, int k,
                      int64_t self_shift, int exclude_self, int64_t index_offset, int out_squared, int32_t* idx,
                      float* dist, cudaStream_t s)
{
    if (nq == 0) return UMAP_OK;
    const int splits = choose_splits(nq, nr);
    int64_t split_len = (nr + splits - 1) / splits;
    split_len = (split_len + BN - 1) / BN * BN;
    const int n_splits = (int)((nr + split_len - 1) / split_len);

    Scratch cand_i, cand_d;
    UMAP_TRY(cand_i.alloc(sizeof(int32_t) * (size_t)n_splits * nq * k, s));
    UMAP_TRY(cand_d.alloc(sizeof(float) * (size_t)n_splits * nq * k, s));
    TileArgs a{};
    a.Xq = Xq; a.nq = nq; a.Xr = Xr; a.nr = nr; a.d = d; a.k = k;
    a.self_shift = self_shift; a.exclude_self = exclude_self; a.index_offset = index_offset;
    a.split_len = split_len;
    a.out_idx = cand_i.as<int32_t>(); a.out_d2 = cand_d.as<float>();
    UMAP_TRY(launch_tiles<EPI_TOPK>(a, n_splits, s));
    if (n_splits == 1) {
        const int64_t total = nq * (int64_t)k;
        finalize_single_kernel<<<ceil_div(total, 256), 256, 0, s>>>(a.out_idx, a.out_d2, total, out_squared,
                                                                     idx, dist);
        UMAP_LAUNCH_CHECK("finalize_single_kernel");
        return UMAP_OK;
    }
    return topk_merge(a.out_idx, a.out_d2, n_splits, nq, k, k, out_squared, idx, dist, s);
}

// Input-space rank counts for trustworthiness: for each query row q (global row
// q + row_offset of X) and each of its k sorted thresholds (thr_d2, thr_id),
// cnt[q][t] = #{ l != self : key(d2(q,l), l) < key(thr_t) and not < key(thr_{t-1}) }.
umap_status rank_count_exact(const float* Xq, int64_t nq, const float* X, int64_t n, int d, int k,
                             int64_t self_offset, const float* thr_d2, const int32_t* thr_id,
                             int32_t* cnt_out /* [nq][k], summed over splits */, Scratch& tmp,
                             int* n_splits_out, cudaStream_t s)
{
    const int splits = choose_splits(nq, n);
    int64_t split_len = (n + splits - 1) / splits;
    split_len = (split_len + BN - 1) / BN * BN;
    const int n_splits = (int)((n + split_len - 1) / split_len);
    *n_splits_out = n_splits;
    TileArgs a{};
    a.Xq = Xq; a.nq = nq; a.Xr = X; a.nr = n; a.d = d; a.k = k;
    a.self_shift = self_offset; a.exclude_self = 1; a.index_offset = 0; a.split_len = split_len;
    a.thr_d2 = thr_d2; a.thr_id = thr_id;
    if (n_splits == 1) {
        a.out_cnt = cnt_out;
    } else {
        UMAP_TRY(tmp.alloc(sizeof(int32_t) * (size_t)n_splits * nq * k, s));
        a.out_cnt = tmp.as<int32_t>();
    }
    return launch_tiles<EPI_RANK>(a, n_splits, s);
}

}  // namespace umapb200
