// sgd.cu -- random init (a7), SGD layout (a6, a8) and transform SGD (a9).
//
// Layout SGD.  One launch per epoch e (1 <= e < N).
// A warp owns 32 consecutive vertices (their CSR rows are contiguous): it streams
// the rows' (col, w) pairs with coalesced loads, evaluates the closed-form schedule
// (R9) per edge, compacts the due edges into a per-warp shared-memory queue and
// processes the queue 32 items at a time, so every lane carries a due edge while
// the expensive part runs (attractive term + m negatives + 2 Philox calls).
//
//  * DETERMINISTIC (R13): reads Y_e only, writes Y_{e+1} (ping-pong).  Each
//    vertex is updated only by the warp that owns it ("owner computes"): because
//    B is bit-exactly symmetric, the tail update of edge (i,j) equals the head
//    update of edge (j,i), so vertex i receives 2 q(g_att) per own due edge plus
//    q(g_rep) per negative, q(g) = round(g 2^32) summed in int64 (order-free, so the
//    result is identical for any launch configuration).  No global atomics.
//  * HOGWILD: in-place.  Each due edge reads the live positions, moves
//    its head in registers through the attractive and the m repulsive updates
//    (the paper's register accumulation) and pushes -g_att to the tail and
//    the accumulated head delta with fp32 vector atomics.
#include "common.cuh"

namespace umapb200 {

namespace {

struct SgdArgs {
    const int64_t* indptr;
    const int32_t* col;
    const float* val;
    const float* w_max;      // device scalar
    int64_t n;
    const float* Yr;         // positions read (Y_e)
    float* Yw;               // positions written (Y_{e+1}, or == Yr in Hogwild)
    float a, b, gamma, alpha0;
    int32_t n_epochs, epoch, m;
    uint32_t key0, key1;
    unsigned long long* positives;  // optional device counter
};

__device__ __forceinline__ float clip4(float v) { return fminf(fmaxf(v, -4.0f), 4.0f); }

// s^b via exp2(b log2 s); s > 0
__device__ __forceinline__ float pow_b(float s, float b) { return exp2f(b * __log2f(s)); }

__device__ __forceinline__ bool edge_due(float r, int e)
{
    return floorf(__fmul_rn((float)e, r)) > floorf(__fmul_rn((float)(e - 1), r));
}

template <int DIM>
__device__ __forceinline__ void load_row(const float* Y, int64_t v, float (&y)[DIM])
{
    if (DIM == 2) {
        const float2 t = *reinterpret_cast<const float2*>(Y + v * 2);
        y[0] = t.x; y[1] = t.y;
    } else if (DIM == 4) {
        const float4 t = *reinterpret_cast<const float4*>(Y + v * 4);
        y[0] = t.x; y[1] = t.y; y[2] = t.z; y[3] = t.w;
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) y[c] = Y[v * DIM + c];
    }
}

constexpr int SGD_WARPS = 8;
constexpr int QCAP = 64;

// Process one due edge (h, t): returns the head delta (deterministic: in fixed point).
template <int DIM, bool DET>
__device__ __forceinline__ void process_edge(const SgdArgs& A, float alpha, int64_t h, int64_t t,
                                             long long (&qacc)[DIM])
{
    float yh[DIM], yt[DIM], g[DIM];
    load_row<DIM>(A.Yr, h, yh);
    load_row<DIM>(A.Yr, t, yt);
    float s = 0.0f;
#pragma unroll
    for (int c = 0; c < DIM; ++c) { const float df = yh[c] - yt[c]; s = fmaf(df, df, s); }
    float coef = 0.0f;
    if (s > 0.0f) {
        const float sb = pow_b(s, A.b);
        coef = __fdividef(-2.0f * A.a * A.b * __fdividef(sb, s), fmaf(A.a, sb, 1.0f));
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) g[c] = clip4(coef * (yh[c] - yt[c])) * alpha;
    float h0[DIM];
    if (DET) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) qacc[c] += 2 * __double2ll_rn((double)g[c] * 4294967296.0);
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) { h0[c] = yh[c]; yh[c] += g[c]; }
        if (DIM == 2) {
            atomicAdd(reinterpret_cast<float2*>(A.Yw + t * 2), make_float2(-g[0], -g[1]));
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) atomicAdd(A.Yw + t * DIM + c, -g[c]);
        }
    }
    // m negative samples, head only; Philox counter (h, t, e, p>>2) (R11)
    u32x4 rnd = {0, 0, 0, 0};
    for (int p = 0; p < A.m; ++p) {
        if ((p & 3) == 0)
            rnd = philox4x32_10((uint32_t)h, (uint32_t)t, (uint32_t)A.epoch, (uint32_t)(p >> 2), A.key0, A.key1);
        const uint32_t u = pick(rnd, p & 3);
        const int64_t v = (int64_t)(((unsigned long long)u * (unsigned long long)A.n) >> 32);
        if (v == h) continue;
        float yv[DIM];
        load_row<DIM>(A.Yr, v, yv);
        float s2 = 0.0f;
#pragma unroll
        for (int c = 0; c < DIM; ++c) { const float df = yh[c] - yv[c]; s2 = fmaf(df, df, s2); }
        if (s2 > 0.0f) {
            const float sb = pow_b(s2, A.b);
            const float cr = __fdividef(2.0f * A.gamma * A.b, (0.001f + s2) * fmaf(A.a, sb, 1.0f));
#pragma unroll
            for (int c = 0; c < DIM; ++c) g[c] = clip4(cr * (yh[c] - yv[c])) * alpha;
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) g[c] = 4.0f * alpha;
        }
        if (DET) {
#pragma unroll
            for (int c = 0; c < DIM; ++c) qacc[c] += __double2ll_rn((double)g[c] * 4294967296.0);
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) yh[c] += g[c];
        }
    }
    if (!DET) {
        if (DIM == 2) {
            atomicAdd(reinterpret_cast<float2*>(A.Yw + h * 2), make_float2(yh[0] - h0[0], yh[1] - h0[1]));
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) atomicAdd(A.Yw + h * DIM + c, yh[c] - h0[c]);
        }
    }
}

template <int DIM, bool DET>
__global__ void __launch_bounds__(32 * SGD_WARPS) sgd_epoch_kernel(SgdArgs A)
{
    __shared__ int32_t q_h[SGD_WARPS][QCAP];   // local owner lane of the queued edge
    __shared__ int32_t q_t[SGD_WARPS][QCAP];   // tail vertex
    __shared__ long long acc[SGD_WARPS][DIM][32];
    __shared__ int64_t ptr_s[SGD_WARPS][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t v0 = ((int64_t)blockIdx.x * SGD_WARPS + warp) * 32;
    if (v0 >= A.n) return;
    const int nv = (int)imin64(32, A.n - v0);
    ptr_s[warp][lane] = A.indptr[v0 + min(lane, nv)];
    if (lane == 0) ptr_s[warp][32] = A.indptr[v0 + nv];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[warp][c][lane] = 0;
    __syncwarp();
    const int64_t e_begin = ptr_s[warp][0], e_end = ptr_s[warp][32];
    const float w_max = *A.w_max;
    const float alpha = __fmul_rn(A.alpha0, __fsub_rn(1.0f, __fdiv_rn((float)A.epoch, (float)A.n_epochs)));
    int qn = 0;
    unsigned long long due_count = 0;

    auto drain = [&](int count) {
        // lanes < count take one queued item each
        if (lane < count) {
            const int hl = q_h[warp][lane];
            long long qa[DIM];
#pragma unroll
            for (int c = 0; c < DIM; ++c) qa[c] = 0;
            process_edge<DIM, DET>(A, alpha, v0 + hl, (int64_t)q_t[warp][lane], qa);
            if (DET) {
#pragma unroll
                for (int c = 0; c < DIM; ++c)
                    atomicAdd(reinterpret_cast<unsigned long long*>(&acc[warp][c][hl]), (unsigned long long)qa[c]);
            }
        }
        __syncwarp();
    };

    for (int64_t base = e_begin; base < e_end; base += 32) {
        const int64_t e = base + lane;
        bool due = false;
        int32_t tail = 0, hl = 0;
        if (e < e_end) {
            const float r = __fdiv_rn(A.val[e], w_max);
            due = edge_due(r, A.epoch);
            tail = A.col[e];
            // owner lane: largest l with ptr_s[l] <= e (binary search over 33 offsets)
            int lo = 0, hi = nv;  // invariant ptr[lo] <= e < ptr[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (ptr_s[warp][mid] <= e) lo = mid; else hi = mid;
            }
            hl = lo;
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, due);
        due_count += __popc(ballot);
        if (due) {
            const int pos = qn + __popc(ballot & ((1u << lane) - 1u));
            q_h[warp][pos] = hl;
            q_t[warp][pos] = tail;
        }
        __syncwarp();
        qn += __popc(ballot);
        if (qn >= 32) {
            drain(32);
            qn -= 32;
            if (lane < qn) {  // move the remainder to the front
                q_h[warp][lane] = q_h[warp][32 + lane];
                q_t[warp][lane] = q_t[warp][32 + lane];
            }
            __syncwarp();
        }
    }
    if (qn > 0) drain(qn);
    if (DET && lane < nv) {
        const int64_t v = v0 + lane;
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            const double upd = (double)acc[warp][c][lane] * (1.0 / 4294967296.0);
            A.Yw[v * DIM + c] = (float)((double)A.Yr[v * DIM + c] + upd);
        }
    }
    if (A.positives && lane == 0 && due_count) atomicAdd(A.positives, due_count);
}

__global__ void wmax_kernel(const float* __restrict__ val, int64_t nnz, float* __restrict__ out)
{
    float m = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
        m = fmaxf(m, val[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));  // m >= 0
}

__global__ void wmax_dense_kernel(const float* __restrict__ val, int64_t m, float* __restrict__ out)
{
    float mx = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmaxf(mx, val[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(mx));
}

__global__ void random_init_kernel(int64_t n, int dim, uint32_t k0, uint32_t k1, float* __restrict__ Y)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * dim) return;
    const int64_t v = i / dim;
    const int c = (int)(i - v * dim);
    const u32x4 r = philox4x32_10((uint32_t)v, (uint32_t)c, 0xFFFFFFFFu, 0u, k0, k1);
    const float f = __fmul_rn((float)(r.x >> 8), 1.0f / 16777216.0f);
    Y[i] = __fadd_rn(-10.0f, __fmul_rn(20.0f, f));
}

// ---------------------------------------------------------------- transform SGD (a9)
// Thread per query row; all epochs in one launch (rows are independent: P:138 only
// the query rows move, the training layout is frozen), so there is no inter-epoch
// barrier and no atomics.  Deterministic by construction.
template <int DIM, int KMAX>
__global__ void __launch_bounds__(128)
transform_sgd_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int64_t nq, int k,
                     const float* __restrict__ Ytr, int64_t ntr, float* __restrict__ Yq, const float* w_max_p,
                     float a, float b, float gamma, float alpha0, int n_epochs_t, int e_begin, int e_end, int m,
                     uint32_t key0, uint32_t key1, int64_t q_offset, int init)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    float y[DIM];
    if (init) {
        // L1-normalised weighted mean of the neighbours' training positions, fp64 in neighbour order
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            double num = 0.0, den = 0.0;
            for (int j = 0; j < k; ++j) {
                const double wj = (double)w[q * k + j];
                num = __dadd_rn(num, __dmul_rn(wj, (double)Ytr[(int64_t)idx[q * k + j] * DIM + c]));
                den = __dadd_rn(den, wj);
            }
            y[c] = den > 0.0 ? (float)__ddiv_rn(num, den) : 0.0f;
        }
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) y[c] = Yq[q * DIM + c];
    }
    const float w_max = *w_max_p;
    float rr[KMAX];
    int32_t tt[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        rr[j] = j < k ? __fdiv_rn(w[q * k + j], w_max) : 0.0f;
        tt[j] = j < k ? idx[q * k + j] : 0;
    }
    const uint32_t head = (uint32_t)(q + q_offset);
    if (e_begin < 1) e_begin = 1;
    if (e_end > n_epochs_t) e_end = n_epochs_t;
    for (int e = e_begin; e < e_end; ++e) {
        const float alpha = __fmul_rn(alpha0, __fsub_rn(1.0f, __fdiv_rn((float)e, (float)n_epochs_t)));
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            if (j >= k || !edge_due(rr[j], e)) continue;
            const int64_t t = tt[j];
            float yt[DIM], g[DIM];
            load_row<DIM>(Ytr, t, yt);
            float s = 0.0f;
#pragma unroll
            for (int c = 0; c < DIM; ++c) { const float df = y[c] - yt[c]; s = fmaf(df, df, s); }
            float coef = 0.0f;
            if (s > 0.0f) {
                const float sb = pow_b(s, b);
                coef = __fdividef(-2.0f * a * b * __fdividef(sb, s), fmaf(a, sb, 1.0f));
            }
#pragma unroll
            for (int c = 0; c < DIM; ++c) { g[c] = clip4(coef * (y[c] - yt[c])) * alpha; }
#pragma unroll
            for (int c = 0; c < DIM; ++c) y[c] += g[c];
            u32x4 rnd = {0, 0, 0, 0};
            for (int p = 0; p < m; ++p) {
                if ((p & 3) == 0) rnd = philox4x32_10(head, (uint32_t)t, (uint32_t)e, (uint32_t)(p >> 2), key0, key1);
                const uint32_t u = pick(rnd, p & 3);
                const int64_t v = (int64_t)(((unsigned long long)u * (unsigned long long)ntr) >> 32);
                float yv[DIM];
                load_row<DIM>(Ytr, v, yv);
                float s2 = 0.0f;
#pragma unroll
                for (int c = 0; c < DIM; ++c) { const float df = y[c] - yv[c]; s2 = fmaf(df, df, s2); }
                if (s2 > 0.0f) {
                    const float sb = pow_b(s2, b);
                    const float cr = __fdividef(2.0f * gamma * b, (0.001f + s2) * fmaf(a, sb, 1.0f));
#pragma unroll
                    for (int c = 0; c < DIM; ++c) g[c] = clip4(cr * (y[c] - yv[c])) * alpha;
                } else {
#pragma unroll
                    for (int c = 0; c < DIM; ++c) g[c] = 4.0f * alpha;
                }
#pragma unroll
                for (int c = 0; c < DIM; ++c) y[c] += g[c];
            }
        }
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) Yq[q * DIM + c] = y[c];
}

template <int DIM>
umap_status launch_epoch(const SgdArgs& A, bool det, cudaStream_t s)
{
    const unsigned grid = ceil_div(A.n, 32 * SGD_WARPS);
    if (det) sgd_epoch_kernel<DIM, true><<<grid, 32 * SGD_WARPS, 0, s>>>(A);
    else sgd_epoch_kernel<DIM, false><<<grid, 32 * SGD_WARPS, 0, s>>>(A);
    UMAP_LAUNCH_CHECK("sgd_epoch_kernel");
    return UMAP_OK;
}

template <int DIM, int KMAX>
umap_status launch_transform_t(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                               float* Yq, const float* wmax, const umap_params* p, int nt, int eb, int ee,
                               int64_t q_offset, int init, cudaStream_t s)
{
    transform_sgd_kernel<DIM, KMAX><<<ceil_div(nq, 128), 128, 0, s>>>(
        idx, w, nq, k, Ytr, ntr, Yq, wmax, p->a, p->b, p->repulsion_strength, p->learning_rate, nt, eb, ee,
        p->negative_sample_rate, (uint32_t)p->seed, (uint32_t)(p->seed >> 32), q_offset, init);
    UMAP_LAUNCH_CHECK("transform_sgd_kernel");
    return UMAP_OK;
}

template <int DIM>
umap_status launch_transform(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                             float* Yq, const float* wmax, const umap_params* p, int nt, int eb, int ee,
                             int64_t q_offset, int init, cudaStream_t s)
{
    if (k <= 16) return launch_transform_t<DIM, 16>(idx, w, nq, k, Ytr, ntr, Yq, wmax, p, nt, eb, ee, q_offset, init, s);
    if (k <= 32) return launch_transform_t<DIM, 32>(idx, w, nq, k, Ytr, ntr, Yq, wmax, p, nt, eb, ee, q_offset, init, s);
    return launch_transform_t<DIM, 64>(idx, w, nq, k, Ytr, ntr, Yq, wmax, p, nt, eb, ee, q_offset, init, s);
}

}  // namespace

bool dim_supported(int dim) { return dim == 1 || dim == 2 || dim == 3 || dim == 4 || dim == 8 || dim == 16; }

umap_status random_init(int64_t n, int dim, uint64_t seed, float* Y, cudaStream_t s)
{
    if (n == 0) return UMAP_OK;
    random_init_kernel<<<ceil_div(n * dim, 256), 256, 0, s>>>(n, dim, (uint32_t)seed, (uint32_t)(seed >> 32), Y);
    UMAP_LAUNCH_CHECK("random_init_kernel");
    return UMAP_OK;
}

umap_status compute_wmax(const float* val, int64_t nnz, float* wmax_dev, cudaStream_t s)
{
    UMAP_CUDA_TRY(cudaMemsetAsync(wmax_dev, 0, sizeof(float), s));
    if (nnz == 0) return UMAP_OK;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(nnz, 256), 4LL * num_sms());
    wmax_kernel<<<grid, 256, 0, s>>>(val, nnz, wmax_dev);
    UMAP_LAUNCH_CHECK("wmax_kernel");
    return UMAP_OK;
}

// Run epochs [e_begin, e_end) on Y (device, in place).  nnz_bound: an upper bound of
// indptr[n] used only to size the w_max pass (the exact value is read from indptr).
umap_status optimize_layout(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, int64_t nnz,
                            float* Y, const umap_params* p, int e_begin, int e_end, int64_t* positives_host,
                            cudaStream_t s)
{
    const int dim = p->n_components;
    if (!dim_supported(dim)) {
        set_last_error("n_components must be one of 1,2,3,4,8,16");
        return UMAP_ERR_UNSUPPORTED;
    }
    if (e_begin < 1) e_begin = 1;
    if (e_end > p->n_epochs) e_end = p->n_epochs;
    Scratch wmax, other, counter;
    UMAP_TRY(wmax.alloc(sizeof(float), s));
    UMAP_TRY(compute_wmax(val, nnz, wmax.as<float>(), s));
    UMAP_TRY(counter.alloc(sizeof(unsigned long long), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), s));
    const bool det = p->sgd_mode == UMAP_SGD_DETERMINISTIC;
    float* bufs[2] = {Y, nullptr};
    if (det) {
        UMAP_TRY(other.alloc(sizeof(float) * (size_t)n * dim, s));
        bufs[1] = other.as<float>();
    }
    SgdArgs A{};
    A.indptr = indptr; A.col = col; A.val = val; A.w_max = wmax.as<float>(); A.n = n;
    A.a = p->a; A.b = p->b; A.gamma = p->repulsion_strength; A.alpha0 = p->learning_rate;
    A.n_epochs = p->n_epochs; A.m = p->negative_sample_rate;
    A.key0 = (uint32_t)p->seed; A.key1 = (uint32_t)(p->seed >> 32);
    A.positives = counter.as<unsigned long long>();
    int cur = 0;
    for (int e = e_begin; e < e_end; ++e) {
        A.epoch = e;
        A.Yr = bufs[cur];
        A.Yw = det ? bufs[cur ^ 1] : bufs[cur];
        umap_status st;
        switch (dim) {
            case 1: st = launch_epoch<1>(A, det, s); break;
            case 2: st = launch_epoch<2>(A, det, s); break;
            case 3: st = launch_epoch<3>(A, det, s); break;
            case 4: st = launch_epoch<4>(A, det, s); break;
            case 8: st = launch_epoch<8>(A, det, s); break;
            default: st = launch_epoch<16>(A, det, s); break;
        }
        if (st != UMAP_OK) return st;
        if (det) cur ^= 1;
    }
    if (cur != 0) {
        UMAP_CUDA_TRY(cudaMemcpyAsync(Y, bufs[cur], sizeof(float) * (size_t)n * dim, cudaMemcpyDeviceToDevice, s));
    }
    if (positives_host) {
        unsigned long long c = 0;
        UMAP_CUDA_TRY(cudaMemcpyAsync(&c, counter.p, sizeof(c), cudaMemcpyDeviceToHost, s));
        UMAP_CUDA_TRY(cudaStreamSynchronize(s));
        *positives_host = (int64_t)c;
    }
    return UMAP_OK;
}

umap_status transform_optimize(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                               float* Yq, const umap_params* p, int n_epochs_t, int e_begin, int e_end,
                               int64_t q_offset, int init, cudaStream_t s)
{
    const int dim = p->n_components;
    if (!dim_supported(dim)) {
        set_last_error("n_components must be one of 1,2,3,4,8,16");
        return UMAP_ERR_UNSUPPORTED;
    }
    if (nq == 0) return UMAP_OK;
    Scratch wmax;
    UMAP_TRY(wmax.alloc(sizeof(float), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(wmax.p, 0, sizeof(float), s));
    const int64_t m = nq * (int64_t)k;
    wmax_dense_kernel<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), 4LL * num_sms()), 256, 0, s>>>(w, m, wmax.as<float>());
    UMAP_LAUNCH_CHECK("wmax_dense_kernel");
    switch (dim) {
        case 1: return launch_transform<1>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 2: return launch_transform<2>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 3: return launch_transform<3>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 4: return launch_transform<4>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 8: return launch_transform<8>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        default: return launch_transform<16>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
    }
}

}  // namespace umapb200
