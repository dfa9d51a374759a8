// transform.cu -- transform SGD (a9; R15): query rows
// move against the frozen training layout.
#include "sgd_common.cuh"

namespace umapb200 {

bool dim_supported(int dim);  // sgd.cu
namespace {
using namespace sgdk;

__global__ void wmax_dense_kernel(const float* __restrict__ val, int64_t m, float* __restrict__ out)
{
    float mx = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmaxf(mx, val[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(mx));
}

// ---------------------------------------------------------------- transform SGD (a9)
// Thread per query row; all epochs in one launch (rows are independent: P:138 only
// the query rows move, the training layout is frozen), so there is no inter-epoch
// barrier and no atomics.  Deterministic by construction.
// F64: the per-edge arithmetic of R12/R15 in fp64 with the position stored back in fp32 after
// every update (the oracle's precision reading, R15): coefficients -2ab s^(b-1) /
// (a s^b + 1) and 2 gamma b / ((0.001 + s)(a s^b + 1)) with IEEE pow and division, products and
// sums in the written order without FMA contraction (measured: equal to the oracle bit for bit,
// teacher-forced; ~8x slower on the C5 transform, an exp2(b log2 s) form in fp64 slower still).
// !F64 (the default): the fp32 MUFU form of the fit SGD.
template <int DIM>
__device__ __forceinline__ void transform_update_f64(float (&y)[DIM], const float (&yo)[DIM], bool attractive,
                                                     double a, double b, double gamma, double alpha)
{
    double df[DIM], s = 0.0;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        df[c] = __dsub_rn((double)y[c], (double)yo[c]);
        s = __dadd_rn(s, __dmul_rn(df[c], df[c]));
    }
    double g[DIM];
    if (attractive) {
        double coef = 0.0;
        if (s > 0.0)
            coef = __ddiv_rn(__dmul_rn(__dmul_rn(-2.0 * a, b), pow(s, b - 1.0)), __dadd_rn(__dmul_rn(a, pow(s, b)), 1.0));
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = __dmul_rn(fmin(fmax(__dmul_rn(coef, df[c]), -4.0), 4.0), alpha);
    } else if (s > 0.0) {
        const double cr = __ddiv_rn(__dmul_rn(2.0 * gamma, b),
                                    __dmul_rn(__dadd_rn(0.001, s), __dadd_rn(__dmul_rn(a, pow(s, b)), 1.0)));
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = __dmul_rn(fmin(fmax(__dmul_rn(cr, df[c]), -4.0), 4.0), alpha);
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = __dmul_rn(4.0, alpha);
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) y[c] = __double2float_rn(__dadd_rn((double)y[c], g[c]));
}

template <int DIM, int KMAX, bool F64>
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
        // unrolled (rr / tt in registers) only for the fp32 mode at k <= 16 (C5's k = 15): the fp64
        // mode's IEEE pow / division bodies and the k <= 64 forms, unrolled KMAX times, took
        // minutes to compile; there rr / tt live in local memory
#pragma unroll (F64 || KMAX > 16 ? 1 : KMAX)
        for (int j = 0; j < KMAX; ++j) {
            if (j >= k || !edge_due(rr[j], e)) continue;
            const int64_t t = tt[j];
            float yt[DIM], g[DIM];
            load_row<DIM>(Ytr, t, yt);
            if constexpr (F64) {
                transform_update_f64<DIM>(y, yt, true, (double)a, (double)b, (double)gamma, (double)alpha);
                u32x4 rnd = {0, 0, 0, 0};
                for (int p = 0; p < m; ++p) {
                    if ((p & 3) == 0) rnd = philox4x32_10(head, (uint32_t)t, (uint32_t)e, (uint32_t)(p >> 2), key0, key1);
                    const uint32_t u = pick(rnd, p & 3);
                    const int64_t v = (int64_t)(((unsigned long long)u * (unsigned long long)ntr) >> 32);
                    float yv[DIM];
                    load_row<DIM>(Ytr, v, yv);
                    transform_update_f64<DIM>(y, yv, false, (double)a, (double)b, (double)gamma, (double)alpha);
                }
                continue;
            }
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

template <int DIM, int KMAX>
umap_status launch_transform_t(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                               float* Yq, const float* wmax, const umap_params* p, int nt, int eb, int ee,
                               int64_t q_offset, int init, cudaStream_t s)
{
    ProfScope ps(PROF_TRANSFORM_SGD, s);
    auto kern = p->transform_precision == 1 ? transform_sgd_kernel<DIM, KMAX, true> : transform_sgd_kernel<DIM, KMAX, false>;
    kern<<<ceil_div(nq, 128), 128, 0, s>>>(
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

