// proj.cu -- orthonormal basis of the leading principal subspace of the centred data, for the
// projected coarse pass of trustworthiness (a10).
//
// For any real d x K matrix P, |P^T v|^2 <= sigma_max(P)^2 |v|^2, so distances between projected
// rows bound the input-space distances from below: a reference tile whose projected distances to
// a row all exceed the row's largest threshold (with the rounding slack of every step) cannot hold
// a column below any of the row's thresholds.  The subspace only decides how many tiles are
// skipped; the bound holds for any P, with sigma_max^2 <= 1 + ||P^T P - I||_F measured here.
//
// Randomised range finder with one power step on a row sample of the centred data (fp32 GEMMs),
// orthonormalised by CholeskyQR in fp64 (Gram matrix, one-CTA Cholesky, row-parallel solve).
#include <cmath>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"

namespace umapb200 {
namespace {

// Xs[s][f] = fl(x_{i_s, f} - mean_f), i_s = s stride
__global__ void pca_sample_kernel(const float* __restrict__ X, int64_t n, int d, const double* __restrict__ colsum,
                                  double inv_n, int S, int64_t stride, float* __restrict__ Xs)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)S * d) return;
    const int64_t s = i / d;
    const int f = (int)(i - s * d);
    const int64_t row = s * stride;
    Xs[i] = X[row * d + f] - (float)(colsum[f] * inv_n);
}

// Omega: d x 128, uniform [-1, 1) in the first K columns, zero after
__global__ void pca_init_kernel(float* __restrict__ V, int d, int K)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d * 128) return;
    const u32x4 r = philox4x32_10((uint32_t)i, 0x5CA1AB1Eu, 0u, 0u, 0x0DDB1A5Eu, 0x7E57AB1Eu);
    V[i] = (i & 127) < K ? (float)(r.x >> 8) * (1.0f / 8388608.0f) - 1.0f : 0.0f;
}

// G = W^T W split over the rows of W: part[z][i][j] = sum over rows f = z, z + nz, ... (fp64),
// then summed in a fixed order (gram_sum_kernel): deterministic, and nz x more CTAs than one
// K x K grid walking all d rows (latency-bound: 84 us at d = 784)
__global__ void gram64_part_kernel(const float* __restrict__ W, int d, int K, int nz, double* __restrict__ part)
{
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x, z = blockIdx.z;
    if (j >= K) return;
    double a0 = 0.0, a1 = 0.0;
    int f = z;
    for (; f + nz < d; f += 2 * nz) {
        a0 += (double)W[(int64_t)f * 128 + i] * (double)W[(int64_t)f * 128 + j];
        a1 += (double)W[(int64_t)(f + nz) * 128 + i] * (double)W[(int64_t)(f + nz) * 128 + j];
    }
    if (f < d) a0 += (double)W[(int64_t)f * 128 + i] * (double)W[(int64_t)f * 128 + j];
    part[((int64_t)z * K + i) * K + j] = a0 + a1;
}
__global__ void gram_sum_kernel(const double* __restrict__ part, int nz, int K, double* __restrict__ G)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= K * K) return;
    double g = 0.0;
    for (int z = 0; z < nz; ++z) g += part[(int64_t)z * K * K + t];
    G[t] = g;
}
// err2 = sum_{i,j} (G_ij - delta_ij)^2, one CTA, fixed-order tree reduction
__global__ void orth_err_from_gram_kernel(const double* __restrict__ G, int K, double* __restrict__ err2)
{
    __shared__ double red[256];
    double e = 0.0;
    for (int t = threadIdx.x; t < K * K; t += blockDim.x) {
        const double v = G[t] - ((t / K) == (t % K) ? 1.0 : 0.0);
        e += v * v;
    }
    red[threadIdx.x] = e;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *err2 = red[0];
}

// Right-looking Cholesky of G (K x K, fp64, symmetric) in one CTA: G + jitter I = L L^T, L (lower,
// row-major, K x K) to Lout.  Per column j: the pivot, the column scaled, then the rank-1 update of
// the trailing triangle spread over the whole CTA (independent FMAs; the left-looking form's
// per-row dot products were one dependent chain per thread: 0.34 ms at K = 122).  ok = 0 when a
// pivot is not positive.
__global__ void __launch_bounds__(512) chol_rl_kernel(const double* __restrict__ G, int K, double* __restrict__ Lout,
                                                      int* __restrict__ ok)
{
    extern __shared__ double A[];  // A[r * K + c]
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < K * K; t += nt) A[t] = G[t];
    __syncthreads();
    __shared__ double jitter;
    if (tid == 0) {
        double m = 0.0;
        for (int t = 0; t < K; ++t) m = fmax(m, A[t * K + t]);
        jitter = 1e-12 * m;
    }
    for (int j = 0; j < K; ++j) {
        __syncthreads();
        if (tid == 0) {
            const double dj = A[j * K + j] + jitter;
            if (!(dj > 0.0)) *ok = 0;
            A[j * K + j] = sqrt(fmax(dj, 1e-300));
        }
        __syncthreads();
        const double inv = 1.0 / A[j * K + j];
        for (int r = j + 1 + tid; r < K; r += nt) A[r * K + j] *= inv;
        __syncthreads();
        // trailing lower triangle: warp w takes rows j+1+w, j+1+w+NW, ..., lane l columns
        // j+1+l, j+1+l+32, ... <= r (no index division)
        const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
        for (int r = j + 1 + w; r < K; r += nw) {
            const double lr = A[r * K + j];
            for (int c = j + 1 + lane; c <= r; c += 32) A[r * K + c] -= lr * A[c * K + j];
        }
    }
    __syncthreads();
    for (int t = tid; t < K * K; t += nt) {
        const int r = t / K, c = t % K;
        Lout[t] = c <= r ? A[t] : 0.0;
    }
}

// V = W L^-T (d x 128 fp32, columns >= K zero): row w of W solves L v^T = w^T by forward
// substitution, one warp per row (lane l holds v_m for m = l mod 32), L broadcast from shared memory
__global__ void __launch_bounds__(256) trsm_rows_kernel(const float* __restrict__ W, int d, int K,
                                                        const double* __restrict__ L, float* __restrict__ V)
{
    extern __shared__ double Ls[];
    for (int t = threadIdx.x; t < K * K; t += blockDim.x) Ls[t] = L[t];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= d) return;
    double v[4] = {0.0, 0.0, 0.0, 0.0};  // v[q] = v_{lane + 32 q}
    for (int i = 0; i < K; ++i) {
        double part = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int m = lane + 32 * q;
            if (m < i) part += Ls[i * K + m] * v[q];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const double vi = ((double)W[(int64_t)row * 128 + i] - part) / Ls[i * K + i];
        if ((i & 31) == lane) v[i >> 5] = vi;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int m = lane + 32 * q;
        V[(int64_t)row * 128 + m] = m < K ? (float)v[q] : 0.0f;
    }
}

constexpr int GRAM_NZ = 16;
umap_status gram64(const float* W, int d, int K, double* G, cudaStream_t s)
{
    Scratch part;
    UMAP_TRY(part.alloc(sizeof(double) * (size_t)GRAM_NZ * K * K, s));
    gram64_part_kernel<<<dim3((unsigned)ceil_div(K, 128), (unsigned)K, GRAM_NZ), 128, 0, s>>>(W, d, K, GRAM_NZ,
                                                                                              part.as<double>());
    UMAP_LAUNCH_CHECK("gram64_part_kernel");
    gram_sum_kernel<<<ceil_div(K * K, 256), 256, 0, s>>>(part.as<double>(), GRAM_NZ, K, G);
    UMAP_LAUNCH_CHECK("gram_sum_kernel");
    return UMAP_OK;
}

// CholeskyQR: V = W L^-T with W^T W = L L^T (W, V: d x 128, columns >= K zero)
umap_status cholqr(const float* W, float* V, int d, int K, double* G, double* L, int* ok, cudaStream_t s)
{
    UMAP_TRY(gram64(W, d, K, G, s));
    chol_rl_kernel<<<1, 512, sizeof(double) * (size_t)K * K, s>>>(G, K, L, ok);
    UMAP_LAUNCH_CHECK("chol_rl_kernel");
    trsm_rows_kernel<<<(unsigned)ceil_div(d, 8), 256, sizeof(double) * (size_t)K * K, s>>>(W, d, K, L, V);
    UMAP_LAUNCH_CHECK("trsm_rows_kernel");
    return UMAP_OK;
}

// sigma[0] = sqrt(1 + sqrt(err2)) (+ slack), or +inf when the basis failed (every tile is then
// kept: the projected pass degrades to no pruning, never to a wrong skip)
__global__ void sigma_kernel(const double* __restrict__ err2, const int* __restrict__ ok, float* __restrict__ sigma)
{
    const double s2 = 1.0 + sqrt(*err2) + 1e-7;
    sigma[0] = (*ok && s2 == s2 && s2 < 1.01) ? (float)(sqrt(s2) * (1.0 + 1e-6)) : INFINITY;
}

}  // namespace

// P (device, d x 128 fp32, row-major, columns >= K zero): an orthonormal-to-fp32 basis of the leading K-dimensional
// principal subspace of the centred rows (colsum = column sums of X, mean = colsum / n), by the
// randomised range finder with one power step on a 4096-row sample: P = orth(Xs^T Xs Omega), one
// CholeskyQR in fp64.  sigma (device, 1 float) = a bound on sigma_max(P) from ||P^T P - I||_F, or
// +inf when the basis failed.  No host synchronisation.
umap_status pca_basis(const float* X, int64_t n, int d, const double* colsum, int K, float* P, float* sigma,
                      cudaStream_t s)
{
    if (K > 128) { set_last_error("pca_basis: K > 128"); return UMAP_ERR_UNSUPPORTED; }
    const int S = (int)std::min<int64_t>(n, 4096);
    Scratch xs, u, w, wp, g, l, okb, err;
    UMAP_TRY(u.alloc(sizeof(float) * (size_t)S * 128, s));
    UMAP_TRY(w.alloc(sizeof(float) * (size_t)d * 128, s));
    UMAP_TRY(xs.alloc(sizeof(float) * (size_t)S * d, s));
    UMAP_TRY(g.alloc(sizeof(double) * (size_t)K * K, s));
    UMAP_TRY(l.alloc(sizeof(double) * (size_t)K * K, s));
    UMAP_TRY(okb.alloc(sizeof(int), s));
    UMAP_TRY(err.alloc(sizeof(double), s));
    static PerDeviceOnce attr;
    if (attr.first()) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(chol_rl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 8));
        UMAP_CUDA_TRY(cudaFuncSetAttribute(trsm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 8));
    }
    const int one = 1;
    UMAP_CUDA_TRY(cudaMemcpyAsync(okb.p, &one, sizeof(int), cudaMemcpyHostToDevice, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(err.p, 0, sizeof(double), s));
    pca_init_kernel<<<(unsigned)ceil_div((int64_t)d * 128, 256), 256, 0, s>>>(P, d, K);  // Omega
    UMAP_LAUNCH_CHECK("pca_init_kernel");
    // U = Xs Omega (S x 128; the sample: rows r * (n / S) of X, centred), Xs materialised for W
    const int64_t stride = n / S;
    tgemm128_kernel<false><<<(unsigned)ceil_div(S, 128), 256, 0, s>>>(X, S, stride, d, d, colsum, 1.0 / (double)n, P,
                                                                      u.as<float>());
    UMAP_LAUNCH_CHECK("tgemm128_kernel");
    pca_sample_kernel<<<(unsigned)ceil_div((int64_t)S * d, 256), 256, 0, s>>>(X, n, d, colsum, 1.0 / (double)n, S,
                                                                               stride, xs.as<float>());
    UMAP_LAUNCH_CHECK("pca_sample_kernel");
    // W = Xs^T U (d x 128), P = orth(W)
    constexpr int KSPLIT = 32;  // the reduction over the sample split over 32 x (d / 128) CTAs
    UMAP_TRY(wp.alloc(sizeof(float) * (size_t)KSPLIT * d * 128, s));
    tgemm128_kernel<true><<<dim3((unsigned)ceil_div(d, 128), KSPLIT), 256, 0, s>>>(
        xs.as<float>(), d, 1, S, d, nullptr, 0.0, u.as<float>(), wp.as<float>());
    UMAP_LAUNCH_CHECK("tgemm128_kernel");
    split_sum_kernel<<<(unsigned)ceil_div((int64_t)d * 128, 256), 256, 0, s>>>(wp.as<float>(), KSPLIT, (int64_t)d * 128,
                                                                              w.as<float>());
    UMAP_LAUNCH_CHECK("split_sum_kernel");
    UMAP_TRY(cholqr(w.as<float>(), P, d, K, g.as<double>(), l.as<double>(), okb.as<int>(), s));
    // ||P^T P - I||_F^2 of the fp32 basis as used (fp64 Gram, fixed-order sums)
    UMAP_TRY(gram64(P, d, K, g.as<double>(), s));
    orth_err_from_gram_kernel<<<1, 256, 0, s>>>(g.as<double>(), K, err.as<double>());
    UMAP_LAUNCH_CHECK("orth_err_from_gram_kernel");
    sigma_kernel<<<1, 1, 0, s>>>(err.as<double>(), okb.as<int>(), sigma);
    UMAP_LAUNCH_CHECK("sigma_kernel");
    return UMAP_OK;
}

}  // namespace umapb200
