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

// G = W^T W (K x K, fp64), W d x K fp32 in rows of 128 (four partial sums per thread)
__global__ void gram64_kernel(const float* __restrict__ W, int d, int K, double* __restrict__ G)
{
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int f = 0;
    for (; f + 4 <= d; f += 4) {
        a0 += (double)W[(int64_t)f * 128 + i] * (double)W[(int64_t)f * 128 + j];
        a1 += (double)W[(int64_t)(f + 1) * 128 + i] * (double)W[(int64_t)(f + 1) * 128 + j];
        a2 += (double)W[(int64_t)(f + 2) * 128 + i] * (double)W[(int64_t)(f + 2) * 128 + j];
        a3 += (double)W[(int64_t)(f + 3) * 128 + i] * (double)W[(int64_t)(f + 3) * 128 + j];
    }
    for (; f < d; ++f) a0 += (double)W[(int64_t)f * 128 + i] * (double)W[(int64_t)f * 128 + j];
    G[i * K + j] = (a0 + a1) + (a2 + a3);
}

// One CTA of 128 threads (K <= 128): G + jitter = L L^T (left-looking Cholesky, thread i owns row i
// of L, stored column-major so that the lanes of a dot product read consecutive words; one
// barrier per column), then Linv = L^-1 in place (columns right to left), written as B = Linv^T in
// rows of 128 (B[j][k] = Linv[k][j], zero past K) so that V = W B is one tgemm128.
// ok = 0 when a pivot is not positive.
__global__ void __launch_bounds__(128) chol_kernel(const double* __restrict__ G, int K, float* __restrict__ Bt,
                                                   int* __restrict__ ok)
{
    extern __shared__ double Lc[];  // L[i][m] at Lc[m * K + i]; then X = L^-1 in place
    const int i = threadIdx.x;
    for (int t = i; t < K * K; t += blockDim.x) Lc[(t % K) * K + t / K] = G[t];  // G symmetric: any layout
    __syncthreads();
    __shared__ double jitter;
    if (i == 0) {
        double m = 0.0;
        for (int t = 0; t < K; ++t) m = fmax(m, Lc[t * K + t]);
        jitter = 1e-12 * m;
    }
    __syncthreads();
    auto dot = [&](int r1, int r2, int len) {  // sum_{m < len} L[r1][m] L[r2][m]
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int m = 0;
        for (; m + 4 <= len; m += 4) {
            a0 += Lc[m * K + r1] * Lc[m * K + r2];
            a1 += Lc[(m + 1) * K + r1] * Lc[(m + 1) * K + r2];
            a2 += Lc[(m + 2) * K + r1] * Lc[(m + 2) * K + r2];
            a3 += Lc[(m + 3) * K + r1] * Lc[(m + 3) * K + r2];
        }
        for (; m < len; ++m) a0 += Lc[m * K + r1] * Lc[m * K + r2];
        return (a0 + a1) + (a2 + a3);
    };
    for (int j = 0; j < K; ++j) {
        if (i == j) {
            const double sdiag = Lc[j * K + j] + jitter - dot(j, j, j);
            if (!(sdiag > 0.0)) *ok = 0;
            Lc[j * K + j] = sqrt(fmax(sdiag, 1e-300));
        }
        __syncthreads();
        if (i > j && i < K) Lc[j * K + i] = (Lc[j * K + i] - dot(i, j, j)) / Lc[j * K + j];
    }
    __syncthreads();
    // X = L^-1 in place, columns right to left: X[j][j] = 1 / L[j][j],
    // X[i][j] = -(sum_{m=j+1}^{i} X[i][m] L[m][j]) / L[j][j] for i > j (row i of X right of j is done,
    // column j of L is still intact until the barrier)
    for (int j = K - 1; j >= 0; --j) {
        double x = 0.0;
        const double ljj = Lc[j * K + j];
        if (i > j && i < K) {
            double a0 = 0.0, a1 = 0.0;
            int m = j + 1;
            for (; m + 2 <= i + 1; m += 2) {
                a0 += Lc[m * K + i] * Lc[j * K + m];
                a1 += Lc[(m + 1) * K + i] * Lc[j * K + m + 1];
            }
            if (m <= i) a0 += Lc[m * K + i] * Lc[j * K + m];
            x = -(a0 + a1) / ljj;
        }
        __syncthreads();
        if (i > j && i < K) Lc[j * K + i] = x;
        if (i == j) Lc[j * K + j] = 1.0 / ljj;
        __syncthreads();
    }
    __syncthreads();
    // Bt[j][k] = X[k][j] (k >= j; X[k][j] at Lc[j * K + k]), rows of 128
    for (int t = i; t < K * 128; t += blockDim.x) {
        const int j = t / 128, k = t % 128;
        Bt[t] = (k < K && k >= j) ? (float)Lc[j * K + k] : 0.0f;
    }
}

// err2 += sum_{i,j} ((P^T P)_ij - delta_ij)^2 (fp64, P the fp32 basis as used)
__global__ void orth_err_kernel(const float* __restrict__ P, int d, int K, double* __restrict__ err2)
{
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int f = 0;
    for (; f + 4 <= d; f += 4) {
        a0 += (double)P[(int64_t)f * 128 + i] * (double)P[(int64_t)f * 128 + j];
        a1 += (double)P[(int64_t)(f + 1) * 128 + i] * (double)P[(int64_t)(f + 1) * 128 + j];
        a2 += (double)P[(int64_t)(f + 2) * 128 + i] * (double)P[(int64_t)(f + 2) * 128 + j];
        a3 += (double)P[(int64_t)(f + 3) * 128 + i] * (double)P[(int64_t)(f + 3) * 128 + j];
    }
    for (; f < d; ++f) a0 += (double)P[(int64_t)f * 128 + i] * (double)P[(int64_t)f * 128 + j];
    const double e = ((a0 + a1) + (a2 + a3)) - (i == j ? 1.0 : 0.0);
    atomicAdd(err2, e * e);
}

// CholeskyQR: V = W L^-T with W^T W = L L^T (W, V: d x 128, columns >= K zero)
umap_status cholqr(const float* W, float* V, int d, int K, double* G, float* Bt, int* ok, cudaStream_t s)
{
    gram64_kernel<<<dim3((unsigned)ceil_div(K, 128), (unsigned)K), 128, 0, s>>>(W, d, K, G);
    UMAP_LAUNCH_CHECK("gram64_kernel");
    chol_kernel<<<1, 128, sizeof(double) * (size_t)K * K, s>>>(G, K, Bt, ok);
    UMAP_LAUNCH_CHECK("chol_kernel");
    tgemm128_kernel<false><<<(unsigned)ceil_div(d, 128), 256, 0, s>>>(W, d, 1, 128, 128, nullptr, 0.0, Bt, V);
    UMAP_LAUNCH_CHECK("tgemm128_kernel");
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
    UMAP_TRY(l.alloc(sizeof(float) * (size_t)128 * 128, s));
    UMAP_TRY(okb.alloc(sizeof(int), s));
    UMAP_TRY(err.alloc(sizeof(double), s));
    static PerDeviceOnce attr;
    if (attr.first()) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 8));
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
    UMAP_TRY(cholqr(w.as<float>(), P, d, K, g.as<double>(), l.as<float>(), okb.as<int>(), s));
    orth_err_kernel<<<dim3((unsigned)ceil_div(K, 128), (unsigned)K), 128, 0, s>>>(P, d, K, err.as<double>());
    UMAP_LAUNCH_CHECK("orth_err_kernel");
    sigma_kernel<<<1, 1, 0, s>>>(err.as<double>(), okb.as<int>(), sigma);
    UMAP_LAUNCH_CHECK("sigma_kernel");
    return UMAP_OK;
}

}  // namespace umapb200
