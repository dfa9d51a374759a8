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

namespace umapb200 {
namespace {

// Xs[s][f] = fl(x_{i_s, f} - mean_f), i_s = floor(s n / S)
__global__ void pca_sample_kernel(const float* __restrict__ X, int64_t n, int d, const double* __restrict__ colsum,
                                  double inv_n, int S, float* __restrict__ Xs)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)S * d) return;
    const int64_t s = i / d;
    const int f = (int)(i - s * d);
    const int64_t row = s * n / S;
    Xs[i] = X[row * d + f] - (float)(colsum[f] * inv_n);
}

__global__ void pca_init_kernel(float* __restrict__ V, int d, int K)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d * K) return;
    const u32x4 r = philox4x32_10((uint32_t)i, 0x5CA1AB1Eu, 0u, 0u, 0x0DDB1A5Eu, 0x7E57AB1Eu);
    V[i] = (float)(r.x >> 8) * (1.0f / 8388608.0f) - 1.0f;
}

// C (M x N) = op(A) B: A row-major M x Kd (transA = 0) or Kd x M (transA = 1), B row-major Kd x N;
// 32 x 32 output tile per CTA, Kd staged through shared memory in slabs of 32
__global__ void __launch_bounds__(1024) gemm32_kernel(const float* __restrict__ A, int transA, const float* __restrict__ B,
                                                      float* __restrict__ C, int M, int N, int Kd)
{
    __shared__ float As[32][33], Bs[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int row = blockIdx.y * 32 + ty, col = blockIdx.x * 32 + tx;
    float acc = 0.0f;
    for (int k0 = 0; k0 < Kd; k0 += 32) {
        const int ka = k0 + tx, kb = k0 + ty;
        if (transA) {
            const int r = blockIdx.y * 32 + tx, kk = k0 + ty;  // coalesced along M
            As[tx][ty] = (r < M && kk < Kd) ? A[(int64_t)kk * M + r] : 0.0f;
        } else {
            As[ty][tx] = (row < M && ka < Kd) ? A[(int64_t)row * Kd + ka] : 0.0f;
        }
        Bs[ty][tx] = (kb < Kd && col < N) ? B[(int64_t)kb * N + col] : 0.0f;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 32; ++k) acc = fmaf(As[ty][k], Bs[k][tx], acc);
        __syncthreads();
    }
    if (row < M && col < N) C[(int64_t)row * N + col] = acc;
}

// G = W^T W (K x K, fp64), W d x K fp32
__global__ void gram64_kernel(const float* __restrict__ W, int d, int K, double* __restrict__ G)
{
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    double acc = 0.0;
    for (int f = 0; f < d; ++f) acc += (double)W[(int64_t)f * K + i] * (double)W[(int64_t)f * K + j];
    G[i * K + j] = acc;
}

// One CTA of 128 threads (K <= 128): G + jitter = L L^T (left-looking Cholesky, thread i owns row
// i of L, one barrier per column; four partial sums break the dot-product dependency chain).
// ok = 0 when a pivot is not positive.
__global__ void __launch_bounds__(128) chol_kernel(const double* __restrict__ G, int K, double* __restrict__ L,
                                                   int* __restrict__ ok)
{
    extern __shared__ double Ls[];  // K x K, row-major; the lower triangle becomes L
    const int i = threadIdx.x;
    for (int t = i; t < K * K; t += blockDim.x) Ls[t] = G[t];
    __syncthreads();
    __shared__ double jitter;
    if (i == 0) {
        double m = 0.0;
        for (int t = 0; t < K; ++t) m = fmax(m, Ls[t * K + t]);
        jitter = 1e-12 * m;
    }
    __syncthreads();
    auto dot = [&](int r1, int r2, int len) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int m = 0;
        for (; m + 4 <= len; m += 4) {
            a0 += Ls[r1 * K + m] * Ls[r2 * K + m];
            a1 += Ls[r1 * K + m + 1] * Ls[r2 * K + m + 1];
            a2 += Ls[r1 * K + m + 2] * Ls[r2 * K + m + 2];
            a3 += Ls[r1 * K + m + 3] * Ls[r2 * K + m + 3];
        }
        for (; m < len; ++m) a0 += Ls[r1 * K + m] * Ls[r2 * K + m];
        return (a0 + a1) + (a2 + a3);
    };
    for (int j = 0; j < K; ++j) {
        if (i == j) {
            const double sdiag = Ls[j * K + j] + jitter - dot(j, j, j);
            if (!(sdiag > 0.0)) *ok = 0;
            Ls[j * K + j] = sqrt(fmax(sdiag, 1e-300));
        }
        __syncthreads();
        if (i > j && i < K) Ls[i * K + j] = (Ls[i * K + j] - dot(i, j, j)) / Ls[j * K + j];
    }
    __syncthreads();
    for (int t = i; t < K * K; t += blockDim.x) L[t] = Ls[t];
}

// V = W L^-T (V L^T = W): thread per row of W, forward substitution against L in shared memory
__global__ void __launch_bounds__(128) trsm_kernel(const float* __restrict__ W, const double* __restrict__ L, int d,
                                                   int K, float* __restrict__ V)
{
    extern __shared__ double Lsh[];
    for (int t = threadIdx.x; t < K * K; t += blockDim.x) Lsh[t] = L[t];
    __syncthreads();
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= d) return;
    double v[128];
    for (int k = 0; k < K; ++k) {
        double acc = (double)W[f * K + k];
        for (int j = 0; j < k; ++j) acc -= Lsh[k * K + j] * v[j];
        v[k] = acc / Lsh[k * K + k];
        V[f * K + k] = (float)v[k];
    }
}

// err2 += sum_{i,j} ((P^T P)_ij - delta_ij)^2 (fp64, P the fp32 basis as used)
__global__ void orth_err_kernel(const float* __restrict__ P, int d, int K, double* __restrict__ err2)
{
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    double acc = 0.0;
    for (int f = 0; f < d; ++f) acc += (double)P[(int64_t)f * K + i] * (double)P[(int64_t)f * K + j];
    const double e = acc - (i == j ? 1.0 : 0.0);
    atomicAdd(err2, e * e);
}

// CholeskyQR: V = W R^-1 with W^T W = R^T R (W, V: d x K)
umap_status cholqr(const float* W, float* V, int d, int K, double* G, double* L, int* ok, cudaStream_t s)
{
    gram64_kernel<<<dim3((unsigned)ceil_div(K, 128), (unsigned)K), 128, 0, s>>>(W, d, K, G);
    UMAP_LAUNCH_CHECK("gram64_kernel");
    chol_kernel<<<1, 128, sizeof(double) * (size_t)K * K, s>>>(G, K, L, ok);
    UMAP_LAUNCH_CHECK("chol_kernel");
    trsm_kernel<<<(unsigned)ceil_div(d, 128), 128, sizeof(double) * (size_t)K * K, s>>>(W, L, d, K, V);
    UMAP_LAUNCH_CHECK("trsm_kernel");
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

// P (device, d x K fp32, row-major): an orthonormal-to-fp32 basis of the leading K-dimensional
// principal subspace of the centred rows (colsum = column sums of X, mean = colsum / n), by the
// randomised range finder with one power step on a 4096-row sample: P = orth(Xs^T Xs Omega), one
// CholeskyQR in fp64.  sigma (device, 1 float) = a bound on sigma_max(P) from ||P^T P - I||_F, or
// +inf when the basis failed.  No host synchronisation.
umap_status pca_basis(const float* X, int64_t n, int d, const double* colsum, int K, float* P, float* sigma,
                      cudaStream_t s)
{
    if (K > 128) { set_last_error("pca_basis: K > 128"); return UMAP_ERR_UNSUPPORTED; }
    const int S = (int)std::min<int64_t>(n, 4096);
    Scratch xs, u, w, g, l, okb, err;
    UMAP_TRY(xs.alloc(sizeof(float) * (size_t)S * d, s));
    UMAP_TRY(u.alloc(sizeof(float) * (size_t)S * K, s));
    UMAP_TRY(w.alloc(sizeof(float) * (size_t)d * K, s));
    UMAP_TRY(g.alloc(sizeof(double) * (size_t)K * K, s));
    UMAP_TRY(l.alloc(sizeof(double) * (size_t)K * K, s));
    UMAP_TRY(okb.alloc(sizeof(int), s));
    UMAP_TRY(err.alloc(sizeof(double), s));
    static PerDeviceOnce attr;
    if (attr.first()) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 8));
        UMAP_CUDA_TRY(cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 8));
    }
    const int one = 1;
    UMAP_CUDA_TRY(cudaMemcpyAsync(okb.p, &one, sizeof(int), cudaMemcpyHostToDevice, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(err.p, 0, sizeof(double), s));
    pca_sample_kernel<<<(unsigned)ceil_div((int64_t)S * d, 256), 256, 0, s>>>(X, n, d, colsum, 1.0 / (double)n, S,
                                                                               xs.as<float>());
    UMAP_LAUNCH_CHECK("pca_sample_kernel");
    pca_init_kernel<<<(unsigned)ceil_div((int64_t)d * K, 256), 256, 0, s>>>(P, d, K);  // Omega
    UMAP_LAUNCH_CHECK("pca_init_kernel");
    // U = Xs Omega (S x K), W = Xs^T U (d x K), P = orth(W)
    gemm32_kernel<<<dim3((unsigned)ceil_div(K, 32), (unsigned)ceil_div(S, 32)), 1024, 0, s>>>(xs.as<float>(), 0, P,
                                                                                            u.as<float>(), S, K, d);
    UMAP_LAUNCH_CHECK("gemm32_kernel");
    gemm32_kernel<<<dim3((unsigned)ceil_div(K, 32), (unsigned)ceil_div(d, 32)), 1024, 0, s>>>(
        xs.as<float>(), 1, u.as<float>(), w.as<float>(), d, K, S);
    UMAP_LAUNCH_CHECK("gemm32_kernel");
    UMAP_TRY(cholqr(w.as<float>(), P, d, K, g.as<double>(), l.as<double>(), okb.as<int>(), s));
    orth_err_kernel<<<dim3((unsigned)ceil_div(K, 128), (unsigned)K), 128, 0, s>>>(P, d, K, err.as<double>());
    UMAP_LAUNCH_CHECK("orth_err_kernel");
    sigma_kernel<<<1, 1, 0, s>>>(err.as<double>(), okb.as<int>(), sigma);
    UMAP_LAUNCH_CHECK("sigma_kernel");
    return UMAP_OK;
}

}  // namespace umapb200
