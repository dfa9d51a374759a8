// spectral.cu -- spectral initialisation of the layout (f3; "computing a spectral
// embedding over the fuzzy union"; reading R18).
//
// The dim eigenvectors of L = I - D^-1/2 B D^-1/2 with the smallest non-trivial eigenvalues,
// by orthogonal (block power) iteration on M = 2I - L = I + D^-1/2 B D^-1/2 with the trivial
// vector v0 = D^1/2 1 / |D^1/2 1| deflated, all in fp64:
//   V0 = U[-1,1) from Philox (row, column, 0xFFFFFFFE, 0)[0];
//   iters times:  W = M V  (CSR SpMM, thread per row),  W -= v0 (v0' W),  G = W'W,
//                 R = chol(G),  V = W R^-1;
// then each column is rescaled affinely to [-scale, scale] and 1e-4 scale U[-1,1) noise
// (counter tag 0xFFFFFFFD) is added.  Reductions are two-level in a fixed order, so the result
// is identical run to run.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace umapb200 {
namespace {

constexpr int SP_THREADS = 256;

__device__ __forceinline__ double uniform_pm1(int64_t i, int c, uint32_t tag, uint32_t k0, uint32_t k1)
{
    const u32x4 r = philox4x32_10((uint32_t)i, (uint32_t)c, tag, 0u, k0, k1);
    return -1.0 + 2.0 * (double)(r.x >> 8) * (1.0 / 16777216.0);
}

template <int NV>
__device__ __forceinline__ void block_partials(double (&v)[NV], double* __restrict__ partials)
{
    __shared__ double red[SP_THREADS / 32][NV];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int m = 0; m < NV; ++m) {
        double x = v[m];
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) red[warp][m] = x;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int w = 0; w < SP_THREADS / 32; ++w) s += red[w][threadIdx.x];
        partials[(int64_t)blockIdx.x * NV + threadIdx.x] = s;
    }
}

// degrees (sequential fp64 row sums of the fp32 weights, CSR order), s = sqrt(deg), dinv, and
// block partials of |s|^2; V0 from Philox
template <int DIM>
__global__ void sp_setup_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ val, int64_t n,
                                uint32_t k0, uint32_t k1, double* __restrict__ sq, double* __restrict__ dinv,
                                double* __restrict__ V, double* __restrict__ partials)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double v[1] = {0.0};
    if (i < n) {
        double deg = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) deg += (double)val[e];
        const double s = sqrt(deg);
        sq[i] = s;
        dinv[i] = s > 0.0 ? 1.0 / s : 0.0;
        v[0] = s * s;
#pragma unroll
        for (int c = 0; c < DIM; ++c) V[i * DIM + c] = uniform_pm1(i, c, 0xFFFFFFFEu, k0, k1);
    }
    block_partials<1>(v, partials);
}

// W = V + dinv (B (dinv V)); block partials of v0'W (DIM) and W'W (upper triangle)
template <int DIM>
__global__ void sp_spmm_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ col,
                               const float* __restrict__ val, int64_t n, const double* __restrict__ dinv,
                               const double* __restrict__ sq, double inv_norm, const double* __restrict__ V,
                               double* __restrict__ W, double* __restrict__ partials)
{
    constexpr int NV = DIM + DIM * (DIM + 1) / 2;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double v[NV];
#pragma unroll
    for (int m = 0; m < NV; ++m) v[m] = 0.0;
    if (i < n) {
        double acc[DIM];
#pragma unroll
        for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            const int64_t j = col[e];
            const double wj = (double)val[e] * dinv[j];
#pragma unroll
            for (int c = 0; c < DIM; ++c) acc[c] += wj * V[j * DIM + c];
        }
        const double di = dinv[i], v0 = sq[i] * inv_norm;
        double w[DIM];
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            w[c] = V[i * DIM + c] + di * acc[c];
            W[i * DIM + c] = w[c];
            v[c] = v0 * w[c];
        }
        int m = DIM;
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
            for (int b = a; b < DIM; ++b) v[m++] = w[a] * w[b];
    }
    block_partials<NV>(v, partials);
}

// one block: sum the partials in block order, G' = G - d0 d0', R = chol(G'), Rinv = R^-1
template <int DIM>
__global__ void sp_coeff_kernel(const double* __restrict__ partials, int nblocks, double* __restrict__ coef)
{
    constexpr int NV = DIM + DIM * (DIM + 1) / 2;
    __shared__ double tot[NV];
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int b = 0; b < nblocks; ++b) s += partials[(int64_t)b * NV + threadIdx.x];
        tot[threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double d0[DIM], G[DIM][DIM], R[DIM][DIM], Ri[DIM][DIM];
        for (int c = 0; c < DIM; ++c) d0[c] = tot[c];
        int m = DIM;
        for (int a = 0; a < DIM; ++a)
            for (int b = a; b < DIM; ++b) { G[a][b] = G[b][a] = tot[m++] - d0[a] * d0[b]; }
        for (int a = 0; a < DIM; ++a)  // Cholesky, G = R'R, R upper
            for (int b = 0; b < DIM; ++b) {
                R[a][b] = 0.0;
                Ri[a][b] = 0.0;
            }
        for (int j = 0; j < DIM; ++j) {
            double s = G[j][j];
            for (int k = 0; k < j; ++k) s -= R[k][j] * R[k][j];
            R[j][j] = sqrt(fmax(s, 1e-300));
            for (int c = j + 1; c < DIM; ++c) {
                double t = G[j][c];
                for (int k = 0; k < j; ++k) t -= R[k][j] * R[k][c];
                R[j][c] = t / R[j][j];
            }
        }
        for (int j = DIM - 1; j >= 0; --j) {  // Ri = R^-1 (upper triangular)
            Ri[j][j] = 1.0 / R[j][j];
            for (int c = j + 1; c < DIM; ++c) {
                double t = 0.0;
                for (int k = j + 1; k <= c; ++k) t += R[j][k] * Ri[k][c];
                Ri[j][c] = -t / R[j][j];
            }
        }
        for (int c = 0; c < DIM; ++c) coef[c] = d0[c];
        for (int a = 0; a < DIM; ++a)
            for (int b = 0; b < DIM; ++b) coef[DIM + a * DIM + b] = Ri[a][b];
    }
}

// V = (W - v0 d0') Ri
template <int DIM>
__global__ void sp_apply_kernel(int64_t n, const double* __restrict__ sq, double inv_norm,
                                const double* __restrict__ W, const double* __restrict__ coef, double* __restrict__ V)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v0 = sq[i] * inv_norm;
    double w[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) w[c] = W[i * DIM + c] - v0 * coef[c];
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a <= c; ++a) s += w[a] * coef[DIM + a * DIM + c];
        V[i * DIM + c] = s;
    }
}

// per-block min / max of each column (warp shuffles, then per-warp results)
template <int DIM>
__global__ void sp_minmax_kernel(const double* __restrict__ V, int64_t n, double* __restrict__ partials)
{
    __shared__ double mn[SP_THREADS / 32][DIM], mx[SP_THREADS / 32][DIM];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        double a = i < n ? V[i * DIM + c] : INFINITY, b = i < n ? V[i * DIM + c] : -INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (lane == 0) { mn[warp][c] = a; mx[warp][c] = b; }
    }
    __syncthreads();
    if (threadIdx.x < DIM) {
        double a = INFINITY, b = -INFINITY;
        for (int w = 0; w < SP_THREADS / 32; ++w) { a = fmin(a, mn[w][threadIdx.x]); b = fmax(b, mx[w][threadIdx.x]); }
        partials[(int64_t)blockIdx.x * 2 * DIM + threadIdx.x] = a;
        partials[(int64_t)blockIdx.x * 2 * DIM + DIM + threadIdx.x] = b;
    }
}

template <int DIM>
__global__ void sp_finish_kernel(const double* __restrict__ V, int64_t n, const double* __restrict__ partials,
                                 int nblocks, double scale, uint32_t k0, uint32_t k1, float* __restrict__ Y)
{
    __shared__ double lo[DIM], hi[DIM];
    if (threadIdx.x < DIM) {
        double a = INFINITY, b = -INFINITY;
        for (int t = 0; t < nblocks; ++t) {
            a = fmin(a, partials[(int64_t)t * 2 * DIM + threadIdx.x]);
            b = fmax(b, partials[(int64_t)t * 2 * DIM + DIM + threadIdx.x]);
        }
        lo[threadIdx.x] = a;
        hi[threadIdx.x] = b;
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const double span = hi[c] > lo[c] ? hi[c] - lo[c] : 1.0;
        const double y = (V[i * DIM + c] - lo[c]) / span * (2.0 * scale) - scale;
        Y[i * DIM + c] = (float)(y + 1e-4 * scale * uniform_pm1(i, c, 0xFFFFFFFDu, k0, k1));
    }
}

template <int DIM>
umap_status spectral_t(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, uint64_t seed,
                       int iters, float* Y, cudaStream_t s)
{
    constexpr int NV = DIM + DIM * (DIM + 1) / 2;
    const int nb = (int)ceil_div(n, SP_THREADS);
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    Scratch sq, dinv, V, W, part, coef;
    UMAP_TRY(sq.alloc(sizeof(double) * (size_t)n, s));
    UMAP_TRY(dinv.alloc(sizeof(double) * (size_t)n, s));
    UMAP_TRY(V.alloc(sizeof(double) * (size_t)n * DIM, s));
    UMAP_TRY(W.alloc(sizeof(double) * (size_t)n * DIM, s));
    UMAP_TRY(part.alloc(sizeof(double) * (size_t)nb * std::max(NV, 2 * DIM), s));
    UMAP_TRY(coef.alloc(sizeof(double) * (DIM + DIM * DIM), s));
    sp_setup_kernel<DIM><<<nb, SP_THREADS, 0, s>>>(indptr, val, n, k0, k1, sq.as<double>(), dinv.as<double>(),
                                                  V.as<double>(), part.as<double>());
    UMAP_LAUNCH_CHECK("sp_setup_kernel");
    std::vector<double> hp((size_t)nb);
    UMAP_CUDA_TRY(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    double ss = 0.0;
    for (double x : hp) ss += x;
    const double inv_norm = ss > 0.0 ? 1.0 / std::sqrt(ss) : 0.0;
    for (int it = 0; it < iters; ++it) {
        sp_spmm_kernel<DIM><<<nb, SP_THREADS, 0, s>>>(indptr, col, val, n, dinv.as<double>(), sq.as<double>(), inv_norm,
                                                     V.as<double>(), W.as<double>(), part.as<double>());
        UMAP_LAUNCH_CHECK("sp_spmm_kernel");
        sp_coeff_kernel<DIM><<<1, 64, 0, s>>>(part.as<double>(), nb, coef.as<double>());
        UMAP_LAUNCH_CHECK("sp_coeff_kernel");
        sp_apply_kernel<DIM><<<nb, SP_THREADS, 0, s>>>(n, sq.as<double>(), inv_norm, W.as<double>(), coef.as<double>(),
                                                      V.as<double>());
        UMAP_LAUNCH_CHECK("sp_apply_kernel");
    }
    sp_minmax_kernel<DIM><<<nb, SP_THREADS, 0, s>>>(V.as<double>(), n, part.as<double>());
    UMAP_LAUNCH_CHECK("sp_minmax_kernel");
    sp_finish_kernel<DIM><<<nb, SP_THREADS, 0, s>>>(V.as<double>(), n, part.as<double>(), nb, 10.0, k0, k1, Y);
    UMAP_LAUNCH_CHECK("sp_finish_kernel");
    return UMAP_OK;
}

}  // namespace

umap_status spectral_init(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, int dim,
                          uint64_t seed, int iters, float* Y, cudaStream_t s)
{
    if (n < dim + 2) { set_last_error("spectral init needs n >= n_components + 2"); return UMAP_ERR_TOO_FEW_ROWS; }
    ProfScope ps(PROF_SPECTRAL, s);
    switch (dim) {
        case 1: return spectral_t<1>(indptr, col, val, n, seed, iters, Y, s);
        case 2: return spectral_t<2>(indptr, col, val, n, seed, iters, Y, s);
        case 3: return spectral_t<3>(indptr, col, val, n, seed, iters, Y, s);
        case 4: return spectral_t<4>(indptr, col, val, n, seed, iters, Y, s);
        case 8: return spectral_t<8>(indptr, col, val, n, seed, iters, Y, s);
        default: return spectral_t<16>(indptr, col, val, n, seed, iters, Y, s);
    }
}

}  // namespace umapb200
