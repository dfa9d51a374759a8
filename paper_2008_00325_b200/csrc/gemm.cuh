// gemm.cuh -- the fp32 SIMT GEMM of the projected trust coarse pass (knn_tensor.cu) and of its
// basis (proj.cu).  Never shared with oracle/.
#pragma once
#include "common.cuh"

namespace umapb200 {
namespace {

// Projected coarse pass: Z = X_c P (n x 128 fp32, original row order), X_c = fl(x -
// mean) as in split_bf16_kernel (rows r * stride: stride > 1 draws the basis sample), P the d x 128
// basis of pca_basis (zero columns past K).  Also the basis sample's W = Xs^T U (TRANS_A: A = Xs^T,
// reduction over the sample).  128 x 128 outputs per CTA, 256 threads with 8 x 8 each, the
// reduction staged in slabs of 16.
template <bool TRANS_A>
__global__ void __launch_bounds__(256, 2) tgemm128_kernel(const float* __restrict__ A, int64_t M, int64_t stride,
                                                       int64_t kdim, int lda, const double* __restrict__ colsum,
                                                       double inv_n, const float* __restrict__ B,
                                                       float* __restrict__ C)
{
    __shared__ __align__(16) float As[16][128 + 4], Bs[16][128];
    const int tid = threadIdx.x;
    const int tr = tid >> 4, tc = tid & 15;  // rows tr * 8 + i, columns tc * 8 + j (vector shared loads)
    const int64_t r0 = (int64_t)blockIdx.x * 128;
    // split reduction (gridDim.y > 1): block y sums k in [k_lo, k_hi) into C + y M 128 (partials
    // added in a fixed order by split_sum_kernel: deterministic)
    const int64_t kchunk = (kdim + gridDim.y - 1) / gridDim.y;
    const int64_t k_lo = (int64_t)blockIdx.y * kchunk, k_hi = k_lo + kchunk < kdim ? k_lo + kchunk : kdim;
    C += (int64_t)blockIdx.y * M * 128;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    // each thread stages 8 A and 8 B values per slab; the next slab is loaded into registers
    // while the current one is multiplied
    float ra[8], rb[8];
    // per-thread bases: (non-TRANS) A rows r0 + tid / 16 + 16 q, column k0 + tid % 16 (the column
    // mean loaded once per slab); (TRANS) A[k0 + tid / 128 + 2 q][r0 + tid % 128]; B[k0 + tid / 128 + 2 q][tid % 128]
    const int64_t a_row = TRANS_A ? r0 + (tid & 127) : r0 + (tid >> 4);
    const int a_k = TRANS_A ? (tid >> 7) : (tid & 15);
    const float* pa = TRANS_A ? A + a_row : A + a_row * stride * lda + a_k;
    const int64_t a_step = TRANS_A ? 2 * (int64_t)lda : 16 * stride * (int64_t)lda;  // per q
    const float* pb = B + (tid >> 7) * 128 + (tid & 127);
    auto load = [&](int64_t k0) {
        if (TRANS_A) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int64_t k = k0 + a_k + 2 * q;
                ra[q] = (a_row < M && k < k_hi) ? pa[k * lda] : 0.0f;
            }
        } else {
            const int64_t k = k0 + a_k;
            const bool kv = k < k_hi;
            const float mean = (kv && colsum) ? (float)(colsum[k] * inv_n) : 0.0f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                ra[q] = (kv && a_row + 16 * q < M) ? pa[q * a_step + k0] - mean : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) rb[q] = (k0 + (tid >> 7) + 2 * q < k_hi) ? pb[(k0 + 2 * q) * 128] : 0.0f;
    };
    auto store = [&]() {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int i = tid + 256 * q;
            if (TRANS_A) As[i >> 7][i & 127] = ra[q];
            else As[i & 15][i >> 4] = ra[q];
            Bs[i >> 7][i & 127] = rb[q];
        }
    };
    if (k_lo < k_hi) load(k_lo);
    for (int64_t k0 = k_lo; k0 < k_hi; k0 += 16) {
        store();
        __syncthreads();
        if (k0 + 16 < k_hi) load(k0 + 16);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a[8], b[8];
            const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][tr * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][tr * 8 + 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tc * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][tc * 8 + 4]);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t r = r0 + tr * 8 + i;
        if (r < M) {
            float4* o = reinterpret_cast<float4*>(C + r * 128 + tc * 8);
            o[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            o[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        }
    }
}

// out[i] = sum_{y < parts} in[y * len + i], in the order y = 0, 1, ...
__global__ void split_sum_kernel(const float* __restrict__ in, int parts, int64_t len, float* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    float acc = 0.0f;
    for (int y = 0; y < parts; ++y) acc += in[y * len + i];
    out[i] = acc;
}

}  // namespace
}  // namespace umapb200
