// knn_lowdim.cu -- exact kNN for the 2-D embedding (trustworthiness, a10; R1/R2 on Y).
//
// The brute-force tile kernel spends O(n^2) compares on a 2-D input.  Here the points are
// bucketed into a uniform grid (counting sort by cell, ~0.15 points per cell) and each query
// scans Chebyshev rings of cells around its own cell, keeping its k best keys (d2, id) in
// registers, until the ring's distance lower bound exceeds the current k-th distance.
// d2 uses the R2 operation order (fmaf over the two coordinates), every point that can
// enter the top-k is examined, so the result is bit-identical to the brute-force
// definition.  The lower bound is taken one ring early to absorb rounding in the cell
// assignment.
#include <cstdlib>

#include "common.cuh"

namespace umapb200 {

umap_status exclusive_scan_i32(const int32_t* in, int64_t n, int64_t* out, cudaStream_t s);

namespace {

__global__ void bbox_kernel(const float* __restrict__ Y, int64_t n, float* __restrict__ box)
{
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 p = reinterpret_cast<const float2*>(Y)[i];
        mnx = fminf(mnx, p.x); mny = fminf(mny, p.y); mxx = fmaxf(mxx, p.x); mxy = fmaxf(mxy, p.y);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // order-preserving int encoding of floats for atomic min/max
        auto enc = [](float f) { int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7fffffff; };
        atomicMin(reinterpret_cast<int*>(box) + 0, enc(mnx));
        atomicMin(reinterpret_cast<int*>(box) + 1, enc(mny));
        atomicMax(reinterpret_cast<int*>(box) + 2, enc(mxx));
        atomicMax(reinterpret_cast<int*>(box) + 3, enc(mxy));
    }
}

__device__ __forceinline__ float dec(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

struct Grid {
    float x0, y0, inv_h, h;
    int G;
};

__device__ __forceinline__ Grid grid_of(const float* box, int G)
{
    const int* b = reinterpret_cast<const int*>(box);
    Grid g;
    g.x0 = dec(b[0]);
    g.y0 = dec(b[1]);
    const float ext = fmaxf(fmaxf(dec(b[2]) - g.x0, dec(b[3]) - g.y0), 1e-30f);
    g.h = ext / (float)G * 1.0001f;
    g.inv_h = 1.0f / g.h;
    g.G = G;
    return g;
}

__device__ __forceinline__ int cell_coord(float v, float v0, float inv_h, int G)
{
    const int c = (int)floorf((v - v0) * inv_h);
    return min(max(c, 0), G - 1);
}

__global__ void cell_count_kernel(const float* __restrict__ Y, int64_t n, const float* __restrict__ box, int G,
                                  int32_t* __restrict__ cell_of, int32_t* __restrict__ cnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Grid g = grid_of(box, G);
    const float2 p = reinterpret_cast<const float2*>(Y)[i];
    const int c = cell_coord(p.y, g.y0, g.inv_h, G) * G + cell_coord(p.x, g.x0, g.inv_h, G);
    cell_of[i] = c;
    atomicAdd(cnt + c, 1);
}

__global__ void cell_fill_kernel(const float* __restrict__ Y, int64_t n, const int32_t* __restrict__ cell_of,
                                 const int64_t* __restrict__ start, int32_t* __restrict__ cursor,
                                 int32_t* __restrict__ pid, float2* __restrict__ pxy)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = cell_of[i];
    const int64_t pos = start[c] + atomicAdd(cursor + c, 1);
    pid[pos] = (int32_t)i;
    pxy[pos] = reinterpret_cast<const float2*>(Y)[i];
}

template <int KC>
__global__ void __launch_bounds__(128) grid_knn_kernel(const float2* __restrict__ pxy, const int32_t* __restrict__ pid,
                                                       const int64_t* __restrict__ start, const float* __restrict__ box,
                                                       int G, int64_t n, int k, int out_squared,
                                                       int32_t* __restrict__ idx, float* __restrict__ dist)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // position in cell order (locality)
    if (s >= n) return;
    const Grid g = grid_of(box, G);
    const float2 p = pxy[s];
    const int self = pid[s];
    const int cx = cell_coord(p.x, g.x0, g.inv_h, G), cy = cell_coord(p.y, g.y0, g.inv_h, G);
    float kd[KC];
    int32_t ki[KC];
#pragma unroll
    for (int i = 0; i < KC; ++i) { kd[i] = INFINITY; ki[i] = INT32_MAX; }
    for (int r = 0; r <= G; ++r) {
        if (r >= 2) {
            const float lb = (float)(r - 2) * g.h;  // one ring of slack for cell-assignment rounding
            if (lb * lb * 0.99999f > kd[k - 1]) break;
        }
        const int ylo = cy - r, yhi = cy + r;
        for (int yy = max(ylo, 0); yy <= min(yhi, G - 1); ++yy) {
            const bool edge_row = (yy == ylo || yy == yhi);
            const int step = edge_row ? 1 : 2 * r;  // ring perimeter only
            for (int xx = cx - r; xx <= cx + r; xx += (step > 0 ? step : 1)) {
                if (xx < 0 || xx >= G) continue;
                const int c = yy * G + xx;
                for (int64_t e = start[c]; e < start[c + 1]; ++e) {
                    const int32_t j = pid[e];
                    if (j == self) continue;
                    const float2 o = pxy[e];
                    const float t0 = __fsub_rn(p.x, o.x), t1 = __fsub_rn(p.y, o.y);
                    float cv = __fmaf_rn(t1, t1, __fmaf_rn(t0, t0, 0.0f));
                    if (!key_less(cv, j, kd[k - 1], ki[k - 1])) continue;
                    int32_t ci = j;
#pragma unroll
                    for (int i = 0; i < KC; ++i) {
                        const bool sw = key_less(cv, ci, kd[i], ki[i]);
                        const float tk = sw ? kd[i] : cv;
                        const int32_t ti = sw ? ki[i] : ci;
                        kd[i] = sw ? cv : kd[i];
                        ki[i] = sw ? ci : ki[i];
                        cv = tk;
                        ci = ti;
                    }
                }
                if (step == 0) break;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < KC; ++i) {
        if (i < k) {
            idx[(int64_t)self * k + i] = ki[i] == INT32_MAX ? -1 : ki[i];
            dist[(int64_t)self * k + i] = out_squared ? kd[i] : __fsqrt_rn(kd[i]);
        }
    }
}

}  // namespace

// exact self-kNN of a 2-D point set (R1/R2), rows sorted by key; k <= 32
umap_status knn_grid2d(const float* Y, int64_t n, int k, int out_squared, int32_t* idx, float* dist, cudaStream_t s)
{
    if (n == 0) return UMAP_OK;
    if (k > 32 || n >= (int64_t)INT32_MAX) {
        set_last_error("grid kNN: k <= 32 and n < 2^31 required");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    // points per cell: fine cells (mostly empty) make the ring lower bound tight, so fewer
    // points are examined; measured at C2 (70k points, k = 15): 4 -> 1.16 ms, 1 -> 0.50,
    // 0.25 -> 0.31, 0.15 -> 0.26, 0.1 -> 0.28
    double ppc = 0.15;
    if (const char* e = getenv("UMAP_GRID_PPC")) ppc = atof(e);  // tuning knob
    int G = (int)std::max<double>(1.0, std::floor(std::sqrt((double)n / ppc)));
    G = std::min(G, 4096);
    const int64_t cells = (int64_t)G * G;
    Scratch box, cell_of, cnt, start, cursor, pid, pxy;
    UMAP_TRY(box.alloc(4 * sizeof(float), s));
    // min slots start at +FLT_MAX, max slots at -FLT_MAX (order-preserving int encoding)
    int h_init[4] = {0x7f7fffff, 0x7f7fffff, (int)(0xff7fffffu ^ 0x7fffffffu), (int)(0xff7fffffu ^ 0x7fffffffu)};
    UMAP_CUDA_TRY(cudaMemcpyAsync(box.p, h_init, sizeof(h_init), cudaMemcpyHostToDevice, s));
    bbox_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 4LL * num_sms()), 256, 0, s>>>(Y, n, box.as<float>());
    UMAP_LAUNCH_CHECK("bbox_kernel");
    UMAP_TRY(cell_of.alloc(sizeof(int32_t) * (size_t)n, s));
    UMAP_TRY(cnt.alloc(sizeof(int32_t) * (size_t)cells, s));
    UMAP_TRY(start.alloc(sizeof(int64_t) * (size_t)(cells + 1), s));
    UMAP_TRY(cursor.alloc(sizeof(int32_t) * (size_t)cells, s));
    UMAP_TRY(pid.alloc(sizeof(int32_t) * (size_t)n, s));
    UMAP_TRY(pxy.alloc(sizeof(float2) * (size_t)n, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * cells, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(cursor.p, 0, sizeof(int32_t) * cells, s));
    cell_count_kernel<<<ceil_div(n, 256), 256, 0, s>>>(Y, n, box.as<float>(), G, cell_of.as<int32_t>(),
                                                        cnt.as<int32_t>());
    UMAP_LAUNCH_CHECK("cell_count_kernel");
    UMAP_TRY(exclusive_scan_i32(cnt.as<int32_t>(), cells, start.as<int64_t>(), s));
    cell_fill_kernel<<<ceil_div(n, 256), 256, 0, s>>>(Y, n, cell_of.as<int32_t>(), start.as<int64_t>(),
                                                       cursor.as<int32_t>(), pid.as<int32_t>(), pxy.as<float2>());
    UMAP_LAUNCH_CHECK("cell_fill_kernel");
    ProfScope ps(PROF_GRID_KNN, s);
    if (k <= 16)
        grid_knn_kernel<16><<<ceil_div(n, 128), 128, 0, s>>>(pxy.as<float2>(), pid.as<int32_t>(), start.as<int64_t>(),
                                                             box.as<float>(), G, n, k, out_squared, idx, dist);
    else
        grid_knn_kernel<32><<<ceil_div(n, 128), 128, 0, s>>>(pxy.as<float2>(), pid.as<int32_t>(), start.as<int64_t>(),
                                                             box.as<float>(), G, n, k, out_squared, idx, dist);
    UMAP_LAUNCH_CHECK("grid_knn_kernel");
    return UMAP_OK;
}

}  // namespace umapb200

// ---------------------------------------------------------------- cluster order of an embedding
// Hilbert (default) or Morton (Z-order, UMAP_ORDER_MORTON) key of each 2-D point on a 2^16 x 2^16 grid over the bounding box, then a
// stable radix sort of (key, row): perm[p] = the row at position p.  Used by the trust path
// to visit rows and columns cluster by cluster (a layout choice; results do not depend on it).
#include <cub/device/device_radix_sort.cuh>

namespace umapb200 {
namespace {

__device__ __forceinline__ uint32_t spread16(uint32_t v)
{
    v &= 0xFFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

// Hilbert index of (x, y) on a 2^16 x 2^16 grid (the classic rotate-and-flip walk): unlike the
// Z order it has no long jumps, so consecutive rows stay inside one 2-D region longer
__device__ __forceinline__ uint32_t hilbert16(uint32_t x, uint32_t y)
{
    uint32_t d = 0;
    for (uint32_t s = 1u << 15; s > 0; s >>= 1) {
        const uint32_t rx = (x & s) > 0, ry = (y & s) > 0;
        d += s * s * ((3 * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) { x = s - 1 - x; y = s - 1 - y; }
            const uint32_t t = x; x = y; y = t;
        }
    }
    return d;
}

__global__ void morton_kernel(const float* __restrict__ Y, int64_t n, const float* __restrict__ box,
                              uint32_t* __restrict__ keys, int32_t* __restrict__ vals, int hilbert)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Grid g = grid_of(box, 65536);
    const float2 p = reinterpret_cast<const float2*>(Y)[i];
    const uint32_t cx = (uint32_t)cell_coord(p.x, g.x0, g.inv_h, 65536);
    const uint32_t cy = (uint32_t)cell_coord(p.y, g.y0, g.inv_h, 65536);
    keys[i] = hilbert ? hilbert16(cx, cy) : (spread16(cx) | (spread16(cy) << 1));
    vals[i] = (int32_t)i;
}

}  // namespace

// in place: sort (keys, vals) by key, stable (LSD radix)
umap_status sort_pairs_u32(uint32_t* keys, int32_t* vals, int64_t n, cudaStream_t s)
{
    if (n <= 1) return UMAP_OK;
    Scratch k2, v2, tmp;
    UMAP_TRY(k2.alloc(sizeof(uint32_t) * (size_t)n, s));
    UMAP_TRY(v2.alloc(sizeof(int32_t) * (size_t)n, s));
    size_t bytes = 0;
    UMAP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, k2.as<uint32_t>(), vals, v2.as<int32_t>(),
                                                  (int)n, 0, 32, s));
    UMAP_TRY(tmp.alloc(bytes, s));
    UMAP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys, k2.as<uint32_t>(), vals, v2.as<int32_t>(),
                                                  (int)n, 0, 32, s));
    count_launch(4);
    UMAP_CUDA_TRY(cudaMemcpyAsync(keys, k2.p, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
    UMAP_CUDA_TRY(cudaMemcpyAsync(vals, v2.p, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
    return UMAP_OK;
}

umap_status cluster_order(const float* Y, int64_t n, int d_emb, int32_t* perm, cudaStream_t s)
{
    if (d_emb != 2) { set_last_error("cluster_order: 2-D embedding required"); return UMAP_ERR_UNSUPPORTED; }
    Scratch box, keys;
    UMAP_TRY(box.alloc(4 * sizeof(float), s));
    int h_init[4] = {0x7f7fffff, 0x7f7fffff, (int)(0xff7fffffu ^ 0x7fffffffu), (int)(0xff7fffffu ^ 0x7fffffffu)};
    UMAP_CUDA_TRY(cudaMemcpyAsync(box.p, h_init, sizeof(h_init), cudaMemcpyHostToDevice, s));
    bbox_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 4LL * num_sms()), 256, 0, s>>>(Y, n, box.as<float>());
    UMAP_LAUNCH_CHECK("bbox_kernel");
    UMAP_TRY(keys.alloc(sizeof(uint32_t) * (size_t)n, s));
    const int hilbert = getenv("UMAP_ORDER_MORTON") ? 0 : 1;  // A/B knob
    morton_kernel<<<ceil_div(n, 256), 256, 0, s>>>(Y, n, box.as<float>(), keys.as<uint32_t>(), perm, hilbert);
    UMAP_LAUNCH_CHECK("morton_kernel");
    return sort_pairs_u32(keys.as<uint32_t>(), perm, n, s);
}

}  // namespace umapb200
