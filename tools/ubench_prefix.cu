// ubench_prefix.cu -- does an smem-resident copy of a prefix of Y (refreshed every epoch by
// bulk copies, optionally multicast across a cluster) take random position gathers off the
// L1TEX/L2 path fast enough to pay for the refresh?  Models the C2 SGD: 500 epochs, a grid
// barrier per epoch, G random 8-byte gathers per thread per epoch (C2: 457k due edges x 6
// gathers / 148 SMs / 1024 threads = 18).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ubp tools/ubench_prefix.cu
//   tools/bin/ubp [n] [gathers_per_thread] [epochs]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t xs(uint32_t x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int k)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned int target = k * gridDim.x;
        unsigned int v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t cluster_ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// mode 0: all gathers global (.ca); mode 1: rows < P from the smem prefix, refreshed per epoch by
// this CTA's own bulk copies; mode 2: the same, the refresh multicast across the cluster
// (each CTA copies 1/csz of the prefix to every CTA of its cluster).
template <int MODE>
__global__ void __launch_bounds__(1024, 1) epochs_kernel(float2* Y, int n, int P, int G, int epochs,
                                                         unsigned int* bar, float* out)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    float2* yp = reinterpret_cast<float2*>(smem + 128);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
    const uint32_t ypa = (uint32_t)__cvta_generic_to_shared(yp);
    const uint32_t bytes = (uint32_t)P * 8u;
    const uint32_t csz = MODE == 2 ? cluster_nctarank() : 1;
    const uint32_t crank = MODE == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (MODE == 2) asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
    __syncthreads();
    uint32_t st = 0x9E3779B9u * (blockIdx.x * 1024 + threadIdx.x + 1);
    float acc = 0.0f;
    uint32_t phase = 0;
    if (MODE >= 1 && threadIdx.x == 0)  // arm for epoch 0
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    if (MODE == 2) asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
    for (int e = 0; e < epochs; ++e) {
        if (MODE >= 1 && threadIdx.x == 0) {
            // refresh: split the prefix into 16 KB pieces; this CTA issues pieces crank, crank+csz, ...
            const uint32_t piece = 16384;
            for (uint32_t off = crank * piece; off < bytes; off += csz * piece) {
                const uint32_t sz = min(piece, bytes - off);
                const char* src = reinterpret_cast<const char*>(Y) + off;
                if (MODE == 1) {
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(ypa + off), "l"(src), "r"(sz), "r"(mb) : "memory");
                } else {
                    const uint16_t mask = (uint16_t)((1u << csz) - 1u);
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                                 ::"r"(ypa + off), "l"(src), "r"(sz), "r"(mb), "h"(mask) : "memory");
                }
            }
        }
        if (MODE >= 1) {
            uint32_t done = 0;
            while (!done) {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(mb), "r"(phase) : "memory");
            }
            phase ^= 1;
        }
        for (int g = 0; g < G; g += 6) {
            float a[6], b[6];
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                st = xs(st);
                const int v = (int)__umulhi(st, (uint32_t)n);
                if (MODE >= 1 && v < P) {
                    const float2 t = yp[v];
                    a[l] = t.x; b[l] = t.y;
                } else {
                    asm volatile("ld.global.ca.v2.f32 {%0, %1}, [%2];" : "=f"(a[l]), "=f"(b[l]) : "l"(Y + v));
                }
            }
#pragma unroll
            for (int l = 0; l < 6; ++l) acc += a[l] * b[l];
        }
        // every thread of the CTA is done reading the prefix of epoch e; arm for e + 1, then
        // the grid barrier (after it, peers may multicast the next prefix into this CTA)
        __syncthreads();
        if (MODE >= 1 && threadIdx.x == 0 && e + 1 < epochs)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        if (e + 1 < epochs) grid_barrier(bar, (unsigned)(e + 1));
    }
    if (MODE == 2) asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
    if (acc == 1.2345f) out[0] = acc;
}

int main(int argc, char** argv)
{
    const int n = argc > 1 ? atoi(argv[1]) : 70000;
    const int G = argc > 2 ? atoi(argv[2]) : 18;
    const int epochs = argc > 3 ? atoi(argv[3]) : 500;
    float2* Y;
    float* out;
    unsigned int* bar;
    CK(cudaMalloc(&Y, sizeof(float2) * n));
    CK(cudaMalloc(&out, 4));
    CK(cudaMalloc(&bar, 4));
    CK(cudaMemset(Y, 0, sizeof(float2) * n));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](auto kern, int P, int csz, const char* name) {
        const size_t smem = 128 + (size_t)P * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(csz);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl <= 0) {
            printf("{\"variant\": \"%s\", \"P\": %d, \"csz\": %d, \"error\": \"no occupancy\"}\n", name, P, csz);
            cudaGetLastError();
            return;
        }
        const int grid = std::min(ncl * csz, (sms / csz) * csz);
        cfg.gridDim = dim3(grid);
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaMemset(bar, 0, 4));
            CK(cudaEventRecord(e0));
            CK(cudaLaunchKernelEx(&cfg, kern, Y, n, P, G, epochs, bar, out));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep) best = ms < best ? ms : best;
        }
        // gathers per epoch scaled to the whole 148-SM problem (fewer CTAs -> same per-CTA G)
        printf("{\"variant\": \"%s\", \"n\": %d, \"P\": %d, \"csz\": %d, \"ctas\": %d, \"G\": %d, \"epochs\": %d, "
               "\"ms\": %.4f, \"us_per_epoch\": %.3f}\n",
               name, n, P, csz, grid, G, epochs, best, best * 1000.0f / epochs);
    };
    run(epochs_kernel<0>, 0, 1, "global");
    for (int P : {8192, 16384, 20480, 24576, 26624}) {
        if (P > n) continue;
        run(epochs_kernel<1>, P, 1, "prefix_unicast");
        for (int csz : {2, 4, 8, 16}) run(epochs_kernel<2>, P, csz, "prefix_multicast");
    }
    return 0;
}
