// ubench_stream.cu -- can every SM receive the whole embedding Y (C2: 70,000 x 2 fp32 =
// 560 KB) once per SGD epoch?  Each CTA (one per SM) streams Y through a ring of NB shared-memory
// slice buffers with TMA bulk copies; in a cluster of C CTAs each CTA issues 1/C of every slice
// with .multicast::cluster to all C CTAs (C = 1: plain unicast).  A grid barrier closes each
// "epoch".  Prints microseconds per epoch and the implied per-SM ingest and L2 read rates.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubs tools/ubench_stream.cu && /tmp/ubs
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) { while (!mbar_try_wait(bar, parity)) {} }
__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_n()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// NT threads: warp 0 lane 0 produces, all threads consume (read a few words of the slice)
template <int NB>
__global__ void __launch_bounds__(512, 1) stream_kernel(const char* Y, int bytes, int slice, int epochs,
                                                         unsigned int* bar, float* out, int touch)
{
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) unsigned long long full[NB], empty[NB];
    const uint32_t C = cluster_n(), r = cluster_rank();
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) { mbar_init(smem_u32(&full[b]), 1); mbar_init(smem_u32(&empty[b]), C); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    const int S = (bytes + slice - 1) / slice;
    const int chunk = slice / (int)C;
    float acc = 0.f;
    uint32_t it0 = 0;  // ring position of the epoch's first slice
    auto issue = [&](int s, uint32_t it) {  // thread 0: slice s of this epoch into ring slot it % NB
        const int b = it % NB;
        const uint32_t ph = (it / NB) & 1;
        if (it >= NB) mbar_wait(smem_u32(&empty[b]), ph ^ 1);
        const int off = s * slice;
        const int len = min(slice, bytes - off);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[b])), "r"(len) : "memory");
        const int my = (int)r * chunk;
        if (my < len) {
            const int ml = min(chunk, len - my);
            const uint32_t dst = smem_u32(sm + (size_t)b * slice + my);
            if (C == 1) {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(dst), "l"(Y + off + my), "r"(ml), "r"(smem_u32(&full[b])) : "memory");
            } else {
                const uint16_t mask = (uint16_t)((1u << C) - 1u);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                             ::"r"(dst), "l"(Y + off + my), "r"(ml), "r"(smem_u32(&full[b])), "h"(mask) : "memory");
            }
        }
    };
    for (int e = 0; e < epochs; ++e) {
        if (threadIdx.x == 0)
            for (int s = 0; s < min(NB, S); ++s) issue(s, it0 + s);
        for (int s = 0; s < S; ++s) {
            const uint32_t it = it0 + s;
            const int b = it % NB;
            const uint32_t ph = (it / NB) & 1;
            mbar_wait(smem_u32(&full[b]), ph);
            if (touch) {
                const float* f = reinterpret_cast<const float*>(sm + (size_t)b * slice);
                for (int i = threadIdx.x; i < slice / 4; i += blockDim.x * touch) acc += f[i];
            }
            __syncthreads();
            if (threadIdx.x < C) {  // release buffer b in CTA threadIdx.x of the cluster
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&empty[b])), "r"((uint32_t)threadIdx.x));
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
            }
            if (threadIdx.x == 0 && s + NB < S) issue(s + NB, it + NB);
        }
        it0 += S;
        // grid barrier
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            const unsigned int target = (unsigned)(e + 1) * gridDim.x;
            unsigned int v;
            do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
        }
        __syncthreads();
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (acc == 1.2345f) out[0] = acc;
}

template <int NB>
void run(const char* Y, int bytes, int slice, int C, int epochs, unsigned int* bar, float* out, int touch)
{
    auto kern = stream_kernel<NB>;
    const int smem = NB * slice;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (C > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at; cfg.numAttrs = 1;
    cfg.gridDim = dim3(C);
    int ncl = 0;
    CK(cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg));
    const int grid = ncl * C;
    cfg.gridDim = dim3(grid);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemset(bar, 0, 4));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        CK(cudaLaunchKernelEx(&cfg, kern, Y, bytes, slice, epochs, bar, out, touch));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double us = best * 1e3 / epochs;
    printf("{\"C\": %d, \"ctas\": %d, \"slice\": %d, \"NB\": %d, \"touch\": %d, \"bytes\": %d, \"us_per_epoch\": %.3f, "
           "\"ingest_GBs_per_sm\": %.1f, \"l2_read_GBs_if_mc_dedups\": %.1f, \"delivered_GBs\": %.1f}\n",
           C, grid, slice, NB, touch, bytes, us, bytes / us * 1e-3, (double)bytes * grid / C / us * 1e-3,
           (double)bytes * grid / us * 1e-3);
    fflush(stdout);
}

int main(int argc, char** argv)
{
    const int bytes = argc > 1 ? atoi(argv[1]) : 560000;
    const int epochs = 200;
    char* Y; unsigned int* bar; float* out;
    CK(cudaMalloc(&Y, 64 << 20)); CK(cudaMemset(Y, 0, 64 << 20));
    CK(cudaMalloc(&bar, 64)); CK(cudaMalloc(&out, 64));
    // barrier-only reference
    run<2>(Y, 0, 16384, 1, epochs, bar, out, 0);
    for (int C : {1, 2, 4, 8, 16}) {
        for (int slice : {8192, 16384, 32768}) {
            run<4>(Y, bytes, slice, C, epochs, bar, out, 0);
            run<6>(Y, bytes, slice, C, epochs, bar, out, 0);
        }
        run<4>(Y, bytes, 32768, C, epochs, bar, out, 4);
    }
    return 0;
}
