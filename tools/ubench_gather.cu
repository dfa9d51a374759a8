// ubench_gather.cu -- throughput of random 8-byte position gathers (the SGD's access pattern)
// from (a) global memory through L1 (.ca) or L2 only (.cg), (b) distributed shared memory
// across a thread-block cluster holding one slice of Y per CTA, (c) a CTA's own shared memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubg tools/ubench_gather.cu && /tmp/ubg [n]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int NL = 6;  // gathers issued together (tail + 5 negatives)

__device__ __forceinline__ uint32_t xs(uint32_t x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

template <int MODE, int NT = 1024, int NLD = NL>  // MODE 0 = .ca, 1 = .cg, 2 = .nc, 3 = .nc.L1::no_allocate, 4 = .lu
__global__ void __launch_bounds__(NT) gather_global(const float2* Y, int n, int iters, float* out)
{
    extern __shared__ float pad_smem[];  // dynamic smem only to shrink L1 (carveout experiments)
    uint32_t st = 0x9E3779B9u * (blockIdx.x * 1024 + threadIdx.x + 1);
    float acc = 0.0f;
    for (int it = 0; it < iters; ++it) {
        float a[NLD], b[NLD];
#pragma unroll
        for (int l = 0; l < NLD; ++l) {
            st = xs(st);
            const int v = (int)__umulhi(st, (uint32_t)n);
            if (MODE == 0) asm volatile("ld.global.ca.v2.f32 {%0, %1}, [%2];" : "=f"(a[l]), "=f"(b[l]) : "l"(Y + v));
            else if (MODE == 1) asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(a[l]), "=f"(b[l]) : "l"(Y + v));
            else if (MODE == 2) asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(a[l]), "=f"(b[l]) : "l"(Y + v));
            else if (MODE == 3) asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(a[l]), "=f"(b[l]) : "l"(Y + v));
            else asm volatile("ld.global.lu.v2.f32 {%0, %1}, [%2];" : "=f"(a[l]), "=f"(b[l]) : "l"(Y + v));
        }
#pragma unroll
        for (int l = 0; l < NLD; ++l) acc += a[l] * b[l];
    }
    if (acc == 1.2345f) out[0] = acc;
}

// cluster of C CTAs; CTA r holds rows [r*slice, (r+1)*slice) of Y in its shared memory
__global__ void __launch_bounds__(1024, 1) gather_dsmem(const float2* Y, int n, int slice, int iters, float* out,
                                                         int local_only)
{
    extern __shared__ float2 ys[];
    cg::cluster_group cl = cg::this_cluster();
    const int r = (int)cl.block_rank();
    for (int i = threadIdx.x; i < slice; i += blockDim.x) {
        const int v = r * slice + i;
        ys[i] = v < n ? Y[v] : make_float2(0.f, 0.f);
    }
    cl.sync();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(ys);
    uint32_t st = 0x9E3779B9u * (blockIdx.x * 1024 + threadIdx.x + 1);
    float acc = 0.0f;
    const int nn = local_only ? slice : n;
    for (int it = 0; it < iters; ++it) {
        float a[NL], b[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            st = xs(st);
            const int v = (int)__umulhi(st, (uint32_t)nn);
            const int owner = local_only ? r : v / slice;
            const int off = local_only ? v : v - owner * slice;
            uint32_t la = base + off * 8, ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(owner));
            asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(a[l]), "=f"(b[l]) : "r"(ra));
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) acc += a[l] * b[l];
    }
    cl.sync();
    if (acc == 1.2345f) out[0] = acc;
}

int main(int argc, char** argv)
{
    const int n = argc > 1 ? atoi(argv[1]) : 70000;
    const int iters = argc > 2 ? atoi(argv[2]) : 1000;
    float2* Y;
    float* out;
    CK(cudaMalloc(&Y, sizeof(float2) * n));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(Y, 0, sizeof(float2) * n));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto report = [&](const char* name, int ctas, float ms) {
        const double g = (double)ctas * 1024 * iters * NL;  // every variant does the same total count
        printf("{\"variant\": \"%s\", \"n\": %d, \"ctas\": %d, \"ms\": %.4f, \"Ggathers_per_s\": %.1f}\n", name, n, ctas,
               ms, g / ms * 1e-6);
    };
    auto timeit = [&](auto kern, int grid, int nt, size_t smem, int it, const char* name) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(e0));
            kern<<<grid, nt, smem>>>(Y, n, it, out);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep) best = ms < best ? ms : best;
        }
        char nm[96];
        snprintf(nm, sizeof nm, "%s_smem%zuK", name, smem / 1024);
        report(nm, sms, best);
    };
    for (size_t smem : {(size_t)0, (size_t)32768, (size_t)98304, (size_t)163840}) {
        timeit(gather_global<0>, sms, 1024, smem, iters, "global_ca");
        timeit(gather_global<1>, sms, 1024, smem, iters, "global_cg");
        timeit(gather_global<2>, sms, 1024, smem, iters, "global_nc");
        timeit(gather_global<3>, sms, 1024, smem, iters, "global_nc_noalloc");
        timeit(gather_global<4>, sms, 1024, smem, iters, "global_lu");
    }
    // more loads in flight per thread (same total), fewer threads per SM
    timeit(gather_global<0, 1024, 12>, sms, 1024, 0, iters / 2, "global_ca_12inflight");
    timeit(gather_global<0, 512, 6>, 2 * sms, 512, 0, iters, "global_ca_2x512");
    timeit(gather_global<0, 256, 6>, 4 * sms, 256, 0, iters, "global_ca_4x256");
    timeit(gather_global<0, 512, 12>, sms * 2, 512, 0, iters / 2, "global_ca_2x512_12inflight");
    CK(cudaFuncSetAttribute(gather_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int C : {2, 3, 4, 6, 8, 16}) {
        for (int local_only = 0; local_only < 2; ++local_only) {
            const int slice = (n + C - 1) / C;
            const size_t smem = sizeof(float2) * slice;
            if (smem > 227 * 1024) continue;
            CK(cudaFuncSetAttribute(gather_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.blockDim = dim3(1024);
            cfg.dynamicSmemBytes = smem;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cfg.gridDim = dim3(C);
            int ncl = 0;
            cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, gather_dsmem, &cfg);
            if (oe != cudaSuccess || ncl <= 0) { printf("{\"variant\": \"dsmem%d\", \"error\": \"occupancy %s\"}\n", C, cudaGetErrorString(oe)); cudaGetLastError(); continue; }
            cfg.gridDim = dim3(ncl * C);
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaEventRecord(e0));
                cudaError_t le = cudaLaunchKernelEx(&cfg, gather_dsmem, (const float2*)Y, n, slice, iters, out, local_only);
                if (le != cudaSuccess) { printf("launch C=%d: %s\n", C, cudaGetErrorString(le)); break; }
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                char name[64];
                snprintf(name, sizeof name, "%s%d", local_only ? "local_smem_c" : "dsmem_c", C);
                if (rep) report(name, ncl * C, ms);
            }
        }
    }
    return 0;
}
