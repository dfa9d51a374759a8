// common.cuh -- shared device helpers of the CUDA path (never shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <string>

#include "../../include/umap_b200.h"

namespace umapb200 {

// ---------------------------------------------------------------- errors
void set_last_error(const std::string& s);
umap_status cuda_status(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define UMAP_CUDA_TRY(expr)                                              \
    do {                                                                 \
        cudaError_t _e = (expr);                                         \
        if (_e != cudaSuccess) return ::umapb200::cuda_status(_e, #expr);\
    } while (0)

#define UMAP_TRY(expr)                                                   \
    do {                                                                 \
        umap_status _s = (expr);                                         \
        if (_s != UMAP_OK) return _s;                                    \
    } while (0)

#define UMAP_LAUNCH_CHECK(name)                                          \
    do {                                                                 \
        ::umapb200::count_launch();                                      \
        cudaError_t _e = cudaGetLastError();                             \
        if (_e != cudaSuccess) return ::umapb200::cuda_status(_e, name); \
    } while (0)

// ---------------------------------------------------------------- live kernel timing
// Optional per-kernel CUDA-event timing (umap_profile_begin / umap_profile_end): when
// enabled, a ProfScope records an event pair around one launch on its stream.
enum ProfSlot {
    PROF_KNN_TC = 0, PROF_RERANK, PROF_TRUST_TC, PROF_RANK_FIX, PROF_THRESHOLDS, PROF_GRID_KNN,
    PROF_SMOOTH_KNN, PROF_UNION, PROF_SGD, PROF_KNN_EXACT, PROF_TRUST_EXACT, PROF_TRANSFORM_SGD,
    PROF_TRUST_COARSE, PROF_SPECTRAL, PROF_TRUST_PROJ, PROF_TRUST_REGROUP, PROF_KNN_PRUNE, PROF_SGD_SCHED, PROF_NSLOTS
};
bool profiling_enabled();
void profile_record(int slot, cudaEvent_t e0, cudaEvent_t e1);
struct ProfScope {
    int slot;
    cudaStream_t s;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ProfScope(int sl, cudaStream_t st) : slot(sl), s(st)
    {
        if (sl >= 0 && profiling_enabled() && cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess)
            cudaEventRecord(e0, s);
        else
            e0 = e1 = nullptr;
    }
    ~ProfScope()
    {
        if (e0) {
            cudaEventRecord(e1, s);
            profile_record(slot, e0, e1);  // ownership of the events moves to the profile table
        }
    }
};

inline int current_device()
{
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

// Function attributes (dynamic shared memory opt-in, carveout) and occupancy are per device:
// `static PerDeviceOnce once; if (once.first()) {...}` runs the block once on every device a
// process uses (a process-wide flag skipped it on the second GPU).
struct PerDeviceOnce {
    std::atomic<uint64_t> mask{0};
    bool first()
    {
        const uint64_t b = 1ull << (current_device() & 63);
        return !(mask.fetch_or(b) & b);
    }
};

inline int num_sms()
{
    static int sms[64] = {0};
    const int dev = current_device() & 63;
    if (!sms[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device());
        sms[dev] = v > 0 ? v : 148;
    }
    return sms[dev];
}

// Stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync): the RMM-pool
// analogue of P:81.  Freed on the same stream when the owner goes out of scope.
struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() { if (p) cudaFreeAsync(p, s); }
    umap_status alloc(size_t bytes, cudaStream_t st)
    {
        s = st;
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMallocAsync(&p, bytes, st);
        if (e != cudaSuccess) { p = nullptr; return cuda_status(e, "cudaMallocAsync"); }
        return UMAP_OK;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al. SC'11; constants of the Random123 reference.  R11.
struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    return {c0, c1, c2, c3};
}

__device__ __forceinline__ uint32_t pick(const u32x4& v, int i)
{
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// key order (d2, id) of R1
__device__ __forceinline__ bool key_less(float da, int32_t ia, float db, int32_t ib)
{
    return da < db || (da == db && ia < ib);
}

template <class T> __device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }


// R2 exact distance: sequential fmaf in ascending feature order (float4 loads when the
// rows are 16-byte aligned; the accumulation order is unchanged).
__device__ __forceinline__ float exact_d2(const float* x, const float* y, int d)
{
    float s = 0.0f;
    int f = 0;
    if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* y4 = reinterpret_cast<const float4*>(y);
        for (; f + 4 <= d; f += 4) {
            const float4 a = __ldg(x4 + (f >> 2)), b = __ldg(y4 + (f >> 2));
            float t = __fsub_rn(a.x, b.x); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.y, b.y); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.z, b.z); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.w, b.w); s = __fmaf_rn(t, t, s);
        }
    }
    for (; f < d; ++f) {
        const float t = __fsub_rn(__ldg(x + f), __ldg(y + f));
        s = __fmaf_rn(t, t, s);
    }
    return s;
}


// ascending bitonic sort of 32 (key, id) pairs across a warp (lane i ends with rank i)
__device__ __forceinline__ void warp_bitonic(float& key, int32_t& id, int lane)
{
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const float ok = __shfl_xor_sync(0xffffffffu, key, stride);
            const int32_t oi = __shfl_xor_sync(0xffffffffu, id, stride);
            const bool up = ((lane & size) == 0);
            const bool lower = (lane & stride) == 0;
            const bool other_less = key_less(ok, oi, key, id);
            const bool take = lower ? (up ? other_less : !other_less) : (up ? !other_less : other_less);
            if (take && !(ok == key && oi == id)) { key = ok; id = oi; }
        }
    }
}


// two independent ascending bitonic sorts of (key, id) over lanes 0..15 and 16..31
__device__ __forceinline__ void warp_bitonic16(float& key, int32_t& id, int lane)
{
#pragma unroll
    for (int size = 2; size <= 16; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const float ok = __shfl_xor_sync(0xffffffffu, key, stride);
            const int32_t oi = __shfl_xor_sync(0xffffffffu, id, stride);
            const bool up = size == 16 || ((lane & size) == 0);
            const bool lower = (lane & stride) == 0;
            const bool other_less = key_less(ok, oi, key, id);
            const bool take = lower ? (up ? other_less : !other_less) : (up ? !other_less : other_less);
            if (take && !(ok == key && oi == id)) { key = ok; id = oi; }
        }
    }
}

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// Measurement knobs that make results invalid or uncertified (margin overrides, disabled
// kernel parts) are read only when UMAP_UNSAFE_EXPERIMENTS is set as well.
inline const char* unsafe_env(const char* name)
{
    return getenv("UMAP_UNSAFE_EXPERIMENTS") ? getenv(name) : nullptr;
}

}  // namespace umapb200
