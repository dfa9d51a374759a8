// bulk.cuh -- mbarrier helpers and the TMA bulk-copy row ring shared by the exact
// distance re-checks (rank_fix, rerank, trust thresholds).  Device code of the CUDA path only.
#pragma once
#include "common.cuh"

namespace umapb200 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// try_wait with a suspend-time hint: the waiting thread is suspended in hardware until the phase
// completes (or the hint, 10 ms, elapses) instead of re-issuing the poll: a spinning producer or
// MMA thread otherwise takes issue slots from the epilogue warps of its scheduler
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity), "r"(10000000u)
            : "memory");
    }
}

// Exact R2 distances of 32 pairs (one query row, one candidate per lane) with the rows staged by the TMA bulk-copy engine: per warp a
// double-buffered smem ring of 33 row segments (32 candidates + the query row) of RB_CH
// floats; lane p issues one cp.async.bulk for its candidate's segment, completion is counted
// on the buffer's mbarrier, and each lane then continues the sequential R2 fmaf chain of its
// pair from shared memory with 16-byte loads (row stride RB_CH = 100 words = 4 mod 32: the
// eight lanes of each LDS.128 phase hit 32 distinct banks).  Requires d % 4 == 0 (16-byte
// aligned rows); the value is bit-identical to exact_d2.  8 warps x 100-float segments
// measured best at C2 (4.3 ms vs 7.2 ms for per-lane LDG streaming; 4 x 196: 4.9, 16 x 52: 4.9).
constexpr int RB_WARPS = 8;
constexpr int RB_CH = 100;
constexpr size_t RB_WARP_FLOATS = 2 * 33 * RB_CH;
constexpr size_t RB_SMEM = RB_WARPS * RB_WARP_FLOATS * sizeof(float) + RB_WARPS * 2 * sizeof(uint64_t);

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// 32 pairs (x, Xr[l_lane]) (l < 0: none) through the warp's bulk ring; returns lane's R2 value.
// ph: per-buffer phase bits of the ring's two mbarriers (updated).
__device__ __forceinline__ float exact_d2_bulk(const float* __restrict__ x, const float* __restrict__ Xr,
                                               int32_t l, int d, float* ring, uint32_t bar0, uint32_t& ph, int lane)
{
    const unsigned act = __ballot_sync(0xffffffffu, l >= 0);
    const int nch = (d + RB_CH - 1) / RB_CH;
    auto issue = [&](int c) {
        const int b = c & 1;
        const int w = min(RB_CH, d - c * RB_CH);
        const uint32_t bytes = (uint32_t)w * 4u;
        const uint32_t bar = bar0 + 8 * b;
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(ring + (size_t)b * 33 * RB_CH);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads vs the async refill
        __syncwarp();
        if (lane == 0) {
            mbar_expect_tx(bar, bytes * (uint32_t)(__popc(act) + 1));
            bulk_g2s(base + 32u * RB_CH * 4u, x + (size_t)c * RB_CH, bytes, bar);
        }
        __syncwarp();
        if (l >= 0) bulk_g2s(base + (uint32_t)lane * RB_CH * 4u, Xr + (int64_t)l * d + (size_t)c * RB_CH, bytes, bar);
    };
    issue(0);
    float s = 0.0f;
    for (int c = 0; c < nch; ++c) {
        const int b = c & 1;
        if (c + 1 < nch) issue(c + 1);
        mbar_wait(bar0 + 8 * b, (ph >> b) & 1u);
        ph ^= 1u << b;
        const float4* rr = reinterpret_cast<const float4*>(ring + (size_t)b * 33 * RB_CH + (size_t)lane * RB_CH);
        const float4* xx = reinterpret_cast<const float4*>(ring + (size_t)b * 33 * RB_CH + 32 * RB_CH);
        const int w4 = min(RB_CH, d - c * RB_CH) >> 2;
        for (int j = 0; j < w4; ++j) {
            const float4 a = xx[j], y = rr[j];
            float t = __fsub_rn(a.x, y.x); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.y, y.y); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.z, y.z); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.w, y.w); s = __fmaf_rn(t, t, s);
        }
        __syncwarp();  // every lane is done with buffer b before it is refilled (iteration c + 1 issues c + 2)
    }
    return s;
}


// Two query rows per warp (k <= 15 candidates each): lanes 0..14 pair x0 with Xr[l_lane], lanes
// 16..30 pair x1 with Xr[l_lane]; x0 goes to the ring's query slot (32), x1 to lane 31's slot (lanes
// 15 and 31 carry no candidate).  Otherwise exact_d2_bulk.
__device__ __forceinline__ float exact_d2_bulk2(const float* __restrict__ x0, const float* __restrict__ x1,
                                                const float* __restrict__ Xr, int32_t l, int d, float* ring,
                                                uint32_t bar0, uint32_t& ph, int lane)
{
    const unsigned act = __ballot_sync(0xffffffffu, l >= 0);
    const int nch = (d + RB_CH - 1) / RB_CH;
    const int qslot = lane < 16 ? 32 : 31;
    auto issue = [&](int c) {
        const int b = c & 1;
        const int w = min(RB_CH, d - c * RB_CH);
        const uint32_t bytes = (uint32_t)w * 4u;
        const uint32_t bar = bar0 + 8 * b;
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(ring + (size_t)b * 33 * RB_CH);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads vs the async refill
        __syncwarp();
        if (lane == 0) {
            mbar_expect_tx(bar, bytes * (uint32_t)(__popc(act) + 2));
            bulk_g2s(base + 32u * RB_CH * 4u, x0 + (size_t)c * RB_CH, bytes, bar);
            bulk_g2s(base + 31u * RB_CH * 4u, x1 + (size_t)c * RB_CH, bytes, bar);
        }
        __syncwarp();
        if (l >= 0) bulk_g2s(base + (uint32_t)lane * RB_CH * 4u, Xr + (int64_t)l * d + (size_t)c * RB_CH, bytes, bar);
    };
    issue(0);
    float s = 0.0f;
    for (int c = 0; c < nch; ++c) {
        const int b = c & 1;
        if (c + 1 < nch) issue(c + 1);
        mbar_wait(bar0 + 8 * b, (ph >> b) & 1u);
        ph ^= 1u << b;
        const float4* rr = reinterpret_cast<const float4*>(ring + (size_t)b * 33 * RB_CH + (size_t)lane * RB_CH);
        const float4* xx = reinterpret_cast<const float4*>(ring + (size_t)b * 33 * RB_CH + (size_t)qslot * RB_CH);
        const int w4 = min(RB_CH, d - c * RB_CH) >> 2;
        for (int j = 0; j < w4; ++j) {
            const float4 a = xx[j], y = rr[j];
            float t = __fsub_rn(a.x, y.x); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.y, y.y); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.z, y.z); s = __fmaf_rn(t, t, s);
            t = __fsub_rn(a.w, y.w); s = __fmaf_rn(t, t, s);
        }
        __syncwarp();  // every lane is done with buffer b before it is refilled
    }
    return s;
}

// per-warp ring of a block of RB_WARPS warps (dynamic smem of RB_SMEM bytes); initialises the
// warp's two mbarriers (lane 0) and returns the ring and the first barrier's address
__device__ __forceinline__ float* bulk_ring_setup(uint32_t& bar0)
{
    extern __shared__ __align__(16) float rb_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(rb_smem + RB_WARPS * RB_WARP_FLOATS);
    bar0 = smem_u32(bars + 2 * warp);
    if (lane == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    return rb_smem + (size_t)warp * RB_WARP_FLOATS;
}

}  // namespace umapb200
