// sgd_common.cuh -- the SGD argument block and the device helpers shared by the layout SGD
// kernels (sgd.cu: the deterministic flat kernels; sgd_persistent.cu: the chunk kernel, Hogwild
// and DIM 8/16) and the transform SGD (transform.cu).  R-numbers: DESIGN.md section 2.
#pragma once
#include "common.cuh"

namespace umapb200 {
namespace sgdk {


struct SgdArgs {
    const int64_t* indptr;
    const int2* edges;       // per CSR entry {col, float_as_int(r)}, r = w / w_max (R9), built once
    int64_t n;
    int64_t n_chunks;        // ceil(n / VPW)
    const int32_t* bounds;   // CPB == 0: CTA b owns chunks [bounds[b], bounds[b+1]) (edge-balanced)
    float* Y0;               // positions (Hogwild: in place)
    float* Y1;               // deterministic: ping-pong partner of Y0
    float a, b, gamma, alpha0;
    int32_t n_epochs, e_begin, e_end, m;
    uint32_t key0, key1;
    unsigned long long* positives;  // device counter of due directed edges
    unsigned int* bar;       // grid barrier counters (BAR_WORDS words)
    const uint8_t* owner;    // per CSR entry: head vertex & 255 (its lane in the owning chunk)
    const uint16_t* hoff;    // flat kernel: per CSR entry, head vertex - first vertex of its piece
    int64_t nnz;
    int32_t vt;              // flat kernel: piece size (vertices whose sums are held in shared memory)
    const int2* prec;        // flat kernel, optional: {col | hoff << 21, r} (n < 2^21, vt <= 2048)
    int debug;               // profiling knob (UMAP_SGD_DEBUG): 1 = barrier only, 2 = no edge work (flat)
    // Philox4x32-10 round keys (R11) precomputed on the host: rk0[r] = key0 + r 0x9E3779B9,
    // rk1[r] = key1 + r 0xBB67AE85.  In the kernel parameter (constant) bank they enter the
    // round's 3-input XOR as an operand, no per-thread key schedule.
    uint32_t rk0[10], rk1[10];
    const int* max_row;      // flat2/3: device max CSR row length (> 65535: 64-bit CAS accumulation)
    int list_cap;            // flat3: due-list capacity (>= every CTA's record count)
    int scan_split_pct;      // flat3: % of the next epoch's scan done before the grid barrier's arrive
    int batch_static;        // flat3: 1 = warp w takes batches w, w + 32, ... (0: claimed dynamically)
    // flat4: the closed-form schedule (R9) materialised before the launch (sgd.cu, flat4): CTA b's
    // records in slots [slot_base[b], slot_base[b + 1]); slot s's epoch lists start at
    // sched + sched_region[s], the padded count of epoch index i at
    // sched_pcnt[NE slot_base[b] + i (slots of b) + (s - slot_base[b])]
    const uint32_t* sched;
    const int64_t* slot_base;
    const int64_t* sched_region;
    const int32_t* sched_pcnt;
};

__device__ __forceinline__ u32x4 philox_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const SgdArgs& A)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned long long p0 = (unsigned long long)0xD2511F53u * c0;
        const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ A.rk0[r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ A.rk1[r];
        c0 = n0; c1 = (uint32_t)p1; c2 = n2; c3 = (uint32_t)p0;
    }
    return {c0, c1, c2, c3};
}

__device__ __forceinline__ float clip4(float v) { return fminf(fmaxf(v, -4.0f), 4.0f); }

// s^b via exp2(b log2 s); s > 0
__device__ __forceinline__ float ex2_approx(float x)
{
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float pow_b(float s, float b) { return ex2_approx(b * __log2f(s)); }

__device__ __forceinline__ bool edge_due(float r, int e)
{
    return floorf(__fmul_rn((float)e, r)) > floorf(__fmul_rn((float)(e - 1), r));
}
// the same test with the epoch conversions hoisted: ef = (float)e, ef1 = (float)(e - 1)
__device__ __forceinline__ bool edge_due_f(float r, float ef, float ef1)
{
    return floorf(__fmul_rn(ef, r)) > floorf(__fmul_rn(ef1, r));
}

// L2-only read (ld.global.cg): the transform's training rows and the piece setup
template <int DIM>
__device__ __forceinline__ void load_row(const float* Y, int64_t v, float (&y)[DIM])
{
    if (DIM == 2) {
        const float2 t = __ldcg(reinterpret_cast<const float2*>(Y + v * 2));
        y[0] = t.x; y[1] = t.y;
    } else if (DIM == 4) {
        const float4 t = __ldcg(reinterpret_cast<const float4*>(Y + v * 4));
        y[0] = t.x; y[1] = t.y; y[2] = t.z; y[3] = t.w;
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) y[c] = __ldcg(Y + v * DIM + c);
    }
}

// streamed once per epoch, kept out of L1 (which holds the gathered positions)
__device__ __forceinline__ int2 ld_stream_i2(const int2* p)
{
    int2 r;
    asm("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ int ld_stream_u16(const uint16_t* p)
{
    unsigned short r;
    asm("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return (int)r;
}

// L1-cached read (ld.global.ca) for the flat deterministic kernel: within an epoch it only
// reads the ping-pong buffer Yr (writes go to Yw), and the grid barrier's gpu-scope fence
// invalidates L1 (CCTL.IVALL) before the next epoch reads what other SMs wrote
template <int DIM>
__device__ __forceinline__ void load_row_ca(const float* Y, int64_t v, float (&y)[DIM])
{
    if (DIM == 2) {
        float a, b;
        asm("ld.global.ca.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "l"(Y + v * 2));
        y[0] = a; y[1] = b;
    } else if (DIM == 4) {
        float a, b, c, d;
        asm("ld.global.ca.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(Y + v * 4));
        y[0] = a; y[1] = b; y[2] = c; y[3] = d;
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            float t;
            asm("ld.global.ca.f32 %0, [%1];" : "=f"(t) : "l"(Y + v * DIM + c));
            y[c] = t;
        }
    }
}

template <int DIM>
__device__ __forceinline__ void load_row_ro(const float* Y, int64_t v, float (&y)[DIM])
{
    if (DIM == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(Y + v * 2));
        y[0] = t.x; y[1] = t.y;
    } else if (DIM == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(Y + v * 4));
        y[0] = t.x; y[1] = t.y; y[2] = t.z; y[3] = t.w;
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) y[c] = __ldg(Y + v * DIM + c);
    }
}

constexpr int SGD_WARPS = 8;  // warps per CTA at MINB = 4; in general 32 / MINB (32 warps per SM)
template <int MINB> constexpr int sgd_warps() { return MINB >= 4 ? SGD_WARPS : 32 / MINB; }
constexpr int QCAP = 64;

// R13 fixed point: q(g) = round(g 2^24) (exact scaling; |g| <= 4 alpha, so |q| <= 2^26 alpha0; a
// due edge's (2 + m) terms fit int32 while (2 + m) alpha0 < 32, enforced by check_params)
__device__ __forceinline__ int qfix(float g) { return __float2int_rn(g * 16777216.0f); }

// One due edge (h, t) at epoch e: attractive update of h (and, Hogwild, t) and M negative
// samples on h.  MC = compile-time M (all negative-sample loads issued before use), or 0
// for a runtime M.  DET: the head contribution is returned in fixed point (qacc); the
// tail contribution is the head contribution of (t, h), computed by t's owner.
template <int DIM, bool DET, int MC, bool L1 = false>
__device__ __forceinline__ void process_edge(const SgdArgs& A, const float* Yr, float* Yw, int epoch, float alpha,
                                             int h, int t, int (&qacc)[DIM])
{
    float yh[DIM], yt[DIM], g[DIM];
    constexpr int MP = MC > 0 ? MC : 1;
    int vv[MP];
    float yv[MP][DIM];
    if (MC > 0) {
        // Philox counter (h, t, e, p>>2) (R11) first, then the head, tail and all M sample
        // rows are requested together: one L2 round trip per due edge
#pragma unroll
        for (int blk = 0; blk < (MP + 3) / 4; ++blk) {
            const u32x4 rnd = philox4x32_10((uint32_t)h, (uint32_t)t, (uint32_t)epoch, (uint32_t)blk, A.key0, A.key1);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int p = 4 * blk + i;
                if (p < MP) vv[p] = (int)__umulhi(pick(rnd, i), (uint32_t)A.n);
            }
        }
    }
    if (L1) {
        load_row_ca<DIM>(Yr, h, yh);
        load_row_ca<DIM>(Yr, t, yt);
    } else {
        load_row<DIM>(Yr, h, yh);
        load_row<DIM>(Yr, t, yt);
    }
    if (MC > 0) {
#pragma unroll
        for (int p = 0; p < MP; ++p) {
            if (L1) load_row_ca<DIM>(Yr, vv[p], yv[p]);
            else load_row<DIM>(Yr, vv[p], yv[p]);
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int c = 0; c < DIM; ++c) { const float df = yh[c] - yt[c]; s = fmaf(df, df, s); }
    float coef = 0.0f;
    if (s > 0.0f) {
        const float sb = pow_b(s, A.b);
        coef = __fdividef(-2.0f * A.a * A.b * __fdividef(sb, s), fmaf(A.a, sb, 1.0f));
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) g[c] = clip4(coef * (yh[c] - yt[c])) * alpha;
    float h0[DIM];
    if (DET) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) qacc[c] += 2 * qfix(g[c]);
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) { h0[c] = yh[c]; yh[c] += g[c]; }
        if (DIM == 2) {
            atomicAdd(reinterpret_cast<float2*>(Yw + t * 2), make_float2(-g[0], -g[1]));
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) atomicAdd(Yw + t * DIM + c, -g[c]);
        }
    }
    const int pend = MC > 0 ? MC : A.m;
    u32x4 rnd = {0, 0, 0, 0};
#pragma unroll
    for (int p = 0; p < pend; ++p) {
        int v;
        float yvv[DIM];
        if (MC > 0) {
            v = vv[MC > 0 ? p : 0];
#pragma unroll
            for (int c = 0; c < DIM; ++c) yvv[c] = yv[MC > 0 ? p : 0][c];
        } else {
            if ((p & 3) == 0)
                rnd = philox4x32_10((uint32_t)h, (uint32_t)t, (uint32_t)epoch, (uint32_t)(p >> 2), A.key0, A.key1);
            v = (int)__umulhi(pick(rnd, p & 3), (uint32_t)A.n);
            if (L1) load_row_ca<DIM>(Yr, v, yvv);
            else load_row<DIM>(Yr, v, yvv);
        }
        if (v == h) continue;
        float s2 = 0.0f;
#pragma unroll
        for (int c = 0; c < DIM; ++c) { const float df = yh[c] - yvv[c]; s2 = fmaf(df, df, s2); }
        if (s2 > 0.0f) {
            const float sb = pow_b(s2, A.b);
            const float cr = __fdividef(2.0f * A.gamma * A.b, (0.001f + s2) * fmaf(A.a, sb, 1.0f));
#pragma unroll
            for (int c = 0; c < DIM; ++c) g[c] = clip4(cr * (yh[c] - yvv[c])) * alpha;
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) g[c] = 4.0f * alpha;
        }
        if (DET) {
#pragma unroll
            for (int c = 0; c < DIM; ++c) qacc[c] += qfix(g[c]);
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) yh[c] += g[c];
        }
    }
    if (!DET) {
        if (DIM == 2) {
            atomicAdd(reinterpret_cast<float2*>(Yw + h * 2), make_float2(yh[0] - h0[0], yh[1] - h0[1]));
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) atomicAdd(Yw + h * DIM + c, yh[c] - h0[c]);
        }
    }
}

// grid-wide barrier between epochs (cooperative launch guarantees co-residency);
// release/acquire at gpu scope order the epoch's writes and invalidate L1.  Monotonic arrival
// counter: barrier number k (1-based) completes when the counter reaches k * gridDim.x (no
// reset, one release-add and acquire polling per CTA).  A two-level variant (8 group
// counters on separate lines) measured no faster at 592 CTAs.
constexpr size_t BAR_WORDS = 2;
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int k)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        // the CTA's writes happen-before thread 0's release through the bar.sync above (release
        // is cumulative), and the acquire poll below invalidates this SM's L1 (CCTL.IVALL)
        // before the next epoch's L1-cached reads: no separate fence.sc needed
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned int target = k * gridDim.x;
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// ---------------------------------------------------------------- flat2: lean deterministic SGD
// The flat kernel's edge work, restructured to issue fewer instructions per due edge (the
// flat kernel issues ~800 thread-instructions per due edge; ncu r01p):
//  * Philox round keys from the kernel parameter bank (philox_rk) instead of a per-thread
//    key schedule;
//  * the piece's own head rows sit in shared memory (loaded once per piece, also the base of
//    the final write), only the tail and the m samples are gathered from global memory, all
//    issued together before any arithmetic (predicated volatile loads: the compiler cannot
//    sink one into a branch);
//  * branch-free terms: alpha 2^24 folded into the coefficient (A24 = alpha 2^24 exactly, so
//    clip4(c d) alpha 2^24 = clamp(c A24 d, +-4 A24) up to the rounding of one product), one
//    MUFU.RCP per term, the s = 0 and v = head cases by selects (v = head gives d = 0, s = 0
//    and a zero kick); packed FADD2/FMUL2 at DIM 2;
//  * fixed-point sums by 32-bit shared reductions of the per-edge sum split at bit 16
//    (lo = q & 0xFFFF summed unsigned, hi = q >> 16 summed signed; exact while a vertex has
//    < 65536 due edges per epoch, i.e. every CSR row shorter than 65536 -- else the 64-bit CAS
//    add), instead of the warp-segmented 64-bit scan.
// The per-term quantisation q = rint(g 2^24) and the integer sums keep the result independent
// of the launch shape and of the order of the work (R13).
template <int DIM>
__device__ __forceinline__ void gather_row_p(const float* Y, int64_t v, bool p, float (&y)[DIM])
{
    const float* a = Y + v * DIM;
    if (DIM == 2) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.global.ca.v2.f32 {%0, %1}, [%2];\n\t}"
                     : "+f"(y[0]), "+f"(y[1]) : "l"(a), "r"((int)p));
    } else if (DIM == 4) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.ca.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
                     : "+f"(y[0]), "+f"(y[1]), "+f"(y[2]), "+f"(y[3]) : "l"(a), "r"((int)p));
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c)
            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.ca.f32 %0, [%1];\n\t}"
                         : "+f"(y[c]) : "l"(a + c), "r"((int)p));
    }
}

__device__ __forceinline__ float lg2_ftz(float x)
{
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_ftz(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

struct TermK {
    float a, b;     // curve (R8)
    float katt;     // -2 a b A24
    float krep;     // 2 gamma b A24
    float c4;       // 4 A24 (the clip bound in fixed-point units)
};

// d = yh - yo, s = |d|^2 in the R12 order (s = fmaf(d_c, d_c, s) over c)
template <int DIM>
__device__ __forceinline__ float diff_sq(const float (&yh)[DIM], const float (&yo)[DIM], float (&d)[DIM])
{
    if (DIM == 2) {
        unsigned long long H, O, D;
        asm("mov.b64 %0, {%1, %2};" : "=l"(H) : "f"(yh[0]), "f"(yh[1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(O) : "f"(yo[0]), "f"(yo[1]));
        asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(D) : "l"(H), "l"(O));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(d[0]), "=f"(d[1]) : "l"(D));
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) d[c] = yh[c] - yo[c];
    }
    float s = 0.0f;
#pragma unroll
    for (int c = 0; c < DIM; ++c) s = fmaf(d[c], d[c], s);
    return s;
}

// q_c += sel ? rint(clamp(k d_c, +-c4)) : rint(alt)
template <int DIM>
__device__ __forceinline__ void quant_add(float k, const float (&d)[DIM], bool sel, float alt, float c4, int mul,
                                          int (&q)[DIM])
{
    float g[DIM];
    if (DIM == 2) {
        unsigned long long D, K, G;
        asm("mov.b64 %0, {%1, %2};" : "=l"(D) : "f"(d[0]), "f"(d[1]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(K) : "f"(k));
        asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(G) : "l"(D), "l"(K));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(g[0]), "=f"(g[1]) : "l"(G));
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = k * d[c];
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const float x = sel ? fminf(fmaxf(g[c], -c4), c4) : alt;
        q[c] += mul * __float2int_rn(x);
    }
}

// Edge work of one due edge (h = v0 + hl, t) at epoch `epoch` for the lean kernels: the head's
// fixed-point contribution qa (2 q(g_att) + sum of the m repulsive q(g), R12/R13).  yhead holds
// the head rows of the vertices [v0, ...).  act = false: the gathers are predicated off and qa is
// meaningless (the caller does not add it).
// XDBG (UMAP_SGD_DEBUG with UMAP_UNSAFE_EXPERIMENTS, flat3 at DIM 2 / M 5 only; results are wrong
// by construction, timing decomposition only): 4 = negatives gathered from the CTA's own 256
// vertices (L1-resident), 8 = the tail too, 16 = a one-multiply hash instead of Philox
template <int DIM, int MC, int XDBG = 0>
__device__ __forceinline__ void edge_terms(const SgdArgs& A, const float* Yr, int epoch, uint32_t nn, const TermK& K,
                                           const float* yhead, int v0, int hl, int t, bool act, int (&qa)[DIM])
{
    const int h = v0 + hl;
    constexpr int MP = MC > 0 ? MC : 1;
    int vv[MP];
    float yt[DIM], yv[MP][DIM], yh[DIM];
    if (MC > 0) {
#pragma unroll
        for (int blk = 0; blk < (MP + 3) / 4; ++blk) {
            u32x4 rnd;
            if constexpr ((XDBG & 16) != 0) {
                const uint32_t x = ((uint32_t)h * 0x9E3779B1u) ^ ((uint32_t)t * 0x85EBCA77u) ^ ((uint32_t)epoch * 0xC2B2AE3Du) ^ blk;
                rnd = {x, x * 0x27D4EB2Fu, x * 0x165667B1u, x * 0xD3A2646Cu};
            } else {
                rnd = philox_rk((uint32_t)h, (uint32_t)t, (uint32_t)epoch, (uint32_t)blk, A);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (4 * blk + i < MP) {
                    vv[4 * blk + i] = (int)__umulhi(pick(rnd, i), nn);
                    if constexpr ((XDBG & 4) != 0) vv[4 * blk + i] = v0 + (int)(pick(rnd, i) & 255u);
                }
        }
    }
    if constexpr ((XDBG & 8) != 0) t = v0 + (t & 255);
#pragma unroll
    for (int c = 0; c < DIM; ++c) yt[c] = 0.0f;
    gather_row_p<DIM>(Yr, t, act, yt);
    if (MC > 0) {
#pragma unroll
        for (int p = 0; p < MP; ++p) {
#pragma unroll
            for (int c = 0; c < DIM; ++c) yv[p][c] = 0.0f;
            gather_row_p<DIM>(Yr, vv[p], act, yv[p]);
        }
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) yh[c] = yhead[hl * DIM + c];
#pragma unroll
    for (int c = 0; c < DIM; ++c) qa[c] = 0;
    {   // attractive: head share 2 q(g) (owner computes, R13)
        float d[DIM];
        const float s = diff_sq<DIM>(yh, yt, d);
        const float sb = ex2_approx(K.b * lg2_ftz(s));
        const float den = s * fmaf(K.a, sb, 1.0f);
        const float k = s > 0.0f ? K.katt * sb * rcp_ftz(den) : 0.0f;
        quant_add<DIM>(k, d, true, 0.0f, K.c4, 2, qa);
    }
    const int pend = MC > 0 ? MC : A.m;
    u32x4 rnd = {0, 0, 0, 0};
#pragma unroll
    for (int p = 0; p < pend; ++p) {
        int v;
        float yvv[DIM];
        if (MC > 0) {
            v = vv[MC > 0 ? p : 0];
#pragma unroll
            for (int c = 0; c < DIM; ++c) yvv[c] = yv[MC > 0 ? p : 0][c];
        } else {
            if ((p & 3) == 0) rnd = philox_rk((uint32_t)h, (uint32_t)t, (uint32_t)epoch, (uint32_t)(p >> 2), A);
            v = (int)__umulhi(pick(rnd, p & 3), nn);
#pragma unroll
            for (int c = 0; c < DIM; ++c) yvv[c] = 0.0f;
            gather_row_p<DIM>(Yr, v, act, yvv);
        }
        float d[DIM];
        const float s2 = diff_sq<DIM>(yh, yvv, d);
        const float sb = ex2_approx(K.b * lg2_ftz(s2));
        const float k = K.krep * rcp_ftz((0.001f + s2) * fmaf(K.a, sb, 1.0f));
        // s2 = 0: +4 alpha per component unless v is the head itself (then d = 0, no term)
        quant_add<DIM>(k, d, s2 > 0.0f, v != h ? K.c4 : 0.0f, K.c4, 1, qa);
    }
}

// add a per-edge fixed-point sum to the head's accumulators (16-bit split, or 64-bit CAS when
// some CSR row has >= 65536 entries)
template <int DIM>
__device__ __forceinline__ void acc_add(uint32_t* acc_lo, int32_t* acc_hi, unsigned long long* acc64, int stride,
                                        int hl, bool wide, const int (&qa)[DIM])
{
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        if (!wide) {
            atomicAdd(acc_lo + c * stride + hl, (uint32_t)qa[c] & 0xFFFFu);
            atomicAdd(acc_hi + c * stride + hl, qa[c] >> 16);
        } else {
            atomicAdd(acc64 + c * stride + hl, (unsigned long long)(long long)qa[c]);
        }
    }
}

__device__ __forceinline__ TermK epoch_terms(const SgdArgs& A, int epoch)
{
    const float alpha = __fmul_rn(A.alpha0, __fsub_rn(1.0f, __fdiv_rn((float)epoch, (float)A.n_epochs)));
    const float a24 = __fmul_rn(alpha, 16777216.0f);  // exact (power-of-two scale)
    TermK K;
    K.a = A.a; K.b = A.b;
    K.katt = __fmul_rn(-2.0f * A.a * A.b, a24);
    K.krep = __fmul_rn(2.0f * A.gamma * A.b, a24);
    K.c4 = __fmul_rn(4.0f, a24);
    return K;
}


// sgd_persistent.cu: the chunk kernel (Hogwild, and deterministic at DIM 8/16)
template <int DIM>
umap_status launch_sgd_persistent(const SgdArgs& A, bool det, cudaStream_t s);

}  // namespace sgdk
}  // namespace umapb200
