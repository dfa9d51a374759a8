// sgd.cu -- random init (a7), SGD layout (a6, a8) and transform SGD (a9).
//
// Layout SGD: all epochs in one cooperative launch, a grid barrier between
// epochs.  A CTA owns a cost-balanced vertex range; the due edges of an epoch (closed-form
// schedule, R9) are compacted so that every lane carries a due edge through the expensive part
// (attractive term + m negatives + 2 Philox calls).
//
//  * DETERMINISTIC (R13): reads Y_e only, writes Y_{e+1} (ping-pong).  Each vertex is
//    updated only by the CTA that owns it ("owner computes"): because B is bit-exactly symmetric,
//    the tail update of edge (i,j) equals the head update of edge (j,i), so vertex i receives
//    2 q(g_att) per own due edge plus q(g_rep) per negative, q(g) = round(g 2^24) per term, the
//    terms of a due edge summed in int32 and added to the head's shared-memory accumulator by
//    32-bit reductions of the sum split at bit 16 (flat2 / flat3) or by 64-bit warp-segment sums
//    (the round-1 flat kernel) -- integer sums, so the result is identical for any launch shape
//    and work order.  No global atomics.  Kernels: sgd_flat3_kernel (default: the whole CTA range
//    in one piece, per-epoch due lists), sgd_flat2_kernel (pieces of vt vertices, e.g. C4),
//    sgd_flat_kernel (round 1, UMAP_SGD_VARIANT=100), sgd_persistent_kernel (DIM 8 / 16).
//  * HOGWILD: in-place.  Each due edge reads the live positions, moves its head in
//    registers through the attractive and the m repulsive updates (the paper's register
//    accumulation) and pushes -g_att to the tail and the accumulated head delta with fp32
//    vector atomics.
// Position gathers go through L1 (ld.global.ca): within an epoch the deterministic kernels read
// only the ping-pong buffer Y_e, and the grid barrier's acquire invalidates L1 before the next
// epoch; Hogwild reads are unsynchronised by definition (staleness bounded to one epoch).
#include <cstdlib>

#include "common.cuh"

namespace umapb200 {

template <class Tin> umap_status exclusive_scan(const Tin* in, int64_t n, int64_t* out, cudaStream_t s);  // graph.cu
namespace {

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

// Persistent SGD: epochs [e_begin, e_end) in one cooperative launch.  A warp work unit
// owns VPW consecutive vertices; their CSR rows are contiguous, so the warp streams the
// (col, r) records with coalesced loads, evaluates the closed-form schedule (R9), and
// compacts due edges into a per-warp queue that is processed 32 at a time (every lane
// carries a due edge during the expensive part).
template <int DIM, bool DET, int MC, int VPW, int MINB, int CPB>
__global__ void __launch_bounds__(32 * sgd_warps<MINB>(), MINB) sgd_persistent_kernel(SgdArgs A)
{
    constexpr int W = sgd_warps<MINB>();
    __shared__ int32_t q_h[W][QCAP];   // owner lane (0..VPW-1) of the queued edge
    __shared__ int32_t q_t[W][QCAP];   // tail vertex
    __shared__ long long acc[W][DIM][VPW];
    __shared__ int s_ctr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = (int)A.n;
    const int n_chunks = (int)A.n_chunks;
    unsigned long long due_count = 0;
    for (int epoch = A.e_begin; epoch < A.e_end; ++epoch) {
        const int par = (epoch - A.e_begin) & 1;
        const float* Yr = (DET && par) ? A.Y1 : A.Y0;
        float* Yw = DET ? (par ? A.Y0 : A.Y1) : A.Y0;
        const float alpha = __fmul_rn(A.alpha0, __fsub_rn(1.0f, __fdiv_rn((float)epoch, (float)A.n_epochs)));
        const float ef = (float)epoch, ef1 = (float)(epoch - 1);
        // a CTA owns CPB consecutive chunks (VPW * CPB vertices); its warps take chunks from
        // the CTA's range through a shared-memory counter (dynamic balance inside the CTA,
        // no global work counter: thousands of grabs per epoch would serialise at L2)
        // (CPB == 0: one edge-balanced range per CTA, precomputed)
        const int n_br = CPB > 0 ? (n_chunks + CPB - 1) / CPB : (int)gridDim.x;
        for (int br = blockIdx.x; br < (A.debug & 1 ? 0 : n_br); br += gridDim.x) {
          const int c_lo = CPB > 0 ? br * CPB : A.bounds[br];
          const int c_hi = CPB > 0 ? min(n_chunks, c_lo + CPB) : A.bounds[br + 1];
          if (threadIdx.x == 0) s_ctr = 0;
          __syncthreads();
          for (;;) {
            int ci = 0;
            if (lane == 0) ci = atomicAdd(&s_ctr, 1);
            ci = __shfl_sync(0xffffffffu, ci, 0);
            const int chunk = c_lo + ci;
            if (chunk >= c_hi) break;
            const int v0 = chunk * VPW;
            const int nv = min(VPW, n - v0);
            // lane l < nv holds indptr[v0 + l]; the end is loaded separately (nv may be 32)
            const int64_t ptr_l = lane < nv ? __ldg(A.indptr + v0 + lane) : 0;
            const int64_t e_lo = __shfl_sync(0xffffffffu, ptr_l, 0);
            const int64_t e_hi = __ldg(A.indptr + v0 + nv);
            if (DET && lane < VPW) {
#pragma unroll
                for (int c = 0; c < DIM; ++c) acc[warp][c][lane] = 0;
            }
            __syncwarp();
            int qn = 0;
            auto drain = [&](int count) {
                const bool act = lane < count;
                const int hl = act ? q_h[warp][lane] : -1;
                int qa[DIM];
#pragma unroll
                for (int c = 0; c < DIM; ++c) qa[c] = 0;
                if (act) process_edge<DIM, DET, MC, true>(A, Yr, Yw, epoch, alpha, v0 + hl, q_t[warp][lane], qa);
                if (DET) {
                    // queued items are in CSR order, so equal owners are contiguous: segmented
                    // sum over the warp, the last lane of each segment adds it (order-free int sum;
                    // measured faster than 64-bit shared atomics)
                    long long sv[DIM];
#pragma unroll
                    for (int c = 0; c < DIM; ++c) sv[c] = qa[c];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int ho = __shfl_up_sync(0xffffffffu, hl, o);
#pragma unroll
                        for (int c = 0; c < DIM; ++c) {
                            const long long so = __shfl_up_sync(0xffffffffu, sv[c], o);
                            if (lane >= o && ho == hl) sv[c] += so;
                        }
                    }
                    const int hn = __shfl_down_sync(0xffffffffu, hl, 1);
                    if (act && (lane == count - 1 || hn != hl)) {
#pragma unroll
                        for (int c = 0; c < DIM; ++c) acc[warp][c][hl] += sv[c];
                    }
                }
                __syncwarp();
            };
            int2 nrec = (e_lo + lane < e_hi) ? __ldg(A.edges + e_lo + lane) : make_int2(0, 0);
            for (int64_t base = e_lo; base < e_hi; base += 32) {
                const int64_t e = base + lane;
                const int2 rec = nrec;  // records are prefetched one 32-edge step ahead
                if (base + 32 + lane < e_hi) nrec = __ldg(A.edges + base + 32 + lane);
                const bool due = e < e_hi && edge_due_f(__int_as_float(rec.y), ef, ef1);
                // owner lane of the edge's head vertex within the chunk (precomputed)
                const int lo = due ? (int)(__ldg(A.owner + e) & (VPW - 1)) : 0;
                const unsigned ballot = __ballot_sync(0xffffffffu, due);
                due_count += __popc(ballot);
                if (due) {
                    const int pos = qn + __popc(ballot & ((1u << lane) - 1u));
                    q_h[warp][pos] = lo;
                    q_t[warp][pos] = rec.x;
                }
                __syncwarp();
                qn += __popc(ballot);
                if (qn >= 32) {
                    drain(32);
                    qn -= 32;
                    if (lane < qn) {
                        q_h[warp][lane] = q_h[warp][32 + lane];
                        q_t[warp][lane] = q_t[warp][32 + lane];
                    }
                    __syncwarp();
                }
            }
            if (qn > 0) drain(qn);
            if (DET && lane < nv) {
                const int v = v0 + lane;
                float yo[DIM];
                load_row<DIM>(Yr, v, yo);
#pragma unroll
                for (int c = 0; c < DIM; ++c) {
                    const double upd = (double)acc[warp][c][lane] * (1.0 / 16777216.0);
                    Yw[(int64_t)v * DIM + c] = (float)((double)yo[c] + upd);
                }
            }
            __syncwarp();
          }
          __syncthreads();
        }
        if (epoch + 1 < A.e_end) grid_barrier(A.bar, (unsigned int)(epoch - A.e_begin + 1));
    }
    // due_count is warp-uniform (every lane added the same ballot counts)
    if (A.positives && lane == 0 && due_count) atomicAdd(A.positives, due_count);
}

// Deterministic SGD with the CTA's records split evenly over its warps.  CTA b owns the
// vertex range [bounds[b], bounds[b+1]) (cost-balanced) and works through it in pieces of
// at most vt vertices.  Within a piece the 32-record steps of the piece's CSR range go to
// the warps round-robin (step s -> warp s mod W), so every warp gets ~1/W of the piece's
// records whatever the degree mix (the chunk kernel above hands out whole 16-vertex chunks,
// about one per warp per epoch at C2, and its warps idle at the CTA barrier).  Head sums:
// warp-segmented int sums as above, then one 64-bit shared atomic per segment into the
// piece's fixed-point accumulators; integer addition is associative, so the result is
// bit-identical to the chunk kernel's whatever the order (R13).
template <int DIM, int MC>
__global__ void __launch_bounds__(1024, 1) sgd_flat_kernel(SgdArgs A)
{
    constexpr int W = 32;
    extern __shared__ __align__(16) unsigned char sgd_smem[];
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(sgd_smem);  // [DIM][vt]
    int32_t* const qh = reinterpret_cast<int32_t*>(acc + (size_t)DIM * A.vt) + (threadIdx.x >> 5) * QCAP;
    int32_t* const qt = qh + W * QCAP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int vt = A.vt;
    const int v_lo = A.bounds[blockIdx.x], v_hi = A.bounds[blockIdx.x + 1];
    unsigned long long due_count = 0;
    for (int epoch = A.e_begin; epoch < A.e_end; ++epoch) {
        const int par = (epoch - A.e_begin) & 1;
        const float* Yr = par ? A.Y1 : A.Y0;
        float* Yw = par ? A.Y0 : A.Y1;
        const float alpha = __fmul_rn(A.alpha0, __fsub_rn(1.0f, __fdiv_rn((float)epoch, (float)A.n_epochs)));
        const float ef = (float)epoch, ef1 = (float)(epoch - 1);
        for (int pv0 = v_lo; pv0 < (A.debug & 1 ? v_lo : v_hi); pv0 += vt) {  // debug: profiling only
            const int np = min(vt, v_hi - pv0);
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
#pragma unroll
                for (int c = 0; c < DIM; ++c) acc[c * vt + i] = 0ull;
            }
            __syncthreads();
            const int64_t E0 = __ldg(A.indptr + pv0), E1 = __ldg(A.indptr + pv0 + np);
            int qn = 0;
            auto drain = [&](int count) {
                const bool act = lane < count;
                const int hl = act ? qh[lane] : -1;
                int qa[DIM];
#pragma unroll
                for (int c = 0; c < DIM; ++c) qa[c] = 0;
                if (act && !(A.debug & 2))
                    process_edge<DIM, true, MC, true>(A, Yr, Yw, epoch, alpha, pv0 + hl, qt[lane], qa);
                long long sv[DIM];
#pragma unroll
                for (int c = 0; c < DIM; ++c) sv[c] = qa[c];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int ho = __shfl_up_sync(0xffffffffu, hl, o);
#pragma unroll
                    for (int c = 0; c < DIM; ++c) {
                        const long long so = __shfl_up_sync(0xffffffffu, sv[c], o);
                        if (lane >= o && ho == hl) sv[c] += so;
                    }
                }
                const int hn = __shfl_down_sync(0xffffffffu, hl, 1);
                if (act && (lane == count - 1 || hn != hl)) {
#pragma unroll
                    for (int c = 0; c < DIM; ++c) atomicAdd(acc + c * vt + hl, (unsigned long long)sv[c]);
                }
                __syncwarp();
            };
            int64_t base = E0 + 32 * warp;
            int2 nrec = make_int2(0, 0);
            int nho = 0;
            // one 8-byte record per step when the head offset is packed above the column
            auto ld_rec = [&](int64_t e, int2& r, int& ho) {
                if (A.prec) {
                    r = ld_stream_i2(A.prec + e);
                    ho = (int)((uint32_t)r.x >> 21);
                    r.x &= 0x1FFFFF;
                } else {
                    r = ld_stream_i2(A.edges + e);
                    ho = ld_stream_u16(A.hoff + e);
                }
            };
            if (base + lane < E1) ld_rec(base + lane, nrec, nho);
            for (; base < E1; base += 32 * W) {
                const int64_t e = base + lane;
                const int2 rec = nrec;  // records and head offsets prefetched one step ahead
                const int ho = nho;
                if (base + 32 * W + lane < E1) ld_rec(base + 32 * W + lane, nrec, nho);
                const bool due = e < E1 && edge_due_f(__int_as_float(rec.y), ef, ef1);
                const unsigned ballot = __ballot_sync(0xffffffffu, due);
                due_count += __popc(ballot);
                if (due) {
                    const int pos = qn + __popc(ballot & ((1u << lane) - 1u));
                    qh[pos] = ho;
                    qt[pos] = rec.x;
                }
                __syncwarp();
                qn += __popc(ballot);
                if (qn >= 32) {
                    drain(32);
                    qn -= 32;
                    if (lane < qn) { qh[lane] = qh[32 + lane]; qt[lane] = qt[32 + lane]; }
                    __syncwarp();
                }
            }
            if (qn > 0) drain(qn);
            __syncthreads();
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
                const int v = pv0 + i;
                float yo[DIM];
                load_row<DIM>(Yr, v, yo);
#pragma unroll
                for (int c = 0; c < DIM; ++c) {
                    const double upd = (double)(long long)acc[c * vt + i] * (1.0 / 16777216.0);
                    Yw[(int64_t)v * DIM + c] = (float)((double)yo[c] + upd);
                }
            }
            __syncthreads();
        }
        if (epoch + 1 < A.e_end) grid_barrier(A.bar, (unsigned int)(epoch - A.e_begin + 1));
    }
    if (A.positives && lane == 0 && due_count) atomicAdd(A.positives, due_count);
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
template <int DIM, int MC>
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
            const u32x4 rnd = philox_rk((uint32_t)h, (uint32_t)t, (uint32_t)epoch, (uint32_t)blk, A);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (4 * blk + i < MP) vv[4 * blk + i] = (int)__umulhi(pick(rnd, i), nn);
        }
    }
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

template <int DIM, int MC>
__global__ void __launch_bounds__(1024, 1) sgd_flat2_kernel(SgdArgs A)
{
    constexpr int W = 32;
    extern __shared__ __align__(16) unsigned char sgd_smem[];
    const int vt = A.vt;
    uint32_t* acc_lo = reinterpret_cast<uint32_t*>(sgd_smem);              // [DIM][vt]
    int32_t* acc_hi = reinterpret_cast<int32_t*>(acc_lo + (size_t)DIM * vt); // [DIM][vt]
    unsigned long long* acc64 = reinterpret_cast<unsigned long long*>(sgd_smem);  // wide mode: [DIM][vt]
    float* yhead = reinterpret_cast<float*>(acc_hi + (size_t)DIM * vt);     // [vt][DIM]
    int32_t* const qh = reinterpret_cast<int32_t*>(yhead + (size_t)DIM * vt) + (threadIdx.x >> 5) * QCAP;
    int32_t* const qt = qh + W * QCAP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int v_lo = A.bounds[blockIdx.x], v_hi = A.bounds[blockIdx.x + 1];
    const bool wide = *A.max_row > 65535;
    const uint32_t nn = (uint32_t)A.n;
    unsigned long long due_count = 0;
    for (int epoch = A.e_begin; epoch < A.e_end; ++epoch) {
        const int par = (epoch - A.e_begin) & 1;
        const float* Yr = par ? A.Y1 : A.Y0;
        float* Yw = par ? A.Y0 : A.Y1;
        const TermK K = epoch_terms(A, epoch);
        const float ef = (float)epoch, ef1 = (float)(epoch - 1);
        for (int pv0 = v_lo; pv0 < v_hi; pv0 += vt) {
            const int np = min(vt, v_hi - pv0);
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
#pragma unroll
                for (int c = 0; c < DIM; ++c) {
                    if (wide) acc64[c * vt + i] = 0ull;
                    else { acc_lo[c * vt + i] = 0u; acc_hi[c * vt + i] = 0; }
                }
            }
            for (int i = threadIdx.x; i < np * DIM; i += blockDim.x) yhead[i] = __ldcg(Yr + (int64_t)pv0 * DIM + i);
            __syncthreads();
            const int64_t E0 = __ldg(A.indptr + pv0), E1 = __ldg(A.indptr + pv0 + np);
            int qn = 0;
            auto drain = [&](int count) {
                const bool act = lane < count;
                const int hl = act ? qh[lane] : 0;
                const int t = act ? qt[lane] : pv0;
                int qa[DIM];
                edge_terms<DIM, MC>(A, Yr, epoch, nn, K, yhead, pv0, hl, t, act, qa);
                if (act) acc_add<DIM>(acc_lo, acc_hi, acc64, vt, hl, wide, qa);
            };
            int64_t base = E0 + 32 * warp;
            int2 nrec = make_int2(0, 0);
            int nho = 0;
            auto ld_rec = [&](int64_t e, int2& r, int& ho) {
                if (A.prec) {
                    r = ld_stream_i2(A.prec + e);
                    ho = (int)((uint32_t)r.x >> 21);
                    r.x &= 0x1FFFFF;
                } else {
                    r = ld_stream_i2(A.edges + e);
                    ho = ld_stream_u16(A.hoff + e);
                }
            };
            if (base + lane < E1) ld_rec(base + lane, nrec, nho);
            for (; base < E1; base += 32 * W) {
                const int64_t e = base + lane;
                const int2 rec = nrec;
                const int ho = nho;
                if (base + 32 * W + lane < E1) ld_rec(base + 32 * W + lane, nrec, nho);
                const bool due = e < E1 && edge_due_f(__int_as_float(rec.y), ef, ef1);
                const unsigned ballot = __ballot_sync(0xffffffffu, due);
                due_count += __popc(ballot);
                if (due) {
                    const int pos = qn + __popc(ballot & ((1u << lane) - 1u));
                    qh[pos] = ho;
                    qt[pos] = rec.x;
                }
                __syncwarp();
                qn += __popc(ballot);
                if (qn >= 32) {
                    drain(32);
                    qn -= 32;
                    __syncwarp();
                    if (lane < qn) { qh[lane] = qh[32 + lane]; qt[lane] = qt[32 + lane]; }
                    __syncwarp();
                }
            }
            if (qn > 0) drain(qn);
            __syncthreads();
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
                const int v = pv0 + i;
#pragma unroll
                for (int c = 0; c < DIM; ++c) {
                    const long long tot = wide ? (long long)acc64[c * vt + i]
                                               : (long long)acc_hi[c * vt + i] * 65536LL + (long long)acc_lo[c * vt + i];
                    Yw[(int64_t)v * DIM + c] = (float)((double)yhead[i * DIM + c] + (double)tot * (1.0 / 16777216.0));
                }
            }
            __syncthreads();
        }
        if (epoch + 1 < A.e_end) grid_barrier(A.bar, (unsigned int)(epoch - A.e_begin + 1));
    }
    if (A.positives && lane == 0 && due_count) atomicAdd(A.positives, due_count);
}

// ---------------------------------------------------------------- flat3: one piece per CTA
// When every CTA's vertex range fits one piece (<= 2048 vertices; n < 2^21 so that a due edge
// packs into 32 bits as hl << 21 | t, the packed record's own layout) the epoch is split into
// two phases that overlap across the epoch boundary:
//   A(e)  scan: warps claim 32-record steps from a shared counter, evaluate the closed-form
//         schedule (R9) and append the due edges to the CTA's due list for epoch e;
//   B(e)  edge work: warps claim 32-edge batches of that list from a shared counter.
// Only the CTA's last batch of an epoch is partial (the flat kernels leave one partial batch
// per warp per piece), the batches balance the warps dynamically, and a warp that finds no
// batch left goes on with A(e+1) into the other list (the scan does not read positions), so
// the tail of B(e) is filled with the next epoch's scan.  The piece's head rows stay in shared
// memory across epochs: the CTA computes Y_{e+1} of its own vertices itself.  Lists hold up to
// the CTA's record count (every record due), so they never overflow.
template <int DIM, int MC>
__global__ void __launch_bounds__(1024, 1) sgd_flat3_kernel(SgdArgs A)
{
    extern __shared__ __align__(16) unsigned char sgd_smem[];
    const int vt = A.vt;        // >= the largest CTA range
    const int cap = A.list_cap;  // >= the largest CTA record count
    uint32_t* acc_lo = reinterpret_cast<uint32_t*>(sgd_smem);                  // [DIM][vt]
    int32_t* acc_hi = reinterpret_cast<int32_t*>(acc_lo + (size_t)DIM * vt);     // [DIM][vt]
    unsigned long long* acc64 = reinterpret_cast<unsigned long long*>(sgd_smem);  // wide mode: [DIM][vt]
    float* yhead = reinterpret_cast<float*>(acc_hi + (size_t)DIM * vt);         // [vt][DIM]
    uint32_t* list0 = reinterpret_cast<uint32_t*>(yhead + (size_t)DIM * vt);    // [2][cap]
    __shared__ int s_step, s_batch, s_cur[2], s_nlist;
    const int lane = threadIdx.x & 31;
    const int v_lo = A.bounds[blockIdx.x], v_hi = A.bounds[blockIdx.x + 1];
    const int np = v_hi - v_lo;
    const bool wide = *A.max_row > 65535;
    const uint32_t nn = (uint32_t)A.n;
    const int64_t E0 = __ldg(A.indptr + v_lo), E1 = __ldg(A.indptr + v_hi);
    const int n_steps = (int)((E1 - E0 + 31) >> 5);
    unsigned long long due_count = 0;

    // A(e): claim groups of SG 32-record steps until `limit` steps are taken; due edges go to list
    // `buf`.  The next group is claimed before the current one is processed and all SG record
    // loads of a group are issued together (the claim and load latencies overlap the work).
    constexpr int SG = 4;
    auto scan = [&](int e, int buf, int limit) {
        const float ef = (float)e, ef1 = (float)(e - 1);
        uint32_t* list = list0 + (size_t)buf * cap;
        int g = 0;
        if (lane == 0) g = atomicAdd(&s_step, SG);
        g = __shfl_sync(0xffffffffu, g, 0);
        while (g < limit) {
            int gn = 0;
            if (lane == 0) gn = atomicAdd(&s_step, SG);
            int2 rec[SG];
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int64_t ei = E0 + 32 * (int64_t)(g + k) + lane;
                rec[k] = make_int2(0, 0);
                if (g + k < limit && ei < E1) {
                    if (A.prec) {
                        rec[k] = ld_stream_i2(A.prec + ei);
                    } else {
                        rec[k] = ld_stream_i2(A.edges + ei);
                        rec[k].x |= ld_stream_u16(A.hoff + ei) << 21;
                    }
                }
            }
            unsigned ballot[SG];
            int tot = 0;
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int64_t ei = E0 + 32 * (int64_t)(g + k) + lane;
                const bool due = g + k < limit && ei < E1 && edge_due_f(__int_as_float(rec[k].y), ef, ef1);
                ballot[k] = __ballot_sync(0xffffffffu, due);
                tot += __popc(ballot[k]);
            }
            due_count += tot;
            int base = 0;
            if (lane == 0 && tot) base = atomicAdd(&s_cur[buf], tot);
            base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                if ((ballot[k] >> lane) & 1u) list[base + __popc(ballot[k] & ((1u << lane) - 1u))] = (uint32_t)rec[k].x;
                base += __popc(ballot[k]);
            }
            g = __shfl_sync(0xffffffffu, gn, 0);
        }
    };
    // the scan of epoch e + 1 is split: steps [0, split) fill the tail of B(e), steps
    // [split, n_steps) overlap the grid barrier
    int split = n_steps;
    {
        const int pct = A.scan_split_pct;
        split = (int)(((int64_t)n_steps * pct / 100 + SG - 1) / SG * SG);
        if (split > n_steps) split = n_steps;
    }

    for (int i = threadIdx.x; i < np * DIM; i += blockDim.x) yhead[i] = __ldcg(A.Y0 + (int64_t)v_lo * DIM + i);
    for (int i = threadIdx.x; i < np; i += blockDim.x) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            if (wide) acc64[c * vt + i] = 0ull;
            else { acc_lo[c * vt + i] = 0u; acc_hi[c * vt + i] = 0; }
        }
    }
    if (threadIdx.x == 0) { s_step = 0; s_batch = 0; s_cur[0] = 0; s_cur[1] = 0; }
    __syncthreads();
    scan(A.e_begin, A.e_begin & 1, n_steps);
    __syncthreads();
    if (threadIdx.x == 0) { s_nlist = s_cur[A.e_begin & 1]; s_step = 0; }
    __syncthreads();

    for (int epoch = A.e_begin; epoch < A.e_end; ++epoch) {
        const int par = (epoch - A.e_begin) & 1;
        const float* Yr = par ? A.Y1 : A.Y0;
        float* Yw = par ? A.Y0 : A.Y1;
        const TermK K = epoch_terms(A, epoch);
        const int buf = epoch & 1;
        const uint32_t* list = list0 + (size_t)buf * cap;
        const int nl = s_nlist;
        const int nb = (nl + 31) >> 5;
        // B(epoch): warp w takes batches w, w + 32, ... (batch_static, the default: 7 % faster than
        // claiming them from a shared counter, the next one before the current one is processed;
        // a software-pipelined variant that preps the next batch's gathers before the current
        // batch's arithmetic measured slower: 8.3-9.0 vs 8.0-8.1 ms)
        const int warp = threadIdx.x >> 5;
        constexpr int NW = 32;
        int b = warp;
        if (!A.batch_static) {
            if (lane == 0) b = atomicAdd(&s_batch, 1);
            b = __shfl_sync(0xffffffffu, b, 0);
        }
        while (b < nb) {
            int bn = b + NW;
            if (!A.batch_static && lane == 0) bn = atomicAdd(&s_batch, 1);
            // batch b takes list entries b, b + nb, b + 2 nb, ...: the list is in CSR order (equal
            // heads adjacent), so a strided batch has 32 different heads and its shared-memory
            // reductions do not serialise on one address (9.3 -> ~1 wavefront per ATOMS)
            const int j = b + lane * nb;
            const bool act = j < nl;
            const uint32_t ent = act ? list[j] : 0u;
            const int hl = (int)(ent >> 21), t = act ? (int)(ent & 0x1FFFFFu) : v_lo;
            int qa[DIM];
            edge_terms<DIM, MC>(A, Yr, epoch, nn, K, yhead, v_lo, hl, t, act, qa);
            if (act) acc_add<DIM>(acc_lo, acc_hi, acc64, vt, hl, wide, qa);
            b = A.batch_static ? bn : __shfl_sync(0xffffffffu, bn, 0);
        }
        // A(epoch + 1), first part: fills the tail of B(epoch)
        if (epoch + 1 < A.e_end) scan(epoch + 1, buf ^ 1, split);
        __syncthreads();
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
            const int v = v_lo + i;
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                long long tot;
                if (wide) { tot = (long long)acc64[c * vt + i]; acc64[c * vt + i] = 0ull; }
                else {
                    tot = (long long)acc_hi[c * vt + i] * 65536LL + (long long)acc_lo[c * vt + i];
                    acc_lo[c * vt + i] = 0u; acc_hi[c * vt + i] = 0;
                }
                const float y = (float)((double)yhead[i * DIM + c] + (double)tot * (1.0 / 16777216.0));
                yhead[i * DIM + c] = y;
                Yw[(int64_t)v * DIM + c] = y;
            }
        }
        if (epoch + 1 < A.e_end) {
            // split grid barrier: arrive, finish the scan of epoch + 1, then wait
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
                s_step = split;
            }
            __syncthreads();
            scan(epoch + 1, buf ^ 1, n_steps);
            __syncthreads();
            if (threadIdx.x == 0) {
                s_nlist = s_cur[buf ^ 1]; s_cur[buf] = 0; s_batch = 0; s_step = 0;
                const unsigned int target = (unsigned int)(epoch - A.e_begin + 1) * gridDim.x;
                unsigned int v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(A.bar) : "memory");
                } while (v < target);
            }
            __syncthreads();
        } else {
            __syncthreads();
        }
    }
    if (A.positives && lane == 0 && due_count) atomicAdd(A.positives, due_count);
}

// Expected per-epoch cost of vertex v's work in the flat kernel, in units of 1/256 record
// scan: every record is scanned each epoch, record e is due in a fraction ~r_e of the epochs
// (R9) and then costs cdue scans' worth (the gathers and the gradient), plus cvert for the
// vertex's own read-modify-write.
__global__ void vertex_cost_kernel(const int64_t* __restrict__ indptr, const int2* __restrict__ edges, int64_t n,
                                   int cdue, int cvert, int64_t* __restrict__ cost, int* __restrict__ max_row)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int64_t len = indptr[v + 1] - indptr[v];
    atomicMax(max_row, len > INT32_MAX ? INT32_MAX : (int)len);
    int64_t c = 256LL * cvert;
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e)
        c += 256 + (int64_t)(256.0f * (float)cdue * __int_as_float(edges[e].y));
    cost[v] = c;
}

// bounds[b] = first v with P(v) >= P(n) b / G  (P = exclusive prefix of the vertex costs)
__global__ void cost_bounds_kernel(const int64_t* __restrict__ P, int64_t n, int G, int32_t* __restrict__ bounds)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > G) return;
    const double target = (double)P[n] * (double)b / (double)G;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((double)P[mid] < target) lo = mid + 1; else hi = mid;
    }
    bounds[b] = b == G ? (int32_t)n : (int32_t)lo;
}

__global__ void pack_records_kernel(const int2* __restrict__ edges, const uint16_t* __restrict__ hoff, int64_t nnz,
                                    int2* __restrict__ out)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nnz) {
        const int2 r = edges[e];
        out[e] = make_int2((int)((uint32_t)r.x | ((uint32_t)hoff[e] << 21)), r.y);
    }
}

// per CSR entry: head vertex - first vertex of its piece (CTA ranges `bounds`, pieces of vt)
__global__ void hoff_kernel(const int64_t* __restrict__ indptr, int64_t n, const int32_t* __restrict__ bounds, int G,
                            int vt, uint16_t* __restrict__ hoff)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int lo = 0, hi = G - 1;  // last b with bounds[b] <= v
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (bounds[mid] <= v) lo = mid; else hi = mid - 1;
    }
    const uint16_t off = (uint16_t)((v - bounds[lo]) % vt);
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) hoff[e] = off;
}

// Edge-balanced CTA ranges for the persistent SGD kernel: CTA b gets the chunks whose
// cost prefix W(c) = indptr[c VPW] + 2 c VPW (edges + per-vertex work) starts in
// [b W / G, (b + 1) W / G).  bounds[0] = 0, bounds[G] = n_chunks.
__global__ void chunk_bounds_kernel(const int64_t* __restrict__ indptr, int64_t n, int vpw, int n_chunks, int G,
                                    int32_t* __restrict__ bounds)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > G) return;
    auto W = [&](int c) -> double {
        const int64_t v = min((int64_t)c * vpw, n);
        return (double)indptr[v] + 2.0 * (double)v;
    };
    const double target = W(n_chunks) * (double)b / (double)G;
    int lo = 0, hi = n_chunks;  // first c with W(c) >= target
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (W(mid) < target) lo = mid + 1; else hi = mid;
    }
    bounds[b] = b == G ? n_chunks : lo;
}

__global__ void owner_kernel(const int64_t* __restrict__ indptr, int64_t n, uint8_t* __restrict__ owner)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) owner[e] = (uint8_t)(v & 255);
}

__global__ void edge_records_kernel(const int32_t* __restrict__ col, const float* __restrict__ val, int64_t nnz,
                                    const float* __restrict__ w_max, int2* __restrict__ out)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nnz) out[e] = make_int2(col[e], __float_as_int(__fdiv_rn(val[e], *w_max)));
}

__global__ void wmax_kernel(const float* __restrict__ val, int64_t nnz, float* __restrict__ out)
{
    float m = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
        m = fmaxf(m, val[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));  // m >= 0
}

__global__ void wmax_dense_kernel(const float* __restrict__ val, int64_t m, float* __restrict__ out)
{
    float mx = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmaxf(mx, val[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(mx));
}

__global__ void random_init_kernel(int64_t n, int dim, uint32_t k0, uint32_t k1, float* __restrict__ Y)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * dim) return;
    const int64_t v = i / dim;
    const int c = (int)(i - v * dim);
    const u32x4 r = philox4x32_10((uint32_t)v, (uint32_t)c, 0xFFFFFFFFu, 0u, k0, k1);
    const float f = __fmul_rn((float)(r.x >> 8), 1.0f / 16777216.0f);
    Y[i] = __fadd_rn(-10.0f, __fmul_rn(20.0f, f));
}

// ---------------------------------------------------------------- transform SGD (a9)
// Thread per query row; all epochs in one launch (rows are independent: P:138 only
// the query rows move, the training layout is frozen), so there is no inter-epoch
// barrier and no atomics.  Deterministic by construction.
// F64: the per-edge arithmetic of R12/R15 in fp64 with the position stored back in fp32 after
// every update (the oracle's precision reading, R15): coefficients -2ab s^(b-1) /
// (a s^b + 1) and 2 gamma b / ((0.001 + s)(a s^b + 1)) with IEEE pow and division, products and
// sums in the written order without FMA contraction (measured: equal to the oracle bit for bit,
// teacher-forced; ~8x slower on the C5 transform, an exp2(b log2 s) form in fp64 slower still).
// !F64 (the default): the fp32 MUFU form of the fit SGD.
template <int DIM>
__device__ __forceinline__ void transform_update_f64(float (&y)[DIM], const float (&yo)[DIM], bool attractive,
                                                     double a, double b, double gamma, double alpha)
{
    double df[DIM], s = 0.0;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        df[c] = __dsub_rn((double)y[c], (double)yo[c]);
        s = __dadd_rn(s, __dmul_rn(df[c], df[c]));
    }
    double g[DIM];
    if (attractive) {
        double coef = 0.0;
        if (s > 0.0)
            coef = __ddiv_rn(__dmul_rn(__dmul_rn(-2.0 * a, b), pow(s, b - 1.0)), __dadd_rn(__dmul_rn(a, pow(s, b)), 1.0));
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = __dmul_rn(fmin(fmax(__dmul_rn(coef, df[c]), -4.0), 4.0), alpha);
    } else if (s > 0.0) {
        const double cr = __ddiv_rn(__dmul_rn(2.0 * gamma, b),
                                    __dmul_rn(__dadd_rn(0.001, s), __dadd_rn(__dmul_rn(a, pow(s, b)), 1.0)));
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = __dmul_rn(fmin(fmax(__dmul_rn(cr, df[c]), -4.0), 4.0), alpha);
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = __dmul_rn(4.0, alpha);
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) y[c] = __double2float_rn(__dadd_rn((double)y[c], g[c]));
}

template <int DIM, int KMAX, bool F64>
__global__ void __launch_bounds__(128)
transform_sgd_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int64_t nq, int k,
                     const float* __restrict__ Ytr, int64_t ntr, float* __restrict__ Yq, const float* w_max_p,
                     float a, float b, float gamma, float alpha0, int n_epochs_t, int e_begin, int e_end, int m,
                     uint32_t key0, uint32_t key1, int64_t q_offset, int init)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    float y[DIM];
    if (init) {
        // L1-normalised weighted mean of the neighbours' training positions, fp64 in neighbour order
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            double num = 0.0, den = 0.0;
            for (int j = 0; j < k; ++j) {
                const double wj = (double)w[q * k + j];
                num = __dadd_rn(num, __dmul_rn(wj, (double)Ytr[(int64_t)idx[q * k + j] * DIM + c]));
                den = __dadd_rn(den, wj);
            }
            y[c] = den > 0.0 ? (float)__ddiv_rn(num, den) : 0.0f;
        }
    } else {
#pragma unroll
        for (int c = 0; c < DIM; ++c) y[c] = Yq[q * DIM + c];
    }
    const float w_max = *w_max_p;
    float rr[KMAX];
    int32_t tt[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        rr[j] = j < k ? __fdiv_rn(w[q * k + j], w_max) : 0.0f;
        tt[j] = j < k ? idx[q * k + j] : 0;
    }
    const uint32_t head = (uint32_t)(q + q_offset);
    if (e_begin < 1) e_begin = 1;
    if (e_end > n_epochs_t) e_end = n_epochs_t;
    for (int e = e_begin; e < e_end; ++e) {
        const float alpha = __fmul_rn(alpha0, __fsub_rn(1.0f, __fdiv_rn((float)e, (float)n_epochs_t)));
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            if (j >= k || !edge_due(rr[j], e)) continue;
            const int64_t t = tt[j];
            float yt[DIM], g[DIM];
            load_row<DIM>(Ytr, t, yt);
            if constexpr (F64) {
                transform_update_f64<DIM>(y, yt, true, (double)a, (double)b, (double)gamma, (double)alpha);
                u32x4 rnd = {0, 0, 0, 0};
                for (int p = 0; p < m; ++p) {
                    if ((p & 3) == 0) rnd = philox4x32_10(head, (uint32_t)t, (uint32_t)e, (uint32_t)(p >> 2), key0, key1);
                    const uint32_t u = pick(rnd, p & 3);
                    const int64_t v = (int64_t)(((unsigned long long)u * (unsigned long long)ntr) >> 32);
                    float yv[DIM];
                    load_row<DIM>(Ytr, v, yv);
                    transform_update_f64<DIM>(y, yv, false, (double)a, (double)b, (double)gamma, (double)alpha);
                }
                continue;
            }
            float s = 0.0f;
#pragma unroll
            for (int c = 0; c < DIM; ++c) { const float df = y[c] - yt[c]; s = fmaf(df, df, s); }
            float coef = 0.0f;
            if (s > 0.0f) {
                const float sb = pow_b(s, b);
                coef = __fdividef(-2.0f * a * b * __fdividef(sb, s), fmaf(a, sb, 1.0f));
            }
#pragma unroll
            for (int c = 0; c < DIM; ++c) { g[c] = clip4(coef * (y[c] - yt[c])) * alpha; }
#pragma unroll
            for (int c = 0; c < DIM; ++c) y[c] += g[c];
            u32x4 rnd = {0, 0, 0, 0};
            for (int p = 0; p < m; ++p) {
                if ((p & 3) == 0) rnd = philox4x32_10(head, (uint32_t)t, (uint32_t)e, (uint32_t)(p >> 2), key0, key1);
                const uint32_t u = pick(rnd, p & 3);
                const int64_t v = (int64_t)(((unsigned long long)u * (unsigned long long)ntr) >> 32);
                float yv[DIM];
                load_row<DIM>(Ytr, v, yv);
                float s2 = 0.0f;
#pragma unroll
                for (int c = 0; c < DIM; ++c) { const float df = y[c] - yv[c]; s2 = fmaf(df, df, s2); }
                if (s2 > 0.0f) {
                    const float sb = pow_b(s2, b);
                    const float cr = __fdividef(2.0f * gamma * b, (0.001f + s2) * fmaf(a, sb, 1.0f));
#pragma unroll
                    for (int c = 0; c < DIM; ++c) g[c] = clip4(cr * (y[c] - yv[c])) * alpha;
                } else {
#pragma unroll
                    for (int c = 0; c < DIM; ++c) g[c] = 4.0f * alpha;
                }
#pragma unroll
                for (int c = 0; c < DIM; ++c) y[c] += g[c];
            }
        }
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) Yq[q * DIM + c] = y[c];
}

template <int DIM, bool DET, int MC, int VPW, int MINB, int CPB>
umap_status launch_sgd_t(SgdArgs A, cudaStream_t s)
{
    auto kern = sgd_persistent_kernel<DIM, DET, MC, VPW, MINB, CPB>;
    A.n_chunks = (A.n + VPW - 1) / VPW;
    static int max_blocks_dev[64] = {0};  // per device (occupancy is a per-device property)
    int& max_blocks = max_blocks_dev[current_device() & 63];
    if (max_blocks <= 0) {
        int per_sm = 0;
        UMAP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * sgd_warps<MINB>(), 0));
        max_blocks = std::max(1, per_sm) * num_sms();
    }
    const int64_t want = CPB > 0 ? (A.n_chunks + CPB - 1) / CPB : A.n_chunks;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, max_blocks));
    Scratch bounds;
    if (CPB == 0) {
        UMAP_TRY(bounds.alloc(sizeof(int32_t) * (size_t)(grid + 1), s));
        chunk_bounds_kernel<<<ceil_div(grid + 1, 256), 256, 0, s>>>(A.indptr, A.n, VPW, (int)A.n_chunks, grid,
                                                                    bounds.as<int32_t>());
        UMAP_LAUNCH_CHECK("chunk_bounds_kernel");
        A.bounds = bounds.as<int32_t>();
    }
    void* args[] = {&A};
    ProfScope ps(PROF_SGD, s);
    UMAP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(32 * sgd_warps<MINB>()), args, 0, s));
    UMAP_LAUNCH_CHECK("sgd_persistent_kernel");
    return UMAP_OK;
}

// largest CTA vertex range and record count of the flat split (flat3 sizing)
__global__ void cta_extent_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ bounds, int G,
                                  int* __restrict__ out)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= G) return;
    const int lo = bounds[b], hi = bounds[b + 1];
    atomicMax(out, hi - lo);
    const int64_t rec = indptr[hi] - indptr[lo];
    atomicMax(out + 1, rec > INT32_MAX ? INT32_MAX : (int)rec);
}

// ver: 1 = the round-1 flat kernel, 2 = flat2, 3 = flat3 when every CTA range fits one piece
// (else flat2)
template <int DIM, int MC>
umap_status launch_sgd_flat(SgdArgs A, int64_t nnz, cudaStream_t s, int ver)
{
    const int grid = num_sms();  // one CTA of 32 warps per SM (checked against the occupancy below)
    A.n_chunks = A.n;
    Scratch bounds, hoff;
    UMAP_TRY(bounds.alloc(sizeof(int32_t) * (size_t)(grid + 1), s));
    {
        static int cdue = -1, cvert = 2;
        if (cdue < 0) {
            const char* e = getenv("UMAP_SGD_CDUE");  // tuning knob (cost model of the CTA balance)
            cdue = e ? atoi(e) : 16;
        }
        Scratch cost, pre;
        UMAP_TRY(cost.alloc(sizeof(int64_t) * (size_t)A.n, s));
        UMAP_TRY(pre.alloc(sizeof(int64_t) * (size_t)(A.n + 1), s));
        UMAP_CUDA_TRY(cudaMemsetAsync(const_cast<int*>(A.max_row), 0, sizeof(int), s));
        vertex_cost_kernel<<<ceil_div(A.n, 256), 256, 0, s>>>(A.indptr, A.edges, A.n, cdue, cvert, cost.as<int64_t>(),
                                                              const_cast<int*>(A.max_row));
        UMAP_LAUNCH_CHECK("vertex_cost_kernel");
        UMAP_TRY(exclusive_scan<int64_t>(cost.as<int64_t>(), A.n, pre.as<int64_t>(), s));
        cost_bounds_kernel<<<ceil_div(grid + 1, 256), 256, 0, s>>>(pre.as<int64_t>(), A.n, grid, bounds.as<int32_t>());
        UMAP_LAUNCH_CHECK("cost_bounds_kernel");
    }
    constexpr size_t QBYTES = 2 * sizeof(int32_t) * 32 * QCAP;
    const int vt_max = std::min(4096, 65536 / (8 * DIM));
    size_t smem = 0;
    if (ver == 3 && A.n < (1 << 21) && !getenv("UMAP_SGD_VT")) {
        Scratch ext;
        UMAP_TRY(ext.alloc(2 * sizeof(int), s));
        UMAP_CUDA_TRY(cudaMemsetAsync(ext.p, 0, 2 * sizeof(int), s));
        cta_extent_kernel<<<ceil_div(grid, 256), 256, 0, s>>>(A.indptr, bounds.as<int32_t>(), grid, ext.as<int>());
        UMAP_LAUNCH_CHECK("cta_extent_kernel");
        int h[2] = {0, 0};
        UMAP_CUDA_TRY(cudaMemcpyAsync(h, ext.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        UMAP_CUDA_TRY(cudaStreamSynchronize(s));
        const int vt3 = std::max(32, (h[0] + 31) & ~31);
        const int cap = std::max(32, (h[1] + 31) & ~31);
        smem = (size_t)(sizeof(unsigned long long) + sizeof(float)) * DIM * vt3 + 2 * sizeof(uint32_t) * (size_t)cap;
        if (vt3 <= 2048 && smem <= 200 * 1024) {
            A.vt = vt3;
            A.list_cap = cap;
            const char* e = getenv("UMAP_SGD_SCAN_SPLIT");  // tuning knob (% of the scan before the barrier)
            A.scan_split_pct = e ? std::max(0, std::min(100, atoi(e))) : 50;
            const char* bs = getenv("UMAP_SGD_BATCH_STATIC");  // tuning knob (1: measured 7 % faster)
            A.batch_static = bs ? atoi(bs) : 1;
        } else {
            ver = 2;
        }
    } else if (ver == 3) {
        ver = 2;
    }
    if (ver != 3) {
        // piece size: ~1.25x the mean vertices per CTA, between 1024 and 4096 (C2: ~470 per CTA,
        // one piece of <= 1024: the fixed-point sums take 16 KB of shared memory at DIM 2 and the
        // max-L1 carveout leaves the rest of the SM's 256 KB to L1, which caches the gathered
        // positions; C4, 1M rows: ~6800 per CTA, two pieces of 4096 instead of seven of 1024)
        const int64_t want_vt = (A.n * 5 / 4) / std::max(1, num_sms()) + 1;
        A.vt = (int)std::min<int64_t>(vt_max, std::max<int64_t>(std::min(1024, vt_max), want_vt));
        if (const char* e = getenv("UMAP_SGD_VT")) A.vt = std::max(1, std::min(vt_max, atoi(e)));  // test knob: piece size
        // flat2 adds the piece's head rows (4 DIM B per vertex) to the fixed-point sums (8 DIM B)
        const size_t per_v = (sizeof(unsigned long long) + (ver == 2 ? sizeof(float) : 0)) * (size_t)DIM;
        smem = per_v * A.vt + QBYTES;
    }
    const int nt = 1024;
    auto kern = ver == 3 ? sgd_flat3_kernel<DIM, MC>
            : ver == 2 ? sgd_flat2_kernel<DIM, MC> : sgd_flat_kernel<DIM, MC>;
    static PerDeviceOnce attr[4];
    if (attr[ver].first()) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           (int)cudaSharedmemCarveoutMaxL1));
    }
    int per_sm = 0;
    UMAP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
    if (per_sm < 1) {
        set_last_error("SGD kernel does not fit one CTA per SM");
        return UMAP_ERR_CUDA;
    }
    UMAP_TRY(hoff.alloc(sizeof(uint16_t) * (size_t)std::max<int64_t>(nnz, 1), s));
    hoff_kernel<<<ceil_div(A.n, 256), 256, 0, s>>>(A.indptr, A.n, bounds.as<int32_t>(), grid, A.vt, hoff.as<uint16_t>());
    UMAP_LAUNCH_CHECK("hoff_kernel");
    A.bounds = bounds.as<int32_t>();
    A.hoff = hoff.as<uint16_t>();
    Scratch prec;
    A.prec = nullptr;
    if (A.n < (1 << 21) && A.vt <= 2048 && nnz > 0 && !getenv("UMAP_SGD_NO_PACK")) {
        UMAP_TRY(prec.alloc(sizeof(int2) * (size_t)nnz, s));
        pack_records_kernel<<<ceil_div(nnz, 256), 256, 0, s>>>(A.edges, A.hoff, nnz, prec.as<int2>());
        UMAP_LAUNCH_CHECK("pack_records_kernel");
        A.prec = prec.as<int2>();
    }
    void* args[] = {&A};
    ProfScope ps(PROF_SGD, s);
    UMAP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(nt), args, smem, s));
    UMAP_LAUNCH_CHECK(ver == 3 ? "sgd_flat3_kernel" : ver == 2 ? "sgd_flat2_kernel" : "sgd_flat_kernel");
    return UMAP_OK;
}

int sgd_variant()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("UMAP_SGD_VARIANT");  // tuning knob: 0 = default
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <int DIM, bool DET, int MC>
umap_status launch_sgd_m(const SgdArgs& A, cudaStream_t s)
{
    if constexpr (DIM == 2) {  // launch-shape variants (tools/sgd_variants.py) only for the 2-D kernels
        switch (DIM == 2 ? sgd_variant() : 0) {
            case 1: return launch_sgd_t<DIM, DET, MC, 32, 3, 8>(A, s);
            case 2: return launch_sgd_t<DIM, DET, MC, 8, 3, 32>(A, s);
            case 3: return launch_sgd_t<DIM, DET, MC, 16, 3, 32>(A, s);
            case 4: return launch_sgd_t<DIM, DET, MC, 32, 3, 16>(A, s);
            case 5: return launch_sgd_t<DIM, DET, MC, 16, 3, 8>(A, s);
            case 6: return launch_sgd_t<DIM, DET, MC, 16, 4, 4>(A, s);
            case 7: return launch_sgd_t<DIM, DET, MC, 8, 3, 8>(A, s);
            case 8: return launch_sgd_t<DIM, DET, MC, 16, 4, 8>(A, s);
            case 9: return launch_sgd_t<DIM, DET, MC, 16, 3, 16>(A, s);  // the round-1 shape
            case 10: return launch_sgd_t<DIM, DET, MC, 8, 4, 0>(A, s);
            case 11: return launch_sgd_t<DIM, DET, MC, 32, 4, 0>(A, s);
            case 12: return launch_sgd_t<DIM, DET, MC, 16, 3, 0>(A, s);
                case 14: return launch_sgd_t<DIM, DET, MC, 16, 2, 0>(A, s);   // 2 CTAs of 16 warps per SM
            case 15: return launch_sgd_t<DIM, DET, MC, 8, 1, 0>(A, s);
            case 16: return launch_sgd_t<DIM, DET, MC, 16, 4, 0>(A, s);  // 4 CTAs of 8 warps per SM
            default: return launch_sgd_t<DIM, DET, MC, 16, 1, 0>(A, s);  // 1 CTA of 32 warps per SM: measured
                                                                         // best at C2 (tools/sgd_variants.py)
        }
    } else {
        return launch_sgd_t<DIM, DET, MC, 16, 4, 0>(A, s);
    }
}

template <int DIM>
umap_status launch_sgd(const SgdArgs& A, bool det, cudaStream_t s)
{
    const int sv = sgd_variant();
    if constexpr (DIM <= 4) {  // DIM 8, 16: 64 registers per thread spill (persistent chunk kernel)
        if (det && (sv == 0 || sv == 100 || sv == 101)) {
            // 100: the round-1 flat kernel, 101: flat2 (A/B comparisons); default flat3 (else flat2)
            const int ver = sv == 100 ? 1 : sv == 101 ? 2 : 3;
            return A.m == 5 ? launch_sgd_flat<DIM, 5>(A, A.nnz, s, ver) : launch_sgd_flat<DIM, 0>(A, A.nnz, s, ver);
        }
    }
    if (A.m == 5) return det ? launch_sgd_m<DIM, true, 5>(A, s) : launch_sgd_m<DIM, false, 5>(A, s);
    return det ? launch_sgd_m<DIM, true, 0>(A, s) : launch_sgd_m<DIM, false, 0>(A, s);
}

template <int DIM, int KMAX>
umap_status launch_transform_t(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                               float* Yq, const float* wmax, const umap_params* p, int nt, int eb, int ee,
                               int64_t q_offset, int init, cudaStream_t s)
{
    ProfScope ps(PROF_TRANSFORM_SGD, s);
    auto kern = p->transform_precision == 1 ? transform_sgd_kernel<DIM, KMAX, true> : transform_sgd_kernel<DIM, KMAX, false>;
    kern<<<ceil_div(nq, 128), 128, 0, s>>>(
        idx, w, nq, k, Ytr, ntr, Yq, wmax, p->a, p->b, p->repulsion_strength, p->learning_rate, nt, eb, ee,
        p->negative_sample_rate, (uint32_t)p->seed, (uint32_t)(p->seed >> 32), q_offset, init);
    UMAP_LAUNCH_CHECK("transform_sgd_kernel");
    return UMAP_OK;
}

template <int DIM>
umap_status launch_transform(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                             float* Yq, const float* wmax, const umap_params* p, int nt, int eb, int ee,
                             int64_t q_offset, int init, cudaStream_t s)
{
    if (k <= 16) return launch_transform_t<DIM, 16>(idx, w, nq, k, Ytr, ntr, Yq, wmax, p, nt, eb, ee, q_offset, init, s);
    if (k <= 32) return launch_transform_t<DIM, 32>(idx, w, nq, k, Ytr, ntr, Yq, wmax, p, nt, eb, ee, q_offset, init, s);
    return launch_transform_t<DIM, 64>(idx, w, nq, k, Ytr, ntr, Yq, wmax, p, nt, eb, ee, q_offset, init, s);
}

}  // namespace

bool dim_supported(int dim) { return dim == 1 || dim == 2 || dim == 3 || dim == 4 || dim == 8 || dim == 16; }

umap_status random_init(int64_t n, int dim, uint64_t seed, float* Y, cudaStream_t s)
{
    if (n == 0) return UMAP_OK;
    random_init_kernel<<<ceil_div(n * dim, 256), 256, 0, s>>>(n, dim, (uint32_t)seed, (uint32_t)(seed >> 32), Y);
    UMAP_LAUNCH_CHECK("random_init_kernel");
    return UMAP_OK;
}

umap_status compute_wmax(const float* val, int64_t nnz, float* wmax_dev, cudaStream_t s)
{
    UMAP_CUDA_TRY(cudaMemsetAsync(wmax_dev, 0, sizeof(float), s));
    if (nnz == 0) return UMAP_OK;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(nnz, 256), 4LL * num_sms());
    wmax_kernel<<<grid, 256, 0, s>>>(val, nnz, wmax_dev);
    UMAP_LAUNCH_CHECK("wmax_kernel");
    return UMAP_OK;
}

// Run epochs [e_begin, e_end) on Y (device, in place).  nnz = indptr[n].
umap_status optimize_layout(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, int64_t nnz,
                            float* Y, const umap_params* p, int e_begin, int e_end, int64_t* positives_host,
                            cudaStream_t s)
{
    const int dim = p->n_components;
    if (!dim_supported(dim)) {
        set_last_error("n_components must be one of 1,2,3,4,8,16");
        return UMAP_ERR_UNSUPPORTED;
    }
    if (e_begin < 1) e_begin = 1;
    if (e_end > p->n_epochs) e_end = p->n_epochs;
    if (positives_host) *positives_host = 0;
    if (e_begin >= e_end || n == 0) return UMAP_OK;
    if (n >= (int64_t)INT32_MAX) { set_last_error("n must be < 2^31"); return UMAP_ERR_INVALID_ARGUMENT; }
    Scratch wmax, other, counter, edges, bar;
    UMAP_TRY(wmax.alloc(sizeof(float), s));
    UMAP_TRY(compute_wmax(val, nnz, wmax.as<float>(), s));
    // a6: per-entry record {col, r = w / w_max}, built once per call
    UMAP_TRY(edges.alloc(sizeof(int2) * (size_t)std::max<int64_t>(nnz, 1), s));
    if (nnz > 0) {
        edge_records_kernel<<<ceil_div(nnz, 256), 256, 0, s>>>(col, val, nnz, wmax.as<float>(), edges.as<int2>());
        UMAP_LAUNCH_CHECK("edge_records_kernel");
    }
    Scratch owner;
    UMAP_TRY(owner.alloc((size_t)std::max<int64_t>(nnz, 1), s));
    owner_kernel<<<ceil_div(n, 256), 256, 0, s>>>(indptr, n, owner.as<uint8_t>());
    UMAP_LAUNCH_CHECK("owner_kernel");
    UMAP_TRY(counter.alloc(sizeof(unsigned long long), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), s));
    UMAP_TRY(bar.alloc(BAR_WORDS * sizeof(unsigned int), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(bar.p, 0, BAR_WORDS * sizeof(unsigned int), s));
    const bool det = p->sgd_mode == UMAP_SGD_DETERMINISTIC;
    if (det) {
        UMAP_TRY(other.alloc(sizeof(float) * (size_t)n * dim, s));
    }
    SgdArgs A{};
    A.indptr = indptr; A.edges = edges.as<int2>(); A.n = n; A.nnz = nnz;
    A.Y0 = Y; A.Y1 = det ? other.as<float>() : Y;
    A.a = p->a; A.b = p->b; A.gamma = p->repulsion_strength; A.alpha0 = p->learning_rate;
    A.n_epochs = p->n_epochs; A.e_begin = e_begin; A.e_end = e_end; A.m = p->negative_sample_rate;
    A.key0 = (uint32_t)p->seed; A.key1 = (uint32_t)(p->seed >> 32);
    for (int r = 0; r < 10; ++r) {
        A.rk0[r] = A.key0 + (uint32_t)r * 0x9E3779B9u;
        A.rk1[r] = A.key1 + (uint32_t)r * 0xBB67AE85u;
    }
    Scratch maxrow;
    UMAP_TRY(maxrow.alloc(sizeof(int), s));
    A.max_row = maxrow.as<int>();
    A.positives = counter.as<unsigned long long>();
    A.bar = bar.as<unsigned int>();
    A.owner = owner.as<uint8_t>();
    {
        const char* dbg = unsafe_env("UMAP_SGD_DEBUG");
        A.debug = dbg ? atoi(dbg) : 0;
    }
    umap_status st;
    switch (dim) {
        case 1: st = launch_sgd<1>(A, det, s); break;
        case 2: st = launch_sgd<2>(A, det, s); break;
        case 3: st = launch_sgd<3>(A, det, s); break;
        case 4: st = launch_sgd<4>(A, det, s); break;
        case 8: st = launch_sgd<8>(A, det, s); break;
        default: st = launch_sgd<16>(A, det, s); break;
    }
    if (st != UMAP_OK) return st;
    if (det && ((e_end - e_begin) & 1)) {  // odd number of epochs: the result sits in the partner buffer
        UMAP_CUDA_TRY(cudaMemcpyAsync(Y, other.p, sizeof(float) * (size_t)n * dim, cudaMemcpyDeviceToDevice, s));
    }
    if (positives_host) {
        unsigned long long c = 0;
        UMAP_CUDA_TRY(cudaMemcpyAsync(&c, counter.p, sizeof(c), cudaMemcpyDeviceToHost, s));
        UMAP_CUDA_TRY(cudaStreamSynchronize(s));
        *positives_host = (int64_t)c;
    }
    return UMAP_OK;
}

umap_status transform_optimize(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                               float* Yq, const umap_params* p, int n_epochs_t, int e_begin, int e_end,
                               int64_t q_offset, int init, cudaStream_t s)
{
    const int dim = p->n_components;
    if (!dim_supported(dim)) {
        set_last_error("n_components must be one of 1,2,3,4,8,16");
        return UMAP_ERR_UNSUPPORTED;
    }
    if (nq == 0) return UMAP_OK;
    Scratch wmax;
    UMAP_TRY(wmax.alloc(sizeof(float), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(wmax.p, 0, sizeof(float), s));
    const int64_t m = nq * (int64_t)k;
    wmax_dense_kernel<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), 4LL * num_sms()), 256, 0, s>>>(w, m, wmax.as<float>());
    UMAP_LAUNCH_CHECK("wmax_dense_kernel");
    switch (dim) {
        case 1: return launch_transform<1>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 2: return launch_transform<2>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 3: return launch_transform<3>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 4: return launch_transform<4>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        case 8: return launch_transform<8>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
        default: return launch_transform<16>(idx, w, nq, k, Ytr, ntr, Yq, wmax.as<float>(), p, n_epochs_t, e_begin, e_end, q_offset, init, s);
    }
}

}  // namespace umapb200
