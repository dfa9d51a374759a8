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

#include "bulk.cuh"
#include "sgd_common.cuh"

namespace umapb200 {

template <class Tin> umap_status exclusive_scan(const Tin* in, int64_t n, int64_t* out, cudaStream_t s);  // graph.cu
using namespace sgdk;
namespace {

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
template <int DIM, int MC, int XDBG = 0>
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
        const int nb = (A.debug & 2) ? 0 : (nl + 31) >> 5;  // debug 2: scan + barriers only (timing)
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
            edge_terms<DIM, MC, XDBG>(A, Yr, epoch, nn, K, yhead, v_lo, hl, t, act, qa);
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

// ---------------------------------------------------------------- flat5: records in shared memory
// flat3 with the CTA's records resident in shared memory for all epochs (SoA: r fp32, packed
// hl << 21 | t), so the per-epoch scan (A) reads shared memory instead of streaming 8 bytes per
// record from L2 every epoch; the due lists hold 16-bit record indices.  Same edge work, batches
// and fixed-point sums as flat3 (R13: Y is bit-identical).
// HOG: the Hogwild mode (R14) on the same structure: positions in place (Y0 == Y1), each due edge
// reads the live head, tail and sample rows (L1-cached: staleness bounded to one epoch by the grid
// barrier's acquire), moves its head through the attractive and the m repulsive updates in
// registers and pushes -g_att to the tail and the head's total delta with fp32 vector atomics
// (process_edge, as the persistent Hogwild kernel); no accumulators, no end-of-epoch vertex pass.
template <int DIM, int MC, int NT = 1024, int MINB = 1, bool HOG = false>
__global__ void __launch_bounds__(NT, MINB) sgd_flat5_kernel(SgdArgs A)
{
    extern __shared__ __align__(16) unsigned char sgd_smem[];
    const int vt = A.vt;         // >= the largest CTA range (multiple of 32)
    const int cap = A.list_cap;  // >= the largest CTA record count (multiple of 32)
    uint32_t* acc_lo = reinterpret_cast<uint32_t*>(sgd_smem);                  // [DIM][vt]
    int32_t* acc_hi = reinterpret_cast<int32_t*>(acc_lo + (size_t)DIM * vt);     // [DIM][vt]
    unsigned long long* acc64 = reinterpret_cast<unsigned long long*>(sgd_smem);  // wide mode: [DIM][vt]
    float* yhead = reinterpret_cast<float*>(acc_hi + (size_t)DIM * vt);         // [vt][DIM]
    float* rr = yhead + (size_t)DIM * vt;                                       // [cap] r
    uint32_t* rx = reinterpret_cast<uint32_t*>(rr + cap);                       // [cap] hl << 21 | t
    uint16_t* list0 = reinterpret_cast<uint16_t*>(rx + cap);                    // [2][cap] record indices
    __shared__ int s_step, s_cur[2], s_nlist;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int v_lo = A.bounds[blockIdx.x], v_hi = A.bounds[blockIdx.x + 1];
    const int np = v_hi - v_lo;
    const bool wide = *A.max_row > 65535;
    const uint32_t nn = (uint32_t)A.n;
    const int64_t E0 = __ldg(A.indptr + v_lo), E1 = __ldg(A.indptr + v_hi);
    const int R = (int)(E1 - E0);
    const int n_steps = (R + 31) >> 5;
    unsigned long long due_count = 0;

    constexpr int SG = 8;
    auto scan = [&](int e, int buf, int limit) {
        const float ef = (float)e, ef1 = (float)(e - 1);
        uint16_t* list = list0 + (size_t)buf * cap;
        int g = 0;
        if (lane == 0) g = atomicAdd(&s_step, SG);
        g = __shfl_sync(0xffffffffu, g, 0);
        while (g < limit) {
            int gn = 0;
            if (lane == 0) gn = atomicAdd(&s_step, SG);
            unsigned ballot[SG];
            int tot = 0;
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int i = 32 * (g + k) + lane;
                const bool due = g + k < limit && i < R && edge_due_f(rr[i], ef, ef1);
                ballot[k] = __ballot_sync(0xffffffffu, due);
                tot += __popc(ballot[k]);
            }
            due_count += tot;
            int base = 0;
            if (lane == 0 && tot) base = atomicAdd(&s_cur[buf], tot);
            base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                if ((ballot[k] >> lane) & 1u) list[base + __popc(ballot[k] & ((1u << lane) - 1u))] = (uint16_t)(32 * (g + k) + lane);
                base += __popc(ballot[k]);
            }
            g = __shfl_sync(0xffffffffu, gn, 0);
        }
    };
    int split = n_steps;
    {
        const int pct = A.scan_split_pct;
        split = (int)(((int64_t)n_steps * pct / 100 + SG - 1) / SG * SG);
        if (split > n_steps) split = n_steps;
    }
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
        int2 rec;
        if (A.prec) {
            rec = ld_stream_i2(A.prec + E0 + i);
        } else {
            rec = ld_stream_i2(A.edges + E0 + i);
            rec.x |= ld_stream_u16(A.hoff + E0 + i) << 21;
        }
        rr[i] = __int_as_float(rec.y);
        rx[i] = (uint32_t)rec.x;
    }
    if (!HOG) {
        for (int i = threadIdx.x; i < np * DIM; i += blockDim.x) yhead[i] = __ldcg(A.Y0 + (int64_t)v_lo * DIM + i);
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                if (wide) acc64[c * vt + i] = 0ull;
                else { acc_lo[c * vt + i] = 0u; acc_hi[c * vt + i] = 0; }
            }
        }
    }
    if (threadIdx.x == 0) { s_step = 0; s_cur[0] = 0; s_cur[1] = 0; }
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
        const uint16_t* list = list0 + (size_t)buf * cap;
        const int nl = s_nlist;
        const int nb = (nl + 31) >> 5;
        // static strided batches (flat3): warp w takes batches w, w + NT / 32, ...
        const float alpha = HOG ? __fmul_rn(A.alpha0, __fsub_rn(1.0f, __fdiv_rn((float)epoch, (float)A.n_epochs))) : 0.0f;
        for (int b = warp; b < nb; b += NT / 32) {
            const int j = b + lane * nb;
            const bool act = j < nl;
            const uint32_t ent = act ? rx[list[j]] : 0u;
            const int hl = (int)(ent >> 21), t = act ? (int)(ent & 0x1FFFFFu) : v_lo;
            int qa[DIM];
            if constexpr (HOG) {
                if (act) process_edge<DIM, false, MC, true>(A, Yr, Yw, epoch, alpha, v_lo + hl, t, qa);
            } else {
                edge_terms<DIM, MC>(A, Yr, epoch, nn, K, yhead, v_lo, hl, t, act, qa);
                if (act) acc_add<DIM>(acc_lo, acc_hi, acc64, vt, hl, wide, qa);
            }
        }
        if (epoch + 1 < A.e_end) scan(epoch + 1, buf ^ 1, split);
        __syncthreads();
        if (!HOG) {
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
        }
        if (epoch + 1 < A.e_end) {
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
                s_step = split;
            }
            __syncthreads();
            scan(epoch + 1, buf ^ 1, n_steps);
            __syncthreads();
            if (threadIdx.x == 0) {
                s_nlist = s_cur[buf ^ 1]; s_cur[buf] = 0; s_step = 0;
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

// ---------------------------------------------------------------- flat4: materialised schedule
// The schedule (R9) does not depend on the positions, so every CTA's due lists are built before
// the launch and the epoch loop streams them instead of scanning every record every epoch
// (flat3's scan: ~1 ms of the 7.4 ms at C2, tools/sgd_decomp.py; the records cost 8 bytes of
// L2->SM traffic per record per epoch, a due entry 4 bytes per due edge).
//
// Layout: a CTA range's records are cut into slots of SK_SLOT consecutive records (CSR order);
// slot s owns a region of the list array, epoch-major: for each epoch its due records (packed
// hl << 21 | t) in CSR order, padded with SK_PAD entries to a multiple of 4 (16-byte bulk copies),
// and pcnt[b][i][s] = that padded count.  The region bound is exact: the records due in epochs
// [e_begin, e_end) number at most floor(fl((e_end - 1) r)) - floor(fl((e_begin - 1) r)) per record
// (fl(e r) is monotone in e; the due test counts the strict increases of its floor).
//
// sgd_flat4_kernel: per epoch, warp 0 fetches the CTA's slot segments of epoch e + 2 into one
// shared-memory list with the TMA bulk-copy engine (one cp.async.bulk per slot, completion on the
// buffer's mbarrier) while epochs e and e + 1 run; the padded counts of epoch e + 2 are fetched by
// LDGSTS at the start of epoch e.  Edge work, batches and fixed-point sums are flat3's (R13: Y is
// bit-identical); padding entries are inactive lanes.
// records per slot: SK_SLOT_MIN x 2^j (tuning knob UMAP_SGD_SLOT; one warp holds a slot's records in registers)
constexpr int SK_SLOT_MIN = 256;
constexpr int SK_MAXSLOTS = 128;    // slots per CTA range handled by flat4 (C2: 42)
constexpr uint32_t SK_PAD = 0xFFFFFFFFu;

// per CTA range b: its slot count
__global__ void sched_slots_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ bounds, int G,
                                   int slot, int32_t* __restrict__ nslots)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= G) return;
    const int64_t R = indptr[bounds[b + 1]] - indptr[bounds[b]];
    nslots[b] = (int32_t)((R + slot - 1) / slot);
}

// per slot (one warp): its CTA range (slot_b) and the region bound (records' due epochs + padding)
__global__ void sched_bound_kernel(const int2* __restrict__ prec, const int64_t* __restrict__ indptr,
                                   const int32_t* __restrict__ bounds, int G, const int64_t* __restrict__ slot_base,
                                   int64_t S, int slot, int e_begin, int e_end, int32_t* __restrict__ slot_b,
                                   int64_t* __restrict__ bound)
{
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= S) return;
    int lo = 0, hi = G - 1;  // last b with slot_base[b] <= gw
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (slot_base[mid] <= gw) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int64_t E0 = indptr[bounds[b]] + (gw - slot_base[b]) * slot;
    const int64_t E1 = min(indptr[bounds[b + 1]], E0 + slot);
    const float ea = (float)(e_begin - 1), ez = (float)(e_end - 1);
    int64_t c = 0;
    for (int64_t e = E0 + lane; e < E1; e += 32) {
        const float r = __int_as_float(prec[e].y);
        c += (int64_t)(floorf(__fmul_rn(ez, r)) - floorf(__fmul_rn(ea, r)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) {
        slot_b[gw] = b;
        bound[gw] = (c + 3LL * (e_end - e_begin) + 3) & ~3LL;  // regions start 16-byte aligned
    }
}

// one warp per slot of 32 MS records: the due lists of every epoch into the slot's region,
// pcnt[b][i][s] = padded count.  Due test: floor(fl(e r)) > floor(fl((e - 1) r))  <=>
// floor(fl(e r)) > fl((e - 1) r).  Branch-free: ballot, prefix popc, predicated store.
template <int MS>
__global__ void __launch_bounds__(256)
sched_fill_kernel(const int2* __restrict__ prec, const int64_t* __restrict__ indptr, const int32_t* __restrict__ bounds,
                  const int64_t* __restrict__ slot_base, const int32_t* __restrict__ slot_b, int64_t S, int e_begin,
                  int NE, const int64_t* __restrict__ region, int32_t* __restrict__ pcnt, uint32_t* __restrict__ out)
{
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= S) return;
    const int b = slot_b[gw];
    const int64_t sb = slot_base[b];
    const int local = (int)(gw - sb), ns = (int)(slot_base[b + 1] - sb);
    const int64_t E0 = indptr[bounds[b]] + (int64_t)local * (32 * MS);
    const int64_t E1 = min(indptr[bounds[b + 1]], E0 + 32 * MS);
    float r[MS], pv[MS];
    uint32_t x[MS];
    const float ef0 = (float)(e_begin - 1);
#pragma unroll
    for (int k = 0; k < MS; ++k) {
        const int64_t e = E0 + 32 * k + lane;
        const int2 rc = e < E1 ? prec[e] : make_int2(0, 0);  // r = 0: never due
        r[k] = __int_as_float(rc.y);
        x[k] = (uint32_t)rc.x;
        pv[k] = __fmul_rn(ef0, r[k]);
    }
    uint32_t* o = out + region[gw];
    int32_t* pc = pcnt + (int64_t)NE * sb + local;
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (int i = 0; i < NE; ++i) {
        const float ef = (float)(e_begin + i);
        int c = 0;
#pragma unroll
        for (int k = 0; k < MS; ++k) {
            const float xe = __fmul_rn(ef, r[k]);
            const bool due = floorf(xe) > pv[k];
            pv[k] = xe;
            const unsigned bal = __ballot_sync(0xffffffffu, due);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p st.global.u32 [%0], %1;\n\t}"
                         ::"l"(o + c + __popc(bal & lt)), "r"(x[k]), "r"((int)due) : "memory");
            c += __popc(bal);
        }
        const int pad = (4 - (c & 3)) & 3;
        if (lane < pad) o[c + lane] = SK_PAD;
        c += pad;
        if (lane == 0) pc[(int64_t)i * ns] = c;
        o += c;
    }
}

template <int DIM, int MC>
__global__ void __launch_bounds__(1024, 1) sgd_flat4_kernel(SgdArgs A)
{
    extern __shared__ __align__(16) unsigned char sgd_smem[];
    const int vt = A.vt;         // >= the largest CTA range, multiple of 32
    const int cap = A.list_cap;  // >= the largest padded epoch list, multiple of 32
    uint32_t* acc_lo = reinterpret_cast<uint32_t*>(sgd_smem);                  // [DIM][vt]
    int32_t* acc_hi = reinterpret_cast<int32_t*>(acc_lo + (size_t)DIM * vt);     // [DIM][vt]
    unsigned long long* acc64 = reinterpret_cast<unsigned long long*>(sgd_smem);  // wide mode: [DIM][vt]
    float* yhead = reinterpret_cast<float*>(acc_hi + (size_t)DIM * vt);         // [vt][DIM]
    uint32_t* list0 = reinterpret_cast<uint32_t*>(yhead + (size_t)DIM * vt);    // [2][cap], 16-byte aligned
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ int64_t s_src[SK_MAXSLOTS];  // next unread entry of each slot's region
    __shared__ int32_t s_pc[2][SK_MAXSLOTS];
    __shared__ int s_nl[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int v_lo = A.bounds[blockIdx.x], v_hi = A.bounds[blockIdx.x + 1];
    const int np = v_hi - v_lo;
    const bool wide = *A.max_row > 65535;
    const uint32_t nn = (uint32_t)A.n;
    const int NE = A.e_end - A.e_begin;
    const int64_t sb = A.slot_base[blockIdx.x];
    const int ns = (int)(A.slot_base[blockIdx.x + 1] - sb);
    const int32_t* pcb = A.sched_pcnt + (int64_t)NE * sb;
    const uint32_t bar0 = smem_u32(&s_bar[0]);
    // warp 0: LDGSTS of the padded counts of epoch index i into s_pc[i & 1]
    auto fetch_counts = [&](int i) {
        for (int s = lane; s < ns; s += 32) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&s_pc[i & 1][s])),
                         "l"(pcb + (int64_t)i * ns + s) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // warp 0: bulk copies of the slot segments of epoch index i into list buffer i & 1 (counts in
    // s_pc[i & 1], complete: cp.async.wait_all + __syncwarp by the caller)
    auto fetch_lists = [&](int i) {
        const int bi = i & 1;
        const uint32_t bar = bar0 + 8u * (uint32_t)bi;
        const uint32_t dst0 = smem_u32(list0 + (size_t)bi * cap);
        int base = 0;
        int pcs[SK_MAXSLOTS / 32], offs[SK_MAXSLOTS / 32];
#pragma unroll
        for (int q = 0; q < SK_MAXSLOTS / 32; ++q) {
            const int s = lane + 32 * q;
            const int c = s < ns ? s_pc[bi][s] : 0;
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            pcs[q] = c;
            offs[q] = base + incl - c;
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            s_nl[bi] = base;
            mbar_expect_tx(bar, (uint32_t)base * 4u);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < SK_MAXSLOTS / 32; ++q) {
            const int s = lane + 32 * q;
            if (pcs[q] > 0) {
                bulk_g2s(dst0 + (uint32_t)offs[q] * 4u, A.sched + s_src[s], (uint32_t)pcs[q] * 4u, bar);
                s_src[s] += pcs[q];
            }
        }
    };
    if (warp == 0) {
        for (int s = lane; s < ns; s += 32) s_src[s] = A.sched_region[sb + s];
        if (lane == 0) {
            mbar_init(bar0, 1);
            mbar_init(bar0 + 8, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        fetch_counts(0);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        fetch_lists(0);
        if (NE > 1) fetch_counts(1);
    }
    for (int i = threadIdx.x; i < np * DIM; i += blockDim.x) yhead[i] = __ldcg(A.Y0 + (int64_t)v_lo * DIM + i);
    for (int i = threadIdx.x; i < np; i += blockDim.x) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            if (wide) acc64[c * vt + i] = 0ull;
            else { acc_lo[c * vt + i] = 0u; acc_hi[c * vt + i] = 0; }
        }
    }
    __syncthreads();
    unsigned long long due_count = 0;
    for (int ie = 0; ie < NE; ++ie) {
        const int epoch = A.e_begin + ie;
        const float* Yr = (ie & 1) ? A.Y1 : A.Y0;
        float* Yw = (ie & 1) ? A.Y0 : A.Y1;
        const TermK K = epoch_terms(A, epoch);
        const uint32_t* list = list0 + (size_t)(ie & 1) * cap;
        const int nl = s_nl[ie & 1];
        const int nb = (nl + 31) >> 5;
        if (warp == 0 && ie + 1 < NE) {
            // list buffer (ie + 1) & 1 was last read in epoch ie - 1 (grid barrier since): order
            // those generic reads before the async-proxy refill; its counts arrived by LDGSTS
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
            fetch_lists(ie + 1);
            if (ie + 2 < NE) fetch_counts(ie + 2);  // s_pc[ie & 1] was consumed by fetch_lists(ie)
        }
        mbar_wait(bar0 + 8u * (uint32_t)(ie & 1), (uint32_t)(ie >> 1) & 1u);
        // warp w takes the strided batches 31 - w, 63 - w, ...: batch b = entries b, b + nb, ...
        // (the slots' CSR order: 32 different heads per batch, flat3); padding entries are
        // inactive; warp 0, which issues the fetches, gets the last batch only when nb % 32 == 0
        for (int b = 31 - warp; b < nb; b += 32) {
            const int j = b + lane * nb;
            const uint32_t ent = j < nl ? list[j] : SK_PAD;
            const bool act = ent != SK_PAD;
            due_count += act;
            const int hl = (int)(ent >> 21), t = act ? (int)(ent & 0x1FFFFFu) : v_lo;
            int qa[DIM];
            edge_terms<DIM, MC>(A, Yr, epoch, nn, K, yhead, v_lo, act ? hl : 0, t, act, qa);
            if (act) acc_add<DIM>(acc_lo, acc_hi, acc64, vt, hl, wide, qa);
        }
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
        if (ie + 1 < NE) grid_barrier(A.bar, (unsigned int)(ie + 1));
        else __syncthreads();
    }
    if (A.positives && due_count) atomicAdd(A.positives, due_count);
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

// tuning knob UMAP_SGD_SCHED: 0 = flat3 (records streamed from L2 every epoch), 1 = flat4
// (materialised schedule), 2 = flat5 (records in shared memory; default)
int sgd_sched_mode()
{
    const char* e = getenv("UMAP_SGD_SCHED");
    return e ? atoi(e) : 2;
}
bool sgd_sched_enabled() { return sgd_sched_mode() == 1; }

// ver: 1 = the round-1 flat kernel, 2 = flat2, 3 = flat3 when every CTA range fits one piece
// (else flat2)
template <int DIM, int MC>
umap_status launch_sgd_flat(SgdArgs A, int64_t nnz, cudaStream_t s, int ver, int cps_req, bool* retry, bool hog = false)
{
    // one CTA of 32 warps per SM, or (flat5, cps_req = 2, the default) two CTAs of 18 warps per SM:
    // 36 warps at <= 56 registers carry 1152 due edges per round instead of 1024 (C2: ~3,090 due
    // edges per SM per epoch take 3 rounds on every SM instead of 4 on about half of them; the
    // grid barrier waits for the slowest).  *retry: the flat5 two-CTA form does not fit, call
    // again with cps_req = 1.
    const int cps = (ver == 3 && sgd_sched_mode() == 2 && cps_req == 2) ? 2 : 1;
    const int grid = num_sms() * cps;
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
    int nt = 1024;
    auto kern = ver == 3 ? sgd_flat3_kernel<DIM, MC>
            : ver == 2 ? sgd_flat2_kernel<DIM, MC> : sgd_flat_kernel<DIM, MC>;
    if constexpr (DIM == 2 && MC == 5) {  // timing-decomposition variants (unsafe experiments only)
        if (ver == 3) {
            switch (A.debug & ~3) {
                case 4: kern = sgd_flat3_kernel<DIM, MC, 4>; break;
                case 8: kern = sgd_flat3_kernel<DIM, MC, 8>; break;
                case 12: kern = sgd_flat3_kernel<DIM, MC, 12>; break;
                case 16: kern = sgd_flat3_kernel<DIM, MC, 16>; break;
                case 28: kern = sgd_flat3_kernel<DIM, MC, 28>; break;
                default: break;
            }
        }
    }
    static PerDeviceOnce attr[5];
    if ((A.debug & ~3) != 0) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           (int)cudaSharedmemCarveoutMaxL1));
    }
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
    // flat4: materialise the schedule (R9) when the packed records exist, every CTA range has at
    // most SK_MAXSLOTS slots and the lists fit in half the free device memory (C2: 0.9 GB); else
    // flat3's in-kernel scan
    Scratch sched, nsl, sbase, slotb, sbound, sregion, pcnt;
    int slot = SK_SLOT_MIN * 2;
    if (const char* e = getenv("UMAP_SGD_SLOT")) slot = atoi(e) >= 1024 ? 1024 : atoi(e) >= 512 ? 512 : 256;  // tuning knob
    if (ver == 3 && A.prec && sgd_sched_enabled() && (int64_t)A.list_cap <= (int64_t)SK_MAXSLOTS * slot) {
        const int NE = A.e_end - A.e_begin;
        UMAP_TRY(nsl.alloc(sizeof(int32_t) * (size_t)grid, s));
        UMAP_TRY(sbase.alloc(sizeof(int64_t) * (size_t)(grid + 1), s));
        int64_t S = 0, total = 0;
        {
            ProfScope pc(PROF_SGD_SCHED, s);
            sched_slots_kernel<<<ceil_div(grid, 256), 256, 0, s>>>(A.indptr, bounds.as<int32_t>(), grid, slot,
                                                                  nsl.as<int32_t>());
            UMAP_LAUNCH_CHECK("sched_slots_kernel");
            UMAP_TRY(exclusive_scan<int32_t>(nsl.as<int32_t>(), grid, sbase.as<int64_t>(), s));
        }
        UMAP_CUDA_TRY(cudaMemcpyAsync(&S, sbase.as<int64_t>() + grid, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        UMAP_CUDA_TRY(cudaStreamSynchronize(s));
        UMAP_TRY(slotb.alloc(sizeof(int32_t) * (size_t)S, s));
        UMAP_TRY(sbound.alloc(sizeof(int64_t) * (size_t)S, s));
        UMAP_TRY(sregion.alloc(sizeof(int64_t) * (size_t)(S + 1), s));
        {
            ProfScope pc(PROF_SGD_SCHED, s);
            sched_bound_kernel<<<ceil_div(S * 32, 256), 256, 0, s>>>(A.prec, A.indptr, bounds.as<int32_t>(), grid,
                                                                    sbase.as<int64_t>(), S, slot, A.e_begin, A.e_end,
                                                                    slotb.as<int32_t>(), sbound.as<int64_t>());
            UMAP_LAUNCH_CHECK("sched_bound_kernel");
            UMAP_TRY(exclusive_scan<int64_t>(sbound.as<int64_t>(), S, sregion.as<int64_t>(), s));
        }
        UMAP_CUDA_TRY(cudaMemcpyAsync(&total, sregion.as<int64_t>() + S, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        UMAP_CUDA_TRY(cudaStreamSynchronize(s));
        size_t free_b = 0, total_b = 0;
        UMAP_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
        const size_t smem4 = smem + 2 * sizeof(uint32_t) * (size_t)(3 * SK_MAXSLOTS + 32);
        if ((size_t)total * 4 <= free_b / 2 && smem4 <= 200 * 1024) {
            UMAP_TRY(sched.alloc(sizeof(uint32_t) * (size_t)total, s));
            UMAP_TRY(pcnt.alloc(sizeof(int32_t) * (size_t)S * NE, s));
            ProfScope pf(PROF_SGD_SCHED, s);
            auto fill = slot == 1024 ? sched_fill_kernel<32> : slot == 512 ? sched_fill_kernel<16> : sched_fill_kernel<8>;
            fill<<<ceil_div(S * 32, 256), 256, 0, s>>>(A.prec, A.indptr, bounds.as<int32_t>(), sbase.as<int64_t>(),
                                                      slotb.as<int32_t>(), S, A.e_begin, NE, sregion.as<int64_t>(),
                                                      pcnt.as<int32_t>(), sched.as<uint32_t>());
            UMAP_LAUNCH_CHECK("sched_fill_kernel");
            A.sched = sched.as<uint32_t>();
            A.slot_base = sbase.as<int64_t>();
            A.sched_region = sregion.as<int64_t>();
            A.sched_pcnt = pcnt.as<int32_t>();
            // a padded epoch list holds at most the CTA's records + 3 per slot
            A.list_cap = (A.list_cap + 3 * SK_MAXSLOTS + 31) & ~31;
            smem = smem4;
            ver = 4;
            kern = sgd_flat4_kernel<DIM, MC>;
            if (attr[4].first()) {
                UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                   (int)cudaSharedmemCarveoutMaxL1));
            }
        }
    }
    if (ver == 3 && sgd_sched_mode() == 2) {
        // flat5: records (8 B) and 16-bit list entries (2 x 2 B) per record instead of 2 x 4 B
        const size_t smem5 = (size_t)(sizeof(unsigned long long) + sizeof(float)) * DIM * A.vt +
                             (size_t)A.list_cap * (sizeof(float) + sizeof(uint32_t) + 2 * sizeof(uint16_t));
        if (smem5 <= 200 * 1024 && A.list_cap <= 65535) {
            smem = smem5;
            ver = 5;
            kern = hog ? (cps == 2 ? sgd_flat5_kernel<DIM, MC, 576, 2, true> : sgd_flat5_kernel<DIM, MC, 1024, 1, true>)
                       : (cps == 2 ? sgd_flat5_kernel<DIM, MC, 576, 2> : sgd_flat5_kernel<DIM, MC>);
            nt = cps == 2 ? 576 : 1024;
            static PerDeviceOnce attr5[4];
            if (attr5[(cps - 1) + (hog ? 2 : 0)].first())
                UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            // carveout: the smallest shared-memory share that holds cps CTAs (the rest is L1, which
            // caches the gathered positions); set per launch (the size depends on the graph)
            const int pct = cps == 1 ? (int)cudaSharedmemCarveoutMaxL1
                                     : std::min(100, (int)((cps * (smem + 2048) * 100 + 228 * 1024 - 1) / (228 * 1024)));
            UMAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
            int per5 = 0;
            UMAP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per5, kern, nt, smem));
            if (per5 < cps) {
                if (retry) *retry = true;
                set_last_error("flat5 SGD kernel: fewer resident CTAs per SM than the launch needs");
                return UMAP_ERR_CUDA;
            }
        }
    }
    if ((cps != 1 || hog) && ver != 5) {
        if (retry) *retry = true;
        set_last_error(hog ? "the flat Hogwild form needs the flat5 layout" : "two CTAs per SM need the flat5 kernel");
        return UMAP_ERR_CUDA;
    }
    void* args[] = {&A};
    ProfScope ps(PROF_SGD, s);
    UMAP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(nt), args, smem, s));
    UMAP_LAUNCH_CHECK(ver == 5 ? "sgd_flat5_kernel" : ver == 4 ? "sgd_flat4_kernel" : ver == 3 ? "sgd_flat3_kernel" : ver == 2 ? "sgd_flat2_kernel" : "sgd_flat_kernel");
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

template <int DIM>
umap_status launch_sgd(const SgdArgs& A, bool det, cudaStream_t s)
{
    const int sv = sgd_variant();
    if constexpr (DIM <= 4) {  // DIM 8, 16: 64 registers per thread spill (persistent chunk kernel)
        if (det && (sv == 0 || sv == 100 || sv == 101)) {
            // 100: the round-1 flat kernel, 101: flat2 (A/B comparisons); default flat3 (else flat2)
            const int ver = sv == 100 ? 1 : sv == 101 ? 2 : 3;
            // tuning knob UMAP_SGD_CPS=1: flat5 as one CTA of 32 warps per SM
            const int cps = (getenv("UMAP_SGD_CPS") && atoi(getenv("UMAP_SGD_CPS")) == 1) ? 1 : 2;
            bool retry = false;
            umap_status st = A.m == 5 ? launch_sgd_flat<DIM, 5>(A, A.nnz, s, ver, cps, &retry)
                                      : launch_sgd_flat<DIM, 0>(A, A.nnz, s, ver, cps, &retry);
            if (st != UMAP_OK && retry)
                st = A.m == 5 ? launch_sgd_flat<DIM, 5>(A, A.nnz, s, ver, 1, nullptr)
                              : launch_sgd_flat<DIM, 0>(A, A.nnz, s, ver, 1, nullptr);
            return st;
        }
        // Hogwild on flat5's structure (default; tuning knob UMAP_SGD_HOG_CHUNK=1: the persistent
        // chunk kernel), falling back to the chunk kernel when the flat5 layout does not fit
        if (!det && (sv == 0) && sgd_sched_mode() == 2 && !getenv("UMAP_SGD_HOG_CHUNK")) {
            bool retry = false;
            umap_status st = A.m == 5 ? launch_sgd_flat<DIM, 5>(A, A.nnz, s, 3, 2, &retry, true)
                                      : launch_sgd_flat<DIM, 0>(A, A.nnz, s, 3, 2, &retry, true);
            if (st != UMAP_OK && retry) {
                retry = false;
                st = A.m == 5 ? launch_sgd_flat<DIM, 5>(A, A.nnz, s, 3, 1, &retry, true)
                              : launch_sgd_flat<DIM, 0>(A, A.nnz, s, 3, 1, &retry, true);
            }
            if (st == UMAP_OK || !retry) return st;
        }
    }
    return launch_sgd_persistent<DIM>(A, det, s);
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

}  // namespace umapb200
