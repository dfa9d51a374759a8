// sgd_persistent.cu -- the persistent chunk SGD kernel (a8): Hogwild at every n_components and
// the deterministic mode at DIM 8 / 16.
#include "sgd_common.cuh"

namespace umapb200 {
namespace sgdk {
namespace {

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

// 1 CTA of 32 warps per SM, 16-vertex chunks: measured best at C2 among 16 launch shapes in
// round 1 (2-4 CTAs per SM, 8/32-vertex chunks, fixed chunks per CTA; tools/sgd_variants.py)
template <int DIM, bool DET, int MC>
umap_status launch_sgd_m(const SgdArgs& A, cudaStream_t s)
{
    if constexpr (DIM <= 4) return launch_sgd_t<DIM, DET, MC, 16, 1, 0>(A, s);
    else return launch_sgd_t<DIM, DET, MC, 16, 4, 0>(A, s);
}

}  // namespace

template <int DIM>
umap_status launch_sgd_persistent(const SgdArgs& A, bool det, cudaStream_t s)
{
    if (A.m == 5) return det ? launch_sgd_m<DIM, true, 5>(A, s) : launch_sgd_m<DIM, false, 5>(A, s);
    return det ? launch_sgd_m<DIM, true, 0>(A, s) : launch_sgd_m<DIM, false, 0>(A, s);
}
template umap_status launch_sgd_persistent<1>(const SgdArgs&, bool, cudaStream_t);
template umap_status launch_sgd_persistent<2>(const SgdArgs&, bool, cudaStream_t);
template umap_status launch_sgd_persistent<3>(const SgdArgs&, bool, cudaStream_t);
template umap_status launch_sgd_persistent<4>(const SgdArgs&, bool, cudaStream_t);
template umap_status launch_sgd_persistent<8>(const SgdArgs&, bool, cudaStream_t);
template umap_status launch_sgd_persistent<16>(const SgdArgs&, bool, cudaStream_t);

}  // namespace sgdk
}  // namespace umapb200
