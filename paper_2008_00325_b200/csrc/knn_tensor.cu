// knn_tensor.cu -- tensor-core candidate kNN (R3) with exact re-rank.
//
// a2 in TENSOR_BF16 mode (north_star "a tcgen05/TMA tensor-core GEMM fused
// with a register/shared-memory top-k select").
//
//  1. prep (a1): column means (fp64), Xc = bf16(X - mean) zero-padded to d_pad =
//     ceil(d/64)*64, row norms ||bf16 xc||^2 in fp32.
//  2. knn_tc_kernel: per CTA one block of 128 query rows against a range of reference
//     rows, 256 references per tile.  Warp-specialised:
//        warp 0  TMA producer: A (128 x 64 bf16) + B (256 x 64 bf16) K-slabs into a
//                3-stage smem ring (SWIZZLE_128B), mbarrier full/empty handshake;
//        warp 1  TMEM owner + MMA issuer: one thread issues tcgen05.mma.kind::f16
//                (M=128, N=256, K=16; BF16 in, FP32 accumulate in TMEM), two 256-column
//                accumulators so tile t+1 is multiplied while tile t is filtered;
//        warps 2-5 epilogue: tcgen05.ld of the accumulator row owned by each thread,
//                d2~ = |q|^2 + |r|^2 - 2 q.r, running top-k' (k' <= 64) per query row
//                sorted in registers (one thread per row).
//  3. rerank_kernel: warp per query, lane per candidate: exact fp32 d2 (R2 definition,
//     sequential fmaf over features), bitonic sort of the k' keys (d2, id), top k.
//     Whenever the candidate set holds the true k nearest the output equals the exact
//     mode bit for bit.
#include <cuda.h>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <cstdio>
#include <algorithm>
#include <cuda_bf16.h>

#include "common.cuh"
#include "bulk.cuh"
#include "gemm.cuh"

namespace umapb200 {

static thread_local int64_t g_last_rank_ambiguous = 0;
static thread_local int64_t g_last_regrouped = 0;
static thread_local bool g_last_projected = false;
static thread_local double g_last_fine_fraction = 1.0;

umap_status topk_merge(const int32_t* idx_in, const float* d2_in, int n_parts, int64_t n, int k_in, int k_out,
                       int out_squared, int32_t* idx, float* dist, cudaStream_t s);

namespace {

constexpr int TC_BM = 128;        // query rows per CTA (TMEM lanes)
constexpr int TC_BN = 256;        // reference rows per tile (UMMA N)
constexpr int TC_BK = 64;         // K slab = 64 bf16 = 128 B (one SWIZZLE_128B atom row)
constexpr int TC_KCMAX = 64;      // max candidates per query row (k')
constexpr int TC_EPI_WARPS = 8;  // two warps per TMEM lane quadrant, each half of the columns
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;   // producer + MMA + epilogue warps
// epilogue warps per MODE: the trust fine pass (MODE 1) is latency-bound in its bucketing,
// so it runs four warps per TMEM lane quadrant (a quarter of the columns each)
template <int MODE> constexpr int tc_epi_warps() { return MODE == 1 ? 16 : TC_EPI_WARPS; }
template <int MODE> constexpr int tc_threads() { return 64 + 32 * tc_epi_warps<MODE>(); }
template <int MODE> constexpr int tc_amb_lists() { return tc_epi_warps<MODE>() / 4; }  // per row
constexpr uint32_t A_BYTES = TC_BM * TC_BK * 2;   // 16 KB
constexpr uint32_t B_BYTES = TC_BN * TC_BK * 2;   // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;

// ----------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(bar)
        : "memory");
}
// TMA with an L2 eviction-priority policy (createpolicy): the CTA's own query tile is
// re-read for every reference tile (evict_last keeps it), reference tiles stream through
__device__ __forceinline__ uint64_t l2_policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar,
                                                 uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst), "l"((uint64_t)map), "r"(x), "r"(y), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart (SBO),
// LBO unused (1), descriptor version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;       // SBO
    d |= (uint64_t)1 << 46;                 // version
    d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
    return d;
}

// instruction descriptor: kind::f16, A=B=BF16, D=F32, both K-major, M=128, N=256
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                           ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// ---- CTA-pair (cta_group::2) helpers: the pair's MMA is issued by the leader CTA (rank 0)
__device__ __forceinline__ uint32_t cluster_ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr)
{
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity), "r"(10000000u)
            : "memory");
    }
}
// TMA load whose completion bytes go to the leader CTA's mbarrier (cluster address)
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar_cluster,
                                                uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(dst), "l"((uint64_t)map), "r"(x), "r"(y), "r"(bar_cluster), "l"(pol)
        : "memory");
}
// instruction descriptor with M = 256 (pair), N = 256
constexpr uint32_t IDESC_PAIR = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                                ((uint32_t)((2 * TC_BM) >> 4) << 24);
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC_PAIR), "r"(accumulate)
        : "memory");
}
// commit: arrive once on the mbarrier at this offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"((uint16_t)3) : "memory");
}
template <int CG> __device__ __forceinline__ void umma_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc)
{
    if constexpr (CG == 2) umma_bf16_pair(tmem_d, adesc, bdesc, acc);
    else umma_bf16(tmem_d, adesc, bdesc, acc);
}
template <int CG> __device__ __forceinline__ void umma_arrive(uint32_t bar)
{
    if constexpr (CG == 2) umma_commit_pair(bar);
    else umma_commit(bar);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// tcgen05.ld of 32 columns without the wait (issue several, then tmem_ld_wait)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, float (&v)[32])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// tcgen05.wait::ld with v as in/out operands, so that no use of v is scheduled before the wait
// (a second call after the first is an immediate no-op that only orders the other array)
__device__ __forceinline__ void tmem_ld_wait(float (&v)[32])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]),
                   "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]), "+f"(v[12]), "+f"(v[13]), "+f"(v[14]), "+f"(v[15]),
                   "+f"(v[16]), "+f"(v[17]), "+f"(v[18]), "+f"(v[19]), "+f"(v[20]), "+f"(v[21]), "+f"(v[22]), "+f"(v[23]),
                   "+f"(v[24]), "+f"(v[25]), "+f"(v[26]), "+f"(v[27]), "+f"(v[28]), "+f"(v[29]), "+f"(v[30]), "+f"(v[31])
                 :
                 : "memory");
}

struct TcArgs {
    float* zout;            // MODE 3: [n_q][128] fp32, the first 128 accumulator columns of each row
    const float* qnorm;     // [n_q]
    const float* rnorm;     // [n_r]
    int64_t nq, nr;
    int kblocks;            // d_pad / 64
    int kc;                 // candidates kept per row (<= 32)
    int64_t split_len;      // reference rows per split (multiple of TC_BN)
    int64_t self_shift;     // local reference j is query q's own row when j == q + self_shift
    int exclude_self;
    int64_t index_offset;   // global id = j + index_offset
    int debug;              // bit0: skip epilogue filtering, bit1: skip MMA issue (profiling only)
    int prefilter;          // MODE 0: skip candidate-free chunks with a max tree first (short K)
    int32_t* cand_idx;      // [split][n_q][kc]
    float* cand_d2;
    // RANK mode (trustworthiness, R16)
    const float* thr_d2;    // [n_q][k] exact sorted thresholds
    int k;
    float margin;           // c: |d2~ - d2_exact| < c (|q|^2 + |r|^2)
    // RANK mode: R2's own rounding relative to d2: R2 lies in
    // [(d2~ - E) r_lo, (d2~ + E) r_hi]; 1 / 1 when the margin includes it
    float r_lo, r_hi;
    int32_t* hist;          // [n_q][k] certain bucket counts (written, not accumulated)
    int32_t* amb;           // per (query row, column half) lists of reference rows to re-check
    int amb_cap;            // capacity per list
    int* amb_count;         // [n_q][2] entries per list (may exceed cap -> overflow)
    const int32_t* self_col;  // RANK mode, optional: reference column of query q's own row
    int dense_min;            // RANK mode: see TC_DENSE_MIN
    // RANK mode, optional: the 256-row query block b (= blockIdx.x / 2) visits only the reference
    // tiles tile_list[b * tile_ld + 0 .. tile_count[b]) -- the tiles the coarse pass flagged
    const int32_t* tile_list;
    const int32_t* tile_count;
    int tile_ld;
    uint8_t* flags;           // MODE 2 (coarse pass): flags[b * tile_ld + t] = 1 if tile t may matter
    uint8_t* rowflags;        // MODE 2, optional: rowflags[q * tile_ld + t] = 1 if tile t may matter for row q
    const int32_t* chunk_block;  // MODE 1, optional: query block of tile-list chunk c (hist / amb_count added atomically)
    int rotate;               // MODE 0 without tile lists: start at the pair's proportional tile and wrap
    // MODE 2 on projected operands: per-row slacks (query / reference order) and
    // the basis bound sigma_max(P); qnorm / rnorm are then the projected norms |z~|^2
    const float* proj_bq;
    const float* proj_br;
    const float* proj_sigma;  // device: bound on sigma_max(P) (+inf if the basis failed: nothing skipped)
    // MODE 2, optional: per 32-column chunk maxima of rnorm and proj_br (one broadcast load per chunk
    // instead of a per-lane load and a warp reduction)
    const float* chunk_rmax;
    const float* chunk_bmax;
};

constexpr int TC_KT = 16;   // max thresholds per row in RANK mode

// #{m : t[m] <= x} for ascending t[0..15] in registers: branch-free binary search over
// t[0..14] (selects instead of dynamic register indexing), then t[15].
__device__ __forceinline__ int cnt_le16(float x, const float (&t)[TC_KT])
{
    int i = (t[7] <= x) ? 8 : 0;
    const float p1 = (i & 8) ? t[11] : t[3];
    i += (p1 <= x) ? 4 : 0;
    const float p2 = (i & 8) ? ((i & 4) ? t[13] : t[9]) : ((i & 4) ? t[5] : t[1]);
    i += (p2 <= x) ? 2 : 0;
    const float q0 = (i & 2) ? t[2] : t[0], q1 = (i & 2) ? t[6] : t[4];
    const float q2 = (i & 2) ? t[10] : t[8], q3 = (i & 2) ? t[14] : t[12];
    const float p3 = (i & 8) ? ((i & 4) ? q3 : q2) : ((i & 4) ? q1 : q0);
    i += (p3 <= x) ? 1 : 0;
    return i + ((t[15] <= x) ? 1 : 0);
}
constexpr int TC_DENSE_MIN = 16;  // a warp whose busiest lane has this many candidates in a chunk
                                  // buckets all 32 columns branch-free instead of one by one

// CG = 1: one CTA, MMA M = 128.  CG = 2: a CTA pair (cluster of 2 along the query blocks)
// runs tcgen05.mma.cta_group::2 with M = 256: each CTA loads its own 128 query rows and
// half (128 rows) of the 256-row reference tile, so the L2 -> SMEM bytes per MMA flop drop
// by a third; the leader (rank 0) issues the MMAs, each CTA's TMEM holds its 128 rows x
// 256 columns, and each CTA's epilogue filters its own rows exactly as for CG = 1.
template <int KC, int TC_STAGES, int MODE, int CG>
__global__ void __launch_bounds__(tc_threads<MODE>(), 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_r, TcArgs a)
{
    constexpr uint32_t B_ROWS = TC_BN / CG;                     // reference rows loaded by this CTA
    constexpr uint32_t STAGE_C = A_BYTES + B_ROWS * TC_BK * 2;  // bytes per stage per CTA
    extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
    // 1024-byte alignment for the SWIZZLE_128B atoms
    uint8_t* smem = (uint8_t*)(((uintptr_t)tc_smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* stage_base = smem;                                     // TC_STAGES x (A | B)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TC_STAGES * STAGE_C);  // full[S], empty[S], tfull[2], tempty[2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * TC_STAGES + 4);
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // chunked fine pass (chunk_block != nullptr): CTA pair c works on tile-list chunk c of the
    // 256-row query block chunk_block[c]; chunks of one block run concurrently and add their counts
    const int64_t q0 = a.chunk_block ? ((int64_t)a.chunk_block[blockIdx.x >> 1] * 2 + (blockIdx.x & 1)) * TC_BM
                                     : (int64_t)blockIdx.x * TC_BM;
    const int64_t r_lo = (int64_t)blockIdx.y * a.split_len;
    const int64_t r_hi = imin64(a.nr, r_lo + a.split_len);
    const int ntiles_all = (int)((r_hi - r_lo + TC_BN - 1) / TC_BN);
    const int pblk = (int)(blockIdx.x >> 1);  // 256-row query block of this CTA (both CTAs of a pair)
    const int ntiles = a.tile_count ? a.tile_count[pblk] : ntiles_all;
    const int32_t* tlist = a.tile_count ? a.tile_list + (int64_t)pblk * a.tile_ld : nullptr;
    // rotate (no tile list): the pair starts at the reference tile proportional to its query rows
    // (in pivot order: its own neighbourhood) and wraps around; the same for both CTAs of a pair
    const int rot0 = (a.rotate && !tlist && ntiles_all > 0)
                         ? (int)(((int64_t)pblk * 2 * TC_BM * ntiles_all / (a.nq > 0 ? a.nq : 1)) % ntiles_all) : 0;
    // (t + rot0 < 2 ntiles_all: one conditional subtraction, no integer division per tile)
    auto tile_at = [&](int t) {
        if (tlist) return (int)tlist[t];
        const int u = t + rot0;
        return u >= ntiles_all ? u - ntiles_all : u;
    };
    const int KB = a.kblocks;
    // short K (single-part operands, KB <= 2 slabs: C4's d = 50, the projected coarse pass): the
    // query block's A slabs are loaded once, with tile 0, into the A regions of stages 0..KB-1 and
    // stay there; later tiles stream only B (halves the L2 -> SMEM bytes per tile at KB = 1)
    const bool res_a = MODE != 1 && MODE != 3 && KB <= 2 && KB <= TC_STAGES;

    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + TC_STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * TC_STAGES), tempty0 = smem_u32(bars + 2 * TC_STAGES + 2);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, CG * tc_epi_warps<MODE>());  // the epilogue warps of every CTA of the pair
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_q) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_r) : "memory");
    }
    if (warp == 1) {  // TMEM: 512 columns = two 128x256 fp32 accumulators (per CTA)
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            // MODE 1 (split operands, rows [hi | lo] of 2 KB columns): per K slab two stages,
            // the hi parts (A_hi, B_hi) then the lo parts (A_lo, B_lo)
            constexpr int PARTS = (MODE == 1 || MODE == 3) ? 2 : 1;
            // queries evict_last, references evict_first (profiling knob UMAP_TC_DEBUG bit 2: references
            // evict_last too, bit 3: both evict_normal; same-box A/B: evict_last references and
            // hint-free polling waits measured no faster for C4 and slower for C2)
            uint64_t pol_a = l2_policy_evict_last();
            uint64_t pol_b = (a.debug & 4) ? l2_policy_evict_last() : l2_policy_evict_first();
            if (a.debug & 8) {
                asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_a));
                pol_b = pol_a;
            }
            int g = 0;
            for (int t = 0; t < ntiles; ++t) {
                const int y_r = (int)(r_lo + (int64_t)tile_at(t) * TC_BN);
                for (int kb = 0; kb < KB; ++kb) {
#pragma unroll
                    for (int part = 0; part < PARTS; ++part, ++g) {
                        const int s = g % TC_STAGES;
                        const uint32_t ph = (g / TC_STAGES) & 1;
                        mbar_wait(empty0 + 8 * s, ph ^ 1);
                        const uint32_t dst = smem_u32(stage_base + s * STAGE_C);
                        const int x = (part * KB + kb) * TC_BK;
                        const bool load_a = !res_a || t == 0;
                        const uint32_t bytes = load_a ? STAGE_C : STAGE_C - A_BYTES;
                        if constexpr (CG == 2) {
                            // both CTAs' bytes complete on the leader's full barrier
                            if (leader) mbar_expect_tx(full0 + 8 * s, CG * bytes);
                            const uint32_t fb = mapa_shared(full0 + 8 * s, 0);
                            if (load_a) tma_load_2d_cg2(dst, &map_q, x, (int)q0, fb, pol_a);
                            tma_load_2d_cg2(dst + A_BYTES, &map_r, x, y_r + (int)(rank * B_ROWS), fb, pol_b);
                        } else {
                            mbar_expect_tx(full0 + 8 * s, bytes);
                            if (load_a) tma_load_2d_hint(dst, &map_q, x, (int)q0, full0 + 8 * s, pol_a);
                            tma_load_2d_hint(dst + A_BYTES, &map_r, x, y_r, full0 + 8 * s, pol_b);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ------------------------------------------------ MMA issuer (leader CTA of a pair)
            int g = 0;
            for (int t = 0; t < ntiles; ++t) {
                const int b = t & 1;
                if constexpr (CG == 2) mbar_wait_cluster(tempty0 + 8 * b, ((t >> 1) & 1) ^ 1);
                else mbar_wait(tempty0 + 8 * b, ((t >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + (uint32_t)(b * TC_BN);
                for (int kb = 0; kb < KB; ++kb) {
                    const int s = g % TC_STAGES;
                    const uint32_t ph = (g / TC_STAGES) & 1;
                    mbar_wait(full0 + 8 * s, ph);
                    tc_fence_after();
                    const uint32_t b_addr = smem_u32(stage_base + s * STAGE_C) + A_BYTES;
                    const uint32_t a_addr = smem_u32(stage_base + (res_a ? kb : s) * STAGE_C);
#pragma unroll
                    for (int kk = 0; kk < TC_BK / 16; ++kk) {
                        if (!(a.debug & 2)) umma_mma<CG>(tmem_d, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                                  (kb | kk) != 0);
                    }
                    ++g;
                    if constexpr (MODE == 1 || MODE == 3) {
                        // lo stage: hi_q . lo_r (A of the hi stage, B of the lo stage) and
                        // lo_q . hi_r (A of the lo stage, B of the hi stage) into the same accumulator
                        const int s2 = g % TC_STAGES;
                        const uint32_t ph2 = (g / TC_STAGES) & 1;
                        mbar_wait(full0 + 8 * s2, ph2);
                        tc_fence_after();
                        const uint32_t a2 = smem_u32(stage_base + s2 * STAGE_C);
                        const uint32_t b2 = a2 + A_BYTES;
#pragma unroll
                        for (int kk = 0; kk < TC_BK / 16; ++kk) {
                            umma_mma<CG>(tmem_d, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b2 + kk * 32), 1u);
                            umma_mma<CG>(tmem_d, umma_desc_sw128(a2 + kk * 32), umma_desc_sw128(b_addr + kk * 32), 1u);
                        }
                        umma_arrive<CG>(empty0 + 8 * s2);
                        ++g;
                    }
                    umma_arrive<CG>(empty0 + 8 * s);  // smem slot free (in both CTAs) once these MMAs have read it
                }
                umma_arrive<CG>(tfull0 + 8 * b);  // accumulator b complete (in both CTAs)
            }
        }
    } else if constexpr (MODE == 1) {
        // ---------------------------------------------------- RANK epilogue (warps 2..9)
        // Trustworthiness input-space ranks (R16).  Thread = query row, its half of the
        // columns.  d2~ approximates the exact R2 value within E = c (|q|^2 + |r|^2); a
        // reference row below threshold t certainly iff d2~ + E < thr_t, certainly not iff
        // d2~ - E > thr_t.  Rows whose bucket is certain are counted in a shared histogram;
        // the rest are appended (warp-aggregated) for an exact re-check.
        const int quad = warp & 3;
        constexpr int NP = tc_amb_lists<MODE>();            // column parts (warps per lane quadrant)
        constexpr int CP = TC_BN / NP;                      // columns per part
        const int half = (warp - 2) >> 2;                   // this warp's part
        const int row = quad * 32 + lane;
        const int64_t q = q0 + row;
        const bool valid = q < a.nq;
        const float qn = valid ? a.qnorm[q] : 0.0f;
        const int64_t self_j = (valid && a.exclude_self) ? (a.self_col ? (int64_t)a.self_col[q] : q + a.self_shift) : -1;
        const int k = a.k;
        float thr[TC_KT];
#pragma unroll
        for (int t = 0; t < TC_KT; ++t) thr[t] = (valid && t < k) ? a.thr_d2[q * k + t] : INFINITY;
        const float thr_max = valid ? thr[0] : -INFINITY;
        float tmax = thr_max;
#pragma unroll
        for (int t = 1; t < TC_KT; ++t) tmax = (t < k) ? thr[t] : tmax;
        const float c_m = a.margin;
        // shared histogram [part][t][row] after the ring region (ring stays untouched)
        int32_t* Hs = reinterpret_cast<int32_t*>(stage_base + TC_STAGES * STAGE_C + 8 * (2 * TC_STAGES + 4) + 16);
#pragma unroll
        for (int t = 0; t < TC_KT; ++t) Hs[(half * TC_KT + t) * TC_BM + row] = 0;
        asm volatile("bar.sync 1, %0;" ::"r"(32 * tc_epi_warps<MODE>()) : "memory");
        int32_t* amb_row = a.amb + (valid ? (q * NP + half) * (int64_t)a.amb_cap : 0);
        int n_amb = 0;
        for (int t = 0; t < ntiles; ++t) {
            const int b = t & 1;
            mbar_wait(tfull0 + 8 * b, (t >> 1) & 1);
            tc_fence_after();
            const int64_t rb = r_lo + (int64_t)tile_at(t) * TC_BN;
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * TC_BN);
#pragma unroll 1
            for (int c = half * CP; c < (half + 1) * CP && !(a.debug & 1); c += 32) {
                float v[32];
                tmem_ld32(taddr + c, v);
                const int64_t jb = rb + c;
                const int valid_cols = (int)imin64(32, r_hi - jb);
                const float rn_l = lane < valid_cols ? __ldg(a.rnorm + jb + lane) : 0.0f;
                // the accumulator holds -d2~/2 (norms folded into the GEMM); pre-filter with the
                // chunk's largest margin: -2 acc - E_max > tmax  =>  above every threshold
                float rmax = rn_l;
#pragma unroll
                for (int o = 16; o; o >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
                const float vlim = -0.5f * (tmax / a.r_lo + c_m * (qn + rmax));
                uint32_t cm = 0;  // columns possibly below the largest threshold
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    v[u] = -2.0f * v[u];  // d2~ (exact scaling)
                    cm |= (uint32_t)(v[u] <= -2.0f * vlim) << u;
                }
                if (valid_cols < 32) cm &= valid_cols > 0 ? (0xffffffffu >> (32 - valid_cols)) : 0u;
                if (!valid) cm = 0;
                if (self_j >= jb && self_j < jb + 32) cm &= ~(1u << (uint32_t)(self_j - jb));
                uint32_t am = 0;  // ambiguous columns of this chunk (re-checked exactly later)
                if (__reduce_max_sync(0xffffffffu, (unsigned)__popc(cm)) >= (unsigned)a.dense_min) {
                    // dense chunk (the row's own cluster): every column bucketed, updates predicated
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        const float rn = __shfl_sync(0xffffffffu, rn_l, u);
                        const float E = c_m * (qn + rn);
                        const int b_lo = cnt_le16((v[u] - E) * a.r_lo, thr), b_hi = cnt_le16((v[u] + E) * a.r_hi, thr);
                        const bool act = (cm >> u) & 1u;
                        if (act && b_hi == b_lo && b_lo < k) Hs[(half * TC_KT + b_lo) * TC_BM + row] += 1;
                        am |= (uint32_t)(act && b_hi != b_lo) << u;
                    }
                    cm = 0;
                }
                while (__any_sync(0xffffffffu, cm != 0)) {
                    const int u = cm ? __ffs(cm) - 1 : 0;
                    const bool has = cm != 0;
                    cm &= cm - 1;
                    float w16[16], w8[8], w4[4], w2[2];
#pragma unroll
                    for (int i = 0; i < 16; ++i) w16[i] = (u & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
                    for (int i = 0; i < 8; ++i) w8[i] = (u & 2) ? w16[2 * i + 1] : w16[2 * i];
#pragma unroll
                    for (int i = 0; i < 4; ++i) w4[i] = (u & 4) ? w8[2 * i + 1] : w8[2 * i];
#pragma unroll
                    for (int i = 0; i < 2; ++i) w2[i] = (u & 8) ? w4[2 * i + 1] : w4[2 * i];
                    const float d2a = (u & 16) ? w2[1] : w2[0];
                    const float rn = __shfl_sync(0xffffffffu, rn_l, u);
                    const float E = c_m * (qn + rn);
                    const float hiv = (d2a + E) * a.r_hi, lov = (d2a - E) * a.r_lo;
                    const int b_hi = cnt_le16(hiv, thr), b_lo = cnt_le16(lov, thr);  // #thresholds <= d2~ +- E
                    const bool amb = has && b_hi != b_lo;
                    if (has && !amb && b_lo < k) Hs[(half * TC_KT + b_lo) * TC_BM + row] += 1;
                    am |= (uint32_t)amb << u;
                }
                // the chunk's ambiguous columns appended at once (one list reservation per lane and
                // chunk instead of one atomic round trip per pair), in column order
                if (am) {
                    const int cnt = __popc(am);
                    const int pos0 = a.chunk_block ? atomicAdd(a.amb_count + q * NP + half, cnt) : n_amb;
                    int pos = pos0;
                    for (uint32_t m = am; m; m &= m - 1, ++pos)
                        if (pos < a.amb_cap) amb_row[pos] = (int32_t)(jb + __ffs(m) - 1);
                    n_amb += cnt;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_remote(mapa_shared(tempty0 + 8 * b, 0));
                else mbar_arrive(tempty0 + 8 * b);
            }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * tc_epi_warps<MODE>()) : "memory");
        if (half == 0 && valid) {
            for (int t = 0; t < k; ++t) {
                int sum = 0;
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) sum += Hs[(pp * TC_KT + t) * TC_BM + row];
                if (a.chunk_block) {
                    if (sum) atomicAdd(a.hist + q * k + t, sum);
                } else {
                    a.hist[q * k + t] = sum;
                }
            }
        }
        if (valid && !a.chunk_block) a.amb_count[q * NP + half] = n_amb;
    } else if constexpr (MODE == 3) {
        // ---------------------------------------------------- GEMM out (warps 2..9)
        // Z = X_c P with split operands (hi.hi + hi.lo + lo.hi, the trust projection): one
        // reference "tile" holds P^T (rows >= 128 zero), the half-0 warps write their row's first
        // 128 accumulator columns as fp32
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int row = quad * 32 + lane;
        const int64_t q = q0 + row;
        for (int t = 0; t < ntiles; ++t) {
            const int b = t & 1;
            mbar_wait(tfull0 + 8 * b, (t >> 1) & 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * TC_BN);
            if (half == 0) {
#pragma unroll 1
                for (int c = 0; c < 128; c += 32) {
                    float v[32];
                    tmem_ld32(taddr + c, v);
                    if (q < a.nq) {
                        float4* o = reinterpret_cast<float4*>(a.zout + q * 128 + c);
#pragma unroll
                        for (int i = 0; i < 8; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_remote(mapa_shared(tempty0 + 8 * b, 0));
                else mbar_arrive(tempty0 + 8 * b);
            }
        }
    } else if constexpr (MODE == 2) {
        // ---------------------------------------------------- coarse tile flags (warps 2..9)
        // Single-BF16 pass over the hi operands (norms folded: accumulator = -d2~/2, error
        // <= a.margin (|q|^2 + |r|^2)).  A tile is flagged for the split-precision pass when
        // some row of the 256-row block may have a column at or below its largest threshold.
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int row = quad * 32 + lane;
        const int64_t q = q0 + row;
        const bool valid = q < a.nq;
        const float qn = valid ? a.qnorm[q] : 0.0f;
        const float tmax = valid ? a.thr_d2[q * a.k + (a.k - 1)] : -INFINITY;
        // projected operands: skip only if |z~_q - z~_r| - E-slack - b_q - b_r > sigma sqrt(tmax / r_lo)
        // (then |x_q - x_r| > sqrt(tmax / r_lo) and R2 >= d2 r_lo > tmax); kept iff
        // d2~_P <= (A_q + b_q + b_r)^2 + E
        const bool proj = a.proj_bq != nullptr;
        const float aq = (proj && valid) ? *a.proj_sigma * sqrtf(tmax / a.r_lo) * 1.000001f + a.proj_bq[q] : 0.0f;
        for (int t = 0; t < ntiles; ++t) {
            const int b = t & 1;
            mbar_wait(tfull0 + 8 * b, (t >> 1) & 1);
            tc_fence_after();
            const int tile = tile_at(t);
            const int64_t rb = r_lo + (int64_t)tile * TC_BN;
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * TC_BN);
            // the thread's 128 columns as four 32-column chunks: all four TMEM loads in flight
            // before one wait, four independent max trees (FMNMX3); the tile is flagged for the
            // row when some column reaches its chunk's limit
            constexpr int NCH = TC_BN / 2 / 32;
            // the per-chunk column bounds first: their load latency overlaps the TMEM loads (each
            // was waited on inside its chunk's step before: ~10 % of the stall samples)
            float rmx[NCH], bmx[NCH];
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
                const int64_t c5 = (rb + half * (TC_BN / 2) + 32 * h) >> 5;
                rmx[h] = a.chunk_rmax ? __ldg(a.chunk_rmax + c5) : 0.0f;
                bmx[h] = (proj && a.chunk_bmax) ? __ldg(a.chunk_bmax + c5) : 0.0f;
            }
            float v[NCH][32];
#pragma unroll
            for (int h = 0; h < NCH; ++h) tmem_ld32_nw(taddr + half * (TC_BN / 2) + 32 * h, v[h]);
#pragma unroll
            for (int h = 0; h < NCH; ++h) tmem_ld_wait(v[h]);
            bool hit = false;
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
                const int64_t jb = rb + half * (TC_BN / 2) + 32 * h;
                const int valid_cols = (int)imin64(32, r_hi - jb);
                // out-of-range columns (zero-filled TMA rows: accumulator 0) never flag
                if (valid_cols < 32) {
#pragma unroll
                    for (int u = 0; u < 32; ++u) v[h][u] = u < valid_cols ? v[h][u] : -INFINITY;
                }
                float rmax;
                if (a.chunk_rmax) {
                    rmax = rmx[h];
                } else {
                    rmax = lane < valid_cols ? __ldg(a.rnorm + jb + lane) : 0.0f;
#pragma unroll
                    for (int o = 16; o; o >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
                }
                float lim = tmax;
                if (proj) {
                    float br;
                    if (a.chunk_bmax) {
                        br = bmx[h];
                    } else {
                        br = lane < valid_cols ? __ldg(a.proj_br + jb + lane) : 0.0f;
#pragma unroll
                        for (int o = 16; o; o >>= 1) br = fmaxf(br, __shfl_xor_sync(0xffffffffu, br, o));
                    }
                    const float sb = aq + br;
                    lim = sb * sb * 1.000001f;
                }
                const float vlim = -0.5f * (lim + a.margin * (qn + rmax));
                float m16[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) m16[i] = fmaxf(v[h][2 * i], v[h][2 * i + 1]);
#pragma unroll
                for (int w = 8; w >= 1; w >>= 1) {
#pragma unroll
                    for (int i = 0; i < w; ++i) m16[i] = fmaxf(m16[i], m16[i + w]);
                }
                hit |= valid && m16[0] >= vlim;
            }
            tc_fence_before();
            __syncwarp();
            if (a.rowflags && hit) a.rowflags[q * a.tile_ld + tile] = 1;  // both column halves may store 1
            if (__any_sync(0xffffffffu, hit) && lane == 0) a.flags[(int64_t)pblk * a.tile_ld + tile] = 1;
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_remote(mapa_shared(tempty0 + 8 * b, 0));
                else mbar_arrive(tempty0 + 8 * b);
            }
        }
    } else {
        // ---------------------------------------------------- epilogue (warps 2..9)
        // Warp w reads TMEM lane quadrant w % 4 (hardware restriction) and half
        // h = (w - 2) / 4 of each tile's 256 columns.  Each thread owns one query row and
        // keeps its k' best approximate keys of its half sorted in registers.  Per 32
        // columns: one tcgen05.ld, 32 independent d2 = |q|^2 + |r|^2 - 2 q.r, one warp vote;
        // only when some lane holds a candidate below its threshold does the warp run the
        // branch-free compare-exchange insertion for that column.  The two halves of a row
        // are merged through shared memory at the end.
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int row = quad * 32 + lane;
        const int64_t q = q0 + row;
        const bool valid = q < a.nq;
        const float qn = valid ? a.qnorm[q] : 0.0f;
        const int64_t self_j =
            (valid && a.exclude_self) ? (a.self_col ? (int64_t)a.self_col[q] : q + a.self_shift) : -1;
        float kd[KC];
        int32_t ki[KC];
#pragma unroll
        for (int i = 0; i < KC; ++i) { kd[i] = INFINITY; ki[i] = -1; }
        float thr = INFINITY;
        const bool prefilter = a.prefilter != 0, dbg_skip = (a.debug & 1) != 0;  // hoisted out of the chunk loop
        for (int t = 0; t < ntiles; ++t) {
            const int b = t & 1;
            mbar_wait(tfull0 + 8 * b, (t >> 1) & 1);
            tc_fence_after();
            const int64_t rb = r_lo + (int64_t)tile_at(t) * TC_BN;
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * TC_BN);
            // one chunk of 32 columns (jb = its first column): the columns that beat the running
            // threshold, then one insertion round per candidate of the busiest lane; each lane
            // inserts its lowest remaining candidate (selected from registers by a 5-level select tree)
            auto chunk = [&](const float (&v)[32], int64_t jb) {
                const float nthr = -0.5f * thr;
                const int valid_cols = (int)imin64(32, r_hi - jb);
                uint32_t cm = 0;  // columns of this chunk that beat the running threshold
#pragma unroll
                for (int u = 0; u < 32; ++u) cm |= (uint32_t)(v[u] > nthr) << u;
                if (valid_cols < 32) cm &= valid_cols > 0 ? (0xffffffffu >> (32 - valid_cols)) : 0u;
                if (!valid) cm = 0;
                if (self_j >= jb && self_j < jb + 32) cm &= ~(1u << (uint32_t)(self_j - jb));
                while (__any_sync(0xffffffffu, cm != 0)) {
                    const int u = cm ? __ffs(cm) - 1 : 0;
                    const bool has = cm != 0;
                    cm &= cm - 1;
                    float w16[16], w8[8], w4[4], w2[2];
#pragma unroll
                    for (int i = 0; i < 16; ++i) w16[i] = (u & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
                    for (int i = 0; i < 8; ++i) w8[i] = (u & 2) ? w16[2 * i + 1] : w16[2 * i];
#pragma unroll
                    for (int i = 0; i < 4; ++i) w4[i] = (u & 4) ? w8[2 * i + 1] : w8[2 * i];
#pragma unroll
                    for (int i = 0; i < 2; ++i) w2[i] = (u & 8) ? w4[2 * i + 1] : w4[2 * i];
                    const float sel = -2.0f * ((u & 16) ? w2[1] : w2[0]);
                    float cv = (has && sel < thr) ? sel : INFINITY;
                    int32_t ci = (int32_t)(jb + u + a.index_offset);
#pragma unroll
                    for (int i = 0; i < KC; ++i) {
                        const bool sw = cv < kd[i];
                        const float tk = sw ? kd[i] : cv;
                        const int32_t ti = sw ? ki[i] : ci;
                        kd[i] = sw ? cv : kd[i];
                        ki[i] = sw ? ci : ki[i];
                        cv = tk;
                        ci = ti;
                    }
                    thr = kd[KC - 1];
                }
            };
            // 32-column chunk maximum (31-op tree): the accumulator holds -d2/2, so a chunk with
            // max <= -thr/2 holds no candidate for this row
            // as a tree of 3-input maxima (FMNMX3): 11 + 4 + 2 + 1 = 18 instructions for 32 values
            auto cmax = [](const float (&v)[32]) {
                float m[11];
#pragma unroll
                for (int i = 0; i < 10; ++i) m[i] = fmaxf(fmaxf(v[3 * i], v[3 * i + 1]), v[3 * i + 2]);
                m[10] = fmaxf(v[30], v[31]);
                const float a0 = fmaxf(fmaxf(m[0], m[1]), m[2]), a1 = fmaxf(fmaxf(m[3], m[4]), m[5]);
                const float a2 = fmaxf(fmaxf(m[6], m[7]), m[8]), a3 = fmaxf(m[9], m[10]);
                return fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
            };
            // two chunks per step: both TMEM loads in flight before one wait, two independent max
            // trees (the short-K prefilter: most chunks hold no candidate for any row of the warp
            // and are skipped after one vote); out-of-range columns (zero-filled TMA rows) are
            // masked by their index
#pragma unroll 1
            for (int c = half * (TC_BN / 2); c < (half + 1) * (TC_BN / 2) && !dbg_skip; c += 64) {
                float v0[32], v1[32];
                tmem_ld32_nw(taddr + c, v0);
                tmem_ld32_nw(taddr + c + 32, v1);
                tmem_ld_wait(v0);
                tmem_ld_wait(v1);
                const int64_t jb = rb + c;
                bool p0 = true, p1 = true;
                if (prefilter) {
                    const float nthr = -0.5f * thr;
                    const float m0 = cmax(v0), m1 = cmax(v1);
                    p0 = __any_sync(0xffffffffu, valid && m0 > nthr);
                    p1 = __any_sync(0xffffffffu, valid && m1 > nthr);
                }
                if (p0) chunk(v0, jb);
                if (p1) chunk(v1, jb + 32);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_remote(mapa_shared(tempty0 + 8 * b, 0));
                else mbar_arrive(tempty0 + 8 * b);
            }
        }
        // merge the two halves of each row: half 1 publishes its list through smem (the
        // stage ring is idle now: every TMA load has been consumed by the last MMA)
        float* xd = reinterpret_cast<float*>(stage_base);
        int32_t* xi = reinterpret_cast<int32_t*>(stage_base) + KC * TC_BM;
        asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");  // all MMAs done reading smem
        if (half == 1) {
#pragma unroll
            for (int i = 0; i < KC; ++i) { xd[i * TC_BM + row] = kd[i]; xi[i * TC_BM + row] = ki[i]; }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");
        if (half == 0) {
            for (int m = 0; m < KC; ++m) {
                float cv = xd[m * TC_BM + row];
                int32_t ci = xi[m * TC_BM + row];
                if (!(cv < kd[KC - 1])) break;  // the other list is sorted: nothing better follows
#pragma unroll
                for (int i = 0; i < KC; ++i) {
                    const bool sw = cv < kd[i];
                    const float tk = sw ? kd[i] : cv;
                    const int32_t ti = sw ? ki[i] : ci;
                    kd[i] = sw ? cv : kd[i];
                    ki[i] = sw ? ci : ki[i];
                    cv = tk;
                    ci = ti;
                }
            }
            if (valid) {
                const int kc = a.kc;
                const int64_t base = ((int64_t)blockIdx.y * a.nq + q) * kc;
#pragma unroll
                for (int t = 0; t < KC; ++t) {
                    if (t < kc) {
                        a.cand_idx[base + t] = ki[t];
                        a.cand_d2[base + t] = kd[t];
                    }
                }
            }
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();  // the pair's MMAs and both epilogues are done
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if constexpr (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

// ----------------------------------------------------------------------------- prep
__global__ void colsum_kernel(const float* __restrict__ X, int64_t n, int d, double* __restrict__ colsum)
{
    // block (32 columns x 8 row lanes); grid (ceil(d/32), row chunks)
    __shared__ double part[8][33];
    const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
    const int col = blockIdx.x * 32 + cx;
    double s = 0.0;
    if (col < d)
        for (int64_t r = (int64_t)blockIdx.y * 8 + ry; r < n; r += (int64_t)gridDim.y * 8) s += (double)X[r * d + col];
    part[ry][cx] = s;
    __syncthreads();
    if (ry == 0 && col < d) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += part[i][cx];
        atomicAdd(colsum + col, t);
    }
}

// the six folded-norm columns at d_pad-6 .. d_pad-1: role 1 (A) [n1 n2 n3 1 1 1], role 2 (B)
// [1 1 1 n1 n2 n3] with n1 + n2 + n3 = -nrm / 2 (three BF16 pieces); lanes 0..5 write
__device__ __forceinline__ void write_norm_extras(__nv_bfloat16* rowp, int d_pad, float nrm, int role, int lane)
{
    if (role == 0 || lane >= 6) return;
    const float nh = -0.5f * nrm;
    const __nv_bfloat16 n1 = __float2bfloat16_rn(nh);
    const float r1 = nh - __bfloat162float(n1);
    const __nv_bfloat16 n2 = __float2bfloat16_rn(r1);
    const __nv_bfloat16 n3 = __float2bfloat16_rn(r1 - __bfloat162float(n2));
    const int j = lane < 3 ? lane : lane - 3;
    const __nv_bfloat16 piece = j == 0 ? n1 : (j == 1 ? n2 : n3);
    const bool norm_slot = (role == 1) == (lane < 3);
    rowp[(d_pad - 6) + lane] = norm_slot ? piece : __float2bfloat16_rn(1.0f);
}

// role 1 (query / A operand): padding columns d_pad-6 .. d_pad-1 = [n1, n2, n3, 1, 1, 1];
// role 2 (reference / B operand): [1, 1, 1, n1, n2, n3], where n1 + n2 + n3 = -|x_c|^2 / 2 in
// three BF16 pieces (24 significant bits).  The GEMM then accumulates
// q.r - |q|^2/2 - |r|^2/2 = -d2/2 directly (norms folded into the padding of the last K slab).
__global__ void center_bf16_kernel(const float* __restrict__ X, int64_t n, int d, int d_pad,
                                   const double* __restrict__ colsum, double inv_n, __nv_bfloat16* __restrict__ Xc,
                                   float* __restrict__ norms, int role, const int32_t* __restrict__ rowmap)
{
    const int64_t orow = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // output row
    const int lane = threadIdx.x & 31;
    if (orow >= n) return;
    const int64_t row = rowmap ? (int64_t)rowmap[orow] : orow;  // input row
    float acc = 0.0f;
#pragma unroll 4
    for (int f = lane; f < d_pad; f += 32) {
        __nv_bfloat16 h = __float2bfloat16_rn(0.0f);
        if (f < d) {
            const float c = X[row * d + f] - (float)(colsum[f] * inv_n);
            h = __float2bfloat16_rn(c);
            const float hv = __bfloat162float(h);
            acc = fmaf(hv, hv, acc);
        }
        Xc[orow * d_pad + f] = h;
    }
    acc = warp_sum(acc);
    if (lane == 0) norms[orow] = acc;
    __syncwarp();
    write_norm_extras(Xc + orow * d_pad, d_pad, acc, role, lane);
}

// out[c] = max of v[32 c .. 32 c + 31] (v >= 0; a missing tail counts as 0)
__global__ void chunk_max_kernel(const float* __restrict__ v, int64_t n, float* __restrict__ out)
{
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c * 32 >= n) return;
    float m = c * 32 + lane < n ? v[c * 32 + lane] : 0.0f;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) out[c] = m;
}

// Projected operand rows in a given order (rowmap: output row -> input row): BF16 z (K columns),
// zeros up to d_pad - 6, the folded norms (role 1 / 2) of zn = |z~|^2 (fp32 of the fp32 z~); and
// the per-row slack bvec = sigma (1.01 u |x_c|) + sqrt(K) gamma_d sigma |x_c| covering the
// centring rounding and the fp32 projection error (|x_c|^2 = xnorm, the split operands' norms).
// P^T (the d x 128 basis, fp32 row-major) as the split B operand of the tensor-core projection:
// row c < 128 = [hi | lo] of column c (bf16(v), bf16(v - hi)), the d_pad - d padding columns and the
// rows >= 128 zero (the caller clears the buffer), so the folded norms of the X operand add nothing
__global__ void pt_split_kernel(const float* __restrict__ P, int d, int d_pad, __nv_bfloat16* __restrict__ Pt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d * 128) return;
    const int f = i >> 7, c = i & 127;
    const float v = P[i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    Pt[(int64_t)c * 2 * d_pad + f] = hi;
    Pt[(int64_t)c * 2 * d_pad + d_pad + f] = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// row of Z (in the reference operand's row order) holding query i: pos_of[qrow[i]], or row_begin + i
__global__ void zrow_map_kernel(const int32_t* __restrict__ qrow, const int32_t* __restrict__ pos_of, int64_t rows,
                                int64_t row_begin, int32_t* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) out[i] = qrow ? pos_of[qrow[i]] : (int32_t)(row_begin + i);
}

__global__ void proj_operand_kernel(const float* __restrict__ Z, int KP, int K, int64_t rows, int d_pad,
                                    const int32_t* __restrict__ rowmap, const float* __restrict__ xnorm,
                                    const float* __restrict__ sigma_p, float gamma_d, int role, __nv_bfloat16* __restrict__ Zb, float* __restrict__ zn,
                                    float* __restrict__ bvec)
{
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int64_t src = rowmap ? (int64_t)rowmap[row] : row;
    __nv_bfloat16* o = Zb + row * (int64_t)d_pad;
    float acc = 0.0f;
    for (int c = lane; c < d_pad - 6; c += 32) {
        const float z = c < K ? Z[src * KP + c] : 0.0f;
        acc = fmaf(z, z, acc);
        o[c] = __float2bfloat16_rn(z);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        zn[row] = acc;
        const float sigma = *sigma_p;
        const float xn = sqrtf(xnorm[row]) * 1.0001f;
        const float u = 5.9604645e-8f;
        bvec[row] = (sigma * 1.01f * u * xn + sqrtf((float)K) * gamma_d * sigma * xn) * 1.01f;
    }
    __syncwarp();
    write_norm_extras(o, d_pad, acc, role, lane);
}

// split-BF16 operands for the RANK mode: x_c = x - mean (fp32), hi = bf16(x_c),
// lo = bf16(x_c - hi), row layout [hi | lo] (2 d_pad columns).  The RANK kernel issues
// hi.hi + hi.lo + lo.hi into one accumulator from the hi and lo K slabs (x.y to ~2^-16
// relative); norms are the fp32 sums of x_c^2.
// wnorm (optional): sum_f x_c,f^2 max(0, KB - 1 - f / 64) (KB = d_pad / 64 K slabs) = sum over
// the first KB - 1 slabs k of the cumulative squared norm through slab k: the weighted norm of the
// fine pass's per-pair accumulation bound
__global__ void split_bf16_kernel(const float* __restrict__ X, int64_t n, int d, int d_pad,
                                  const double* __restrict__ colsum, double inv_n,
                                  __nv_bfloat16* __restrict__ Xs, float* __restrict__ norms,
                                  const int32_t* __restrict__ rowmap, int role, float* __restrict__ wnorm = nullptr)
{
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int64_t src = rowmap ? (int64_t)rowmap[row] : row;  // output row `row` holds input row `src`
    float acc = 0.0f, accw = 0.0f;
    const int kbm1 = d_pad / TC_BK - 1;
    __nv_bfloat16* o = Xs + row * (int64_t)(2 * d_pad);
    if ((d & 1) == 0 && ((uintptr_t)X & 7) == 0) {
        // feature pairs (2 lane, 2 lane + 1) + 64 i: 8-byte row loads, 4-byte bf16x2 stores; per lane
        // d_pad / 32 terms in each sum, as in the scalar loop (the norm bound of DESIGN.md 7.1)
        const float2* xr = reinterpret_cast<const float2*>(X + src * d);
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(o);
        __nv_bfloat162* ol = reinterpret_cast<__nv_bfloat162*>(o + d_pad);
#pragma unroll 4
        for (int f = 2 * lane; f < d_pad; f += 64) {
            float2 c = make_float2(0.0f, 0.0f);
            if (f < d) {
                const float2 x = xr[f >> 1];
                c.x = x.x - (float)(colsum[f] * inv_n);
                c.y = x.y - (float)(colsum[f + 1] * inv_n);
                const float wgt = (float)max(0, kbm1 - f / TC_BK);  // f, f + 1 in one K slab
                acc = fmaf(c.x, c.x, acc);
                acc = fmaf(c.y, c.y, acc);
                accw = fmaf(c.x * c.x, wgt, accw);
                accw = fmaf(c.y * c.y, wgt, accw);
            }
            const __nv_bfloat162 hi = __floats2bfloat162_rn(c.x, c.y);
            const float2 hf = __bfloat1622float2(hi);
            oh[f >> 1] = hi;
            ol[f >> 1] = __floats2bfloat162_rn(c.x - hf.x, c.y - hf.y);
        }
    } else {
#pragma unroll 4
        for (int f = lane; f < d_pad; f += 32) {
            __nv_bfloat16 hi = __float2bfloat16_rn(0.0f), lo = hi;
            if (f < d) {
                const float c = X[src * d + f] - (float)(colsum[f] * inv_n);
                hi = __float2bfloat16_rn(c);
                lo = __float2bfloat16_rn(c - __bfloat162float(hi));
                acc = fmaf(c, c, acc);
                accw = fmaf(c * c, (float)max(0, kbm1 - f / TC_BK), accw);
            }
            o[f] = hi;
            o[d_pad + f] = lo;
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) norms[row] = acc;
    if (wnorm) {
        accw = warp_sum(accw);
        if (lane == 0) wnorm[row] = accw;
    }
    __syncwarp();
    write_norm_extras(o, d_pad, acc, role, lane);  // folded norms in the hi part; lo stays 0 there
}

// per-row error budget of the fine pass: e = cS |x_c|^2 + cW wnorm (E(q, r) = e_q + e_r)
__global__ void err_budget_kernel(const float* __restrict__ nrm, const float* __restrict__ wn, int64_t n, float cS,
                                  float cW, float* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (cS * nrm[i] + cW * wn[i]) * 1.0001f;
}

// out[0] += sum of the per-(row, part) ambiguous counts, out[1] |= any count > cap
__global__ void amb_reduce_kernel(const int* __restrict__ cnt, int64_t m, int cap, unsigned long long* __restrict__ out)
{
    unsigned long long sum = 0;
    int over = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = cnt[i];
        sum += (unsigned long long)c;
        over |= c > cap;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        over |= __shfl_xor_sync(0xffffffffu, over, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (sum) atomicAdd(out, sum);
        if (over) atomicOr(out + 1, 1ull);
    }
}

// query i's squared norm and weighted norm from the reference pass: row pos_of[qrow[i]]
__global__ void gather_norms_kernel(const int32_t* __restrict__ qrow, const int32_t* __restrict__ pos_of, int64_t rows,
                                    const float* __restrict__ rn, const float* __restrict__ rw, float* __restrict__ qn,
                                    float* __restrict__ qw)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int32_t p = pos_of[qrow[i]];
    qn[i] = rn[p];
    qw[i] = rw[p];
}

// ----------------------------------------------------------------------------- re-rank
// warp per query row; candidates t and t + 32 on lane t (kc <= 64); exact fp32 d2 (R2),
// a bitonic sort of each 32-wide half by key (d2, id), then the two sorted halves are
// merged by rank (keys are distinct: ids differ) and the first k written.
// Exact re-check of the RANK mode's ambiguous pairs (R16).  Warp per query row: the
// row's two lists (one per column half) hold reference ids; each lane takes pairs,
// computes the exact R2 key and its bucket (first threshold it is below), the warp
// accumulates a shared histogram and adds it to the row's certain counts.
// Exact re-check of the RANK mode's ambiguous pairs (R16).  Warp per query row: the
// row's two lists (one per column half) hold reference ids; each lane takes pairs,
// computes the exact R2 key (its own sequential fmaf chain, float4 loads) and its bucket
// (first threshold it is below), the warp accumulates a shared histogram and adds it to
// the row's certain counts.  (A warp-cooperative variant that stages the 32 candidate
// rows through shared memory with coalesced loads / cp.async measured 2x slower at C2:
// 4-byte LDGSTS and per-row LDG+STS are LSU-issue bound.)
constexpr int RF_WARPS = 8;
__global__ void __launch_bounds__(32 * RF_WARPS)
rank_fix_kernel(const float* __restrict__ Xq, const float* __restrict__ Xr, int d, int64_t nq,
                const int32_t* __restrict__ amb, const int* __restrict__ amb_count, int cap_row,
                const float* __restrict__ thr_d2, const int32_t* __restrict__ thr_id, int k,
                int64_t index_offset, int32_t* __restrict__ hist, const int32_t* __restrict__ qrow,
                const int32_t* __restrict__ colmap)
{
    __shared__ int h[RF_WARPS][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * RF_WARPS + warp;
    if (q >= nq) return;
    if (lane < 16) h[warp][lane] = 0;
    __syncwarp();
    const float* x = Xq + (qrow ? (int64_t)qrow[q] : q) * (int64_t)d;  // qrow: query q is input row qrow[q]
    float td[16];
    int32_t ti[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        td[t] = t < k ? thr_d2[q * k + t] : INFINITY;
        ti[t] = t < k ? thr_id[q * k + t] : INT32_MAX;
    }
    constexpr int NL = tc_amb_lists<1>();
    for (int hf = 0; hf < NL; ++hf) {
        const int cnt = min(amb_count[q * NL + hf], cap_row);
        const int32_t* list = amb + (q * NL + hf) * (int64_t)cap_row;
        for (int e = lane; e < cnt; e += 32) {
            const int32_t l = colmap ? colmap[list[e]] : list[e];  // colmap: column -> input row
            const float v = exact_d2(x, Xr + (int64_t)l * d, d);
            const int32_t gid = (int32_t)(l + index_offset);
            int b = 0;
#pragma unroll
            for (int t = 0; t < 16; ++t) b += (t < k) && !key_less(v, gid, td[t], ti[t]);
            if (b < k) atomicAdd(&h[warp][b], 1);
        }
    }
    __syncwarp();
    if (lane < k) hist[q * k + lane] += h[warp][lane];
}

__global__ void __launch_bounds__(32 * RB_WARPS, 1)
rank_fix_bulk_kernel(const float* __restrict__ Xq, const float* __restrict__ Xr, int d, int64_t nq,
                     const int32_t* __restrict__ amb, const int* __restrict__ amb_count, int cap_row,
                     const float* __restrict__ thr_d2, const int32_t* __restrict__ thr_id, int k,
                     int64_t index_offset, int32_t* __restrict__ hist, const int32_t* __restrict__ qrow,
                     const int32_t* __restrict__ colmap)
{
    __shared__ int h[RB_WARPS][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t bar0;
    float* ring = bulk_ring_setup(bar0);
    if (lane < 16) h[warp][lane] = 0;
    __syncwarp();
    uint32_t ph = 0;
    // persistent over query rows: warp w of block b takes rows b * RB_WARPS + w, + grid stride
    for (int64_t q = (int64_t)blockIdx.x * RB_WARPS + warp; q < nq; q += (int64_t)gridDim.x * RB_WARPS) {
        const float* x = Xq + (qrow ? (int64_t)qrow[q] : q) * (int64_t)d;
        float td[16];
        int32_t ti[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            td[t] = t < k ? thr_d2[q * k + t] : INFINITY;
            ti[t] = t < k ? thr_id[q * k + t] : INT32_MAX;
        }
        // the row's lists (one per column part) taken as one sequence, 32 entries at a time
        constexpr int NL = tc_amb_lists<1>();
        int cnt[NL], tot = 0;
#pragma unroll
        for (int h = 0; h < NL; ++h) { cnt[h] = min(amb_count[q * NL + h], cap_row); tot += cnt[h]; }
        const int32_t* lists = amb + (q * NL) * (int64_t)cap_row;
        for (int base = 0; base < tot; base += 32) {
            const int e = base + lane;
            int32_t l = -1;
            if (e < tot) {
                int h = 0, off = e;
#pragma unroll
                for (int hh = 0; hh < NL - 1; ++hh)
                    if (h == hh && off >= cnt[hh]) { off -= cnt[hh]; h = hh + 1; }
                const int32_t col = lists[(int64_t)h * cap_row + off];
                l = colmap ? colmap[col] : col;
            }
            const float v = exact_d2_bulk(x, Xr, l, d, ring, bar0, ph, lane);
            if (l >= 0) {
                const int32_t gid = (int32_t)(l + index_offset);
                int b = 0;
#pragma unroll
                for (int t = 0; t < 16; ++t) b += (t < k) && !key_less(v, gid, td[t], ti[t]);
                if (b < k) atomicAdd(&h[warp][b], 1);
            }
        }
        __syncwarp();
        if (lane < k) {
            hist[q * k + lane] += h[warp][lane];
            h[warp][lane] = 0;
        }
        __syncwarp();
    }
}

// bulk != 0 (d % 4 == 0, blockDim = 32 RB_WARPS, RB_SMEM dynamic smem): the candidate rows
// go through the TMA bulk ring (exact_d2_bulk), else each lane streams its row (exact_d2)
__global__ void rerank_kernel(const float* __restrict__ Xq, const float* __restrict__ Xr, int d, int64_t nq,
                              const int32_t* __restrict__ cand, int kc, int64_t index_offset, int k, int out_squared,
                              int32_t* __restrict__ idx, float* __restrict__ dist, int bulk)
{
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    uint32_t bar0 = 0, ph = 0;
    float* ring = bulk ? bulk_ring_setup(bar0) : nullptr;
    if (q >= nq) return;
    const float* x = Xq + q * (int64_t)d;
    float key[2] = {INFINITY, INFINITY};
    int32_t id[2] = {INT32_MAX, INT32_MAX};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int t = lane + 32 * h;
        const int32_t c = t < kc ? cand[q * kc + t] : -1;
        if (bulk) {
            if (h == 1 && kc <= 32) break;  // warp-uniform
            const float v = exact_d2_bulk(x, Xr, c >= 0 ? (int32_t)(c - index_offset) : -1, d, ring, bar0, ph, lane);
            if (c >= 0) { key[h] = v; id[h] = c; }
        } else if (c >= 0) {
            key[h] = exact_d2(x, Xr + (int64_t)(c - index_offset) * d, d);
            id[h] = c;
        }
    }
    warp_bitonic(key[0], id[0], lane);
    if (kc > 32) {
        warp_bitonic(key[1], id[1], lane);
        // position of each element in the merged order: own index + rank in the other half
        int pos0 = lane, pos1 = lane;
        for (int j = 0; j < 32; ++j) {  // ballot-free: compare against every element of the other half
            const float ok1 = __shfl_sync(0xffffffffu, key[1], j);
            const int32_t oi1 = __shfl_sync(0xffffffffu, id[1], j);
            const float ok0 = __shfl_sync(0xffffffffu, key[0], j);
            const int32_t oi0 = __shfl_sync(0xffffffffu, id[0], j);
            pos0 += key_less(ok1, oi1, key[0], id[0]);
            pos1 += key_less(ok0, oi0, key[1], id[1]);
        }
        if (pos0 < k) {
            idx[q * k + pos0] = id[0] == INT32_MAX ? -1 : id[0];
            dist[q * k + pos0] = out_squared ? key[0] : (isinf(key[0]) ? key[0] : __fsqrt_rn(key[0]));
        }
        if (pos1 < k) {
            idx[q * k + pos1] = id[1] == INT32_MAX ? -1 : id[1];
            dist[q * k + pos1] = out_squared ? key[1] : (isinf(key[1]) ? key[1] : __fsqrt_rn(key[1]));
        }
        return;
    }
    if (lane < k) {
        idx[q * k + lane] = id[0] == INT32_MAX ? -1 : id[0];
        dist[q * k + lane] = out_squared ? key[0] : (isinf(key[0]) ? key[0] : __fsqrt_rn(key[0]));
    }
}

// ----------------------------------------------------------------------------- host
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

umap_status get_encode(EncodeTiledFn* fn)
{
    static EncodeTiledFn cached = nullptr;
    if (!cached) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        UMAP_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) {
            set_last_error("cuTensorMapEncodeTiled unavailable");
            return UMAP_ERR_CUDA;
        }
        cached = (EncodeTiledFn)p;
    }
    *fn = cached;
    return UMAP_OK;
}

umap_status make_map(CUtensorMap* m, const __nv_bfloat16* base, int64_t rows, int d_pad, int box_rows)
{
    EncodeTiledFn enc;
    UMAP_TRY(get_encode(&enc));
    cuuint64_t dims[2] = {(cuuint64_t)d_pad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d_pad * 2};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_last_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
        return UMAP_ERR_CUDA;
    }
    return UMAP_OK;
}

// centred BF16 copy + norms of X (rows n) with the given column mean (colsum / n_mean)
// ---------------------------------------------------------------- kNN pivot order (round 2)
// Short-K kNN (d_pad <= 256, e.g. C4's d = 50) is bounded by the top-k' epilogue, whose cost is
// set by how often a column beats a row's running k'-th best.  With queries and references in
// pivot order (each row next to the rows nearest the same sampled pivot) every query block meets
// its own neighbourhood early, the running thresholds tighten sooner and fewer columns enter the
// insertion loop.  The result does not depend on the order.

// rows[i] = X[i * stride] (the pivot sample)
__global__ void gather_rows_kernel(const float* __restrict__ X, int64_t m, int64_t stride, int d, float* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m * d) return;
    const int64_t r = i / d;
    out[i] = X[r * stride * d + (i - r * d)];
}

// keys[i] = pivot of row i (the first candidate), vals[i] = i
__global__ void pivot_keys_kernel(const int32_t* __restrict__ piv, int64_t n, uint32_t* __restrict__ keys,
                                  int32_t* __restrict__ vals)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = (uint32_t)max(piv[i], 0);
    vals[i] = (int32_t)i;
}

// candidates of query-operand row i (reference-operand ids) -> the caller's order and ids
__global__ void unpermute_cand_kernel(const int32_t* __restrict__ ci, const float* __restrict__ cd,
                                      const int32_t* __restrict__ qperm, const int32_t* __restrict__ rperm, int64_t nq,
                                      int kc, int64_t index_offset, int32_t* __restrict__ oi, float* __restrict__ od)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq * kc) return;
    const int64_t row = i / kc;
    const int t = (int)(i - row * kc);
    const int32_t c = ci[i];
    const int64_t o = (int64_t)qperm[row] * kc + t;
    oi[o] = c >= 0 ? (int32_t)(rperm[c] + index_offset) : -1;
    od[o] = cd[i];
}

umap_status prep_bf16(const float* X, int64_t n, int d, int d_pad, const double* colsum, int64_t n_mean,
                      __nv_bfloat16* Xc, float* norms, int role, cudaStream_t s, const int32_t* rowmap = nullptr)
{
    if (n == 0) return UMAP_OK;
    center_bf16_kernel<<<ceil_div(n * 32, 256), 256, 0, s>>>(X, n, d, d_pad, colsum, 1.0 / (double)n_mean, Xc, norms,
                                                             role, rowmap);
    UMAP_LAUNCH_CHECK("center_bf16_kernel");
    return UMAP_OK;
}

}  // namespace

template <int KC, int ST, int MODE, int CG>
size_t knn_tc_smem_bytes()
{
    const size_t stage = A_BYTES + (size_t)(TC_BN / CG) * TC_BK * 2;
    return 1024 + ST * stage + 8 * (2 * ST + 4) + 16 + (MODE == 1 ? tc_amb_lists<MODE>() * TC_KT * TC_BM * 4 + 16 : 0);
}

// CTA-pair MMA (cta_group::2) unless UMAP_TC_CG=1 (A/B comparison knob)
int tc_cg()
{
    static int cg = 0;
    if (!cg) {
        const char* e = getenv("UMAP_TC_CG");
        cg = (e && atoi(e) == 1) ? 1 : 2;
    }
    return cg;
}

template <int KC, int ST, int MODE, int CG>
umap_status launch_tc_t(const CUtensorMap& mq, const CUtensorMap& mr, const TcArgs& a, dim3 grid, cudaStream_t s)
{
    const size_t smem = knn_tc_smem_bytes<KC, ST, MODE, CG>();
    static PerDeviceOnce configured;
    if (configured.first()) {
        UMAP_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<KC, ST, MODE, CG>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    // MODE 3 runs inside the caller's projection scope (PROF_TRUST_PROJ)
    ProfScope ps(MODE == 0 ? PROF_KNN_TC : (MODE == 1 ? PROF_TRUST_TC : (MODE == 2 ? PROF_TRUST_COARSE : -1)), s);
    if constexpr (CG == 2) {
        grid.x = (grid.x + 1) & ~1u;  // whole pairs; a pair's second block may lie past n_q (masked)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(tc_threads<MODE>());
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        UMAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, knn_tc_kernel<KC, ST, MODE, CG>, mq, mr, a));
    } else {
        knn_tc_kernel<KC, ST, MODE, CG><<<grid, tc_threads<MODE>(), smem, s>>>(mq, mr, a);
    }
    UMAP_LAUNCH_CHECK("knn_tc_kernel");
    return UMAP_OK;
}

template <int KC, int MODE>
umap_status launch_tc(const CUtensorMap& mq, const CUtensorMap& mr, const TcArgs& a, dim3 grid, cudaStream_t s)
{
    if (tc_cg() == 2) return launch_tc_t<KC, MODE == 1 ? 5 : 6, MODE, 2>(mq, mr, a, grid, s);
    return launch_tc_t<KC, 4, MODE, 1>(mq, mr, a, grid, s);
}

// Tensor-core candidate kNN + exact re-rank.  Centring uses the column means of the
// reference set (R3).  kc = candidates per row (k <= kc <= 32).
static umap_status knn_tensor_impl(const float* Xq, int64_t nq, const float* Xr, int64_t nr, int d, int k, int kc,
                                   int64_t self_shift, int exclude_self, int64_t index_offset, int out_squared,
                                   int32_t* idx, float* dist, cudaStream_t s, bool order_ok);
namespace {
// tile-major chunk order: key = the chunk's middle tile (its lists ascend), value = descriptor index
__global__ void chunk_keys_kernel(const int32_t* __restrict__ desc, int64_t nchunks, const int32_t* __restrict__ tl,
                                  int nt, uint32_t* __restrict__ keys, int32_t* __restrict__ idx)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const int b = desc[3 * c], off = desc[3 * c + 1], len = desc[3 * c + 2];
    keys[c] = len > 0 ? (uint32_t)tl[(int64_t)b * nt + off + (len - 1) / 2] : 0u;
    idx[c] = (int32_t)c;
}

__global__ void order_maps_kernel(const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ pos_of);
}  // namespace
umap_status sort_pairs_u32(uint32_t* keys, int32_t* vals, int64_t n, cudaStream_t s);

umap_status knn_tensor(const float* Xq, int64_t nq, const float* Xr, int64_t nr, int d, int k, int kc,
                       int64_t self_shift, int exclude_self, int64_t index_offset, int out_squared, int32_t* idx,
                       float* dist, cudaStream_t s)
{
    return knn_tensor_impl(Xq, nq, Xr, nr, d, k, kc, self_shift, exclude_self, index_offset, out_squared, idx, dist, s,
                           true);
}

// self-column of query-operand row i in reference-operand order (-1: none)
__global__ void self_col_kernel(const int32_t* __restrict__ qperm, const int32_t* __restrict__ rpos, int64_t nq,
                                int64_t nr, int64_t self_shift, int32_t* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const int64_t r = (int64_t)qperm[i] + self_shift;
    out[i] = (r >= 0 && r < nr) ? rpos[r] : -1;
}

static umap_status knn_tensor_impl(const float* Xq, int64_t nq, const float* Xr, int64_t nr, int d, int k, int kc,
                                   int64_t self_shift, int exclude_self, int64_t index_offset, int out_squared,
                                   int32_t* idx, float* dist, cudaStream_t s, bool order_ok)
{
    if (nq == 0) return UMAP_OK;
    kc = std::min(TC_KCMAX, std::max(kc, 2 * k));
    if (k >= TC_KCMAX) {
        set_last_error("tensor kNN supports k < 64");
        return UMAP_ERR_K_OUT_OF_RANGE;
    }
    if (nr >= (int64_t)INT32_MAX || nq >= (int64_t)INT32_MAX) {
        set_last_error("tensor kNN: row count exceeds the TMA coordinate range");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    const int d_pad = (d + 6 + TC_BK - 1) / TC_BK * TC_BK;  // >= 6 padding columns for the folded norms
    Scratch colsum, xr16, rn, xq16, qn;
    UMAP_TRY(colsum.alloc(sizeof(double) * d, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(colsum.p, 0, sizeof(double) * d, s));
    {
        dim3 grid(ceil_div(d, 32), (unsigned)std::min<int64_t>(std::max<int64_t>(1, nr / 64), 512));
        colsum_kernel<<<grid, 256, 0, s>>>(Xr, nr, d, colsum.as<double>());
        UMAP_LAUNCH_CHECK("colsum_kernel");
    }
    // pivot order for short K (see gather_rows_kernel); off for small problems and the nested
    // pivot searches
    const bool self_case = Xq == Xr && nq == nr && self_shift == 0;
    // (long K, e.g. C2: measured slower, 6.3 -> 7.2 ms with the pivot search; the MMA bounds the tile there)
    bool pivot_order = order_ok && (d_pad <= 256 || getenv("UMAP_TC_KNN_ORDER_ALL")) && nr >= 64 * (int64_t)TC_BN &&
                       nq >= 16 * (int64_t)TC_BN && !getenv("UMAP_TC_KNN_NO_ORDER");
    Scratch rperm, qperm_s, pivots, pidx, pdist, keys, rposs, selfc;
    const int32_t* qperm = nullptr;
    if (pivot_order) {
        ProfScope ps_pr(PROF_KNN_PRUNE, s);
        const int64_t P = std::min<int64_t>(4096, std::max<int64_t>(16, nr / TC_BN));
        const int64_t stride = nr / P;
        UMAP_TRY(pivots.alloc(sizeof(float) * (size_t)P * d, s));
        gather_rows_kernel<<<(unsigned)ceil_div(P * d, 256), 256, 0, s>>>(Xr, P, stride, d, pivots.as<float>());
        UMAP_LAUNCH_CHECK("gather_rows_kernel");
        const int64_t nmax = std::max(nq, nr);
        UMAP_TRY(pidx.alloc(sizeof(int32_t) * (size_t)nmax, s));
        UMAP_TRY(pdist.alloc(sizeof(float) * (size_t)nmax, s));
        UMAP_TRY(keys.alloc(sizeof(uint32_t) * (size_t)nmax, s));
        auto order = [&](const float* Xs, int64_t ns, Scratch& perm) -> umap_status {
            // nearest pivot (BF16 candidates + exact re-rank, k = 1), then rows sorted by pivot
            UMAP_TRY(knn_tensor_impl(Xs, ns, pivots.as<float>(), P, d, 1, 2, 0, 0, 0, 1, pidx.as<int32_t>(),
                                     pdist.as<float>(), s, false));
            UMAP_TRY(perm.alloc(sizeof(int32_t) * (size_t)ns, s));
            pivot_keys_kernel<<<ceil_div(ns, 256), 256, 0, s>>>(pidx.as<int32_t>(), ns, keys.as<uint32_t>(),
                                                               perm.as<int32_t>());
            UMAP_LAUNCH_CHECK("pivot_keys_kernel");
            return sort_pairs_u32(keys.as<uint32_t>(), perm.as<int32_t>(), ns, s);
        };
        UMAP_TRY(order(Xr, nr, rperm));
        if (self_case) {
            qperm = rperm.as<int32_t>();
        } else {
            UMAP_TRY(order(Xq, nq, qperm_s));
            qperm = qperm_s.as<int32_t>();
        }
        if (exclude_self && !self_case) {
            UMAP_TRY(rposs.alloc(sizeof(int32_t) * (size_t)nr, s));
            order_maps_kernel<<<ceil_div(nr, 256), 256, 0, s>>>(rperm.as<int32_t>(), nr, rposs.as<int32_t>());
            UMAP_LAUNCH_CHECK("order_maps_kernel");
            UMAP_TRY(selfc.alloc(sizeof(int32_t) * (size_t)nq, s));
            self_col_kernel<<<ceil_div(nq, 256), 256, 0, s>>>(qperm, rposs.as<int32_t>(), nq, nr, self_shift,
                                                              selfc.as<int32_t>());
            UMAP_LAUNCH_CHECK("self_col_kernel");
        }
    }
    UMAP_TRY(xr16.alloc(sizeof(__nv_bfloat16) * (size_t)nr * d_pad, s));
    UMAP_TRY(rn.alloc(sizeof(float) * (size_t)nr, s));
    UMAP_TRY(prep_bf16(Xr, nr, d, d_pad, colsum.as<double>(), nr, xr16.as<__nv_bfloat16>(), rn.as<float>(), 2, s,
                       pivot_order ? rperm.as<int32_t>() : nullptr));
    // queries always get their own copy (A role; for a self-kNN the same rows in the other role)
    UMAP_TRY(xq16.alloc(sizeof(__nv_bfloat16) * (size_t)nq * d_pad, s));
    UMAP_TRY(qn.alloc(sizeof(float) * (size_t)nq, s));
    UMAP_TRY(prep_bf16(Xq, nq, d, d_pad, colsum.as<double>(), nr, xq16.as<__nv_bfloat16>(), qn.as<float>(), 1, s,
                       pivot_order ? qperm : nullptr));
    const __nv_bfloat16* q16 = xq16.as<__nv_bfloat16>();
    const float* qnp = qn.as<float>();
    CUtensorMap map_q, map_r;
    UMAP_TRY(make_map(&map_q, q16, nq, d_pad, TC_BM));
    UMAP_TRY(make_map(&map_r, xr16.as<__nv_bfloat16>(), nr, d_pad, TC_BN / tc_cg()));

    // reference splits so that the grid covers the GPU (split-R, like the exact kernel); none in
    // pivot order (the self-column table indexes the whole reference range)
    const int64_t qblocks = (nq + TC_BM - 1) / TC_BM;
    int64_t splits = std::max<int64_t>(1, (num_sms() + qblocks - 1) / qblocks);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, nr / (4 * TC_BN)));
    if (const char* e = getenv("UMAP_TC_KNN_SPLITS")) splits = std::max(1, atoi(e));  // tuning knob
    if (pivot_order) splits = 1;
    int64_t split_len = (nr + splits - 1) / splits;
    split_len = (split_len + TC_BN - 1) / TC_BN * TC_BN;
    const int n_splits = (int)((nr + split_len - 1) / split_len);

    Scratch ci, cd;
    UMAP_TRY(ci.alloc(sizeof(int32_t) * (size_t)n_splits * nq * kc, s));
    UMAP_TRY(cd.alloc(sizeof(float) * (size_t)n_splits * nq * kc, s));
    TcArgs a{};
    a.qnorm = qnp; a.rnorm = rn.as<float>(); a.nq = nq; a.nr = nr; a.kblocks = d_pad / TC_BK; a.kc = kc;
    a.prefilter = a.kblocks <= 4 ? 1 : 0;  // K <= 256: the epilogue, not the MMA, bounds the tile
    if (const char* e = getenv("UMAP_TC_PREFILTER")) a.prefilter = atoi(e);  // tuning knob
    a.split_len = split_len; a.self_shift = self_shift; a.exclude_self = exclude_self;
    a.index_offset = pivot_order ? 0 : index_offset; a.cand_idx = ci.as<int32_t>(); a.cand_d2 = cd.as<float>();
    if (pivot_order) {
        a.self_shift = 0;  // self case: the same order on both sides; otherwise the self-column table
        a.self_col = (exclude_self && !self_case) ? selfc.as<int32_t>() : nullptr;
        a.rotate = getenv("UMAP_TC_KNN_NO_ROT") ? 0 : 1;  // A/B knob
    }
    {
        const char* dbg = unsafe_env("UMAP_TC_DEBUG");
        a.debug = dbg ? atoi(dbg) : 0;
    }
    const dim3 grid((unsigned)qblocks, n_splits);
    if (kc <= 32) UMAP_TRY((launch_tc<32, 0>(map_q, map_r, a, grid, s)));
    else UMAP_TRY((launch_tc<64, 0>(map_q, map_r, a, grid, s)));
    const int32_t* cand = ci.as<int32_t>();
    Scratch mi, md;
    if (pivot_order) {  // candidates back to the caller's row order and ids
        UMAP_TRY(mi.alloc(sizeof(int32_t) * (size_t)nq * kc, s));
        UMAP_TRY(md.alloc(sizeof(float) * (size_t)nq * kc, s));
        unpermute_cand_kernel<<<(unsigned)ceil_div(nq * kc, 256), 256, 0, s>>>(
            ci.as<int32_t>(), cd.as<float>(), qperm, rperm.as<int32_t>(), nq, kc, index_offset, mi.as<int32_t>(),
            md.as<float>());
        UMAP_LAUNCH_CHECK("unpermute_cand_kernel");
        cand = mi.as<int32_t>();
    } else if (n_splits > 1) {  // merge the per-split candidate lists by approximate key
        UMAP_TRY(mi.alloc(sizeof(int32_t) * (size_t)nq * kc, s));
        UMAP_TRY(md.alloc(sizeof(float) * (size_t)nq * kc, s));
        UMAP_TRY(topk_merge(ci.as<int32_t>(), cd.as<float>(), n_splits, nq, kc, kc, 1, mi.as<int32_t>(),
                            md.as<float>(), s));
        cand = mi.as<int32_t>();
    }
    ProfScope ps(PROF_RERANK, s);
    const bool bulk = (d % 4 == 0) && ((uintptr_t)Xq % 16 == 0) && ((uintptr_t)Xr % 16 == 0);
    if (bulk) {
        static PerDeviceOnce cfg;
        if (cfg.first()) {
            UMAP_CUDA_TRY(cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RB_SMEM));
        }
    }
    rerank_kernel<<<ceil_div(nq * 32, 32 * RB_WARPS), 32 * RB_WARPS, bulk ? RB_SMEM : 0, s>>>(
        Xq, Xr, d, nq, cand, kc, index_offset, k, out_squared, idx, dist, bulk ? 1 : 0);
    UMAP_LAUNCH_CHECK("rerank_kernel");
    return UMAP_OK;
}


// Input-space rank counts of trustworthiness with the tensor-core GEMM (R16): queries =
// rows [row_begin, row_end) of X, references = all of X.  Exact thresholds in, exact
// non-cumulative bucket counts out (hist [rows][k]); the approximate pass only decides
// pairs whose bucket is certain under the error bound, the rest are re-checked exactly.
// *overflow != 0 tells the caller to fall back to the exact SIMT kernel.
namespace {

// flags [nb][nt] -> ordered list of the tiles flagged by any block of block b's group of `grp`
// consecutive blocks (one CTA per block).  grp = 1 (per-block lists) measured best at C2: the
// union over 4 / 8 Morton-consecutive blocks grows the lists from 94 to 188 / 245 of 274 tiles,
// more than the L2 sharing of identical lists gains back (the per-block fine pass runs at a 52%
// L2 hit rate)
__global__ void compact_flags_kernel(const uint8_t* __restrict__ flags, int64_t nb, int nt, int grp,
                                     int32_t* __restrict__ list, int32_t* __restrict__ count, int rot)
{
    // rot: block b's list starts at its diagonal tile b nt / nb and wraps around (rows and
    // columns share the Hilbert order, so concurrently running neighbour blocks start on
    // neighbouring tiles); 0: ascending
    const int start = rot ? (int)((int64_t)blockIdx.x * nt / nb) : 0;
    __shared__ int base;
    const int64_t b = blockIdx.x;
    const int64_t g0 = b / grp * grp, g1 = g0 + grp < nb ? g0 + grp : nb;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int t0 = 0; t0 < nt; t0 += blockDim.x) {
        const int tt = t0 + threadIdx.x;
        const int t = tt < nt ? (tt + start) % nt : tt;
        bool f = false;
        if (tt < nt)
            for (int64_t bb = g0; bb < g1 && !f; ++bb) f = flags[bb * nt + t] != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        __shared__ int wcnt[32];
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) wcnt[warp] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int w = 0; w < warp; ++w) off += wcnt[w];
        if (f) list[b * nt + off + __popc(bal & ((1u << lane) - 1u))] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += wcnt[w];
            base += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) count[b] = base;
}

// Row regrouping of the trust fine pass: a few rows have an embedding neighbour
// far away in input space, so their largest threshold covers most reference tiles, and every
// 256-row block holding one of them is flagged for most tiles.  The coarse pass records the
// tiles of every row (rowflags); rows with many tiles are moved behind the others (both groups
// keep their cluster order), and each new block's tile list is the union of its rows' tiles.
__global__ void row_tiles_kernel(const uint8_t* __restrict__ rowflags, int64_t rows, int nt, int32_t* __restrict__ cnt)
{
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= rows) return;
    int c = 0;
    for (int t = lane; t < nt; t += 32) c += rowflags[i * nt + t];
    c = warp_sum(c);
    if (lane == 0) cnt[i] = c;
}

// histogram of the rows' tile counts (0..nt), privatised in shared memory
__global__ void tile_hist_kernel(const int32_t* __restrict__ cnt, int64_t rows, int nt, int32_t* __restrict__ hist)
{
    extern __shared__ int32_t hs[];
    for (int v = threadIdx.x; v <= nt; v += blockDim.x) hs[v] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hs[min(cnt[i], nt)], 1);
    __syncthreads();
    for (int v = threadIdx.x; v <= nt; v += blockDim.x)
        if (hs[v]) atomicAdd(&hist[v], hs[v]);
}

// out[0] = the regroup cut max(8, 2 median) (median = the element of rank rows / 2, as
// std::nth_element), out[1] = rows above the cut; one thread
__global__ void regroup_cut_kernel(const int32_t* __restrict__ hist, int nt, int64_t rows, int32_t* __restrict__ out)
{
    int64_t cum = 0;
    int med = nt;
    for (int v = 0; v <= nt; ++v) {
        cum += hist[v];
        if (cum > rows / 2) { med = v; break; }
    }
    const int cut = max(8, 2 * med);
    int64_t above = 0;
    for (int v = cut + 1; v <= nt; ++v) above += hist[v];
    out[0] = cut;
    out[1] = (int32_t)above;
}

__global__ void regroup_keys_kernel(const int32_t* __restrict__ cnt, int64_t rows, const int32_t* __restrict__ cutp,
                                    uint32_t* __restrict__ keys, int32_t* __restrict__ vals)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int cut = *cutp;
    keys[i] = (cnt[i] > cut ? 0x80000000u : 0u) | (uint32_t)i;
    vals[i] = (int32_t)i;
}

__global__ void compose_perm_kernel(const int32_t* __restrict__ qperm, const int32_t* __restrict__ pos2, int64_t rows,
                                    int32_t* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) out[i] = qperm[pos2[i]];
}

// flags[b][t] = OR over the rows r' of new block b (256 rows) of rowflags[pos2[r']][t]
__global__ void block_flags_kernel(const uint8_t* __restrict__ rowflags, const int32_t* __restrict__ pos2, int64_t rows,
                                   int nt, uint8_t* __restrict__ flags)
{
    const int64_t b = blockIdx.x;
    const int64_t r0 = b * 256, r1 = r0 + 256 < rows ? r0 + 256 : rows;
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        // OR over the block's rows, 16 independent loads in flight (an early-exit loop was one
        // dependent L2 round trip per row: 0.145 ms at C2)
        uint32_t f = 0;
        for (int64_t r = r0; r < r1; r += 16) {
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (r + u < r1) f |= rowflags[(int64_t)pos2[r + u] * nt + t];
        }
        flags[b * nt + t] = f ? 1 : 0;
    }
}

// chunk c = (block, offset, length) of descriptor order[c] (identity without order): its own tile
// list (row c of lists, length <= ch)
__global__ void chunk_lists_kernel(const int32_t* __restrict__ desc, const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ tl, int nt, int ch, int32_t* __restrict__ cblock,
                                   int32_t* __restrict__ lists, int32_t* __restrict__ cnt)
{
    const int64_t c = blockIdx.x;
    const int64_t e = order ? order[c] : c;
    const int b = desc[3 * e], off = desc[3 * e + 1], len = desc[3 * e + 2];
    for (int i = threadIdx.x; i < len; i += blockDim.x) lists[c * ch + i] = tl[(int64_t)b * nt + off + i];
    if (threadIdx.x == 0) { cblock[c] = b; cnt[c] = len; }
}

__global__ void order_maps_kernel(const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ pos_of)
{
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) pos_of[perm[p]] = (int32_t)p;
}

// queries of a row shard in cluster order: qrow[i] = input row, selfc[i] = its column, and the
// shard's thresholds gathered into that order
__global__ void shard_order_kernel(const int32_t* __restrict__ qperm, int64_t rows, int64_t row_begin,
                                   const int32_t* __restrict__ pos_of, int k, const float* __restrict__ thr_d2,
                                   const int32_t* __restrict__ thr_id, int32_t* __restrict__ qrow,
                                   int32_t* __restrict__ selfc, float* __restrict__ thr_p, int32_t* __restrict__ thri_p)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int64_t r = qperm[i];
    qrow[i] = (int32_t)(row_begin + r);
    selfc[i] = pos_of[row_begin + r];
    for (int t = 0; t < k; ++t) {
        thr_p[i * k + t] = thr_d2[r * k + t];
        thri_p[i * k + t] = thr_id[r * k + t];
    }
}

__global__ void shard_keys_kernel(const int32_t* __restrict__ pos_of, int64_t row_begin, int64_t rows,
                                  uint32_t* __restrict__ keys, int32_t* __restrict__ vals)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    keys[r] = (uint32_t)pos_of[row_begin + r];
    vals[r] = (int32_t)r;
}

__global__ void unscatter_hist_kernel(const int32_t* __restrict__ qperm, int64_t rows, int k,
                                      const int32_t* __restrict__ hist_p, int32_t* __restrict__ hist)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int64_t r = qperm[i];
    for (int t = 0; t < k; ++t) hist[r * k + t] = hist_p[i * k + t];
}

}  // namespace

umap_status cluster_order(const float* Y, int64_t n, int d_emb, int32_t* perm, cudaStream_t s);
umap_status sort_pairs_u32(uint32_t* keys, int32_t* vals, int64_t n, cudaStream_t s);
umap_status pca_basis(const float* X, int64_t n, int d, const double* colsum, int K, float* P, float* sigma,
                      cudaStream_t s);

// Input-space rank counts of trustworthiness with the tensor-core GEMM (R16): queries =
// rows [row_begin, row_end) of X, references = all of X.  Exact thresholds in, exact
// non-cumulative bucket counts out (hist [rows][k]); the approximate pass only decides
// pairs whose bucket is certain under the error bound, the rest are re-checked exactly.
// Y (optional, n x 2): the embedding; rows and columns are then processed in the Hilbert
// order of Y (counts do not depend on the order), which groups each query block with the
// reference tiles of its own cluster: most column chunks then hold no candidate for any
// row of a warp, and the others hold candidates for all of them.
// *overflow != 0 tells the caller to fall back to the exact SIMT kernel.
umap_status rank_count_tc(const float* X, int64_t n, int d, int64_t row_begin, int64_t rows, int k,
                          const float* thr_d2, const int32_t* thr_id, int32_t* hist, int* overflow,
                          const float* Y, int d_emb, const int32_t* perm_in, cudaStream_t s)
{
    *overflow = 0;
    if (rows == 0) return UMAP_OK;
    if (k > TC_KT) { *overflow = 1; return UMAP_OK; }
    const int d_pad = (d + 6 + TC_BK - 1) / TC_BK * TC_BK;  // >= 6 padding columns for the folded norms
    const int dk = 2 * d_pad;
    Scratch colsum, xr, rn, xq, qn, amb, ambc, rw, qw, er, eq;
    Scratch perm, pos_of, keys, qperm, qrow, selfc, thr_p, thri_p, hist_p;
    const bool ordered = Y != nullptr && d_emb == 2 && n < (int64_t)INT32_MAX;
    if (ordered) {
        UMAP_TRY(perm.alloc(sizeof(int32_t) * (size_t)n, s));
        UMAP_TRY(pos_of.alloc(sizeof(int32_t) * (size_t)n, s));
        if (perm_in)  // the caller's Hilbert order of Y (trust_penalty computed it for the thresholds)
            UMAP_CUDA_TRY(cudaMemcpyAsync(perm.p, perm_in, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
        else
            UMAP_TRY(cluster_order(Y, n, d_emb, perm.as<int32_t>(), s));
        order_maps_kernel<<<ceil_div(n, 256), 256, 0, s>>>(perm.as<int32_t>(), n, pos_of.as<int32_t>());
        UMAP_LAUNCH_CHECK("order_maps_kernel");
        UMAP_TRY(keys.alloc(sizeof(uint32_t) * (size_t)rows, s));
        UMAP_TRY(qperm.alloc(sizeof(int32_t) * (size_t)rows, s));
        shard_keys_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(pos_of.as<int32_t>(), row_begin, rows,
                                                              keys.as<uint32_t>(), qperm.as<int32_t>());
        UMAP_LAUNCH_CHECK("shard_keys_kernel");
        UMAP_TRY(sort_pairs_u32(keys.as<uint32_t>(), qperm.as<int32_t>(), rows, s));
        UMAP_TRY(qrow.alloc(sizeof(int32_t) * (size_t)rows, s));
        UMAP_TRY(selfc.alloc(sizeof(int32_t) * (size_t)rows, s));
        UMAP_TRY(thr_p.alloc(sizeof(float) * (size_t)rows * k, s));
        UMAP_TRY(thri_p.alloc(sizeof(int32_t) * (size_t)rows * k, s));
        UMAP_TRY(hist_p.alloc(sizeof(int32_t) * (size_t)rows * k, s));
        shard_order_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(qperm.as<int32_t>(), rows, row_begin,
                                                               pos_of.as<int32_t>(), k, thr_d2, thr_id,
                                                               qrow.as<int32_t>(), selfc.as<int32_t>(),
                                                               thr_p.as<float>(), thri_p.as<int32_t>());
        UMAP_LAUNCH_CHECK("shard_order_kernel");
    }
    UMAP_TRY(colsum.alloc(sizeof(double) * d, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(colsum.p, 0, sizeof(double) * d, s));
    {
        dim3 grid(ceil_div(d, 32), (unsigned)std::min<int64_t>(std::max<int64_t>(1, n / 64), 512));
        colsum_kernel<<<grid, 256, 0, s>>>(X, n, d, colsum.as<double>());
        UMAP_LAUNCH_CHECK("colsum_kernel");
    }
    UMAP_TRY(xr.alloc(sizeof(__nv_bfloat16) * (size_t)n * dk, s));
    UMAP_TRY(rn.alloc(sizeof(float) * (size_t)n, s));
    UMAP_TRY(rw.alloc(sizeof(float) * (size_t)n, s));
    UMAP_TRY(qw.alloc(sizeof(float) * (size_t)rows, s));
    split_bf16_kernel<<<ceil_div(n * 32, 256), 256, 0, s>>>(X, n, d, d_pad, colsum.as<double>(), 1.0 / (double)n,
                                                          xr.as<__nv_bfloat16>(), rn.as<float>(),
                                                          ordered ? perm.as<int32_t>() : nullptr, 2, rw.as<float>());
    UMAP_LAUNCH_CHECK("split_bf16_kernel");
    UMAP_TRY(xq.alloc(sizeof(__nv_bfloat16) * (size_t)rows * dk, s));
    UMAP_TRY(qn.alloc(sizeof(float) * (size_t)rows, s));
    // the query operand (role 1): in an ordered run its rows are reference rows (pos_of[qrow[i]]), so
    // the norms are gathered from the reference pass and the operand itself is built only when a
    // pass reads it (the projected coarse pass does not; the regroup rebuilds it in its own order)
    bool xq_built = false;
    auto build_xq = [&]() -> umap_status {
        split_bf16_kernel<<<ceil_div(rows * 32, 256), 256, 0, s>>>(ordered ? X : X + row_begin * (int64_t)d, rows, d,
                                                                 d_pad, colsum.as<double>(), 1.0 / (double)n,
                                                                 xq.as<__nv_bfloat16>(), qn.as<float>(),
                                                                 ordered ? qrow.as<int32_t>() : nullptr, 1,
                                                                 qw.as<float>());
        UMAP_LAUNCH_CHECK("split_bf16_kernel");
        xq_built = true;
        return UMAP_OK;
    };
    if (ordered) {
        gather_norms_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(qrow.as<int32_t>(), pos_of.as<int32_t>(), rows,
                                                               rn.as<float>(), rw.as<float>(), qn.as<float>(),
                                                               qw.as<float>());
        UMAP_LAUNCH_CHECK("gather_norms_kernel");
    } else {
        UMAP_TRY(build_xq());
    }
    CUtensorMap map_q, map_r;
    UMAP_TRY(make_map(&map_q, xq.as<__nv_bfloat16>(), rows, dk, TC_BM));
    UMAP_TRY(make_map(&map_r, xr.as<__nv_bfloat16>(), n, dk, TC_BN / tc_cg()));
    const int64_t qblocks = (rows + TC_BM - 1) / TC_BM;
    constexpr int NL = tc_amb_lists<1>();  // ambiguous-pair lists per row (one per column part)
    int cap = 4096 / NL;
    if (const char* e = getenv("UMAP_TC_AMB_CAP")) cap = std::max(1, atoi(e));  // test knob: force the overflow path
    UMAP_TRY(amb.alloc(sizeof(int32_t) * (size_t)rows * NL * cap, s));
    UMAP_TRY(ambc.alloc(sizeof(int) * (size_t)rows * NL, s));
    const float* thr_use = ordered ? thr_p.as<float>() : thr_d2;
    const int32_t* thri_use = ordered ? thri_p.as<int32_t>() : thr_id;
    int32_t* hist_use = ordered ? hist_p.as<int32_t>() : hist;
    TcArgs a{};
    a.qnorm = qn.as<float>(); a.rnorm = rn.as<float>(); a.nq = rows; a.nr = n; a.kblocks = d_pad / TC_BK; a.kc = 0;
    a.split_len = (n + TC_BN - 1) / TC_BN * TC_BN; a.self_shift = row_begin; a.exclude_self = 1; a.index_offset = 0;
    a.self_col = ordered ? selfc.as<int32_t>() : nullptr;
    // certification margin c: |d2~ - R2(q, r)| <= c (|q|^2 + |r|^2) under any
    // accumulation order with round-to-nearest or truncating fp32 adds (u = 2^-24):
    // tuning/A-B knob UMAP_TC_FLAT_MARGIN=1: the uniform margin c (|q|^2 + |r|^2) of round 1
    bool per_pair = !getenv("UMAP_TC_FLAT_MARGIN");
    float cS_f = 0.0f, cW_f = 0.0f;
    // split representation + accumulation of 3 d_pad products + norms + R2's own error + final ops,
    // times 1.1 (C2: 2.94e-4)
    {
        const double u = std::ldexp(1.0, -24);
        // + the folded norms (BF16-piece representation u S / 2; the adds of the last hi MMA and
        //   the 8 lo-stage MMAs after them onto partial sums up to S: 144 products)
        // (+ the centring roundings, 4u S)
        const double c = 3.0 * std::ldexp(1.0, -16) * 0.5 + 3.0 * d_pad * 2.0 * u * 0.5 +
                         ((d + 31) / 32 + 5) * u + 2.0 * u + 0.5 * u + 144.0 * 2.0 * u + 4.0 * u;
        a.margin = (float)(1.1 * c);
        // per-pair form (round 2, the default): the MMAs accumulate slab by slab, so the adds of
        // slab k < KB land on partial sums bounded by the products of slabs 1..k,
        // 1.016 (Q_k + R_k) / 2 (Q_k = |q|^2 through slab k): 192 adds x 2u each; only the last
        // slab (with the folded norms) adds onto partial sums up to 1.008 S.  So
        // E(q, r) = 1.1 (cS S + cW (Qw_q + Qw_r)), Qw = sum_{k < KB} Q_k (split_bf16's wnorm),
        // cS = split representation + last slab 192 x 2u x 1.008 + norms + final ops + centring,
        // cW = 192 x 2u x 1.016 / 2 -- instead of 2496 adds onto partial sums up to S / 2 each
        // (C2: E ~ 1.35e-4 S instead of 2.10e-4 S for rows with their mass spread over the features)
        cS_f = (float)(1.1 * (3.0 * std::ldexp(1.0, -16) * 0.5 + 192.0 * 2.0 * u * 1.008 + ((d + 31) / 32 + 5) * u +
                              2.0 * u + 0.5 * u + 4.0 * u));
        cW_f = (float)(1.1 * 192.0 * 2.0 * u * 1.016 * 0.5);
        // R2's own error, relative to d2 itself rather than 2S: |R2 - d2| <= gamma_{d+1} d2, times
        // 1.1, plus 4u for the fp32 difference and product that apply the factors and the
        // factors' own rounding
        const double g = 1.1 * (d + 1.0) * u / (1.0 - (d + 1.0) * u) + 4.0 * u;
        a.r_lo = (float)(1.0 - g);
        a.r_hi = (float)(1.0 + g);
        if (unsafe_env("UMAP_TC_R2_IN_MARGIN")) {  // measurement only: the round-1 form (R2 term in c)
            a.margin = (float)(1.1 * (c + (d + 1.0) * u * 2.0 - 4.0 * u));
            a.r_lo = a.r_hi = 1.0f;
        }
    }
    if (const char* mg = unsafe_env("UMAP_TRUST_MARGIN_EXPERIMENT")) {  // measurement only (uniform form)
        a.margin = (float)atof(mg);
        per_pair = false;
    }
    if (per_pair) {
        // E(q, r) = e_q + e_r through the kernel's c_m (qnorm + rnorm) with c_m = 1
        UMAP_TRY(er.alloc(sizeof(float) * (size_t)n, s));
        UMAP_TRY(eq.alloc(sizeof(float) * (size_t)rows, s));
        err_budget_kernel<<<ceil_div(n, 256), 256, 0, s>>>(rn.as<float>(), rw.as<float>(), n, cS_f, cW_f, er.as<float>());
        UMAP_LAUNCH_CHECK("err_budget_kernel");
        err_budget_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(qn.as<float>(), qw.as<float>(), rows, cS_f, cW_f,
                                                             eq.as<float>());
        UMAP_LAUNCH_CHECK("err_budget_kernel");
        a.qnorm = eq.as<float>();
        a.rnorm = er.as<float>();
        a.margin = 1.0f;
    }
    a.thr_d2 = thr_use; a.k = k;
    a.hist = hist_use; a.amb = amb.as<int32_t>(); a.amb_cap = cap;
    if (const char* dbg = unsafe_env("UMAP_TC_DEBUG")) a.debug = atoi(dbg);  // profiling only (results invalid)
    a.dense_min = TC_DENSE_MIN;
    if (const char* dm = getenv("UMAP_TC_DENSE_MIN")) a.dense_min = atoi(dm);  // tuning knob
    a.amb_count = ambc.as<int>();
    // coarse pass (ordered runs): single-BF16 GEMM over the hi operands flags the
    // reference tiles where some row of a 256-row block may reach its largest threshold; the
    // split-precision pass then visits only those tiles (the others are certainly above every
    // threshold of every row of the block and add nothing to any count)
    Scratch flags, tl, tcnt, rowfl, rcnt, rkeys, pos2, qperm2, rhist, rcut;
    const int64_t nqb = (qblocks + 1) / 2, ntl = (n + TC_BN - 1) / TC_BN;
    g_last_regrouped = 0;
    if (ordered && !getenv("UMAP_TC_NO_COARSE")) {
        UMAP_TRY(flags.alloc((size_t)nqb * ntl, s));
        UMAP_CUDA_TRY(cudaMemsetAsync(flags.p, 0, (size_t)nqb * ntl, s));
        UMAP_TRY(tl.alloc(sizeof(int32_t) * (size_t)nqb * ntl, s));
        UMAP_TRY(tcnt.alloc(sizeof(int32_t) * (size_t)nqb, s));
        TcArgs ac = a;
        ac.qnorm = qn.as<float>();  // the coarse pass's own margin applies to the squared norms
        ac.rnorm = rn.as<float>();
        ac.kblocks = d_pad / TC_BK;   // hi part only
        ac.flags = flags.as<uint8_t>();
        ac.tile_ld = (int)ntl;
        const bool regroup = !getenv("UMAP_TC_NO_REGROUP");  // A/B knob
        if (regroup) {
            UMAP_TRY(rowfl.alloc((size_t)rows * ntl, s));
            UMAP_CUDA_TRY(cudaMemsetAsync(rowfl.p, 0, (size_t)rows * ntl, s));
            ac.rowflags = rowfl.as<uint8_t>();
        }
        {
            // single BF16 product with folded norms: representation (2 * 2^-8 + 2^-16) S / 2,
            // accumulation of d_pad products onto partial sums up to S, R2's own error, norms
            const double u = std::ldexp(1.0, -24);
            const double c = (2.0 * std::ldexp(1.0, -8) + std::ldexp(1.0, -16)) * 0.5 + d_pad * 2.0 * u +
                             (d + 1.0) * u * 2.0 + ((d + 31) / 32 + 5) * u + 3.0 * u;
            ac.margin = (float)(1.1 * c);
        }
        if (const char* mg = unsafe_env("UMAP_TC_COARSE_MARGIN")) ac.margin = (float)atof(mg);  // measurement only
        // projected coarse pass (d >= 256): the same test on z = P^T x_c, K = 122 principal
        // directions (+ 6 folded-norm columns = 2 K slabs instead of d_pad / 64), with the slack of
        // every rounding step in the per-row bound; any failure of the basis keeps
        // the full-dimensional pass
        constexpr int KPG = 128;
        int KPJ = 122, DPZ = 128;  // projected dimensions (+ 6 folded-norm columns = DPZ)
        if (const char* e = getenv("UMAP_TC_PROJ_K")) {  // tuning knob: 58 (one K slab) or 122 (two)
            KPJ = atoi(e) <= 58 ? 58 : 122;
            DPZ = KPJ + 6;
        }
        Scratch pbp, zf, zq, zr, znq, znr, pbq, pbr, cmr, cmb, psig, pts, zrm;
        CUtensorMap map_zq, map_zr;
        bool projected = false;
        if (d >= 256 && !getenv("UMAP_TC_NO_PROJ")) {
            ProfScope ps_proj(PROF_TRUST_PROJ, s);
            UMAP_TRY(pbp.alloc(sizeof(float) * (size_t)d * KPG, s));
            UMAP_TRY(psig.alloc(sizeof(float), s));
            const float* sigma = psig.as<float>();
            if (pca_basis(X, n, d, colsum.as<double>(), KPJ, pbp.as<float>(), psig.as<float>(), s) == UMAP_OK) {
                // Z = X_c P on the tensor cores: the split reference operand (rows [hi | lo] of x_c, in
                // its own row order) times the split P^T (one 256-row "tile", rows >= 128 zero), three
                // products per K slab (MODE 3); per component |z~ - z| <= gamma_tc sigma |x_c| with
                // gamma_tc = (3 2^-16 representation + 3 d_pad products x 2u accumulated onto sums up to
                // 1.016 |x_c| sigma) x 1.05
                UMAP_TRY(zf.alloc(sizeof(float) * (size_t)n * KPG, s));
                UMAP_TRY(pts.alloc(sizeof(__nv_bfloat16) * (size_t)256 * dk, s));
                UMAP_CUDA_TRY(cudaMemsetAsync(pts.p, 0, sizeof(__nv_bfloat16) * (size_t)256 * dk, s));
                pt_split_kernel<<<ceil_div(d * 128, 256), 256, 0, s>>>(pbp.as<float>(), d, d_pad, pts.as<__nv_bfloat16>());
                UMAP_LAUNCH_CHECK("pt_split_kernel");
                CUtensorMap map_xa, map_pt;
                UMAP_TRY(make_map(&map_xa, xr.as<__nv_bfloat16>(), n, dk, TC_BM));
                UMAP_TRY(make_map(&map_pt, pts.as<__nv_bfloat16>(), 256, dk, TC_BN / tc_cg()));
                TcArgs az{};
                az.zout = zf.as<float>();
                az.nq = n; az.nr = 256; az.kblocks = d_pad / TC_BK; az.split_len = 256;
                UMAP_TRY((launch_tc<32, 3>(map_xa, map_pt, az, dim3((unsigned)((n + TC_BM - 1) / TC_BM), 1), s)));
                const double u = std::ldexp(1.0, -24);
                const float gamma_d = (float)((3.0 * std::ldexp(1.0, -16) + 6.0 * d_pad * u * 1.016) * 1.05);
                UMAP_TRY(zrm.alloc(sizeof(int32_t) * (size_t)rows, s));
                zrow_map_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(ordered ? qrow.as<int32_t>() : nullptr,
                                                                   ordered ? pos_of.as<int32_t>() : nullptr, rows,
                                                                   row_begin, zrm.as<int32_t>());
                UMAP_LAUNCH_CHECK("zrow_map_kernel");
                UMAP_TRY(zq.alloc(sizeof(__nv_bfloat16) * (size_t)rows * DPZ, s));
                UMAP_TRY(znq.alloc(sizeof(float) * (size_t)rows, s));
                UMAP_TRY(pbq.alloc(sizeof(float) * (size_t)rows, s));
                proj_operand_kernel<<<ceil_div(rows * 32, 256), 256, 0, s>>>(
                    zf.as<float>(), KPG, KPJ, rows, DPZ, zrm.as<int32_t>(), qn.as<float>(), sigma, gamma_d, 1,
                    zq.as<__nv_bfloat16>(), znq.as<float>(), pbq.as<float>());
                UMAP_LAUNCH_CHECK("proj_operand_kernel");
                UMAP_TRY(zr.alloc(sizeof(__nv_bfloat16) * (size_t)n * DPZ, s));
                UMAP_TRY(znr.alloc(sizeof(float) * (size_t)n, s));
                UMAP_TRY(pbr.alloc(sizeof(float) * (size_t)n, s));
                proj_operand_kernel<<<ceil_div(n * 32, 256), 256, 0, s>>>(
                    zf.as<float>(), KPG, KPJ, n, DPZ, nullptr, rn.as<float>(), sigma, gamma_d, 2,
                    zr.as<__nv_bfloat16>(), znr.as<float>(), pbr.as<float>());
                UMAP_LAUNCH_CHECK("proj_operand_kernel");
                UMAP_TRY(make_map(&map_zq, zq.as<__nv_bfloat16>(), rows, DPZ, TC_BM));
                UMAP_TRY(make_map(&map_zr, zr.as<__nv_bfloat16>(), n, DPZ, TC_BN / tc_cg()));
                ac.kblocks = DPZ / TC_BK;
                ac.qnorm = znq.as<float>();
                ac.rnorm = znr.as<float>();
                ac.proj_bq = pbq.as<float>();
                ac.proj_br = pbr.as<float>();
                ac.proj_sigma = sigma;
                UMAP_TRY(cmr.alloc(sizeof(float) * (size_t)(n / 32 + 1), s));
                UMAP_TRY(cmb.alloc(sizeof(float) * (size_t)(n / 32 + 1), s));
                chunk_max_kernel<<<(unsigned)ceil_div(n / 32 + 1, 8), 256, 0, s>>>(znr.as<float>(), n, cmr.as<float>());
                UMAP_LAUNCH_CHECK("chunk_max_kernel");
                chunk_max_kernel<<<(unsigned)ceil_div(n / 32 + 1, 8), 256, 0, s>>>(pbr.as<float>(), n, cmb.as<float>());
                UMAP_LAUNCH_CHECK("chunk_max_kernel");
                ac.chunk_rmax = cmr.as<float>();
                ac.chunk_bmax = cmb.as<float>();
                // BF16 representation + accumulation of DPZ products + norms + final ops (no R2 term:
                // R2 enters through tmax / r_lo), times 1.1
                ac.margin = (float)(1.1 * ((2.0 * std::ldexp(1.0, -8) + std::ldexp(1.0, -16)) * 0.5 + DPZ * 2.0 * u +
                                           ((KPJ + 31) / 32 + 5) * u + 3.0 * u));
                projected = true;
            }
        }
        g_last_projected = projected;
        if (projected) {
            UMAP_TRY((launch_tc<32, 2>(map_zq, map_zr, ac, dim3((unsigned)qblocks, 1), s)));
        } else {
            if (!xq_built) UMAP_TRY(build_xq());
            UMAP_TRY((launch_tc<32, 2>(map_q, map_r, ac, dim3((unsigned)qblocks, 1), s)));
        }
        if (regroup) {
            ProfScope ps_rg(PROF_TRUST_REGROUP, s);
            // rows whose own tile count exceeds twice the median go behind the others
            UMAP_TRY(rcnt.alloc(sizeof(int32_t) * (size_t)rows, s));
            row_tiles_kernel<<<ceil_div(rows, 8), 256, 0, s>>>(rowfl.as<uint8_t>(), rows, (int)ntl, rcnt.as<int32_t>());
            UMAP_LAUNCH_CHECK("row_tiles_kernel");
            // the cut (twice the median tile count) on the device: no host round trip; the
            // regroup kernels always run (with no row above the cut the order is unchanged)
            UMAP_TRY(rhist.alloc(sizeof(int32_t) * (size_t)(ntl + 1), s));
            UMAP_TRY(rcut.alloc(sizeof(int32_t) * 2, s));
            UMAP_CUDA_TRY(cudaMemsetAsync(rhist.p, 0, sizeof(int32_t) * (size_t)(ntl + 1), s));
            tile_hist_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows, 256), 4 * num_sms()), 256,
                               sizeof(int32_t) * (size_t)(ntl + 1), s>>>(rcnt.as<int32_t>(), rows, (int)ntl,
                                                                         rhist.as<int32_t>());
            UMAP_LAUNCH_CHECK("tile_hist_kernel");
            regroup_cut_kernel<<<1, 1, 0, s>>>(rhist.as<int32_t>(), (int)ntl, rows, rcut.as<int32_t>());
            UMAP_LAUNCH_CHECK("regroup_cut_kernel");
            {
                UMAP_TRY(rkeys.alloc(sizeof(uint32_t) * (size_t)rows, s));
                UMAP_TRY(pos2.alloc(sizeof(int32_t) * (size_t)rows, s));
                UMAP_TRY(qperm2.alloc(sizeof(int32_t) * (size_t)rows, s));
                regroup_keys_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(rcnt.as<int32_t>(), rows, rcut.as<int32_t>(),
                                                                       rkeys.as<uint32_t>(), pos2.as<int32_t>());
                UMAP_LAUNCH_CHECK("regroup_keys_kernel");
                UMAP_TRY(sort_pairs_u32(rkeys.as<uint32_t>(), pos2.as<int32_t>(), rows, s));
                compose_perm_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(qperm.as<int32_t>(), pos2.as<int32_t>(), rows,
                                                                       qperm2.as<int32_t>());
                UMAP_LAUNCH_CHECK("compose_perm_kernel");
                UMAP_CUDA_TRY(cudaMemcpyAsync(qperm.p, qperm2.p, sizeof(int32_t) * (size_t)rows,
                                              cudaMemcpyDeviceToDevice, s));
                // queries, their thresholds and self columns in the new row order
                shard_order_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(qperm.as<int32_t>(), rows, row_begin,
                                                                       pos_of.as<int32_t>(), k, thr_d2, thr_id,
                                                                       qrow.as<int32_t>(), selfc.as<int32_t>(),
                                                                       thr_p.as<float>(), thri_p.as<int32_t>());
                UMAP_LAUNCH_CHECK("shard_order_kernel");
                split_bf16_kernel<<<ceil_div(rows * 32, 256), 256, 0, s>>>(X, rows, d, d_pad, colsum.as<double>(),
                                                                         1.0 / (double)n, xq.as<__nv_bfloat16>(),
                                                                         qn.as<float>(), qrow.as<int32_t>(), 1,
                                                                         qw.as<float>());
                UMAP_LAUNCH_CHECK("split_bf16_kernel");
                xq_built = true;
                if (per_pair) {
                    err_budget_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(qn.as<float>(), qw.as<float>(), rows, cS_f,
                                                                         cW_f, eq.as<float>());
                    UMAP_LAUNCH_CHECK("err_budget_kernel");
                }
                block_flags_kernel<<<(unsigned)nqb, 256, 0, s>>>(rowfl.as<uint8_t>(), pos2.as<int32_t>(), rows,
                                                                 (int)ntl, flags.as<uint8_t>());
                UMAP_LAUNCH_CHECK("block_flags_kernel");
            }
        }
        int grp = 1;
        if (const char* g = getenv("UMAP_TC_LIST_GROUP")) grp = std::max(1, atoi(g));  // tuning knob
        int rot = 0;
        if (const char* r = getenv("UMAP_TC_LIST_ROT")) rot = atoi(r);  // tuning knob
        compact_flags_kernel<<<(unsigned)nqb, 256, 0, s>>>(flags.as<uint8_t>(), nqb, (int)ntl, grp, tl.as<int32_t>(),
                                                          tcnt.as<int32_t>(), rot);
        UMAP_LAUNCH_CHECK("compact_flags_kernel");
        a.tile_list = tl.as<int32_t>();
        a.tile_count = tcnt.as<int32_t>();
        a.tile_ld = (int)ntl;
        // chunk the tile lists: a CTA pair walks at most CH tiles, so the block of regrouped rows
        // (most tiles) is spread over several pairs instead of being the launch's long pole; and
        // tile-major: the chunks of all blocks launched in the order of their middle tile, so the
        // pairs resident at one time walk the same reference tiles while those are in L2 (C2,
        // same box: DRAM per launch 6.45 -> 2.76 GB, L2 hit rate 58 -> 76 %, 3.73 -> 3.57 ms;
        // CH = 16: 4.28 GB, 3.57 ms; CH = 4: 1.80 GB but 3.74 ms, the per-chunk A reloads and
        // pair start-up dominate)
        std::vector<int32_t> cn((size_t)nqb);
        int32_t cut_h[2] = {0, 0};
        if (regroup) UMAP_CUDA_TRY(cudaMemcpyAsync(cut_h, rcut.p, sizeof(cut_h), cudaMemcpyDeviceToHost, s));
        UMAP_CUDA_TRY(cudaMemcpyAsync(cn.data(), tcnt.p, sizeof(int32_t) * nqb, cudaMemcpyDeviceToHost, s));
        UMAP_CUDA_TRY(cudaStreamSynchronize(s));
        if (regroup) g_last_regrouped = cut_h[1];
        int tmaj = 1;  // tile-major chunk order (all blocks chunked, chunks sorted by their middle tile)
        if (const char* e = getenv("UMAP_TC_TILE_MAJOR")) tmaj = atoi(e);  // tuning knob
        int CH = tmaj ? 8 : 32;
        if (const char* e = getenv("UMAP_TC_CHUNK")) CH = std::max(1, atoi(e));  // tuning knob
        int maxc = 0;
        for (int32_t x : cn) maxc = std::max(maxc, (int)x);
        Scratch cdesc, cblock, ctl, ccnt, ckey, cord;
        int64_t nchunks = qblocks / 2 + (qblocks & 1);
        if (maxc > CH || tmaj) {
            std::vector<int32_t> desc;  // (block, offset, length) per chunk
            for (int64_t b = 0; b < nqb; ++b) {
                const int c = cn[(size_t)b];
                for (int o = 0; o < std::max(1, c); o += CH) {
                    desc.push_back((int32_t)b); desc.push_back(o); desc.push_back(std::min(CH, c - o));
                }
            }
            nchunks = (int64_t)desc.size() / 3;
            UMAP_TRY(cdesc.alloc(sizeof(int32_t) * desc.size(), s));
            UMAP_TRY(cblock.alloc(sizeof(int32_t) * (size_t)nchunks, s));
            UMAP_TRY(ctl.alloc(sizeof(int32_t) * (size_t)nchunks * CH, s));
            UMAP_TRY(ccnt.alloc(sizeof(int32_t) * (size_t)nchunks, s));
            UMAP_CUDA_TRY(cudaMemcpyAsync(cdesc.p, desc.data(), sizeof(int32_t) * desc.size(), cudaMemcpyHostToDevice, s));
            if (tmaj) {
                UMAP_TRY(ckey.alloc(sizeof(uint32_t) * (size_t)nchunks, s));
                UMAP_TRY(cord.alloc(sizeof(int32_t) * (size_t)nchunks, s));
                chunk_keys_kernel<<<ceil_div(nchunks, 256), 256, 0, s>>>(cdesc.as<int32_t>(), nchunks, tl.as<int32_t>(),
                                                                         (int)ntl, ckey.as<uint32_t>(), cord.as<int32_t>());
                UMAP_LAUNCH_CHECK("chunk_keys_kernel");
                UMAP_TRY(sort_pairs_u32(ckey.as<uint32_t>(), cord.as<int32_t>(), nchunks, s));
            }
            chunk_lists_kernel<<<(unsigned)nchunks, 64, 0, s>>>(cdesc.as<int32_t>(), tmaj ? cord.as<int32_t>() : nullptr,
                                                               tl.as<int32_t>(), (int)ntl, CH, cblock.as<int32_t>(),
                                                               ctl.as<int32_t>(), ccnt.as<int32_t>());
            UMAP_LAUNCH_CHECK("chunk_lists_kernel");
            a.chunk_block = cblock.as<int32_t>();
            a.tile_list = ctl.as<int32_t>();
            a.tile_count = ccnt.as<int32_t>();
            a.tile_ld = CH;
            // chunks of one block add into the same rows
            UMAP_CUDA_TRY(cudaMemsetAsync(hist_use, 0, sizeof(int32_t) * (size_t)rows * k, s));
            UMAP_CUDA_TRY(cudaMemsetAsync(ambc.p, 0, sizeof(int) * (size_t)rows * NL, s));
        }
        if (!xq_built) UMAP_TRY(build_xq());
        UMAP_TRY((launch_tc<32, 1>(map_q, map_r, a, dim3((unsigned)(a.chunk_block ? 2 * nchunks : qblocks), 1), s)));
        double m = 0;
        for (int32_t x : cn) m += x;
        g_last_fine_fraction = m / ((double)nqb * (double)ntl);
        if (getenv("UMAP_TC_COARSE_DEBUG"))
            fprintf(stderr, "[coarse] %.1f of %lld tiles kept per block\n", m / nqb, (long long)ntl);
    } else {
        g_last_fine_fraction = 1.0;
        if (!xq_built) UMAP_TRY(build_xq());
        UMAP_TRY((launch_tc<32, 1>(map_q, map_r, a, dim3((unsigned)qblocks, 1), s)));
    }
    {
        ProfScope ps(PROF_RANK_FIX, s);
        const float* xq = ordered ? X : X + row_begin * (int64_t)d;
        const int32_t* qmap = ordered ? qrow.as<int32_t>() : nullptr;
        const int32_t* cmap = ordered ? perm.as<int32_t>() : nullptr;
        if (d % 4 == 0 && (uintptr_t)X % 16 == 0 && !getenv("UMAP_RANKFIX_LDG")) {  // TMA bulk staging (16-byte aligned rows)
            static PerDeviceOnce cfg;
            if (cfg.first()) {
                UMAP_CUDA_TRY(cudaFuncSetAttribute(rank_fix_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)RB_SMEM));
            }
            const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(rows, RB_WARPS), num_sms());
            rank_fix_bulk_kernel<<<grid, 32 * RB_WARPS, RB_SMEM, s>>>(xq, X, d, rows, amb.as<int32_t>(),
                                                                     ambc.as<int>(), cap, thr_use, thri_use, k, 0,
                                                                     hist_use, qmap, cmap);
            UMAP_LAUNCH_CHECK("rank_fix_bulk_kernel");
        } else {
            rank_fix_kernel<<<ceil_div(rows, RF_WARPS), 32 * RF_WARPS, 0, s>>>(xq, X, d, rows, amb.as<int32_t>(),
                                                                              ambc.as<int>(), cap, thr_use, thri_use,
                                                                              k, 0, hist_use, qmap, cmap);
            UMAP_LAUNCH_CHECK("rank_fix_kernel");
        }
    }
    if (ordered) {
        unscatter_hist_kernel<<<ceil_div(rows, 256), 256, 0, s>>>(qperm.as<int32_t>(), rows, k, hist_p.as<int32_t>(),
                                                                  hist);
        UMAP_LAUNCH_CHECK("unscatter_hist_kernel");
    }
    // the re-checked pair total and the list overflow flag, reduced on the device (16 bytes back
    // instead of the rows x NL counts)
    Scratch red;
    UMAP_TRY(red.alloc(sizeof(unsigned long long) * 2, s));
    UMAP_CUDA_TRY(cudaMemsetAsync(red.p, 0, sizeof(unsigned long long) * 2, s));
    amb_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * NL, 256), 4 * num_sms()), 256, 0, s>>>(
        ambc.as<int>(), rows * NL, cap, red.as<unsigned long long>());
    UMAP_LAUNCH_CHECK("amb_reduce_kernel");
    unsigned long long hr[2] = {0, 0};
    UMAP_CUDA_TRY(cudaMemcpyAsync(hr, red.p, sizeof(hr), cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    if (hr[1]) *overflow = 1;
    g_last_rank_ambiguous = (int64_t)hr[0];
    return UMAP_OK;
}

int64_t last_rank_ambiguous() { return g_last_rank_ambiguous; }
int64_t last_regrouped_rows() { return g_last_regrouped; }
double last_fine_fraction() { return g_last_fine_fraction; }

}  // namespace umapb200
