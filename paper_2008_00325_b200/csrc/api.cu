// api.cu -- the C ABI (include/umap_b200.h): validation, host/device staging,
// the fit / transform / trustworthiness pipelines and the host-side a,b fit.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace umapb200 {

// ---- kernels / stage drivers from the other translation units
umap_status knn_exact(const float* Xq, int64_t nq, const float* Xr, int64_t nr, int d, int k, int64_t self_shift,
                      int exclude_self, int64_t index_offset, int out_squared, int32_t* idx, float* dist,
                      cudaStream_t s);
umap_status knn_tensor(const float* Xq, int64_t nq, const float* Xr, int64_t nr, int d, int k, int kc,
                       int64_t self_shift, int exclude_self, int64_t index_offset, int out_squared, int32_t* idx,
                       float* dist, cudaStream_t s);
umap_status knn_grid2d(const float* Y, int64_t n, int k, int out_squared, int32_t* idx, float* dist, cudaStream_t s);
umap_status topk_merge(const int32_t* idx_in, const float* d2_in, int n_parts, int64_t n, int k_in, int k_out,
                       int out_squared, int32_t* idx, float* dist, cudaStream_t s);
umap_status smooth_knn(const float* dist, const int32_t* idx, int64_t n, int k, float* rho, float* sigma, float* w,
                       int32_t* col_sorted, cudaStream_t s);
umap_status fuzzy_union(const int32_t* acol, const float* aw, int64_t n, int k, int64_t* indptr, int32_t* col,
                        float* val, int64_t capacity, int64_t* nnz_host, cudaStream_t s);
umap_status random_init(int64_t n, int dim, uint64_t seed, float* Y, cudaStream_t s);
umap_status optimize_layout(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, int64_t nnz,
                            float* Y, const umap_params* p, int e_begin, int e_end, int64_t* positives_host,
                            cudaStream_t s);
umap_status transform_optimize(const int32_t* idx, const float* w, int64_t nq, int k, const float* Ytr, int64_t ntr,
                               float* Yq, const umap_params* p, int n_epochs_t, int e_begin, int e_end,
                               int64_t q_offset, int init, cudaStream_t s);
umap_status trust_penalty(const float* X, int64_t n, int d, const int32_t* emb_idx, int k, int64_t row_begin,
                          int64_t row_end, int64_t* row_pen, int64_t* penalty_host, int knn_mode, const float* Y,
                          int d_emb, cudaStream_t s);
bool dim_supported(int dim);
umap_status spectral_init(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, int dim,
                          uint64_t seed, int iters, float* Y, cudaStream_t s);
umap_status supervised_adjust(const int64_t* indptr, const int32_t* col, const float* val, int64_t n,
                              const int32_t* labels, float far_dist, float unknown_dist, int64_t* out_indptr,
                              int32_t* out_col, float* out_val, int64_t capacity, int64_t* nnz_host, cudaStream_t s);
int64_t last_rank_ambiguous();
double last_fine_fraction();

// ---- error state
static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;

void set_last_error(const std::string& s) { g_last_error = s; }

// ---- live per-kernel timing (ProfScope, common.cuh)
struct ProfRec { int slot; cudaEvent_t e0, e1; };
static thread_local bool g_prof_on = false;
static thread_local std::vector<ProfRec> g_prof;
bool profiling_enabled() { return g_prof_on; }
void profile_record(int slot, cudaEvent_t e0, cudaEvent_t e1) { g_prof.push_back({slot, e0, e1}); }
static const char* const k_prof_names[PROF_NSLOTS] = {
    "knn_tc_kernel (kNN candidates)", "rerank_kernel", "knn_tc_kernel (trust ranks)", "rank_fix_kernel",
    "thresholds_warp_kernel", "grid_knn_kernel", "smooth_knn_kernel", "fuzzy union (5 kernels)",
    "sgd_kernel", "dist_tile_kernel (kNN, exact)", "dist_tile_kernel (trust, exact)",
    "transform_sgd_kernel", "knn_tc_kernel (trust coarse)", "spectral init (3 kernels x iterations)",
    "trust projection (basis + operands)", "trust regroup + chunking", "kNN pivot order (short K)",
    "sgd schedule (count + fill)"};
void count_launch(int n) { g_launches += n; }

umap_status cuda_status(cudaError_t e, const char* what)
{
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    cudaGetLastError();  // clear sticky-free errors
    return e == cudaErrorMemoryAllocation ? UMAP_ERR_OUT_OF_MEMORY : UMAP_ERR_CUDA;
}

namespace {

__global__ void nonfinite_kernel(const float* __restrict__ x, int64_t m, int* __restrict__ flag)
{
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

umap_status any_nonfinite(const float* x, int64_t m, bool* out, cudaStream_t s)
{
    Scratch flag;
    UMAP_TRY(flag.alloc(sizeof(int), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    if (m > 0) {
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(m, 256), 8LL * num_sms());
        nonfinite_kernel<<<grid, 256, 0, s>>>(x, m, flag.as<int>());
        UMAP_LAUNCH_CHECK("nonfinite_kernel");
    }
    int h = 0;
    UMAP_CUDA_TRY(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    *out = h != 0;
    return UMAP_OK;
}

// f1 input check (umap_fit_knn): thread per row; flag bit 1 = id out of [0, n) or the row
// itself, 2 = an id twice in the row, 4 = a distance not finite or negative.  The graph stages
// index arrays by these ids (indeg/scatter) and assume k distinct neighbours per row.
__global__ void validate_knn_kernel(const int32_t* __restrict__ idx, const float* __restrict__ dist, int64_t n, int k,
                                    int* __restrict__ flag)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t* row = idx + i * k;
    int bad = 0;
    for (int j = 0; j < k; ++j) {
        const int32_t c = row[j];
        if (c < 0 || (int64_t)c >= n || (int64_t)c == i) bad |= 1;
        for (int l = 0; l < j; ++l) bad |= (row[l] == c) ? 2 : 0;
        const float dv = dist[i * k + j];
        if (!isfinite(dv) || dv < 0.0f) bad |= 4;
    }
    if (bad) atomicOr(flag, bad);
}

umap_status validate_knn(const int32_t* idx, const float* dist, int64_t n, int k, cudaStream_t s)
{
    Scratch flag;
    UMAP_TRY(flag.alloc(sizeof(int), s));
    UMAP_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    if (n > 0) {
        validate_knn_kernel<<<ceil_div(n, 128), 128, 0, s>>>(idx, dist, n, k, flag.as<int>());
        UMAP_LAUNCH_CHECK("validate_knn_kernel");
    }
    int h = 0;
    UMAP_CUDA_TRY(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    if (h) {
        std::string m = "knn graph rejected:";
        if (h & 1) m += " id out of [0, n) or equal to its row;";
        if (h & 2) m += " duplicate id within a row;";
        if (h & 4) m += " distance not finite or negative;";
        set_last_error(m);
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    return UMAP_OK;
}

bool is_device_ptr(const void* p)
{
    if (!p) return false;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

umap_status require_device(const void* p, const char* name)
{
    if (p && !is_device_ptr(p)) {
        set_last_error(std::string(name) + " is not a device pointer");
        return UMAP_ERR_NOT_DEVICE_POINTER;
    }
    return UMAP_OK;
}

umap_status require_cuda()
{
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        set_last_error("no CUDA device: this library has no CPU fallback");
        return UMAP_ERR_CUDA;
    }
    // Keep freed stream-ordered scratch in the device pool instead of unmapping it at
    // every synchronisation (the default release threshold is 0): the single
    // per-process memory pool of P:81 / P:105.  Once per device.
    static thread_local int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
        configured_dev = dev;
    }
    return UMAP_OK;
}

// a host-or-device input array made available on the device
struct DevIn {
    const float* p = nullptr;
    Scratch buf;
    umap_status make(const float* src, size_t count, cudaStream_t s)
    {
        if (is_device_ptr(src)) { p = src; return UMAP_OK; }
        UMAP_TRY(buf.alloc(count * sizeof(float), s));
        UMAP_CUDA_TRY(cudaMemcpyAsync(buf.p, src, count * sizeof(float), cudaMemcpyHostToDevice, s));
        p = buf.as<float>();
        return UMAP_OK;
    }
};

struct DevOut {
    float* p = nullptr;
    float* host = nullptr;
    size_t count = 0;
    Scratch buf;
    umap_status make(float* dst, size_t n, cudaStream_t s)
    {
        count = n;
        if (is_device_ptr(dst)) { p = dst; return UMAP_OK; }
        host = dst;
        UMAP_TRY(buf.alloc(n * sizeof(float), s));
        p = buf.as<float>();
        return UMAP_OK;
    }
    umap_status finish(cudaStream_t s)
    {
        if (host) UMAP_CUDA_TRY(cudaMemcpyAsync(host, p, count * sizeof(float), cudaMemcpyDeviceToHost, s));
        return UMAP_OK;
    }
};

// Stage timer without host synchronisation: lap(&field) records an event on the stream and
// remembers where its milliseconds go; resolve() (after the call's final stream synchronisation)
// writes every lap's device time and returns their sum.  (A synchronising lap left the GPU idle
// at every stage boundary while the host enqueued the next stage.)
struct Timer {
    cudaStream_t s;
    std::vector<cudaEvent_t> ev;
    std::vector<double*> dst;
    explicit Timer(cudaStream_t st) : s(st) { mark(nullptr); }
    ~Timer()
    {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
    void mark(double* d)
    {
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.push_back(e);
        dst.push_back(d);
    }
    void lap(double* d) { mark(d); }
    double resolve()
    {
        double tot = 0.0;
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            cudaEventSynchronize(ev[i]);
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            if (dst[i]) *dst[i] = ms;
            tot += ms;
        }
        return tot;
    }
};

umap_status check_params(const umap_params* p)
{
    if (!p || p->struct_size != sizeof(umap_params)) {
        set_last_error("umap_params missing or struct_size mismatch (call umap_params_default)");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    if (!dim_supported(p->n_components)) {
        set_last_error("n_components must be one of 1,2,3,4,8,16");
        return UMAP_ERR_UNSUPPORTED;
    }
    if (p->negative_sample_rate < 0 || p->n_epochs < 0 || !(p->spread > 0.f) || !(p->min_dist >= 0.f)) {
        set_last_error("invalid n_epochs / negative_sample_rate / spread / min_dist");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    if (p->knn_mode != UMAP_KNN_EXACT_FP32 && p->knn_mode != UMAP_KNN_TENSOR_BF16) {
        set_last_error("unknown knn_mode");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    if (p->init != 0 && p->init != 1) {
        set_last_error("init must be 0 (random) or 1 (spectral)");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    if (p->transform_precision != 0 && p->transform_precision != 1) {
        set_last_error("transform_precision must be 0 (fp32) or 1 (fp64)");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    // R13: a due edge's fixed-point contributions (2 q(g_att) + sum of m q(g_rep), each |q| <=
    // 4 alpha 2^24) are summed in int32 before the segment sums widen to int64
    if (p->sgd_mode == UMAP_SGD_DETERMINISTIC &&
        !((2.0 + (double)p->negative_sample_rate) * (double)p->learning_rate < 32.0)) {
        set_last_error("deterministic SGD needs (2 + negative_sample_rate) * learning_rate < 32 (R13 fixed point)");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    if (!(p->learning_rate >= 0.f) || !(p->repulsion_strength >= 0.f)) {
        set_last_error("learning_rate and repulsion_strength must be finite and >= 0");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    return UMAP_OK;
}

// resolved copy: a, b fitted if absent, n_epochs defaulted
umap_status resolve(const umap_params* in, int64_t n, umap_params* out)
{
    *out = *in;
    if (!(out->a > 0.f) || !(out->b > 0.f)) UMAP_TRY(umap_fit_ab(out->min_dist, out->spread, &out->a, &out->b));
    if (out->n_epochs == 0) out->n_epochs = n <= 10000 ? 500 : 200;
    if (out->knn_candidates < out->n_neighbors) out->knn_candidates = std::max(out->n_neighbors, 32);
    return UMAP_OK;
}

umap_status trust_device(const float* X, int d, const float* Y, int d_emb, int64_t n, int k, int knn_mode,
                         double* T, int64_t* penalty, cudaStream_t s);

umap_status run_knn(const umap_params* p, const float* Xq, int64_t nq, const float* Xr, int64_t nr, int d, int k,
                    int64_t self_shift, int exclude_self, int64_t index_offset, int out_squared, int32_t* idx,
                    float* dist, cudaStream_t s)
{
    // 2-D self-kNN (the embedding side of trustworthiness): exact uniform-grid search
    if (d == 2 && Xq == Xr && nq == nr && exclude_self && self_shift == 0 && index_offset == 0 && k <= 32)
        return knn_grid2d(Xq, nq, k, out_squared, idx, dist, s);
    if (p->knn_mode == UMAP_KNN_TENSOR_BF16)
        return knn_tensor(Xq, nq, Xr, nr, d, k, std::min(64, std::max(k, p->knn_candidates)), self_shift,
                          exclude_self, index_offset, out_squared, idx, dist, s);
    return knn_exact(Xq, nq, Xr, nr, d, k, self_shift, exclude_self, index_offset, out_squared, idx, dist, s);
}

}  // namespace
}  // namespace umapb200

using namespace umapb200;

extern "C" {

const char* umap_version(void) { return "umap-b200 0.2 (sm_100a)"; }

double umap_trust_from_penalty(int64_t penalty, int64_t n, int32_t k)
{
    const double nn = (double)n, kk = (double)k;
    const double den = nn * kk * (2.0 * nn - 3.0 * kk - 1.0);
    if (k < 1 || !(den > 0.0)) return std::nan("");
    return 1.0 - (2.0 / den) * (double)penalty;
}

int32_t umap_transform_epoch_count(int32_t n_epochs, int32_t transform_epochs, int64_t n_train)
{
    if (transform_epochs > 0) return transform_epochs;
    const int32_t N = n_epochs > 0 ? n_epochs : (n_train <= 10000 ? 500 : 200);
    return (N + 2) / 3;
}

int64_t umap_kernel_launch_count(void) { return g_launches; }

int64_t umap_trust_ambiguous_count(void) { return last_rank_ambiguous(); }

double umap_trust_fine_fraction(void) { return last_fine_fraction(); }

void umap_profile_begin(void)
{
    for (auto& r : g_prof) { cudaEventDestroy(r.e0); cudaEventDestroy(r.e1); }
    g_prof.clear();
    g_prof_on = true;
}

int32_t umap_profile_end(double* ms, int64_t* launches, int32_t n_slots)
{
    g_prof_on = false;
    for (int i = 0; i < n_slots; ++i) { if (ms) ms[i] = 0.0; if (launches) launches[i] = 0; }
    for (auto& r : g_prof) {
        float t = 0.f;
        if (cudaEventSynchronize(r.e1) == cudaSuccess && cudaEventElapsedTime(&t, r.e0, r.e1) == cudaSuccess &&
            r.slot < n_slots) {
            if (ms) ms[r.slot] += t;
            if (launches) launches[r.slot] += 1;
        }
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    cudaGetLastError();
    g_prof.clear();
    return PROF_NSLOTS;
}

const char* umap_profile_slot_name(int32_t slot)
{
    return (slot >= 0 && slot < PROF_NSLOTS) ? k_prof_names[slot] : "";
}

const char* umap_last_error(void) { return g_last_error.c_str(); }

const char* umap_status_string(umap_status s)
{
    switch (s) {
        case UMAP_OK: return "UMAP_OK";
        case UMAP_ERR_INVALID_ARGUMENT: return "UMAP_ERR_INVALID_ARGUMENT";
        case UMAP_ERR_NOT_DEVICE_POINTER: return "UMAP_ERR_NOT_DEVICE_POINTER";
        case UMAP_ERR_TOO_FEW_ROWS: return "UMAP_ERR_TOO_FEW_ROWS";
        case UMAP_ERR_K_OUT_OF_RANGE: return "UMAP_ERR_K_OUT_OF_RANGE";
        case UMAP_ERR_NONFINITE_INPUT: return "UMAP_ERR_NONFINITE_INPUT";
        case UMAP_ERR_NONFINITE_EMBEDDING: return "UMAP_ERR_NONFINITE_EMBEDDING";
        case UMAP_ERR_FIT_AB_NO_CONVERGENCE: return "UMAP_ERR_FIT_AB_NO_CONVERGENCE";
        case UMAP_ERR_CUDA: return "UMAP_ERR_CUDA";
        case UMAP_ERR_OUT_OF_MEMORY: return "UMAP_ERR_OUT_OF_MEMORY";
        case UMAP_ERR_UNSUPPORTED: return "UMAP_ERR_UNSUPPORTED";
    }
    return "UMAP_ERR_UNKNOWN";
}

void umap_params_default(umap_params* p)
{
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->struct_size = sizeof(umap_params);
    p->n_neighbors = 15;
    p->n_components = 2;
    p->n_epochs = 0;
    p->min_dist = 0.1f;
    p->spread = 1.0f;
    p->negative_sample_rate = 5;
    p->learning_rate = 1.0f;
    p->repulsion_strength = 1.0f;
    p->a = 0.f;
    p->b = 0.f;
    p->seed = 0;
    p->sgd_mode = UMAP_SGD_DETERMINISTIC;
    p->knn_mode = UMAP_KNN_EXACT_FP32;
    p->knn_candidates = 32;
    p->transform_epochs = 0;
    p->trust_k = 0;
    p->far_dist = 5.0f;
    p->unknown_dist = 1.0f;
    p->init = 0;
    p->spectral_iters = 0;
    p->transform_precision = 0;
}

// R8: Levenberg-Marquardt least squares of Phi(x) = 1/(1 + a x^{2b}) against the
// min_dist curve on linspace(0, 3 spread, 300), from (a, b) = (1, 1).
umap_status umap_fit_ab(float min_dist, float spread, float* a_out, float* b_out)
{
    if (!(spread > 0.f) || !(min_dist >= 0.f) || !a_out || !b_out) {
        set_last_error("fit_ab: spread > 0 and min_dist >= 0 required");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    const int N = 300;
    std::vector<double> x(N), y(N);
    for (int i = 0; i < N; ++i) {
        x[i] = 3.0 * spread * (double)i / (double)(N - 1);
        y[i] = x[i] < min_dist ? 1.0 : std::exp(-(x[i] - min_dist) / spread);
    }
    auto cost = [&](double a, double b) {
        double c = 0;
        for (int i = 0; i < N; ++i) {
            const double xb = x[i] > 0 ? std::pow(x[i], 2 * b) : 0.0;
            const double r = 1.0 / (1.0 + a * xb) - y[i];
            c += r * r;
        }
        return c;
    };
    double a = 1.0, b = 1.0, lam = 1e-3;
    double c = cost(a, b);
    bool converged = false;
    for (int it = 0; it < 2000; ++it) {
        double jtj00 = 0, jtj01 = 0, jtj11 = 0, g0 = 0, g1 = 0;
        for (int i = 0; i < N; ++i) {
            if (x[i] <= 0) continue;
            const double xb = std::pow(x[i], 2 * b);
            const double den = 1.0 + a * xb;
            const double f = 1.0 / den;
            const double r = f - y[i];
            const double da = -xb / (den * den);
            const double db = -a * xb * 2.0 * std::log(x[i]) / (den * den);
            jtj00 += da * da; jtj01 += da * db; jtj11 += db * db;
            g0 += da * r; g1 += db * r;
        }
        bool accepted = false;
        for (int tries = 0; tries < 60 && !accepted; ++tries) {
            const double m00 = jtj00 * (1 + lam), m11 = jtj11 * (1 + lam), m01 = jtj01;
            const double det = m00 * m11 - m01 * m01;
            if (det == 0) { lam *= 10; continue; }
            const double da = -(m11 * g0 - m01 * g1) / det;
            const double db = -(-m01 * g0 + m00 * g1) / det;
            const double na = a + da, nb = b + db;
            const double nc = (nb > 0) ? cost(na, nb) : INFINITY;
            if (nc <= c) {
                const double rel = std::fabs(da) / std::max(1e-300, std::fabs(a)) + std::fabs(db) / std::fabs(b);
                a = na; b = nb;
                const double dc = c - nc;
                c = nc;
                lam = std::max(lam / 10, 1e-15);
                accepted = true;
                if (rel < 1e-14 || dc <= 1e-18 * std::max(c, 1e-300)) converged = true;
            } else {
                lam *= 10;
            }
        }
        if (!accepted) converged = true;  // no descent direction left: at the minimum
        if (converged) break;
    }
    if (!std::isfinite(a) || !std::isfinite(b) || !(a > 0) || !(b > 0)) {
        set_last_error("fit_ab did not converge");
        return UMAP_ERR_FIT_AB_NO_CONVERGENCE;
    }
    *a_out = (float)a;
    *b_out = (float)b;
    return UMAP_OK;
}

umap_status umap_knn(const float* X_q, int64_t n_q, const float* X_r, int64_t n_r, int32_t d, int32_t k,
                     int64_t query_offset, int64_t index_offset, int32_t exclude_self, int32_t knn_mode,
                     int32_t out_squared, int32_t* idx, float* dist, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    if (n_q < 0 || n_r < 1 || d < 1) { set_last_error("bad shapes"); return UMAP_ERR_INVALID_ARGUMENT; }
    if (k < 1 || k > 64 || k > n_r - (exclude_self ? 1 : 0)) {
        set_last_error("k out of range (1 <= k <= 64, k <= n_r - exclude_self)");
        return UMAP_ERR_K_OUT_OF_RANGE;
    }
    if (n_q == 0) return UMAP_OK;
    if (!X_q || !X_r || !idx || !dist) { set_last_error("null array"); return UMAP_ERR_INVALID_ARGUMENT; }
    UMAP_TRY(require_device(X_q, "X_q"));
    UMAP_TRY(require_device(X_r, "X_r"));
    UMAP_TRY(require_device(idx, "idx"));
    UMAP_TRY(require_device(dist, "dist"));
    umap_params p;
    umap_params_default(&p);
    p.knn_mode = knn_mode;
    p.n_neighbors = k;
    UMAP_TRY(run_knn(&p, X_q, n_q, X_r, n_r, d, k, query_offset - index_offset, exclude_self != 0, index_offset,
                     out_squared, idx, dist, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_topk_merge(const int32_t* idx_in, const float* d2_in, int32_t n_parts, int64_t n, int32_t k_in,
                            int32_t k_out, int32_t out_squared, int32_t* idx, float* dist, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    UMAP_TRY(require_device(idx_in, "idx_in"));
    UMAP_TRY(require_device(d2_in, "d2_in"));
    UMAP_TRY(require_device(idx, "idx"));
    UMAP_TRY(require_device(dist, "dist"));
    if (k_out > k_in * n_parts) { set_last_error("k_out > n_parts * k_in"); return UMAP_ERR_K_OUT_OF_RANGE; }
    UMAP_TRY(topk_merge(idx_in, d2_in, n_parts, n, k_in, k_out, out_squared, idx, dist, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_smooth_knn(const float* dist, const int32_t* idx, int64_t n, int32_t k, float* rho, float* sigma,
                            float* w, int32_t* col_sorted_idx, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    if (k < 1 || k > 64) { set_last_error("1 <= k <= 64"); return UMAP_ERR_K_OUT_OF_RANGE; }
    if (!dist || !w || (col_sorted_idx && !idx)) { set_last_error("dist, w (and idx) required"); return UMAP_ERR_INVALID_ARGUMENT; }
    UMAP_TRY(require_device(dist, "dist"));
    UMAP_TRY(require_device(idx, "idx"));
    UMAP_TRY(require_device(rho, "rho"));
    UMAP_TRY(require_device(sigma, "sigma"));
    UMAP_TRY(require_device(w, "w"));
    UMAP_TRY(require_device(col_sorted_idx, "col_sorted_idx"));
    UMAP_TRY(smooth_knn(dist, idx, n, k, rho, sigma, w, col_sorted_idx, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_fuzzy_union(const int32_t* idx, const float* w, int64_t n, int32_t k, int64_t* indptr, int32_t* col,
                             float* val, int64_t capacity, int64_t* nnz, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    if (n < 1 || k < 1) { set_last_error("n >= 1, k >= 1"); return UMAP_ERR_INVALID_ARGUMENT; }
    UMAP_TRY(require_device(idx, "idx"));
    UMAP_TRY(require_device(w, "w"));
    UMAP_TRY(require_device(indptr, "indptr"));
    UMAP_TRY(require_device(col, "col"));
    UMAP_TRY(require_device(val, "val"));
    UMAP_TRY(fuzzy_union(idx, w, n, k, indptr, col, val, capacity, nnz, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_random_init(int64_t n, int32_t dim, uint64_t seed, float* Y, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    UMAP_TRY(require_device(Y, "Y"));
    if (dim < 1) { set_last_error("dim >= 1"); return UMAP_ERR_INVALID_ARGUMENT; }
    UMAP_TRY(random_init(n, dim, seed, Y, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_optimize(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, float* Y,
                          const umap_params* p, int32_t e_begin, int32_t e_end, int64_t* positives, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    UMAP_TRY(check_params(p));
    if (!(p->a > 0.f) || !(p->b > 0.f) || p->n_epochs < 1) {
        set_last_error("umap_optimize needs a > 0, b > 0, n_epochs >= 1");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    UMAP_TRY(require_device(indptr, "indptr"));
    UMAP_TRY(require_device(col, "col"));
    UMAP_TRY(require_device(val, "val"));
    UMAP_TRY(require_device(Y, "Y"));
    int64_t nnz = 0;
    UMAP_CUDA_TRY(cudaMemcpyAsync(&nnz, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    UMAP_TRY(optimize_layout(indptr, col, val, n, nnz, Y, p, e_begin, e_end, positives, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_transform_optimize(const int32_t* idx, const float* w, int64_t n_q, int32_t k, const float* Y_train,
                                    int64_t n_train, float* Y_q, const umap_params* p, int32_t n_epochs_t,
                                    int32_t e_begin, int32_t e_end, int64_t q_offset, int32_t init, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    UMAP_TRY(check_params(p));
    if (!(p->a > 0.f) || !(p->b > 0.f) || k < 1 || k > 64) {
        set_last_error("needs a > 0, b > 0, 1 <= k <= 64");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    UMAP_TRY(require_device(idx, "idx"));
    UMAP_TRY(require_device(w, "w"));
    UMAP_TRY(require_device(Y_train, "Y_train"));
    UMAP_TRY(require_device(Y_q, "Y_q"));
    UMAP_TRY(transform_optimize(idx, w, n_q, k, Y_train, n_train, Y_q, p, n_epochs_t, e_begin, e_end, q_offset, init, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_trust_penalty(const float* X, int64_t n, int32_t d, const int32_t* emb_idx, int32_t k,
                               int64_t row_begin, int64_t row_end, int32_t knn_mode, const float* Y, int32_t d_emb,
                               int64_t* row_pen, int64_t* penalty, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    if (k < 1 || k > 64 || row_begin < 0 || row_end > n || row_begin > row_end) {
        set_last_error("bad k or row range");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    UMAP_TRY(require_device(X, "X"));
    UMAP_TRY(require_device(emb_idx, "emb_idx"));
    UMAP_TRY(require_device(row_pen, "row_pen"));
    UMAP_TRY(require_device(Y, "Y"));
    UMAP_TRY(trust_penalty(X, n, d, emb_idx, k, row_begin, row_end, row_pen, penalty, knn_mode, Y, d_emb, s));
    return UMAP_OK;
}

}  // extern "C"

namespace umapb200 {
namespace {

// a3..a8 from a kNN graph already on the device (idx int32, dist fp32, n x k, rows sorted).
umap_status fit_from_knn(const int32_t* idx, const float* dist, int64_t n, const umap_params& p, float* Yd,
                         umap_fit_stats& st, Timer& tm, cudaStream_t s, const int32_t* labels = nullptr)
{
    const int k = p.n_neighbors, dim = p.n_components;
    // a3 + a4
    Scratch acol, aw;
    UMAP_TRY(acol.alloc(sizeof(int32_t) * (size_t)n * k, s));
    UMAP_TRY(aw.alloc(sizeof(float) * (size_t)n * k, s));
    UMAP_TRY(smooth_knn(dist, idx, n, k, nullptr, nullptr, aw.as<float>(), acol.as<int32_t>(), s));
    tm.lap(&st.ms_smooth);
    // a5
    const int64_t cap = 2 * n * (int64_t)k;
    Scratch indptr, col, val;
    UMAP_TRY(indptr.alloc(sizeof(int64_t) * (size_t)(n + 1), s));
    UMAP_TRY(col.alloc(sizeof(int32_t) * (size_t)cap, s));
    UMAP_TRY(val.alloc(sizeof(float) * (size_t)cap, s));
    int64_t nnz = 0;
    UMAP_TRY(fuzzy_union(acol.as<int32_t>(), aw.as<float>(), n, k, indptr.as<int64_t>(), col.as<int32_t>(),
                         val.as<float>(), cap, &nnz, s));
    Scratch sindptr, scol, sval;
    const int64_t* g_indptr = indptr.as<int64_t>();
    const int32_t* g_col = col.as<int32_t>();
    const float* g_val = val.as<float>();
    if (labels) {  // supervised: label-adjusted B (R17)
        UMAP_TRY(sindptr.alloc(sizeof(int64_t) * (size_t)(n + 1), s));
        UMAP_TRY(scol.alloc(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1), s));
        UMAP_TRY(sval.alloc(sizeof(float) * (size_t)std::max<int64_t>(nnz, 1), s));
        UMAP_TRY(supervised_adjust(g_indptr, g_col, g_val, n, labels, p.far_dist, p.unknown_dist,
                                   sindptr.as<int64_t>(), scol.as<int32_t>(), sval.as<float>(), nnz, &nnz, s));
        g_indptr = sindptr.as<int64_t>();
        g_col = scol.as<int32_t>();
        g_val = sval.as<float>();
    }
    tm.lap(&st.ms_union);
    // a7 (random, R11, or spectral on the graph the SGD uses, R18)
    if (p.init == 1)
        UMAP_TRY(spectral_init(g_indptr, g_col, g_val, n, dim, p.seed, p.spectral_iters > 0 ? p.spectral_iters : 300,
                               Yd, s));
    else
        UMAP_TRY(random_init(n, dim, p.seed, Yd, s));
    tm.lap(&st.ms_init);
    // a6 + a8
    int64_t positives = 0;
    UMAP_TRY(optimize_layout(g_indptr, g_col, g_val, n, nnz, Yd, &p, 1, p.n_epochs, &positives, s));
    tm.lap(&st.ms_sgd);
    bool bad = false;
    UMAP_TRY(any_nonfinite(Yd, n * (int64_t)dim, &bad, s));
    if (bad) { set_last_error("embedding became non-finite"); return UMAP_ERR_NONFINITE_EMBEDDING; }
    st.nnz = nnz;
    st.positives = positives;
    st.w_max = 1.0f;
    st.a = p.a;
    st.b = p.b;
    st.n_epochs = p.n_epochs;
    return UMAP_OK;
}

}  // namespace
}  // namespace umapb200

extern "C" {

static umap_status fit_impl(const float* X, int64_t n, int32_t d, const int32_t* labels, const umap_params* p_in,
                            float* Y, umap_fit_stats* stats, void* stream);

umap_status umap_fit(const float* X, int64_t n, int32_t d, const umap_params* p_in, float* Y, umap_fit_stats* stats,
                     void* stream)
{
    return fit_impl(X, n, d, nullptr, p_in, Y, stats, stream);
}

umap_status umap_fit_supervised(const float* X, int64_t n, int32_t d, const int32_t* labels, const umap_params* p,
                                float* Y, umap_fit_stats* stats, void* stream)
{
    if (!labels) { set_last_error("labels required"); return UMAP_ERR_INVALID_ARGUMENT; }
    return fit_impl(X, n, d, labels, p, Y, stats, stream);
}

umap_status umap_spectral_init(const int64_t* indptr, const int32_t* col, const float* val, int64_t n, int32_t dim,
                               uint64_t seed, int32_t iters, float* Y, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    if (!dim_supported(dim) || iters < 0 || !indptr || !col || !val || !Y) {
        set_last_error("spectral_init: dim in {1,2,3,4,8,16}, iters >= 0, arrays required");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    UMAP_TRY(require_device(indptr, "indptr"));
    UMAP_TRY(require_device(col, "col"));
    UMAP_TRY(require_device(val, "val"));
    UMAP_TRY(require_device(Y, "Y"));
    UMAP_TRY(spectral_init(indptr, col, val, n, dim, seed, iters, Y, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_supervised_adjust(const int64_t* indptr, const int32_t* col, const float* val, int64_t n,
                                   const int32_t* labels, float far_dist, float unknown_dist, int64_t* out_indptr,
                                   int32_t* out_col, float* out_val, int64_t capacity, int64_t* nnz, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    if (n < 1 || !indptr || !col || !val || !labels || !out_indptr || !out_col || !out_val) {
        set_last_error("null array or n < 1");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    UMAP_TRY(require_device(indptr, "indptr"));
    UMAP_TRY(require_device(col, "col"));
    UMAP_TRY(require_device(val, "val"));
    UMAP_TRY(require_device(labels, "labels"));
    UMAP_TRY(require_device(out_indptr, "out_indptr"));
    UMAP_TRY(require_device(out_col, "out_col"));
    UMAP_TRY(require_device(out_val, "out_val"));
    UMAP_TRY(supervised_adjust(indptr, col, val, n, labels, far_dist, unknown_dist, out_indptr, out_col, out_val,
                               capacity, nnz, s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

static umap_status fit_impl(const float* X, int64_t n, int32_t d, const int32_t* labels, const umap_params* p_in,
                            float* Y, umap_fit_stats* stats, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    UMAP_TRY(check_params(p_in));
    const int64_t launches0 = g_launches;
    umap_params p;
    UMAP_TRY(resolve(p_in, n, &p));
    const int k = p.n_neighbors, dim = p.n_components;
    if (!X || !Y || d < 1) { set_last_error("X, Y required, d >= 1"); return UMAP_ERR_INVALID_ARGUMENT; }
    if (k < 2 || k > 64) { set_last_error("2 <= n_neighbors <= 64"); return UMAP_ERR_K_OUT_OF_RANGE; }
    if (n <= k) { set_last_error("n must exceed n_neighbors"); return UMAP_ERR_TOO_FEW_ROWS; }

    Timer tm(s);
    DevIn Xd;
    UMAP_TRY(Xd.make(X, (size_t)n * d, s));
    DevOut Yd;
    UMAP_TRY(Yd.make(Y, (size_t)n * dim, s));
    bool bad = false;
    UMAP_TRY(any_nonfinite(Xd.p, n * (int64_t)d, &bad, s));
    if (bad) { set_last_error("X contains NaN or Inf"); return UMAP_ERR_NONFINITE_INPUT; }
    umap_fit_stats st{};
    tm.lap(nullptr);  // staging + input check
    // a2 kNN
    Scratch idx, dist;
    UMAP_TRY(idx.alloc(sizeof(int32_t) * (size_t)n * k, s));
    UMAP_TRY(dist.alloc(sizeof(float) * (size_t)n * k, s));
    UMAP_TRY(run_knn(&p, Xd.p, n, Xd.p, n, d, k, 0, 1, 0, 0, idx.as<int32_t>(), dist.as<float>(), s));
    tm.lap(&st.ms_knn);
    // labels on the device (staged if given in host memory)
    const int32_t* lab_d = labels;
    Scratch lab_buf;
    if (labels && !is_device_ptr(labels)) {
        UMAP_TRY(lab_buf.alloc(sizeof(int32_t) * (size_t)n, s));
        UMAP_CUDA_TRY(cudaMemcpyAsync(lab_buf.p, labels, sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice, s));
        lab_d = lab_buf.as<int32_t>();
    }
    UMAP_TRY(fit_from_knn(idx.as<int32_t>(), dist.as<float>(), n, p, Yd.p, st, tm, s, lab_d));
    if (p.trust_k > 0) {  // a10 on the device-resident X and Y (no second staging of X)
        if (2 * (int64_t)p.trust_k >= n || p.trust_k > 64) {
            set_last_error("trust_k: 1 <= trust_k < n/2, trust_k <= 64");
            return UMAP_ERR_K_OUT_OF_RANGE;
        }
        UMAP_TRY(trust_device(Xd.p, d, Yd.p, dim, n, p.trust_k, p.knn_mode, &st.trustworthiness, &st.trust_penalty, s));
        tm.lap(&st.ms_trust);
    }
    UMAP_TRY(Yd.finish(s));
    tm.lap(nullptr);
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    st.ms_total = tm.resolve();
    st.gpu_launches = (int32_t)(g_launches - launches0);
    if (stats) *stats = st;
    return UMAP_OK;
}

umap_status umap_fit_knn(const int32_t* knn_idx, const float* knn_dist, int64_t n, const umap_params* p_in, float* Y,
                         umap_fit_stats* stats, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    UMAP_TRY(check_params(p_in));
    const int64_t launches0 = g_launches;
    umap_params p;
    UMAP_TRY(resolve(p_in, n, &p));
    const int k = p.n_neighbors, dim = p.n_components;
    if (!knn_idx || !knn_dist || !Y) { set_last_error("null array"); return UMAP_ERR_INVALID_ARGUMENT; }
    if (k < 2 || k > 64) { set_last_error("2 <= n_neighbors <= 64"); return UMAP_ERR_K_OUT_OF_RANGE; }
    if (n <= k) { set_last_error("n must exceed n_neighbors"); return UMAP_ERR_TOO_FEW_ROWS; }
    Timer tm(s);
    const int32_t* idx_d = knn_idx;
    Scratch idx_buf;
    if (!is_device_ptr(knn_idx)) {
        UMAP_TRY(idx_buf.alloc(sizeof(int32_t) * (size_t)n * k, s));
        UMAP_CUDA_TRY(cudaMemcpyAsync(idx_buf.p, knn_idx, sizeof(int32_t) * (size_t)n * k, cudaMemcpyHostToDevice, s));
        idx_d = idx_buf.as<int32_t>();
    }
    DevIn dist_d;
    UMAP_TRY(dist_d.make(knn_dist, (size_t)n * k, s));
    UMAP_TRY(validate_knn(idx_d, dist_d.p, n, k, s));
    DevOut Yd;
    UMAP_TRY(Yd.make(Y, (size_t)n * dim, s));
    umap_fit_stats st{};
    tm.lap(nullptr);
    UMAP_TRY(fit_from_knn(idx_d, dist_d.p, n, p, Yd.p, st, tm, s));
    UMAP_TRY(Yd.finish(s));
    tm.lap(nullptr);
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    st.ms_total = tm.resolve();
    st.gpu_launches = (int32_t)(g_launches - launches0);
    if (stats) *stats = st;
    return UMAP_OK;
}

umap_status umap_transform(const float* X_train, const float* Y_train, int64_t n_train, int32_t d, const float* X_q,
                           int64_t n_q, int64_t q_offset, const umap_params* p_in, float* Y_q, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    UMAP_TRY(check_params(p_in));
    umap_params p;
    UMAP_TRY(resolve(p_in, n_train, &p));
    const int k = p.n_neighbors, dim = p.n_components;
    if (!X_train || !Y_train || !X_q || !Y_q || d < 1) { set_last_error("null array"); return UMAP_ERR_INVALID_ARGUMENT; }
    if (k < 1 || k > 64 || k > n_train) { set_last_error("1 <= k <= min(64, n_train)"); return UMAP_ERR_K_OUT_OF_RANGE; }
    if (n_q == 0) return UMAP_OK;
    const int n_t = umap_transform_epoch_count(p.n_epochs, p.transform_epochs, n_train);
    DevIn Xtr, Ytr, Xq;
    UMAP_TRY(Xtr.make(X_train, (size_t)n_train * d, s));
    UMAP_TRY(Ytr.make(Y_train, (size_t)n_train * dim, s));
    UMAP_TRY(Xq.make(X_q, (size_t)n_q * d, s));
    DevOut Yq;
    UMAP_TRY(Yq.make(Y_q, (size_t)n_q * dim, s));
    bool bad = false;
    UMAP_TRY(any_nonfinite(Xq.p, n_q * (int64_t)d, &bad, s));
    if (bad) { set_last_error("X_q contains NaN or Inf"); return UMAP_ERR_NONFINITE_INPUT; }
    Scratch idx, dist, w;
    UMAP_TRY(idx.alloc(sizeof(int32_t) * (size_t)n_q * k, s));
    UMAP_TRY(dist.alloc(sizeof(float) * (size_t)n_q * k, s));
    UMAP_TRY(w.alloc(sizeof(float) * (size_t)n_q * k, s));
    UMAP_TRY(run_knn(&p, Xq.p, n_q, Xtr.p, n_train, d, k, 0, 0, 0, 0, idx.as<int32_t>(), dist.as<float>(), s));
    UMAP_TRY(smooth_knn(dist.as<float>(), idx.as<int32_t>(), n_q, k, nullptr, nullptr, w.as<float>(), nullptr, s));
    UMAP_TRY(transform_optimize(idx.as<int32_t>(), w.as<float>(), n_q, k, Ytr.p, n_train, Yq.p, &p, n_t, 1, n_t,
                                q_offset, 1, s));
    UMAP_TRY(Yq.finish(s));
    UMAP_CUDA_TRY(cudaStreamSynchronize(s));
    return UMAP_OK;
}

umap_status umap_trustworthiness(const float* X, int32_t d, const float* Y, int32_t d_emb, int64_t n, int32_t k,
                                 int32_t knn_mode, double* T, int64_t* penalty, void* stream)
{
    UMAP_TRY(require_cuda());
    cudaStream_t s = (cudaStream_t)stream;
    if (!X || !Y || !T || d < 1 || d_emb < 1) { set_last_error("null array"); return UMAP_ERR_INVALID_ARGUMENT; }
    if (k < 1 || k > 64 || 2 * (int64_t)k >= n) { set_last_error("1 <= k < n/2, k <= 64"); return UMAP_ERR_K_OUT_OF_RANGE; }
    if (knn_mode != UMAP_KNN_EXACT_FP32 && knn_mode != UMAP_KNN_TENSOR_BF16) {
        set_last_error("unknown knn_mode");
        return UMAP_ERR_INVALID_ARGUMENT;
    }
    DevIn Xd, Yd;
    UMAP_TRY(Xd.make(X, (size_t)n * d, s));
    UMAP_TRY(Yd.make(Y, (size_t)n * d_emb, s));
    return trust_device(Xd.p, d, Yd.p, d_emb, n, k, knn_mode, T, penalty, s);
}

}  // extern "C"

namespace umapb200 {
namespace {

// a10 on device-resident X (n x d) and Y (n x d_emb): embedding kNN, then the input-space
// rank penalty S and T = 1 - 2 S / (n k (2n - 3k - 1)) (R16).
umap_status trust_device(const float* Xd, int d, const float* Yd, int d_emb, int64_t n, int k, int knn_mode,
                         double* T, int64_t* penalty, cudaStream_t s)
{
    Scratch eidx, edist;
    UMAP_TRY(eidx.alloc(sizeof(int32_t) * (size_t)n * k, s));
    UMAP_TRY(edist.alloc(sizeof(float) * (size_t)n * k, s));
    {
        umap_params pe;
        umap_params_default(&pe);
        UMAP_TRY(run_knn(&pe, Yd, n, Yd, n, d_emb, k, 0, 1, 0, 1, eidx.as<int32_t>(), edist.as<float>(), s));
    }
    int64_t S = 0;
    UMAP_TRY(trust_penalty(Xd, n, d, eidx.as<int32_t>(), k, 0, n, nullptr, &S, knn_mode, Yd, d_emb, s));
    *T = umap_trust_from_penalty(S, n, k);
    if (penalty) *penalty = S;
    return UMAP_OK;
}

}  // namespace
}  // namespace umapb200
