// lj_core.cu -- library plumbing, data-prep kernels, device sort and the
// RMI fit / predict kernels (K10).  Reference paths are relative to
// /root/reference/pkg/src/learned_joins/.
#include <cub/cub.cuh>

#include <cstdio>
#include <mutex>

#include "lj_common.cuh"

namespace lj {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    char buf[512];
    snprintf(buf, sizeof(buf), "CUDA error %d (%s) in %s at %s:%d", (int)e, cudaGetErrorString(e),
             what, file, line);
    g_err = buf;
    return LJ_E_CUDA;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

struct MaxOp {
    __device__ __forceinline__ i64 operator()(const i64 &a, const i64 &b) const {
        return a > b ? a : b;
    }
};

// ----------------------------------------------------------- data prep

__global__ void k_fill_payloads(u64 *out, i64 n, i64 offset, u64 base) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = mix64((u64)(offset + i) + base) | 1ULL;
}

__global__ void k_fill_mix64(u64 *out, i64 n, i64 offset, u64 seed) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = mix64(seed ^ (u64)(offset + i));
}

__global__ void k_gather_uniform(u64 *out, i64 n, i64 offset, u64 seed, const u64 *src, i64 src_n) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        u64 r = mix64(seed ^ (u64)(offset + i));
        out[i] = src[__umul64hi(r, (u64)src_n)];
    }
}

// ----------------------------------------------------------- RMI predict

__global__ void k_rmi_predict(RmiDev r, const u64 *keys, i64 nk, i64 *pos, i64 *lo, i64 *hi,
                              i64 *leaf) {
    i64 last = r.n - 1;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nk; i += (i64)gridDim.x * blockDim.x) {
        double x = u64_to_f64(keys[i]);
        i64 l = r.route(x);
        i64 p = rmi_leaf_pos(load_leaf(r.leaves, l), x);
        if (pos) pos[i] = p;
        if (lo) lo[i] = clip_i64(p + r.err[2 * l], 0, last);
        if (hi) hi[i] = clip_i64(p + r.err[2 * l + 1], 0, last);
        if (leaf) leaf[i] = l;
    }
}

__global__ void k_rmi_partition(RmiDev r, const u64 *keys, i64 nk, i64 P, i64 *out) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nk; i += (i64)gridDim.x * blockDim.x)
        out[i] = scale_bucket(r.pos(u64_to_f64(keys[i])), P, r.n);
}

// ------------------------------------------------------------- RMI fit (K10)
//
// models.py:57-110 on device.  Reductions use a fixed partition of the
// input and a fixed combine order, so a fit is deterministic run to run.
// (Summation order differs from numpy's pairwise sums, so parameters agree
// with the reference to rounding; join results do not depend on them.)

constexpr int FIT_GRID = 1024;
constexpr int FIT_THREADS = 256;

// first-occurrence flag -> index, max-scanned into the rank (models.py:65)
__global__ void k_first_occurrence(const u64 *k, i64 n, i64 *r) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        r[i] = (i == 0 || k[i] != k[i - 1]) ? i : 0;
}

template <int NT>
__device__ __forceinline__ void block_sum2(double &a, double &b) {
    __shared__ double sa[NT], sb[NT];
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
#pragma unroll
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            sa[threadIdx.x] += sa[threadIdx.x + s];
            sb[threadIdx.x] += sb[threadIdx.x + s];
        }
        __syncthreads();
    }
    a = sa[0];
    b = sb[0];
    __syncthreads();
}

__device__ __forceinline__ double root_y(i64 rank, i64 n, i64 m) {
    // ranks / n * m (models.py:67)
    return __dmul_rn(__ddiv_rn(i64_to_f64(rank), i64_to_f64(n)), i64_to_f64(m));
}

// pass 1: partial sums of x and y over a fixed block partition
__global__ void k_root_sum(const u64 *k, const i64 *rank, i64 n, i64 m, double *part) {
    double sx = 0.0, sy = 0.0;
    for (i64 i = blockIdx.x * (i64)FIT_THREADS + threadIdx.x; i < n; i += (i64)FIT_GRID * FIT_THREADS) {
        sx = __dadd_rn(sx, u64_to_f64(k[i]));
        sy = __dadd_rn(sy, root_y(rank[i], n, m));
    }
    block_sum2<FIT_THREADS>(sx, sy);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = sx;
        part[2 * blockIdx.x + 1] = sy;
    }
}

// combine partials (fixed order) -> means
__global__ void k_root_mean(const double *part, i64 n, double *means) {
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < FIT_GRID; i += FIT_THREADS) {
        a = __dadd_rn(a, part[2 * i]);
        b = __dadd_rn(b, part[2 * i + 1]);
    }
    block_sum2<FIT_THREADS>(a, b);
    if (threadIdx.x == 0) {
        means[0] = __ddiv_rn(a, i64_to_f64(n));
        means[1] = __ddiv_rn(b, i64_to_f64(n));
    }
}

// pass 2: partial centred moments
__global__ void k_root_moments(const u64 *k, const i64 *rank, i64 n, i64 m, const double *means,
                               double *part) {
    double mx = means[0], my = means[1];
    double var = 0.0, cov = 0.0;
    for (i64 i = blockIdx.x * (i64)FIT_THREADS + threadIdx.x; i < n; i += (i64)FIT_GRID * FIT_THREADS) {
        double dx = __dsub_rn(u64_to_f64(k[i]), mx);
        var = __dadd_rn(var, __dmul_rn(dx, dx));
        cov = __dadd_rn(cov, __dmul_rn(dx, __dsub_rn(root_y(rank[i], n, m), my)));
    }
    block_sum2<FIT_THREADS>(var, cov);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = var;
        part[2 * blockIdx.x + 1] = cov;
    }
}

// models.py:28-36 centred least squares, slope clamped >= 0
__global__ void k_root_finish(const double *part, const double *means, double *root) {
    double var = 0.0, cov = 0.0;
    for (int i = threadIdx.x; i < FIT_GRID; i += FIT_THREADS) {
        var = __dadd_rn(var, part[2 * i]);
        cov = __dadd_rn(cov, part[2 * i + 1]);
    }
    block_sum2<FIT_THREADS>(var, cov);
    if (threadIdx.x == 0) {
        double slope = var > 0.0 ? __ddiv_rn(cov, var) : 0.0;
        if (slope < 0.0) slope = 0.0;
        root[0] = slope;
        root[1] = __dsub_rn(means[1], __dmul_rn(slope, means[0]));
    }
}

// starts[l] = first i with route(x_i) >= l, l in [0, m] (leaf ids are
// nondecreasing over sorted keys, models.py:70-72)
__global__ void k_leaf_starts(const u64 *k, i64 n, i64 m, const double *root, i64 *starts) {
    double rs = root[0], ri = root[1];
    for (i64 l = blockIdx.x * (i64)blockDim.x + threadIdx.x; l <= m; l += (i64)gridDim.x * blockDim.x) {
        i64 lo = 0, hi = n;
        while (lo < hi) {
            i64 mid = (lo + hi) >> 1;
            if (rmi_route(rs, ri, m, u64_to_f64(k[mid])) < l) lo = mid + 1; else hi = mid;
        }
        starts[l] = lo;
    }
}

// One block per leaf: means, centred moments, slope/intercept, clamps
// (models.py:75-98) and the exact residual bounds (:101-108).
__global__ void __launch_bounds__(FIT_THREADS) k_leaf_fit(const u64 *k, const i64 *rank, i64 n, i64 m,
                                                          const i64 *starts, LjLeaf *leaves, i64 *err) {
    for (i64 l = blockIdx.x; l < m; l += gridDim.x) {
        i64 a = starts[l], b = starts[l + 1];
        bool ne = b > a;
        double sx = 0.0, sy = 0.0;
        for (i64 i = a + threadIdx.x; i < b; i += FIT_THREADS) {
            sx = __dadd_rn(sx, u64_to_f64(k[i]));
            sy = __dadd_rn(sy, i64_to_f64(rank[i]));
        }
        block_sum2<FIT_THREADS>(sx, sy);
        double c = i64_to_f64(b - a);
        double d = c > 1.0 ? c : 1.0;
        double mx = ne ? __ddiv_rn(sx, d) : 0.0, my = ne ? __ddiv_rn(sy, d) : 0.0;
        double var = 0.0, cov = 0.0;
        for (i64 i = a + threadIdx.x; i < b; i += FIT_THREADS) {
            double cx = __dsub_rn(u64_to_f64(k[i]), mx);
            double cy = __dsub_rn(i64_to_f64(rank[i]), my);
            var = __dadd_rn(var, __dmul_rn(cx, cx));
            cov = __dadd_rn(cov, __dmul_rn(cx, cy));
        }
        block_sum2<FIT_THREADS>(var, cov);
        double slope = var > 0.0 ? __ddiv_rn(cov, var) : 0.0;
        if (slope < 0.0) slope = 0.0;
        double icpt = __dsub_rn(my, __dmul_rn(slope, mx));
        i64 seg = a < n - 1 ? a : n - 1;
        LjLeaf lf;
        lf.slope = ne ? slope : 0.0;
        lf.icpt = ne ? icpt : i64_to_f64(seg);
        lf.clamp_lo = ne ? a : seg;
        lf.clamp_hi = ne ? b - 1 : seg;
        // residual bounds
        __shared__ i64 s_lo[FIT_THREADS], s_hi[FIT_THREADS];
        i64 elo = 0, ehi = 0;
        for (i64 i = a + threadIdx.x; i < b; i += FIT_THREADS) {
            i64 resid = rank[i] - rmi_leaf_pos(lf, u64_to_f64(k[i]));
            elo = resid < elo ? resid : elo;
            ehi = resid > ehi ? resid : ehi;
        }
        s_lo[threadIdx.x] = elo;
        s_hi[threadIdx.x] = ehi;
        __syncthreads();
        for (int s = FIT_THREADS / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                s_lo[threadIdx.x] = min(s_lo[threadIdx.x], s_lo[threadIdx.x + s]);
                s_hi[threadIdx.x] = max(s_hi[threadIdx.x], s_hi[threadIdx.x + s]);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            leaves[l] = lf;
            err[2 * l] = s_lo[0];
            err[2 * l + 1] = s_hi[0];
        }
        __syncthreads();
    }
}

static size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

static size_t rank_scan_temp_bytes(i64 n) {
    size_t t = 0;
    cub::DeviceScan::InclusiveScan((void *)nullptr, t, (i64 *)nullptr, (i64 *)nullptr, MaxOp(), (int64_t)n);
    return t;
}

}  // namespace lj

using namespace lj;

extern "C" {

const char *lj_last_error(void) { return lj::g_err.c_str(); }

int lj_version(void) { return 1; }

int lj_device_ok(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return 0;
    }
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    return major == 10 ? 1 : 0;
}

int lj_fill_payloads(uint64_t *out, int64_t n, int64_t offset, uint64_t seed, void *stream) {
    LJ_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return LJ_OK;
    k_fill_payloads<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(out, n, offset, mix64(seed));
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_fill_mix64(uint64_t *out, int64_t n, int64_t offset, uint64_t seed, void *stream) {
    LJ_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return LJ_OK;
    k_fill_mix64<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(out, n, offset, seed);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_gather_uniform(uint64_t *out, int64_t n, int64_t offset, uint64_t seed, const uint64_t *src,
                      int64_t src_n, void *stream) {
    LJ_REQUIRE(n >= 0 && src_n > 0, "need n >= 0 and a nonempty source");
    if (n == 0) return LJ_OK;
    k_gather_uniform<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(out, n, offset, seed, src, src_n);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

size_t lj_sort_pairs_workspace_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceRadixSort::SortPairs((void *)nullptr, t, (const u64 *)nullptr, (u64 *)nullptr,
                                    (const u64 *)nullptr, (u64 *)nullptr, (int64_t)n, 0, 64);
    return t + 256;
}

int lj_sort_pairs(const uint64_t *keys_in, const uint64_t *pay_in, uint64_t *keys_out,
                  uint64_t *pay_out, int64_t n, int begin_bit, int end_bit, void *ws,
                  size_t ws_bytes, void *stream) {
    LJ_REQUIRE(n >= 0, "n must be >= 0");
    LJ_REQUIRE(0 <= begin_bit && begin_bit < end_bit && end_bit <= 64, "bad bit range");
    if (n == 0) return LJ_OK;
    size_t t = 0;
    LJ_CK(cub::DeviceRadixSort::SortPairs((void *)nullptr, t, keys_in, keys_out, pay_in, pay_out,
                                          (int64_t)n, begin_bit, end_bit, as_stream(stream)));
    if (t > ws_bytes) {
        set_error("lj_sort_pairs: workspace too small");
        return LJ_E_WORKSPACE;
    }
    LJ_CK(cub::DeviceRadixSort::SortPairs(ws, t, keys_in, keys_out, pay_in, pay_out, (int64_t)n,
                                          begin_bit, end_bit, as_stream(stream)));
    return LJ_OK;
}

size_t lj_rmi_fit_workspace_bytes(int64_t n, int64_t m) {
    return align_up(sizeof(i64) * (size_t)n) + align_up(sizeof(i64) * (size_t)(m + 1)) +
           align_up(sizeof(double) * 2 * FIT_GRID) + align_up(sizeof(double) * 2) +
           align_up(rank_scan_temp_bytes(n));
}

int lj_rmi_fit(const uint64_t *k, int64_t n, int64_t m, double *root, LjLeaf *leaves, int64_t *err,
               void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(n >= 1, "cannot train on an empty key array");
    LJ_REQUIRE(m >= 1, "fanout must be >= 1");
    if (ws_bytes < lj_rmi_fit_workspace_bytes(n, m)) {
        set_error("lj_rmi_fit: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    char *p = (char *)ws;
    i64 *rank = (i64 *)p;
    p += align_up(sizeof(i64) * (size_t)n);
    i64 *starts = (i64 *)p;
    p += align_up(sizeof(i64) * (size_t)(m + 1));
    double *part = (double *)p;
    p += align_up(sizeof(double) * 2 * FIT_GRID);
    double *means = (double *)p;
    p += align_up(sizeof(double) * 2);
    size_t scan_bytes = rank_scan_temp_bytes(n);

    k_first_occurrence<<<grid_for(n, 256, 8), 256, 0, st>>>(k, n, rank);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceScan::InclusiveScan(p, scan_bytes, rank, rank, MaxOp(), (int64_t)n, st));
    k_root_sum<<<FIT_GRID, FIT_THREADS, 0, st>>>(k, rank, n, m, part);
    k_root_mean<<<1, FIT_THREADS, 0, st>>>(part, n, means);
    k_root_moments<<<FIT_GRID, FIT_THREADS, 0, st>>>(k, rank, n, m, means, part);
    k_root_finish<<<1, FIT_THREADS, 0, st>>>(part, means, root);
    k_leaf_starts<<<grid_for(m + 1, 256, 8), 256, 0, st>>>(k, n, m, root, starts);
    unsigned g = (unsigned)(m < 65535 * 4 ? m : 65535 * 4);
    k_leaf_fit<<<g, FIT_THREADS, 0, st>>>(k, rank, n, m, starts, leaves, err);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_rmi_predict(const LjRmi *model, const uint64_t *keys, int64_t nk, int64_t *pos, int64_t *lo,
                   int64_t *hi, int64_t *leaf, void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n >= 1, "model is not fitted");
    LJ_REQUIRE(model->err || (!lo && !hi), "lo/hi need the model's error bounds");
    if (nk <= 0) return LJ_OK;
    k_rmi_predict<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(RmiDev(*model), keys, nk, pos,
                                                                        lo, hi, leaf);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_rmi_partition_index(const LjRmi *model, const uint64_t *keys, int64_t nk, int64_t P,
                           int64_t *out, void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n >= 1, "model is not fitted");
    LJ_REQUIRE(P >= 1, "num_partitions must be >= 1");
    if (nk <= 0) return LJ_OK;
    k_rmi_partition<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(RmiDev(*model), keys, nk, P, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

}  // extern "C"
