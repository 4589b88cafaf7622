// lj_core.cu -- library plumbing, data-prep kernels, device sort and the
// RMI fit / predict kernels (K10).  Reference paths are relative to
// /root/reference/pkg/src/learned_joins/.
#include <cub/cub.cuh>

#include <cstdio>
#include <mutex>

#include "lj_common.cuh"
#include "../../include/lj_gen.h"

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

// portable normal / lognormal / cluster draws (include/lj_gen.h): the same
// bits as the host generator oracle/lj_gen.c
__global__ void k_fill_normal(double *out, i64 n, i64 offset, u64 seed) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = ljg_normal(seed, (u64)(offset + i));
}

__global__ void k_fill_lognormal(i64 *out, i64 n, i64 offset, u64 seed, double sigma, double scale, double maxv) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = ljg_lognormal_key(seed, (u64)(offset + i), sigma, scale, maxv);
}

// key = centre[cluster] + sigma * normal, or -1 when outside [0, maxv)
__global__ void k_fill_cluster(i64 *out, i64 n, i64 offset, u64 seed, const double *centres, int ncent,
                               double sigma, double maxv) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = ljg_cluster_key(seed, (u64)(offset + i), centres, ncent, sigma, maxv);
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

// Leaf fit (models.py:75-108) over "pieces": leaf l's key range [a, b) is
// cut into ceil((b-a)/FIT_PIECE) pieces (at least one), one block per piece,
// and every per-leaf quantity is combined from its pieces in a fixed order,
// so the fit is deterministic and a leaf holding half of a skewed sample no
// longer serialises on one block.
constexpr i64 FIT_PIECE = 8192;

__global__ void k_piece_count(const i64 *starts, i64 m, i64 *pc) {
    for (i64 l = blockIdx.x * (i64)blockDim.x + threadIdx.x; l <= m; l += (i64)gridDim.x * blockDim.x) {
        if (l == m) {
            pc[l] = 0;
            continue;
        }
        const i64 len = starts[l + 1] - starts[l];
        pc[l] = len <= FIT_PIECE ? 1 : (len + FIT_PIECE - 1) / FIT_PIECE;
    }
}

__device__ __forceinline__ i64 piece_leaf(const i64 *pbase, i64 m, i64 q) {
    i64 lo = 0, hi = m;  // last l with pbase[l] <= q
    while (hi - lo > 1) {
        const i64 mid = (lo + hi) >> 1;
        if (pbase[mid] <= q) lo = mid; else hi = mid;
    }
    return lo;
}

// phase 0: sums of x and rank; phase 1: centred moments around the leaf
// means; phase 2: residual bounds of the finished leaf model
template <int PHASE>
__global__ void __launch_bounds__(FIT_THREADS) k_leaf_piece(const u64 *k, const i64 *rank, i64 m, const i64 *starts,
                                                            const i64 *pbase, const i64 *npieces_dev,
                                                            const double *means, const LjLeaf *leaves, double *part,
                                                            i64 *ipart) {
    const i64 npieces = *npieces_dev;  // pbase[m], on the device: no readback
    for (i64 q = blockIdx.x; q < npieces; q += gridDim.x) {
        const i64 l = piece_leaf(pbase, m, q);
        const i64 j = q - pbase[l];
        const i64 a = starts[l] + j * FIT_PIECE, b = min(starts[l + 1], a + FIT_PIECE);
        if (PHASE < 2) {
            const double mx = PHASE ? means[2 * l] : 0.0, my = PHASE ? means[2 * l + 1] : 0.0;
            double s0 = 0.0, s1 = 0.0;
            for (i64 i = a + threadIdx.x; i < b; i += FIT_THREADS) {
                if (PHASE == 0) {
                    s0 = __dadd_rn(s0, u64_to_f64(k[i]));
                    s1 = __dadd_rn(s1, i64_to_f64(rank[i]));
                } else {
                    const double cx = __dsub_rn(u64_to_f64(k[i]), mx);
                    const double cy = __dsub_rn(i64_to_f64(rank[i]), my);
                    s0 = __dadd_rn(s0, __dmul_rn(cx, cx));
                    s1 = __dadd_rn(s1, __dmul_rn(cx, cy));
                }
            }
            block_sum2<FIT_THREADS>(s0, s1);
            if (threadIdx.x == 0) {
                part[2 * q] = s0;
                part[2 * q + 1] = s1;
            }
        } else {
            __shared__ i64 s_lo[FIT_THREADS], s_hi[FIT_THREADS];
            const LjLeaf lf = leaves[l];
            i64 elo = 0, ehi = 0;
            for (i64 i = a + threadIdx.x; i < b; i += FIT_THREADS) {
                const i64 resid = rank[i] - rmi_leaf_pos(lf, u64_to_f64(k[i]));
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
                ipart[2 * q] = s_lo[0];
                ipart[2 * q + 1] = s_hi[0];
            }
            __syncthreads();
        }
    }
}

// per leaf, pieces combined in order: phase 0 -> means; phase 1 -> the leaf
// (slope clamped >= 0, empty leaves constant at the segment start, clamps);
// phase 2 -> residual bounds
template <int PHASE>
__global__ void k_leaf_combine(const i64 *starts, i64 n, i64 m, const i64 *pbase, const double *part,
                               const i64 *ipart, double *means, LjLeaf *leaves, i64 *err) {
    for (i64 l = blockIdx.x * (i64)blockDim.x + threadIdx.x; l < m; l += (i64)gridDim.x * blockDim.x) {
        const i64 a = starts[l], b = starts[l + 1];
        const bool ne = b > a;
        if (PHASE == 2) {
            i64 elo = 0, ehi = 0;
            for (i64 q = pbase[l]; q < pbase[l + 1]; ++q) {
                elo = min(elo, ipart[2 * q]);
                ehi = max(ehi, ipart[2 * q + 1]);
            }
            err[2 * l] = elo;
            err[2 * l + 1] = ehi;
            continue;
        }
        double s0 = 0.0, s1 = 0.0;
        for (i64 q = pbase[l]; q < pbase[l + 1]; ++q) {
            s0 = __dadd_rn(s0, part[2 * q]);
            s1 = __dadd_rn(s1, part[2 * q + 1]);
        }
        if (PHASE == 0) {
            const double c = i64_to_f64(b - a), d = c > 1.0 ? c : 1.0;
            means[2 * l] = ne ? __ddiv_rn(s0, d) : 0.0;
            means[2 * l + 1] = ne ? __ddiv_rn(s1, d) : 0.0;
            continue;
        }
        const double mx = means[2 * l], my = means[2 * l + 1];
        double slope = s0 > 0.0 ? __ddiv_rn(s1, s0) : 0.0;
        if (slope < 0.0) slope = 0.0;
        const double icpt = __dsub_rn(my, __dmul_rn(slope, mx));
        const i64 seg = a < n - 1 ? a : n - 1;
        LjLeaf lf;
        lf.slope = ne ? slope : 0.0;
        lf.icpt = ne ? icpt : i64_to_f64(seg);
        lf.clamp_lo = ne ? a : seg;
        lf.clamp_hi = ne ? b - 1 : seg;
        leaves[l] = lf;
    }
}

// K12 (rmi-inlj): baselines.py:96-157 over the SORTED R.
// predict_many (models.py:126-135) gives [lo, hi]; the lower bound in
// [lo, hi+1) costs one step per bisection plus one verification compare
// (_bounded_binary_search); a hit emits the whole equal run.  One lane per
// probe, checksum + steps reduced on device.
__global__ void k_rmi_probe(RmiDev r, const u64 *__restrict__ rk, const u64 *__restrict__ rp, i64 n,
                            const u64 *__restrict__ sk, const u64 *__restrict__ sp, i64 ns, u64 *out) {
    u64 cnt = 0, sum = 0, x = 0, steps = 0;
    const i64 last = r.n - 1;
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < ns; t += (i64)gridDim.x * blockDim.x) {
        const u64 key = ld_stream(sk + t), ps = ld_stream(sp + t);
        const double xf = u64_to_f64(key);
        const i64 l = r.route(xf);
        const i64 p = rmi_leaf_pos(load_leaf(r.leaves, l), xf);
        i64 left = clip_i64(p + __ldg(r.err + 2 * l), 0, last);
        i64 right = clip_i64(p + __ldg(r.err + 2 * l + 1), 0, last) + 1;
        while (left < right) {
            const i64 mid = (left + right) >> 1;
            ++steps;
            if (ldg(rk + mid) < key) left = mid + 1; else right = mid;
        }
        ++steps;
        for (i64 i = left; i < n && ldg(rk + i) == key; ++i) {
            const u64 v = ldg(rp + i) + ps;
            ++cnt;
            sum += v;
            x ^= v;
        }
    }
    reduce_checksum(cnt, sum, x, steps, out);
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

int lj_fill_normal(double *out, int64_t n, int64_t offset, uint64_t seed, void *stream) {
    LJ_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return LJ_OK;
    k_fill_normal<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(out, n, offset, seed);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_fill_lognormal(int64_t *out, int64_t n, int64_t offset, uint64_t seed, double sigma, double scale,
                      double maxv, void *stream) {
    LJ_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return LJ_OK;
    k_fill_lognormal<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(out, n, offset, seed, sigma, scale, maxv);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_fill_cluster(int64_t *out, int64_t n, int64_t offset, uint64_t seed, const double *centres, int ncent,
                    double sigma, double maxv, void *stream) {
    LJ_REQUIRE(n >= 0 && ncent >= 1 && (ncent & (ncent - 1)) == 0, "need n >= 0 and a power-of-two centre count");
    if (n == 0) return LJ_OK;
    k_fill_cluster<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(out, n, offset, seed, centres, ncent, sigma,
                                                                        maxv);
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

static i64 max_pieces(i64 n, i64 m) { return m + n / FIT_PIECE + 1; }

static size_t piece_scan_bytes(i64 m) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (i64 *)nullptr, (i64 *)nullptr, (int64_t)(m + 1));
    return t;
}

size_t lj_rmi_fit_workspace_bytes(int64_t n, int64_t m) {
    const size_t r = rank_scan_temp_bytes(n), q = piece_scan_bytes(m);
    return align_up(sizeof(i64) * (size_t)n) + align_up(sizeof(i64) * (size_t)(m + 1)) +
           align_up(sizeof(double) * 2 * FIT_GRID) + align_up(sizeof(double) * 2) +
           2 * align_up(sizeof(i64) * (size_t)(m + 1)) +                       // piece counts / bases
           align_up(sizeof(double) * 2 * (size_t)m) +                          // leaf means
           align_up(sizeof(double) * 2 * (size_t)max_pieces(n, m)) +            // piece sums
           align_up(sizeof(i64) * 2 * (size_t)max_pieces(n, m)) + align_up(r > q ? r : q);
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
    i64 *pcnt = (i64 *)p;
    p += align_up(sizeof(i64) * (size_t)(m + 1));
    i64 *pbase = (i64 *)p;
    p += align_up(sizeof(i64) * (size_t)(m + 1));
    double *lmeans = (double *)p;
    p += align_up(sizeof(double) * 2 * (size_t)m);
    double *ppart = (double *)p;
    p += align_up(sizeof(double) * 2 * (size_t)max_pieces(n, m));
    i64 *ipart = (i64 *)p;
    p += align_up(sizeof(i64) * 2 * (size_t)max_pieces(n, m));
    size_t scan_bytes = rank_scan_temp_bytes(n);

    k_first_occurrence<<<grid_for(n, 256, 8), 256, 0, st>>>(k, n, rank);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceScan::InclusiveScan(p, scan_bytes, rank, rank, MaxOp(), (int64_t)n, st));
    k_root_sum<<<FIT_GRID, FIT_THREADS, 0, st>>>(k, rank, n, m, part);
    k_root_mean<<<1, FIT_THREADS, 0, st>>>(part, n, means);
    k_root_moments<<<FIT_GRID, FIT_THREADS, 0, st>>>(k, rank, n, m, means, part);
    k_root_finish<<<1, FIT_THREADS, 0, st>>>(part, means, root);
    k_leaf_starts<<<grid_for(m + 1, 256, 8), 256, 0, st>>>(k, n, m, root, starts);
    k_piece_count<<<grid_for(m + 1, 256, 8), 256, 0, st>>>(starts, m, pcnt);
    LJ_CK_LAUNCH();
    size_t pq = piece_scan_bytes(m);
    LJ_CK(cub::DeviceScan::ExclusiveSum(p, pq, pcnt, pbase, (int64_t)(m + 1), st));
    // the piece count stays on the device (pbase[m]): a grid-stride launch
    // at its bound keeps the fit asynchronous on the stream
    const i64 pmax = max_pieces(n, m), pcap = (i64)sm_count() * 16;
    const unsigned gp = (unsigned)(pmax < pcap ? pmax : pcap);
    const i64 *npieces = pbase + m;
    const unsigned gl = grid_for(m, 256, 8);
    k_leaf_piece<0><<<gp, FIT_THREADS, 0, st>>>(k, rank, m, starts, pbase, npieces, lmeans, leaves, ppart, ipart);
    k_leaf_combine<0><<<gl, 256, 0, st>>>(starts, n, m, pbase, ppart, ipart, lmeans, leaves, err);
    k_leaf_piece<1><<<gp, FIT_THREADS, 0, st>>>(k, rank, m, starts, pbase, npieces, lmeans, leaves, ppart, ipart);
    k_leaf_combine<1><<<gl, 256, 0, st>>>(starts, n, m, pbase, ppart, ipart, lmeans, leaves, err);
    k_leaf_piece<2><<<gp, FIT_THREADS, 0, st>>>(k, rank, m, starts, pbase, npieces, lmeans, leaves, ppart, ipart);
    k_leaf_combine<2><<<gl, 256, 0, st>>>(starts, n, m, pbase, ppart, ipart, lmeans, leaves, err);
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

int lj_rmi_probe(const LjRmi *model, const uint64_t *r_keys, const uint64_t *r_pay, int64_t nr,
                 const uint64_t *s_keys, const uint64_t *s_pay, int64_t ns, uint64_t *out, int accumulate,
                 void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n == nr, "model must be fitted on the nr sorted R keys");
    cudaStream_t st = as_stream(stream);
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (ns <= 0 || nr <= 0) return LJ_OK;
    k_rmi_probe<<<grid_for(ns, 256, 8), 256, 0, st>>>(RmiDev(*model), r_keys, r_pay, nr, s_keys, s_pay, ns, out);
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
