// lj_common.cuh -- shared device code of the learned-join library (sm_100a).
//
// Bit-exact model evaluation: numpy evaluates `a*x + b` as a rounded
// multiply then a rounded add, so every model expression below uses the
// explicit __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn intrinsics, which nvcc
// never contracts into DFMA.  Reference paths are relative to
// /root/reference/pkg/src/learned_joins/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "../../include/lj_b200.h"

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;
typedef uint16_t u16;

namespace lj {

// --------------------------------------------------------------- errors
void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define LJ_CK(call)                                                                \
    do {                                                                           \
        cudaError_t _e = (call);                                                   \
        if (_e != cudaSuccess) return ::lj::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)
#define LJ_CK_LAUNCH() LJ_CK(cudaGetLastError())
#define LJ_REQUIRE(cond, msg)                  \
    do {                                       \
        if (!(cond)) {                         \
            ::lj::set_error(msg);              \
            return LJ_E_INVALID;               \
        }                                      \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// True the first time it is called for the current device (bit in `mask`):
// kernel attributes (dynamic shared memory) are set per device.
inline bool once_per_device(unsigned long long &mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ULL << (dev & 63);
    if (mask & bit) return false;
    mask |= bit;
    return true;
}

// Number of SMs of the current device (cached per process).
int sm_count();
// Grid for a grid-stride kernel: enough blocks to fill every SM
// `per_sm` times, never more than needed.
inline unsigned grid_for(i64 n, int threads, int per_sm) {
    i64 need = (n + threads - 1) / threads;
    i64 cap = (i64)sm_count() * per_sm;
    if (need < 1) need = 1;
    return (unsigned)(need < cap ? need : cap);
}

// ------------------------------------------------------------ bit helpers

// util.py:30-44 SplitMix64 finaliser
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z = z + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// numpy float64 -> int64 cast as executed on x86-64 (cvttsd2si): truncation,
// INT64_MIN ("integer indefinite") for NaN / out of range.  The reference
// hits that path for far-out probe keys (models.py:123).
__device__ __forceinline__ i64 f64_to_i64(double d) {
    return (d >= -9223372036854775808.0 && d < 9223372036854775808.0) ? (i64)d : INT64_MIN;
}
__device__ __forceinline__ double u64_to_f64(u64 k) { return __ull2double_rn(k); }
__device__ __forceinline__ double i64_to_f64(i64 k) { return __ll2double_rn(k); }
__device__ __forceinline__ i64 clip_i64(i64 v, i64 lo, i64 hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}
// np.clip(v, lo, hi) == minimum(maximum(v, lo), hi), NaN-propagating
__device__ __forceinline__ double clip_f64(double v, double lo, double hi) {
    double t = v > lo ? v : lo;
    if (v != v) t = v;
    return t < hi ? t : hi;
}

// Read-only loads through the non-coherent path.
__device__ __forceinline__ u64 ldg(const u64 *p) { return __ldg(reinterpret_cast<const unsigned long long *>(p)); }
__device__ __forceinline__ ulonglong2 ldg2(const u64 *p) {
    return __ldg(reinterpret_cast<const ulonglong2 *>(p));
}
// Streaming (evict-first) loads for data read exactly once.
__device__ __forceinline__ u64 ld_stream(const u64 *p) {
    return __ldcs(reinterpret_cast<const unsigned long long *>(p));
}

// ------------------------------------------------------------------ RMI

// models.py:112-114: leaf = clip(floor(rs*x + ri), 0, m-1)
// floor + clip in f64 + x86 cast == saturating cvt.rmi + integer clamp for
// every raw (NaN: both end at 0 after the clamp; NaN parameters would index
// out of bounds in the reference, the clamp keeps the device safe)
__device__ __forceinline__ i64 rmi_route(double rs, double ri, i64 m, double x) {
    const double raw = __dadd_rn(__dmul_rn(rs, x), ri);
    const i64 l = __double2ll_rd(raw);
    return l < 0 ? 0 : (l >= m ? m - 1 : l);
}

// models.py:121-124: pos = clip(rint(slope*x + icpt), clamp_lo, clamp_hi)
// (x86 cast of rint(raw)) == cvt.rni(raw) whenever raw is in [-2^63, 2^63)
// (doubles that close to 2^63 are integers); else the cast's INT64_MIN
__device__ __forceinline__ i64 rmi_leaf_pos(const LjLeaf &lf, double x) {
    const double raw = __dadd_rn(__dmul_rn(lf.slope, x), lf.icpt);
    const i64 p = (raw >= -9223372036854775808.0 && raw < 9223372036854775808.0) ? __double2ll_rn(raw) : INT64_MIN;
    return clip_i64(p, lf.clamp_lo, lf.clamp_hi);
}

// The same position with a SATURATING cast: a raw prediction beyond the
// int64 range clamps to the leaf's bound instead of the x86 cast's
// INT64_MIN (which sends keys far above the training range to clamp_lo).
// Monotone in the key everywhere; the LSJ's internal bins use it (any
// monotone bin function gives the same join), the reference-facing
// predictions keep the reference's cast.
__device__ __forceinline__ i64 rmi_leaf_pos_sat(const LjLeaf &lf, double x) {
    const double raw = __dadd_rn(__dmul_rn(lf.slope, x), lf.icpt);
    if (raw >= 9223372036854775808.0) return lf.clamp_hi;
    if (!(raw >= -9223372036854775808.0)) return lf.clamp_lo;
    return clip_i64(__double2ll_rn(raw), lf.clamp_lo, lf.clamp_hi);
}

__device__ __forceinline__ LjLeaf load_leaf(const LjLeaf *leaves, i64 l) {
    const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(leaves + l);
    ulonglong2 a = __ldg(p), b = __ldg(p + 1);
    LjLeaf lf;
    lf.slope = __longlong_as_double((long long)a.x);
    lf.icpt = __longlong_as_double((long long)a.y);
    lf.clamp_lo = (i64)b.x;
    lf.clamp_hi = (i64)b.y;
    return lf;
}

struct RmiDev {
    double rs, ri;
    i64 m, n;
    const LjLeaf *leaves;
    const i64 *err;
    const double *rootp;  // root {slope, intercept} in device memory, or null
    __host__ RmiDev() {}
    __host__ explicit RmiDev(const LjRmi &r)
        : rs(r.root_slope), ri(r.root_icpt), m(r.m), n(r.n), leaves(r.leaves), err(r.err), rootp(r.root_dev) {}
    // a model fitted on the stream (lj_lsj_run) keeps its root on the device:
    // kernels take it from there before the first evaluation
    __device__ __forceinline__ void fix() {
        if (rootp) {
            rs = rootp[0];
            ri = rootp[1];
        }
    }
    __device__ __forceinline__ i64 route(double x) const { return rmi_route(rs, ri, m, x); }
    __device__ __forceinline__ i64 pos(double x) const {
        return rmi_leaf_pos(load_leaf(leaves, route(x)), x);
    }
    __device__ __forceinline__ i64 pos_sat(double x) const {
        return rmi_leaf_pos_sat(load_leaf(leaves, route(x)), x);
    }
};

// models.py:297: bucket = clip(pos*P // trained_len, 0, P-1), exact int64
// (pos >= 0, so C division is numpy floor division).
__device__ __forceinline__ i64 scale_bucket(i64 pos, i64 P, i64 trained_len) {
    i64 b = pos * P;
    i64 q = b / trained_len;
    if ((b % trained_len != 0) && ((b < 0) != (trained_len < 0))) --q;
    return clip_i64(q, 0, P - 1);
}

// gapped.py:258-261: slot0 = clip(rint(pos / n * L), 0, L-1)
__device__ __forceinline__ i64 grmi_slot_of_pos(i64 pos, i64 n, i64 L) {
    double s = rint(__dmul_rn(__ddiv_rn(i64_to_f64(pos), i64_to_f64(n)), i64_to_f64(L)));
    return f64_to_i64(clip_f64(s, 0.0, i64_to_f64(L - 1)));
}

// The same slot without the division on the common path.  Both the
// reference's RN(RN(pos/n)*L) and z = RN(pos*RN(L/n)) lie within
// 2^-50*L of r = pos*L/n (pos is an integer < 2^53, r <= L).  When z is
// more than g = 2^-47*L away from every half-integer, r is too, and both
// round to the same integer; otherwise (never when n divides L) the
// reference's own operations run.
struct SlotMap {
    i64 n, L;
    double c, g, top;
    __host__ SlotMap() {}
    __host__ SlotMap(i64 n_, i64 L_)
        : n(n_), L(L_), c(n_ > 0 ? (double)L_ / (double)n_ : 0.0),
          g(L_ < ((i64)1 << 52) ? ldexp((double)L_, -47) : INFINITY), top((double)(L_ - 1)) {}
    __device__ __forceinline__ i64 operator()(i64 pos) const {
        const double z = __dmul_rn(i64_to_f64(pos), c);
        const double f = __dadd_rn(z, -floor(z));
        if (fabs(__dadd_rn(f, -0.5)) > g) {  // rint + clip + cast, z finite, L - 1 exact
            const i64 r = __double2ll_rn(z);
            return r < 0 ? 0 : (r > L - 1 ? L - 1 : r);
        }
        return grmi_slot_of_pos(pos, n, L);
    }
};

// ------------------------------------------------------------ L2 policies

// Read-only loads of small, hot structures (models, tables): plain __ldg,
// or with an L2 evict_last policy so a stream of random, touched-once
// index lines (evict_first) does not push them out of L2.
struct LdNc {
    __device__ __forceinline__ u64 u(const u64 *p) const { return ldg(p); }
    __device__ __forceinline__ u32 w(const u32 *p) const { return __ldg(p); }
    __device__ __forceinline__ double d(const double *p) const { return __ldg(p); }
};
struct LdKeep {
    u64 pol;
    __device__ __forceinline__ static LdKeep make() {
        LdKeep l;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(l.pol));
        return l;
    }
    __device__ __forceinline__ u64 u(const u64 *p) const {
        u64 v;
        asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
        return v;
    }
    __device__ __forceinline__ u32 w(const u32 *p) const {
        u32 v;
        asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
        return v;
    }
    __device__ __forceinline__ double d(const double *p) const {
        double v;
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
        return v;
    }
};
// touched-once random lines: evict_first in L2
struct LdOnce {
    u64 pol;
    __device__ __forceinline__ static LdOnce make() {
        LdOnce l;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(l.pol));
        return l;
    }
    __device__ __forceinline__ u32 w(const u32 *p) const {
        u32 v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
        return v;
    }
    __device__ __forceinline__ ulonglong2 q(const ulonglong2 *p) const {
        ulonglong2 v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                     : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol));
        return v;
    }
};

// ------------------------------------------------------------ RadixSpline

struct SplineDev {
    i64 K, n, max_error, radix_bits;
    u64 shift;
    const u64 *keys;
    const double *ranks;
    const u32 *radix;
    const u64 *aux;
    const u32 *sub;
    __host__ SplineDev() {}
    __host__ explicit SplineDev(const LjSpline &s)
        : K(s.npts), n(s.n), max_error(s.max_error), radix_bits(s.radix_bits), shift(s.shift),
          keys(s.keys), ranks(s.ranks), radix(s.radix), aux(s.aux), sub(s.sub) {}

    // first spline point of k's (sub-)radix bucket: a cheap, monotone
    // approximation of where k lands (no search, no division)
    template <class L = LdNc>
    __device__ __forceinline__ i64 bucket_first_point(u64 k, const L &ld = L()) const {
        if (K <= 1) return 0;
        const i64 rmax = ((i64)1 << radix_bits) - 1;
        const u64 raw = shift >= 64 ? 0 : (k >> shift);
        i64 lo;
        const u64 ax = (aux && raw <= (u64)rmax) ? ld.u(aux + raw) : 0;
        if (ax & 0xFF) {
            const int bits = (int)(ax & 0xFF);
            const u64 q = (k >> (shift - (u64)bits)) & ((1ULL << bits) - 1ULL);
            lo = (i64)ld.w(sub + (ax >> 8) + q);
        } else {
            lo = (i64)ld.w(radix + (raw > (u64)rmax ? rmax : (i64)raw));
        }
        return lo < 0 ? 0 : (lo > K - 1 ? K - 1 : lo);
    }

    // models.py:221-248 + _bounded_first_geq :263-282
    template <class L = LdNc>
    __device__ __forceinline__ i64 pos(u64 k, const L &ld = L()) const {
        i64 p;
        if (K == 1) {
            p = (i64)ld.d(ranks);
        } else {
            i64 rmax = ((i64)1 << radix_bits) - 1;
            // np.minimum((k >> shift).astype(int64), rmax); negative values
            // (probe >= 2^63 with shift 0) index from the table's end as
            // Python indexing does
            i64 len = rmax + 2;
            i64 prefix = (i64)(shift >= 64 ? 0 : (k >> shift));
            if (prefix > rmax) prefix = rmax;
            i64 a = prefix < 0 ? prefix + len : prefix;
            i64 b = prefix + 1 < 0 ? prefix + 1 + len : prefix + 1;
            i64 lo, hi;
            const u64 raw = shift >= 64 ? 0 : (k >> shift);
            u64 ax = 0;
            if (aux && raw <= (u64)rmax) ax = ld.u(aux + raw);  // unclamped prefix: sub-table is exact
            if (ax & 0xFF) {
                const int bits = (int)(ax & 0xFF);
                const u64 q = (k >> (shift - (u64)bits)) & ((1ULL << bits) - 1ULL);
                const u32 *s = sub + (ax >> 8) + q;
                lo = (i64)ld.w(s);
                hi = (i64)ld.w(s + 1);
            } else {
                lo = (i64)ld.w(radix + (a < 0 ? 0 : a));
                hi = (i64)ld.w(radix + (b < 0 ? 0 : b));
            }
            if (hi < lo) hi = lo;
            if (hi > K) hi = K;
            while (lo < hi) {
                i64 mid = (lo + hi) >> 1;
                if (ld.u(keys + mid) < k) lo = mid + 1; else hi = mid;
            }
            i64 j = clip_i64(lo, 1, K - 1 > 1 ? K - 1 : 1);
            double x0 = u64_to_f64(ld.u(keys + j - 1)), x1 = u64_to_f64(ld.u(keys + j));
            double kf = u64_to_f64(k);
            double d = __dsub_rn(x1, x0);
            double t = clip_f64(__ddiv_rn(__dsub_rn(kf, x0), d > 1.0 ? d : 1.0), 0.0, 1.0);
            double r0 = ld.d(ranks + j - 1), r1 = ld.d(ranks + j);
            p = f64_to_i64(rint(__dadd_rn(r0, __dmul_rn(t, __dsub_rn(r1, r0)))));
        }
        return clip_i64(p, 0, n - 1);
    }
};

// ------------------------------------------------------------ reductions

// Warp-reduce the 4 checksum words and fold one atomic per warp leader
// of each block into out[4] = {count, sum, xor, steps}.
__device__ __forceinline__ void reduce_checksum(u64 cnt, u64 sum, u64 x, u64 steps, u64 *out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        x ^= __shfl_xor_sync(0xffffffffu, x, o);
        steps += __shfl_xor_sync(0xffffffffu, steps, o);
    }
    __shared__ u64 s_part[4][32];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_part[0][warp] = cnt;
        s_part[1][warp] = sum;
        s_part[2][warp] = x;
        s_part[3][warp] = steps;
    }
    __syncthreads();
    if (warp == 0) {
        int nw = (blockDim.x + 31) >> 5;
        cnt = lane < nw ? s_part[0][lane] : 0;
        sum = lane < nw ? s_part[1][lane] : 0;
        x = lane < nw ? s_part[2][lane] : 0;
        steps = lane < nw ? s_part[3][lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            sum += __shfl_xor_sync(0xffffffffu, sum, o);
            x ^= __shfl_xor_sync(0xffffffffu, x, o);
            steps += __shfl_xor_sync(0xffffffffu, steps, o);
        }
        if (lane == 0) {
            if (cnt) atomicAdd((unsigned long long *)&out[0], (unsigned long long)cnt);
            if (sum) atomicAdd((unsigned long long *)&out[1], (unsigned long long)sum);
            if (x) atomicXor((unsigned long long *)&out[2], (unsigned long long)x);
            if (steps) atomicAdd((unsigned long long *)&out[3], (unsigned long long)steps);
        }
    }
}

}  // namespace lj
