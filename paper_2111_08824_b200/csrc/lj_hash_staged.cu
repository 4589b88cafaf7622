// lj_hash_staged.cu -- the grouped learned-hash probe (C3 hot path).
// Reference: learned_hash.py:81-96 (probe_batch), models.py:221-248
// (RadixSpline predict), bench.py:202-221 (_run_spline_hash_inlj).
//
// Two structures beside the reference's chains (lj_spline.cu):
//
// 1. The PROBE TABLE ("slots"), built once with the index (untimed, as the
//    reference's build): the entries in key order, entry j at
//        slot_j = max(2 * pos_j, slot_{j-1} + 1),   pos_j = spline pos of key_j
//    (a prefix max: slot_j = j + max_{i<=j}(2 pos_i - i)), gap slots holding
//    the key to their left with payload 0 (leading gaps: key_0), then a
//    terminating pair of reserved keys ~0.  A key k lies at or after slot
//    2*pos(k) (pos is monotone, so every earlier entry has a smaller key and
//    a slot no later), every slot before it holds a smaller key, equal keys
//    are adjacent REAL slots: the probe reads the 32-B aligned slot pair at
//    2*pos(k) and scans forward over keys < k, counting keys == k with a
//    nonzero payload, until a key > k.  The match set is exactly the chain
//    scan's -- every R entry whose key equals k, since the chain of pos(k)
//    holds every entry with key k -- so the checksum words are identical;
//    one dependent 32-B load replaces starts[pos], starts[pos+1] and the
//    chain entries.  Needs every build payload != 0 (the gap marker);
//    otherwise the index keeps the chains only and the chained probe runs.
//
// 2. WINDOW STAGING: S arrives grouped into equi-depth KEY windows (the
//    one-pass claims partition of lj_part_est.cuh with the key-range bins
//    of lj_keybin.cuh).  Per window, a tiny kernel records the spline points
//    the window's keys can need (the lower bound of every key in [klo, khi]
//    and its predecessor) and a 1024-cell table over [klo, khi] giving each
//    cell's lower-bound range.  The probe CTA bulk-copies a window's points
//    (keys u64 + ranks f64) and cells into shared memory once per window
//    and evaluates models.py:221-248 there -- the same first spline key >= k
//    (hence the same pos, bit for bit, with the reference's float64
//    operations) without a global load; records outside the staged range
//    (overflow area, unstageable windows) take the global evaluation.
//
// Work is handed out in window order (pieces of HS_PIECE records) from one
// counter, so all SMs work in the same one or two windows and their slot
// lines stay in L2.
#include <cub/cub.cuh>

#include "lj_common.cuh"
#include "lj_keybin.cuh"
#include "lj_pipe.cuh"

namespace lj {

static inline size_t part_align_c(size_t v) { return (v + 255) & ~(size_t)255; }

// tuning constants (build-time; tools/gpu_hash_variants.sh measures variants)
#ifndef LJ_HS_NT
#define LJ_HS_NT 1024
#endif
#ifndef LJ_HS_CTAS
#define LJ_HS_CTAS 1
#endif
#ifndef LJ_HS_U
#define LJ_HS_U 3
#endif
#ifndef LJ_HS_D
#define LJ_HS_D 1
#endif
#ifndef LJ_HS_PIECE
#define LJ_HS_PIECE 98304  // a multiple of HS_NT * HS_U (no partly filled last iteration); about 15 M records in flight
                           // over the GPU keep the live windows of the probe table in L2 (73728: 20.16, 98304: 19.97,
                           // 122880: 20.05 ms)
#endif
#ifndef LJ_HS_NC
#define LJ_HS_NC 32768  // lower-bound cells per window (64 KB of shared memory; 4096 / 8192 / 16384 / 32768: 18.63 / 18.51 / 18.34 / 18.22 ms)
#endif
#ifndef LJ_HS_SPREAD
#define LJ_HS_SPREAD 2  // probe-table slots per position (the first slot of a position is even: one 32-B pair)
#endif
#ifndef LJ_HS_ROUNDS
#define LJ_HS_ROUNDS 3  // forward slot scan: 3 = one pair per LANE per round (the lane's first unfinished probe selected
                        // into one register set and followed to its end: a round is one pair scan, not one per probe
                        // position u at 3-9 active lanes; 22.07 ms with 2048 cells), 1 = one pair per unfinished probe
                        // of the thread per round (22.84 ms), 2 = unfinished probes compacted across the warp (29.9 ms: a
                        // lane's dependent loads no longer overlap), 0 = slot by slot
#endif
#ifndef LJ_HS_LDV
#define LJ_HS_LDV 1
#endif
// the 32-B slot-pair load (LJ_HS_LDV: cache-hint variants, measured)
#if LJ_HS_LDV == 1
#define LJ_HS_LD "ld.global.nc.L1::no_allocate.v4.u64"
#elif LJ_HS_LDV == 2
#define LJ_HS_LD "ld.global.nc.L1::evict_first.v4.u64"
#elif LJ_HS_LDV == 3
#define LJ_HS_LD "ld.global.nc.L1::evict_last.v4.u64"
#elif LJ_HS_LDV == 4
#define LJ_HS_LD "ld.global.v4.u64"
#elif LJ_HS_LDV == 5
#define LJ_HS_LD "ld.global.L1::no_allocate.v4.u64"
#else
#define LJ_HS_LD "ld.global.nc.v4.u64"
#endif
#ifndef LJ_HS_PADB
#define LJ_HS_PADB 0  // (diagnostic) unused shared memory: a larger carve-out leaves less L1 for the slot loads in flight
#endif
#ifndef LJ_HS_LAYOUT
#define LJ_HS_LAYOUT 0  // probe table: 0 = entries pushed forward in key order; 1 (ablation) = home pairs + tails: no
                        // displacement, but 18.4 % of C3's probes go on to a tail (chains >= 3, rank >= 1) against 16.1 %
                        // past the first pair here, and a tail is another line: 23.6 vs 22.8 ms
#endif
#if LJ_HS_LAYOUT == 1 && ((LJ_HS_ROUNDS != 1 && LJ_HS_ROUNDS != 3) || LJ_HS_SPREAD != 2)
#error "the home-pair probe table is probed in rounds of pairs at two slots per position"
#endif
constexpr int HS_NT = LJ_HS_NT;
constexpr int HS_CTAS = LJ_HS_CTAS;  // CTAs per SM
constexpr int HS_U = LJ_HS_U;        // probes per thread per iteration
constexpr int HS_D = LJ_HS_D;        // iterations of records in flight (cp.async)
constexpr int HS_TT = HS_NT * HS_U;  // records per iteration
// Tuning builds whose record ring (HS_D stages x HS_TT records) holds a power-of-two record count (256 / 512 /
// 1024 threads x 2 or 4 probes x 2 stages, 1024 x 2 x 4, ...) stop with "illegal instruction" on sm_100a (CUDA
// 12.9), unexplained: the same source with 3 probes per thread or 3 stages passes every test, padding the
// shared-memory layout changes nothing.  Such shapes are refused at build time.
static_assert(((HS_D * HS_TT) & (HS_D * HS_TT - 1)) != 0, "see the note above: pick another HS_NT x HS_U x HS_D");
constexpr int HS_CAP = 1024;         // staged spline points per window
constexpr int HS_NC = LJ_HS_NC;      // lower-bound cells per window
constexpr i64 HS_PIECE = LJ_HS_PIECE;  // records per work item
constexpr int HS_MAXWIN = 2048;
constexpr int HS_WPT = (HS_MAXWIN + HS_NT - 1) / HS_NT;  // windows per thread in the piece prefix
constexpr int HS_QCAP = 32 * HS_U;   // unfinished probes a warp can queue per iteration
static_assert(((HS_NC + 8) * 2) % 8 == 0, "the piece prefix and the queues follow the cells 8-B aligned");
// dynamic shared memory for nb windows: record stages, staged points + segments, cells, piece prefix, queues
__host__ __device__ constexpr size_t hs_ip_words(int nb) { return (size_t)((nb + 3) & ~1); }
__host__ __device__ constexpr size_t hs_smem(int nb) {
    return (size_t)HS_D * HS_U * HS_NT * 16 + (size_t)HS_CAP * (8 + 32) + (HS_NC + 8) * 2 + hs_ip_words(nb) * 4 +
           (LJ_HS_ROUNDS == 2 ? (size_t)(HS_NT / 32) * HS_QCAP * (8 + 2) : 0) + LJ_HS_PADB;
}

// first slot of position p in the probe table (monotone, even)
__host__ __device__ __forceinline__ i64 slot_of_pos(i64 p) { return (p * LJ_HS_SPREAD) & ~(i64)1; }

struct WinMeta {
    u64 klo, khi;
    int a0, npts, cshift, ok;
};

inline size_t hs_meta_bytes(int nb) {
    return (((size_t)nb * sizeof(WinMeta) + 255) & ~(size_t)255) + (size_t)nb * (HS_NC + 8) * sizeof(u16);
}

__device__ __forceinline__ i64 lower_bound_u64(const u64 *a, i64 n, u64 k) {
    i64 lo = 0, hi = n;
    while (lo < hi) {
        const i64 mid = (lo + hi) >> 1;
        if (__ldg(reinterpret_cast<const unsigned long long *>(a) + mid) < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ------------------------------------------------------------ probe table

#if LJ_HS_LAYOUT == 0
// t_j = 2 pos_j - j over the sorted build keys; cnt[0] counts zero
// payloads, cnt[1] equal adjacent keys
__global__ void k_slots_t(SplineDev m, const u64 *sk, const u64 *sp, i64 n, i64 *t, unsigned long long *cnt) {
    u32 z = 0, d = 0;
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x) {
        t[j] = slot_of_pos(m.pos(sk[j])) - j;
        z += sp[j] == 0;
        d += j > 0 && sk[j] == sk[j - 1];
    }
    if (z) atomicAdd(cnt, (unsigned long long)z);
    if (d) atomicAdd(cnt + 1, (unsigned long long)d);
}

struct MaxI64 {
    __device__ __forceinline__ i64 operator()(const i64 &a, const i64 &b) const { return a > b ? a : b; }
};
using SlotScanOp = MaxI64;

// plan[0] = slots needed (even, incl. the terminating pair), plan[1] = zero
// payloads, plan[2] = duplicate build keys
__global__ void k_slots_size(const i64 *M, i64 n, unsigned long long *zero, i64 *plan) {
    const i64 last = (n - 1) + M[n - 1];
    i64 L = last + 1;
    if (L < slot_of_pos(n - 1) + 2) L = slot_of_pos(n - 1) + 2;
    L = (L + 1) & ~(i64)1;
    plan[0] = L + 2;
    plan[1] = (i64)zero[0];
    plan[2] = (i64)zero[1];
}

// slot s: the last entry j with slot_j = j + M_j <= s (slot_j is strictly
// increasing) -> (key_j, s == slot_j ? payload_j : 0); before entry 0:
// (key_0, 0); the final pair: (~0, 0)
__global__ void k_slots_fill(const i64 *M, const u64 *sk, const u64 *sp, i64 n, i64 L, ulonglong2 *slots) {
    for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < L; s += (i64)gridDim.x * blockDim.x) {
        if (s >= L - 2) {
            slots[s] = make_ulonglong2(~0ULL, 0ULL);
            continue;
        }
        i64 lo = 0, hi = n;  // first j with slot_j > s
        while (lo < hi) {
            const i64 mid = (lo + hi) >> 1;
            if (mid + __ldg(reinterpret_cast<const long long *>(M) + mid) <= s) lo = mid + 1;
            else hi = mid;
        }
        const i64 j = lo - 1;
        if (j < 0) {
            slots[s] = make_ulonglong2(sk[0], 0ULL);
        } else {
            const bool real = j + M[j] == s;
            slots[s] = make_ulonglong2(sk[j], real ? sp[j] : 0ULL);
        }
    }
}
#else
// Home pairs + tails (layout 1).  All entries with key k share pos(k), so a
// probe needs the chain of ITS position only (learned_hash.py:81-96).  Chain
// C_p = the entries of position p in key order (contiguous in the sorted
// build keys):
//   |C_p| <= 2: the home pair (slots 2p, 2p + 1) holds the chain, empty slots
//               are {~0, 0};
//   |C_p| >= 3: slot 2p = the first entry, slot 2p + 1 = {~0, tail} with
//               tail the (even, >= 2n) slot where entries 1.. of the chain
//               follow in key order, closed by at least one {~0, 0} and
//               padded to whole pairs.
// No entry is displaced by its neighbours' chains: a probe whose key is
// among the first two of its chain (or absent from a short chain) is done
// after ONE 32-B load; the others continue at the tail.  P[j] = pos of the
// sorted build key j; cnt as in layout 0.
__global__ void k_slots_t(SplineDev m, const u64 *sk, const u64 *sp, i64 n, i64 *P, unsigned long long *cnt) {
    u32 z = 0, d = 0;
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x) {
        P[j] = m.pos(sk[j]);
        z += sp[j] == 0;
        d += j > 0 && sk[j] == sk[j - 1];
    }
    if (z) atomicAdd(cnt, (unsigned long long)z);
    if (d) atomicAdd(cnt + 1, (unsigned long long)d);
}

__device__ __forceinline__ i64 first_pos_geq(const i64 *P, i64 n, i64 p) {
    i64 lo = 0, hi = n;
    while (lo < hi) {
        const i64 mid = (lo + hi) >> 1;
        if (__ldg(reinterpret_cast<const long long *>(P) + mid) < p) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// A[j] = tail slots of the chain headed by entry j (0 unless j heads a chain
// of >= 3): its |C| - 1 further entries + a closing {~0, 0}, rounded up to pairs
__global__ void k_slots_tail(const i64 *P, i64 n, i64 *A) {
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x) {
        const i64 p = P[j];
        i64 a = 0;
        if ((j == 0 || P[j - 1] != p) && j + 2 < n && P[j + 2] == p) {
            const i64 c = first_pos_geq(P, n, p + 1) - j;
            a = (c + 1) & ~(i64)1;
        }
        A[j] = a;
    }
}

struct SumI64 {
    __device__ __forceinline__ i64 operator()(const i64 &a, const i64 &b) const { return a + b; }
};
using SlotScanOp = SumI64;  // the plan's scan: inclusive tail-slot sums M[j]

// plan[0] = slots needed: 2n home slots + the tails + a closing pair
__global__ void k_slots_size(const i64 *M, i64 n, unsigned long long *zero, i64 *plan) {
    plan[0] = 2 * n + M[n - 1] + 2;
    plan[1] = (i64)zero[0];
    plan[2] = (i64)zero[1];
}

__global__ void k_slots_fill(const i64 *M, const i64 *P, const u64 *sk, const u64 *sp, i64 n, i64 L,
                             ulonglong2 *slots) {
    const ulonglong2 none = make_ulonglong2(~0ULL, 0ULL);
    for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < L; s += (i64)gridDim.x * blockDim.x) {
        if (s < 2 * n) {
            const i64 p = s >> 1;
            const i64 h = first_pos_geq(P, n, p);
            ulonglong2 v = none;
            if (h < n && P[h] == p) {
                if (!(s & 1)) v = make_ulonglong2(sk[h], sp[h]);
                else if (h + 2 < n && P[h + 2] == p) v = make_ulonglong2(~0ULL, (u64)(2 * n + (h > 0 ? M[h - 1] : 0)));
                else if (h + 1 < n && P[h + 1] == p) v = make_ulonglong2(sk[h + 1], sp[h + 1]);
            }
            slots[s] = v;
            continue;
        }
        const i64 t = s - 2 * n;
        ulonglong2 v = none;
        if (t < M[n - 1]) {
            i64 lo = 0, hi = n;  // the head h whose tail [M[h-1], M[h]) holds t: first j with M[j] > t
            while (lo < hi) {
                const i64 mid = (lo + hi) >> 1;
                if (__ldg(reinterpret_cast<const long long *>(M) + mid) <= t) lo = mid + 1;
                else hi = mid;
            }
            const i64 h = lo, j = h + 1 + (t - (h > 0 ? M[h - 1] : 0));
            if (j < n && P[j] == P[h]) v = make_ulonglong2(sk[j], sp[j]);
        }
        slots[s] = v;
    }
}
#endif

// ------------------------------------------------------------ windows

// one block per window: the spline points [a0, a0 + npts) and the cells
__global__ void __launch_bounds__(1024) k_hash_windows(SplineDev m, const u64 *lay, int nb, u64 kmin, WinMeta *meta,
                                                      u16 *cells) {
    const int w = blockIdx.x;
    const u64 *B = lay + 4;
    __shared__ WinMeta s;
    if (threadIdx.x == 0) {
        const u64 kfirst = __ldg(reinterpret_cast<const unsigned long long *>(m.keys));
        const u64 klast = __ldg(reinterpret_cast<const unsigned long long *>(m.keys) + m.K - 1);
        u64 klo = w == 0 ? kmin : B[w];
        u64 khi = w + 1 < nb ? (B[w + 1] == 0 ? 0 : B[w + 1] - 1) : klast;
        if (klo < kfirst) klo = kfirst;
        if (khi > klast) khi = klast;
        WinMeta t;
        t.klo = klo;
        t.khi = khi;
        t.ok = (m.K >= 2 && klo <= khi && (w + 1 >= nb || B[w + 1] > klo)) ? 1 : 0;
        t.a0 = 0;
        t.npts = 0;
        t.cshift = 0;
        if (t.ok) {
            const i64 lbl = lower_bound_u64(m.keys, m.K, klo);
            const i64 lbh = lower_bound_u64(m.keys, m.K, khi);
            i64 a = lbl - 1 < 0 ? 0 : lbl - 1;
            const i64 b = lbh < 1 ? 1 : (lbh > m.K - 1 ? m.K - 1 : lbh);
            a &= ~(i64)1;
            t.a0 = (int)a;
            t.npts = (int)(b - a + 1);
            if (t.npts > HS_CAP || m.K >= ((i64)1 << 31)) t.ok = 0;
            int sh = 0;
            while (sh < 63 && ((khi - klo) >> sh) >= (u64)HS_NC) ++sh;
            t.cshift = sh;
        }
        s = t;
        meta[w] = t;
    }
    __syncthreads();
    if (!s.ok) return;
    u16 *cw = cells + (size_t)w * (HS_NC + 8);
    for (int c = threadIdx.x; c <= HS_NC; c += blockDim.x) {
        const u64 off = (u64)c << s.cshift;
        const bool past = (s.cshift > 0 && (u64)c > ((s.khi - s.klo) >> s.cshift)) || off > s.khi - s.klo;
        const u64 L = past ? s.khi : s.klo + off;
        // (over the window's own points: the clamp below makes it equal to the search over all K)
        i64 i = lower_bound_u64(m.keys + s.a0, s.npts, L);
        if (past) i = s.npts - 1;
        cw[c] = (u16)(i < 0 ? 0 : (i > s.npts - 1 ? s.npts - 1 : i));
    }
}

// ------------------------------------------------------------ probe

// One staged spline segment [point li-1, point li]: the operands of
// models.py:240-244 -- x0 = float64(key[li-1]), inv = RN(1 / max(x1 - x0, 1)),
// r0 = rank[li-1], dr = RN(r1 - r0) -- precomputed per window in shared
// memory.
struct Seg {
    double x0, inv, r0, dr;
};

struct StagedSpline {
    const u64 *sk;
    const Seg *seg;
    const u16 *cells;
    u64 klo, span;  // staged key range [klo, klo + span]
    int cshift;
    int li_lo, li_hi;  // the staged image of clamping the point index to [1, K-1]
    int nm1;           // n - 1 (the staged path needs n < 2^31)
    double guard;      // 0.5 - (n + 1) * 2^-49: see pos()
    // models.py:221-248 for k in [klo, klo + span]: the first spline key >= k
    // over the staged points (the cell bounds its range), then the
    // reference's operations.  t = (k - x0) / d is taken as (k - x0) *
    // RN(1/d): both are within 3.01 * 2^-53 of the true quotient (t <= 1), so
    // the two values of r0 + t*dr differ by at most 2^-50 * (r1 + 1) <=
    // 2^-50 * (n + 1); rint only jumps at half-integers, so unless the fast
    // value lies within (n + 1) * 2^-49 (twice that) of one, both round to
    // the same integer -- else the reference's division runs.  Every operand
    // is finite and t in [0, 1] keeps z in [0, n), so np.clip's NaN rule and
    // the cast's range rule never apply; z is within 0.5 of the rounded p, so
    // "near a half-integer" is |z - p| >= guard.
    __device__ __forceinline__ int pos(u64 k) const {
        const int c = (int)((k - klo) >> cshift);
        int lo = cells[c], hi = cells[c + 1];
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sk[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        const int li = min(max(lo, li_lo), li_hi);
        const Seg g = seg[li];
        const double a = __dsub_rn(u64_to_f64(k), g.x0);
        double z = __dadd_rn(g.r0, __dmul_rn(fmin(fmax(__dmul_rn(a, g.inv), 0.0), 1.0), g.dr));
        int p = __double2int_rn(z);
        if (fabs(__dsub_rn(z, (double)p)) >= guard) {
            const double d = __dsub_rn(u64_to_f64(sk[li]), g.x0);
            z = __dadd_rn(g.r0, __dmul_rn(fmin(fmax(__ddiv_rn(a, d > 1.0 ? d : 1.0), 0.0), 1.0), g.dr));
            p = __double2int_rn(z);
        }
        return min(max(p, 0), nm1);
    }
};

struct Acc3 {
    u64 c, s, x;
    __device__ __forceinline__ void add(u64 pr, u64 ps) {
        const u64 v = pr + ps;
        ++c;
        s += v;
        x ^= v;
    }
};

// One aligned slot pair {key0, pay0, key1, pay1} of a probe for key k; slot
// keys are non-decreasing.  Matches (key == k, payload != 0) are added;
// returns true when the scan must go on to the next pair (no key > k seen
// and, with unique build keys, no match yet).  UNIQUE is branch-free: at
// most one slot matches, its payload is selected and added under one
// predicate.
template <bool UNIQUE>
__device__ __forceinline__ bool pair_scan(const u64 (&e)[4], u64 k, u64 ps, Acc3 &acc) {
    if (UNIQUE) {
        const u64 h = (e[0] == k && e[1]) ? e[1] : ((e[2] == k && e[3]) ? e[3] : 0ULL);
        if (h) acc.add(h, ps);
        return h == 0 && e[2] <= k;
    }
    if (e[0] > k) return false;
    if (e[0] == k && e[1]) acc.add(e[1], ps);
    if (e[2] > k) return false;
    if (e[2] == k && e[3]) acc.add(e[3], ps);
    return true;
}

#if LJ_HS_LAYOUT == 1
// The HOME pair of a probe for key k (layout 1): its chain's first two
// entries, or the first entry and {~0, tail}.  Matches are added; returns
// true when the chain goes on in its tail (e[3]) and may still hold k (the
// tail's keys are >= e[0]; with unique build keys a match ends the probe).
template <bool UNIQUE>
__device__ __forceinline__ bool pair_first(const u64 (&e)[4], u64 k, u64 ps, Acc3 &acc) {
    const bool tail = e[2] == ~0ULL && e[3] != 0;
    if (UNIQUE) {
        const u64 h = (e[0] == k && e[1]) ? e[1] : ((e[2] == k && e[3]) ? e[3] : 0ULL);
        if (h) acc.add(h, ps);
        return tail && e[0] < k;
    }
    if (e[0] == k && e[1]) acc.add(e[1], ps);
    if (tail) return e[0] <= k;
    if (e[2] == k && e[3]) acc.add(e[3], ps);
    return false;
}
#endif

// 16-B asynchronous global -> shared copy with an L2 cache policy
__device__ __forceinline__ void cp_async16_ef(void *dst, const void *src, u64 pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "l"(pol)
                 : "memory");
}

// global (unstaged) evaluation: the overflow area and windows whose points
// exceed the staging capacity
__device__ __forceinline__ i64 spline_pos_global(const SplineDev &m, u64 k) { return m.pos(k); }

// Per thread, a software pipeline over iterations of HS_U records (one
// per HS_NT-strided lane position): the records of iteration i + HS_D - 1
// are copied into this thread's own shared-memory slots (cp.async, 16 B,
// coalesced across the warp) while iteration i is probed, so no barrier
// is needed inside a work item; every probe's first slot is loaded before
// any is compared (HS_U independent L2 loads in flight per thread).
template <bool UNIQUE>
__global__ void __launch_bounds__(HS_NT, HS_CTAS) k_hash_probe_staged(SplineDev m, const ulonglong2 *__restrict__ slots,
                                                                     const ulonglong2 *__restrict__ rec,
                                                                     const i64 *__restrict__ reg, int nb,
                                                                     const WinMeta *__restrict__ meta,
                                                                     const u16 *__restrict__ cells_g,
                                                                     const Seg *__restrict__ segs_g,
                                                                     unsigned long long *ctr, u64 *out) {
    extern __shared__ __align__(128) unsigned char smem_h[];
    ulonglong2 *rbuf = reinterpret_cast<ulonglong2 *>(smem_h);  // [HS_D][HS_U][HS_NT]
    u64 *sk = reinterpret_cast<u64 *>(smem_h + (size_t)HS_D * HS_U * HS_NT * 16);
    Seg *seg = reinterpret_cast<Seg *>(reinterpret_cast<unsigned char *>(sk) + (size_t)HS_CAP * 8);
    u16 *cells = reinterpret_cast<u16 *>(reinterpret_cast<unsigned char *>(seg) + (size_t)HS_CAP * sizeof(Seg));
    int *ip = reinterpret_cast<int *>(reinterpret_cast<unsigned char *>(cells) + (HS_NC + 8) * 2);  // [nb + 1]
#if LJ_HS_ROUNDS == 2
    // per-warp queue of unfinished probes: next slot + record index in the stage
    u64 *wq_slot = reinterpret_cast<u64 *>(ip + hs_ip_words(nb));
    u16 *wq_idx = reinterpret_cast<u16 *>(wq_slot + (HS_NT / 32) * HS_QCAP);
#endif
    __shared__ int s_item[2], s_tot;
    __shared__ WinMeta s_m;
    __shared__ int s_wsum[HS_NT / 32];
    __shared__ __align__(8) uint64_t sbar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const i64 *rend = reg + nb + 1;
    // pieces per window, exclusive prefix (HS_WPT windows per thread)
    {
        int v[HS_WPT], tot = 0;
#pragma unroll
        for (int q = 0; q < HS_WPT; ++q) {
            const int w = tid * HS_WPT + q;
            v[q] = w < nb ? (int)((rend[w] - reg[w] + HS_PIECE - 1) / HS_PIECE) : 0;
            tot += v[q];
        }
        int inc = tot;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += y;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const int x = lane < HS_NT / 32 ? s_wsum[lane] : 0;
            int xi = x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, xi, d);
                if (lane >= d) xi += y;
            }
            if (lane < HS_NT / 32) s_wsum[lane] = xi - x;
        }
        __syncthreads();
        int run = s_wsum[warp] + inc - tot;
#pragma unroll
        for (int q = 0; q < HS_WPT; ++q) {
            const int w = tid * HS_WPT + q;
            if (w < nb) ip[w] = run;
            run += v[q];
        }
        if (tid * HS_WPT <= nb - 1 && nb - 1 < tid * HS_WPT + HS_WPT) {
            ip[nb] = run;
            s_tot = run + (int)((reg[2 * nb + 1] + HS_PIECE - 1) / HS_PIECE);
        }
    }
    if (tid == 0) {
        mbar_init(&sbar, 1);
        mbar_init_fence();
    }
    __syncthreads();
    const int total = s_tot;
    unsigned sphase = 0;
    int cur = -1;
    bool staged = false;
    StagedSpline ss;
    ss.sk = sk;
    ss.seg = seg;
    ss.cells = cells;
    ss.nm1 = (int)(m.n - 1);
    ss.guard = 0.5 - ((double)m.n + 1.0) * 1.7763568394002505e-15;  // 2^-49
    Acc3 acc = {0, 0, 0};
    u64 pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int it = 0;; ++it) {
        if (tid == 0) s_item[it & 1] = (int)atomicAdd(ctr, 1ULL);
        __syncthreads();
        const int item = s_item[it & 1];
        if (item >= total) break;
        int w;
        i64 lo, hi;
        if (item >= ip[nb]) {  // overflow area: any window
            w = nb;
            lo = reg[nb] + (i64)(item - ip[nb]) * HS_PIECE;
            hi = min(lo + HS_PIECE, reg[nb] + reg[2 * nb + 1]);
        } else {
            int a = 0, b = nb - 1;  // last window with ip[w] <= item
            while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if (ip[mid] <= item) a = mid;
                else b = mid - 1;
            }
            w = a;
            lo = reg[w] + (i64)(item - ip[w]) * HS_PIECE;
            hi = min(lo + HS_PIECE, rend[w]);
        }
        if (w != cur) {
            // restage (every thread is past the previous item: barrier above)
            cur = w;
            staged = false;
            if (w < nb) {
                const WinMeta mw = meta[w];
                if (mw.ok) {
                    if (tid == 0) {
                        const unsigned nbk = ((unsigned)mw.npts * 8u + 15u) & ~15u;
                        const unsigned nbs = (unsigned)mw.npts * (unsigned)sizeof(Seg);
                        const unsigned nbc = (unsigned)(HS_NC + 8) * 2u;
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        mbar_arrive_expect_tx(&sbar, nbk + nbs + nbc);
                        bulk_g2s(sk, m.keys + mw.a0, nbk, &sbar);
                        bulk_g2s(seg, segs_g + mw.a0, nbs, &sbar);
                        bulk_g2s(cells, cells_g + (size_t)w * (HS_NC + 8), nbc, &sbar);
                    }
                    mbar_wait(&sbar, sphase);
                    sphase ^= 1u;
                    staged = true;
                    ss.klo = mw.klo;
                    ss.span = mw.khi - mw.klo;
                    ss.cshift = mw.cshift;
                    // point index j = a0 + lo clamped to [1, K-1], staged-relative
                    ss.li_lo = mw.a0 >= 1 ? 0 : 1;
                    ss.li_hi = (int)min((i64)mw.npts, m.K - 1 - (i64)mw.a0);
                }
            }
        }
        const int niter = (int)((hi - lo + HS_TT - 1) / HS_TT);
        // records of iteration i -> this thread's slots of stage i % HS_D
        // (evict-first in L2: read once; the slot lines are what L2 keeps).
        // HS_D == 1: ONE stage -- a thread reads its records of iteration i
        // into registers and only then starts the copies of iteration i + 1
        // into the same slots (its own: no other thread touches them), so
        // the copies still have a whole iteration to land, at half the
        // shared memory (more L1 for the slot loads in flight).
#pragma unroll
        for (int i = 0; i < (HS_D == 1 ? 1 : HS_D - 1); ++i) {
            if (i < niter) {
#pragma unroll
                for (int u = 0; u < HS_U; ++u) {
                    const i64 j = lo + (i64)i * HS_TT + u * HS_NT + tid;
                    if (j < hi) cp_async16_ef(rbuf + ((size_t)(i % HS_D) * HS_U + u) * HS_NT + tid, rec + j, pol);
                }
            }
            cp_async_commit();
        }
        for (int i = 0; i < niter; ++i) {
            if (HS_D > 1) {
                const int f = i + HS_D - 1;
                if (f < niter) {
#pragma unroll
                    for (int u = 0; u < HS_U; ++u) {
                        const i64 j = lo + (i64)f * HS_TT + u * HS_NT + tid;
                        if (j < hi) cp_async16_ef(rbuf + ((size_t)(f % HS_D) * HS_U + u) * HS_NT + tid, rec + j, pol);
                    }
                }
                cp_async_commit();
            }
            asm volatile("cp.async.wait_group %0;" ::"n"(HS_D > 1 ? HS_D - 1 : 0) : "memory");
            u64 k[HS_U], ps[HS_U];
            i64 s0[HS_U];
#pragma unroll
            for (int u = 0; u < HS_U; ++u) {
                const i64 j = lo + (i64)i * HS_TT + u * HS_NT + tid;
                if (j < hi) {
                    const ulonglong2 r = rbuf[((size_t)(i % HS_D) * HS_U + u) * HS_NT + tid];
                    k[u] = r.x;
                    ps[u] = r.y;
                } else {
                    k[u] = ~0ULL;
                    ps[u] = 0;
                }
            }
            if (HS_D == 1) {
                if (i + 1 < niter) {
#pragma unroll
                    for (int u = 0; u < HS_U; ++u) {
                        const i64 j = lo + (i64)(i + 1) * HS_TT + u * HS_NT + tid;
                        // (the record just read is an operand: the copy issues after its load has returned)
                        if (j < hi) {
                            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;  // after %3 %4" ::"r"(
                                             smem_u32(rbuf + (size_t)u * HS_NT + tid)),
                                         "l"(rec + j), "l"(pol), "l"(k[u]), "l"(ps[u])
                                         : "memory");
                        }
                    }
                }
                cp_async_commit();
            }
#pragma unroll
            for (int u = 0; u < HS_U; ++u) {
                // (one unsigned compare covers klo <= k <= khi; the reserved
                // key of gap records / past the item lies outside every window)
                if (staged && k[u] - ss.klo <= ss.span) s0[u] = slot_of_pos((i64)ss.pos(k[u]));
                else if (k[u] == ~0ULL) s0[u] = -1;
                else s0[u] = slot_of_pos(spline_pos_global(m, k[u]));
            }
            // every probe's first slot PAIR (32 B, aligned: one sector) in flight at once
            u64 e[HS_U][4];
#pragma unroll
            for (int u = 0; u < HS_U; ++u) {
                if (s0[u] >= 0) {
                    asm volatile(LJ_HS_LD " {%0, %1, %2, %3}, [%4];"
                                 : "=l"(e[u][0]), "=l"(e[u][1]), "=l"(e[u][2]), "=l"(e[u][3])
                                 : "l"(slots + s0[u]));
                } else {
                    e[u][0] = e[u][2] = ~0ULL;
                    e[u][1] = e[u][3] = 0;
                }
            }
            // the slot scan (see the header): keys < k skipped, keys == k
            // with a nonzero payload counted (unique build keys: the first
            // is the only one), stop at the first key > k.  About a quarter
            // of the probes go past their first pair (crowded positions push
            // entries forward); their following pairs are fetched in rounds
            // -- one more pair for EVERY unfinished probe of the thread in
            // flight at once -- instead of one dependent 16-B load at a time.
            unsigned need = 0;
#pragma unroll
            for (int u = 0; u < HS_U; ++u) {
                // (a skipped probe's pair {~0, 0, ~0, 0} matches nothing)
#if LJ_HS_LAYOUT == 1
                const bool go = pair_first<UNIQUE>(e[u], k[u], ps[u], acc) && s0[u] >= 0;
                if (go) s0[u] = (i64)e[u][3] - 2;  // round r reads the tail pair r - 1
                need |= (unsigned)go << u;
#else
                need |= (unsigned)(pair_scan<UNIQUE>(e[u], k[u], ps[u], acc) && s0[u] >= 0) << u;
#endif
            }
#if LJ_HS_ROUNDS == 0
            // (ablation) one dependent 16-B slot at a time, probe by probe
#pragma unroll
            for (int u = 0; u < HS_U; ++u) {
                if (!(need >> u & 1u)) continue;
                for (i64 sl = s0[u] + 2;; ++sl) {
                    const ulonglong2 ev = __ldg(slots + sl);
                    if (ev.x > k[u]) break;
                    if (ev.x == k[u] && ev.y) {
                        acc.add(ev.y, ps[u]);
                        if (UNIQUE) break;
                    }
                }
            }
            need = 0;
#endif
#if LJ_HS_ROUNDS == 2
            // Compacted forward scan: the warp's unfinished probes (about a
            // quarter of its HS_U * 32) are queued in shared memory and taken
            // one per lane, so the scan's rounds run with full warps instead
            // of the 3-9 lanes whose own probes are unfinished.
            {
                u64 *qs = wq_slot + warp * HS_QCAP;
                u16 *qi = wq_idx + warp * HS_QCAP;
                const unsigned lt = (1u << lane) - 1u;
                int nq = 0;
#pragma unroll
                for (int u = 0; u < HS_U; ++u) {
                    const bool nd = need >> u & 1u;
                    const unsigned bal = __ballot_sync(0xffffffffu, nd);
                    if (nd) {
                        const int r = nq + __popc(bal & lt);
                        qs[r] = (u64)(s0[u] + 2);
                        qi[r] = (u16)(u * HS_NT + tid);
                    }
                    nq += __popc(bal);
                }
                __syncwarp();
                const ulonglong2 *rb = rbuf + (size_t)(i % HS_D) * HS_U * HS_NT;
                for (int q = lane; q < nq; q += 32) {
                    const ulonglong2 r = rb[qi[q]];
                    const ulonglong2 *sl = slots + qs[q];
                    u64 ee[4];
                    do {
                        asm volatile(LJ_HS_LD " {%0, %1, %2, %3}, [%4];"
                                     : "=l"(ee[0]), "=l"(ee[1]), "=l"(ee[2]), "=l"(ee[3])
                                     : "l"(sl));
                        sl += 2;
                    } while (pair_scan<UNIQUE>(ee, r.x, r.y, acc));
                }
                __syncwarp();
                need = 0;
            }
#endif
#if LJ_HS_ROUNDS == 3
            // One pair per LANE per round: the lane's first unfinished probe
            // is selected into (kq, pq, sq) and followed to its end, then the
            // next -- a round costs one pair scan instead of one per probe
            // position u (whose blocks run at 3-9 active lanes each).
            {
                u64 kq = 0, pq = 0;
                i64 sq = 0;
                bool fresh = true;
#pragma unroll 1
                while (need) {
                    if (fresh) {
                        const int u0 = __ffs(need) - 1;
                        kq = k[0], pq = ps[0], sq = s0[0];
#pragma unroll
                        for (int u = 1; u < HS_U; ++u) {
                            if (u0 == u) kq = k[u], pq = ps[u], sq = s0[u];
                        }
                    }
                    sq += 2;
                    u64 ee[4];
                    asm volatile(LJ_HS_LD " {%0, %1, %2, %3}, [%4];"
                                 : "=l"(ee[0]), "=l"(ee[1]), "=l"(ee[2]), "=l"(ee[3])
                                 : "l"(slots + sq));
                    fresh = !pair_scan<UNIQUE>(ee, kq, pq, acc);
                    if (fresh) need &= need - 1u;
                }
            }
#endif
#pragma unroll 1
            for (int r = 1; need; ++r) {
#pragma unroll
                for (int u = 0; u < HS_U; ++u) {
                    if (need >> u & 1u) {
                        asm volatile(LJ_HS_LD " {%0, %1, %2, %3}, [%4];"
                                     : "=l"(e[u][0]), "=l"(e[u][1]), "=l"(e[u][2]), "=l"(e[u][3])
                                     : "l"(slots + s0[u] + 2 * r));
                    }
                }
#pragma unroll
                for (int u = 0; u < HS_U; ++u) {
                    if (need >> u & 1u) {
                        if (!pair_scan<UNIQUE>(e[u], k[u], ps[u], acc)) need &= ~(1u << u);
                    }
                }
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    reduce_checksum(acc.c, acc.s, acc.x, 0, out);
}

}  // namespace lj

using namespace lj;

extern "C" {

size_t lj_spline_slots_workspace_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceScan::InclusiveScan((void *)nullptr, t, (const i64 *)nullptr, (i64 *)nullptr, SlotScanOp(), (int64_t)n);
    return part_align_c(sizeof(i64) * (size_t)(n > 0 ? n : 1)) * 2 + part_align_c(t) + 256;
}

int lj_spline_slots_plan(const LjSpline *model, const uint64_t *sorted_keys, const uint64_t *sorted_pay, int64_t n,
                         int64_t *plan, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(model && model->npts >= 1 && model->n == n && n >= 1, "model is not fitted on these keys");
    LJ_REQUIRE(ws_bytes >= lj_spline_slots_workspace_bytes(n), "workspace too small");
    cudaStream_t st = as_stream(stream);
    char *q = (char *)ws;
    i64 *t = (i64 *)q;
    q += part_align_c(sizeof(i64) * (size_t)n);
    i64 *M = (i64 *)q;
    q += part_align_c(sizeof(i64) * (size_t)n);
    unsigned long long *zero = (unsigned long long *)q;
    q += 256;
    LJ_CK(cudaMemsetAsync(zero, 0, 2 * sizeof(unsigned long long), st));
    k_slots_t<<<grid_for(n, 256, 8), 256, 0, st>>>(SplineDev(*model), sorted_keys, sorted_pay, n, t, zero);
    LJ_CK_LAUNCH();
#if LJ_HS_LAYOUT == 1
    // t = P (positions) stays for the fill; the tail sizes are scanned in place in M
    k_slots_tail<<<grid_for(n, 256, 8), 256, 0, st>>>(t, n, M);
    LJ_CK_LAUNCH();
    t = M;
#endif
    size_t tb = 0;
    cub::DeviceScan::InclusiveScan(nullptr, tb, t, M, SlotScanOp(), (int64_t)n);
    LJ_CK(cub::DeviceScan::InclusiveScan(q, tb, t, M, SlotScanOp(), (int64_t)n, st));
    k_slots_size<<<1, 1, 0, st>>>(M, n, zero, plan);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_spline_slots_fill(const uint64_t *sorted_keys, const uint64_t *sorted_pay, int64_t n, uint64_t *slots,
                         int64_t nslots, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(n >= 1 && nslots >= 2 * n, "need n >= 1 and the planned slot count");
    LJ_REQUIRE(ws_bytes >= lj_spline_slots_workspace_bytes(n), "workspace too small");
    const i64 *M = (const i64 *)((char *)ws + part_align_c(sizeof(i64) * (size_t)n));
#if LJ_HS_LAYOUT == 1
    k_slots_fill<<<grid_for(nslots, 256, 16), 256, 0, as_stream(stream)>>>(
        M, (const i64 *)ws, sorted_keys, sorted_pay, n, nslots, reinterpret_cast<ulonglong2 *>(slots));
#else
    k_slots_fill<<<grid_for(nslots, 256, 16), 256, 0, as_stream(stream)>>>(
        M, sorted_keys, sorted_pay, n, nslots, reinterpret_cast<ulonglong2 *>(slots));
#endif
    LJ_CK_LAUNCH();
    return LJ_OK;
}

// per spline point li >= 1: Seg{x0, RN(1/max(x1 - x0, 1)), r0, RN(r1 - r0)}
// of the segment ending at li (seg[0] unused)
__global__ void k_spline_segs(SplineDev m, Seg *seg) {
    for (i64 li = blockIdx.x * (i64)blockDim.x + threadIdx.x; li < m.K; li += (i64)gridDim.x * blockDim.x) {
        Seg g;
        if (li == 0) {
            g.x0 = g.inv = g.r0 = g.dr = 0.0;
        } else {
            g.x0 = u64_to_f64(m.keys[li - 1]);
            const double d = __dsub_rn(u64_to_f64(m.keys[li]), g.x0);
            g.inv = __drcp_rn(d > 1.0 ? d : 1.0);
            g.r0 = m.ranks[li - 1];
            g.dr = __dsub_rn(m.ranks[li], g.r0);
        }
        seg[li] = g;
    }
}

int lj_spline_segments(const LjSpline *model, double *segs, void *stream) {
    LJ_REQUIRE(model && model->npts >= 1, "model is not fitted");
    k_spline_segs<<<grid_for(model->npts, 256, 4), 256, 0, as_stream(stream)>>>(SplineDev(*model),
                                                                                reinterpret_cast<Seg *>(segs));
    LJ_CK_LAUNCH();
    return LJ_OK;
}

}  // extern "C"

namespace lj {

size_t hash_staged_meta_bytes(int nb) { return hs_meta_bytes(nb); }

// window metadata for the key-range windows in `lay` (lj_keybin layout)
int hash_windows(const LjSpline &model, const u64 *lay, int nb, u64 kmin, void *meta_ws, cudaStream_t st) {
    WinMeta *meta = reinterpret_cast<WinMeta *>(meta_ws);
    u16 *cells = reinterpret_cast<u16 *>((char *)meta_ws + (((size_t)nb * sizeof(WinMeta) + 255) & ~(size_t)255));
    k_hash_windows<<<nb, 1024, 0, st>>>(SplineDev(model), lay, nb, kmin, meta, cells);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int hash_probe_staged(const LjSplineHash &idx, const ulonglong2 *rec, const i64 *reg, int nb, const void *meta_ws,
                      unsigned long long *ctr, u64 *out, cudaStream_t st) {
    if (!idx.segs) {
        set_error("hash_probe_staged: the index has no segment table");
        return LJ_E_INVALID;
    }
    if (nb > HS_MAXWIN) {
        set_error("hash_probe_staged: at most 2048 windows");
        return LJ_E_INVALID;
    }
    const WinMeta *meta = reinterpret_cast<const WinMeta *>(meta_ws);
    const u16 *cells =
        reinterpret_cast<const u16 *>((const char *)meta_ws + (((size_t)nb * sizeof(WinMeta) + 255) & ~(size_t)255));
    static_assert(sizeof(Seg) == 32, "HS_SMEM assumes 32-B segments");
    const size_t sm = hs_smem(nb);
    if (idx.model.n >= ((i64)1 << 31)) {
        set_error("hash_probe_staged: at most 2^31 - 1 build keys");
        return LJ_E_INVALID;
    }
    static unsigned long long attr = 0;  // one bit per device
    if (once_per_device(attr)) {
        const int mx = (int)hs_smem(HS_MAXWIN);
        LJ_CK(cudaFuncSetAttribute(k_hash_probe_staged<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        LJ_CK(cudaFuncSetAttribute(k_hash_probe_staged<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    }
    LJ_CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    if (idx.slots_unique)
        k_hash_probe_staged<true><<<HS_CTAS * sm_count(), HS_NT, sm, st>>>(
            SplineDev(idx.model), reinterpret_cast<const ulonglong2 *>(idx.slots), rec, reg, nb, meta, cells,
            reinterpret_cast<const Seg *>(idx.segs), ctr, out);
    else
        k_hash_probe_staged<false><<<HS_CTAS * sm_count(), HS_NT, sm, st>>>(
            SplineDev(idx.model), reinterpret_cast<const ulonglong2 *>(idx.slots), rec, reg, nb, meta, cells,
            reinterpret_cast<const Seg *>(idx.segs), ctr, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

}  // namespace lj
