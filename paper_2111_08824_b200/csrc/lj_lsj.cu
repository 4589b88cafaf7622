// lj_lsj.cu -- learned sort-join (LSJ) on the GPU.  Reference: lsj.py:95-405.
//
//   smpl  stratified sample (lj_lsj_sample) -> RMI fit (K10, lj_rmi_fit) ->
//         equi-depth bins over the model's predicted positions (lj_lsj_bins):
//         bin(key) = table[pos(key)], with bin boundaries at equally spaced
//         SAMPLE ranks.  The reference partitions uniformly in predicted
//         position (partition_index, models.py:285-299); on skewed keys the
//         2-level linear RMI predicts positions badly (its linear root sends
//         most lognormal keys to a few leaves) and uniform position buckets
//         vary by >8x.  Cutting the same monotone position axis at sample
//         quantiles keeps every bin near n/nbins.  Monotone in the key, so
//         the buckets are relatively sorted exactly as the reference's.
//   part  K6/K7: shared-memory-privatised histogram + scatter into <= 32768
//         bins (lj_part.cuh), 16-B interleaved records.
//   sort  K8: one CTA per bucket, in shared memory, MODEL-PLACED: every key's
//         unrounded prediction y (slope*x + icpt clamped to its leaf's rank
//         range, monotone non-decreasing in the key) is mapped to one of m
//         slots of the bucket; a counting sort by slot puts each key within
//         a few places of its final position; runs sharing a slot are
//         insertion-sorted; a verification pass falls back to a full
//         in-smem bitonic sort of the bucket if anything is out of order.
//         Buckets above shared-memory capacity (hot duplicate keys) are
//         re-partitioned by y at finer resolution through global memory and
//         sorted the same way; sub-buckets of one repeated key are copied.
//   join  K9: per S tile of 1024 sorted tuples, the R bucket range of the
//         tile's first/last key through R's model (chunked_join's
//         [f_R, l_R], lsj.py:343-346) bounds a binary search for the exact
//         R slice, which is staged in shared memory and merge-searched;
//         emits the checksum (or per-tuple counts / pairs).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "lj_common.cuh"
#include "lj_keybin.cuh"
#include "lj_pipe.cuh"
#include "lj_part.cuh"
#include "lj_part_est.cuh"

namespace lj {

#ifndef LJ_SORT_CTAS
#define LJ_SORT_CTAS 5
#endif
#ifndef LJ_SORT_NT
#define LJ_SORT_NT 256
#endif
#ifndef LJ_SORT_E
#define LJ_SORT_E 8
#endif
constexpr int SORT_CTAS = LJ_SORT_CTAS;  // sort CTAs per SM (their barrier waits overlap)
constexpr int SORT_NT = LJ_SORT_NT;
// largest bucket sorted in shared memory by the main instance: every thread
// owns LJ_SORT_E tuples (keys and slots in registers); 14 B of shared memory
// per tuple (8 B key + 4 B slot counter + u16 index)
constexpr int CAP = SORT_NT * LJ_SORT_E;
static_assert((size_t)CAP * 14 * SORT_CTAS + 1024 * SORT_CTAS <= 233472, "sort CTAs exceed the SM's shared memory");
constexpr int RUN_SMALL = 64;     // equal-slot runs ranked element by element
constexpr int MAX_RUNS = 64;      // longer mixed runs sorted block-wide per bucket
#ifndef LJ_SORT_U
#define LJ_SORT_U 4
#endif
constexpr int SORT_U = LJ_SORT_U;  // tuples in flight per thread in the load / write-out phases (8: -0.6 %, 12: +0.6 %)
#ifndef LJ_SUB_DIV
#define LJ_SUB_DIV 2
#endif
constexpr int SUB = CAP / LJ_SUB_DIV;  // mean tuples per sub-bucket: sample-quantile slices stay below CAP
constexpr int SPLIT_NT = 1024;
#ifndef LJ_SPLIT_U
#define LJ_SPLIT_U 4
#endif
#ifndef LJ_SPLIT_CH
#define LJ_SPLIT_CH 262144
#endif
#ifndef LJ_SPLIT_MINB
#define LJ_SPLIT_MINB 1  // resident split-scatter CTAs per SM the register budget allows
#endif
constexpr int SPLIT_U = LJ_SPLIT_U;    // tuple groups in flight per warp step
constexpr i64 SPLIT_CH = LJ_SPLIT_CH;  // tuples per split work item (C4 sort phase: 64 Ki 17.10, 128 Ki 16.90, 256 Ki 16.77, 512 Ki 16.95 ms)
constexpr int SPLIT_MAXF = 2048;  // slices per coarse bucket (point mode: 2x-1 slots)
#ifndef LJ_JOIN_T
#define LJ_JOIN_T 512
#endif
#ifndef LJ_JOIN_WCAP
#define LJ_JOIN_WCAP 1920
#endif
#ifndef LJ_JOIN_NT
#define LJ_JOIN_NT 128
#endif
#ifndef LJ_JOIN_MINB
#define LJ_JOIN_MINB 1  // resident join CTAs per SM the register budget must allow
#endif
constexpr int JOIN_T = LJ_JOIN_T;
constexpr int JOIN_NT = LJ_JOIN_NT;
constexpr int WCAP = LJ_JOIN_WCAP;  // R slice keys staged per tile (+ the S tile: < 48 KB static)

// ------------------------------------------------------------------ model

// RMI + equi-depth bin table over predicted positions.
struct LsjDev {
    RmiDev m;
    const u32 *table;  // [m.n] predicted position -> bin
    const i64 *pb;     // [nb+1] first position of each bin
    int nb;
    const u64 *sample;  // sorted fit sample (split points) or nullptr
    i64 nsample;
    // monotone over the whole key domain (saturating cast, lj_common.cuh):
    // the key-range bounds found by search, the partition and the join's
    // window lookup all see the same bins
    __device__ __forceinline__ i64 pos(u64 k) const { return m.pos_sat(u64_to_f64(k)); }
    __device__ __forceinline__ int bin(u64 k) const { return (int)__ldg(table + pos(k)); }
    // Unrounded placement key y in [pos-0.5, pos+0.5], monotone in the key:
    // within a leaf slope*x + icpt is non-decreasing; clamping to the leaf's
    // disjoint, ordered rank range [clamp_lo-0.5, clamp_hi+0.5] keeps order
    // across leaves; flat (slope 0, e.g. empty) leaves sit at clamp_lo-0.5.
    __device__ __forceinline__ double y(u64 k) const {
        const double x = u64_to_f64(k);
        const LjLeaf lf = load_leaf(m.leaves, m.route(x));
        const double lo = i64_to_f64(lf.clamp_lo) - 0.5;
        // flat leaves sit at clamp_lo - 0.5, except at the top: an empty
        // leaf past the last training key has its segment start clamped to
        // n - 1 (models.py:87-93), and keys routed there (larger than every
        // training key) must not sort below the last leaf's y <= n - 0.5
        if (!(lf.slope > 0.0)) return lf.clamp_lo >= m.n - 1 ? i64_to_f64(m.n) - 0.5 : lo;
        const double raw = __dadd_rn(__dmul_rn(lf.slope, x), lf.icpt);
        const double hi = i64_to_f64(lf.clamp_hi) + 0.5;
        return raw < lo ? lo : (raw > hi ? hi : raw);
    }
};

static LsjDev make_lsj(const LjLsjModel &md) {
    LsjDev d;
    d.m = RmiDev(md.rmi);
    d.table = md.table;
    d.pb = md.pb;
    d.nb = (int)md.nbins;
    d.sample = md.sample;
    d.nsample = md.sample ? md.nsample : 0;
    return d;
}

struct LsjBin : NoTable {
    LsjDev d;
    int shift = 0;
    __device__ __forceinline__ u32 code(u64 k) const { return (u32)d.bin(k); }
    __device__ __forceinline__ LsjBin at(u64 *) const { return *this; }
};

// Key boundaries of the bins: B[j] = the first key whose predicted position
// reaches pb[j] (pos() is monotone in the key, so bin(k) = table[pos(k)] =
// #{ j : pb[j] <= pos(k) } = #{ j : B[j] <= k }); a 64-step search over the
// key domain per boundary.  Written as lay[4 + j] (lj_keybin.cuh).
__global__ void k_lsj_key_bounds(LsjDev d, u64 *lay) {
    d.m.fix();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d.nb) return;
    if (j == 0) {
        lay[4] = 0;
        return;
    }
    const i64 target = d.pb[j];
    u64 lo = 0, hi = ~0ULL;  // invariant: pos(hi) >= target or hi == max
    if (d.pos(hi) < target) {
        lay[4 + j] = hi;
        return;
    }
    while (lo < hi) {
        const u64 mid = lo + ((hi - lo) >> 1);
        if (d.pos(mid) >= target) hi = mid;
        else lo = mid + 1;
    }
    lay[4 + j] = lo;
}

// spos[i] = pos(sample[i]) (sample sorted -> spos non-decreasing)
__global__ void k_sample_pos(RmiDev m, const u64 *sample, i64 total, i64 *spos) {
    m.fix();
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x)
        spos[i] = m.pos_sat(u64_to_f64(sample[i]));
}

// pb[0] = 0, pb[j] = spos[floor(j*S/nb)], pb[nb] = trained_len.  A key
// repeated so often that it spans several sample quantiles repeats its
// position v as a boundary; the repeats move to v + 1 (capped by the next
// distinct boundary), so the bin that starts at v holds position v alone --
// the hot key -- and the keys after it get a bin of ordinary size instead of
// sharing one giant bucket, where the split's slice cap left them in slices
// far above the sort's capacity (C4's S: 13 M tuples through the big
// instance).  Still non-decreasing; the bins in between are empty.
__global__ void k_bin_bounds(const i64 *spos, i64 total, int nb, i64 tl, i64 *pb) {
    auto raw = [&](int j) -> i64 {
        if (j <= 0) return 0;
        if (j >= nb) return tl;
        return spos[(i64)(((unsigned __int128)j * (u64)total) / (u64)nb)];
    };
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= nb; j += gridDim.x * blockDim.x) {
        i64 v = raw(j);
        if (j >= 1 && j < nb && raw(j - 1) == v) {
            i64 nx = tl;
            for (int q = j + 1; q < nb; ++q) {
                const i64 r = raw(q);
                if (r > v) {
                    nx = r;
                    break;
                }
            }
            v = v + 1 < nx ? v + 1 : nx;
        }
        pb[j] = v;
    }
}

// table[p] = #{ j in [1, nb-1] : pb[j] <= p }
__global__ void k_bin_table(const i64 *pb, int nb, i64 tl, u32 *table) {
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < tl; p += (i64)gridDim.x * blockDim.x) {
        int lo = 1, hi = nb;  // upper_bound over pb[1..nb-1]
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (pb[mid] <= p) lo = mid + 1; else hi = mid;
        }
        table[p] = (u32)(lo - 1);
    }
}

// ------------------------------------------------------------------- sort

struct SortCtl {
    unsigned long long next;
    unsigned long long n_over;
    unsigned long long n_fallback;
    unsigned long long n_const;
};

// bucket descriptor: [in_base, in_base + m) -> [out_base, out_base + m),
// placement range y in [ybase, ybase + yspan)
struct Bucket {
    i64 in_base, m, out_base;
    double ybase, yspan;
    bool point;  // a point slice (one repeated key), already written in place
};

// Sub-buckets written by k_lsj_split: y-slices of the coarse buckets, in
// place (sub-bucket g covers [sub_starts[g], sub_starts[g+1]) of both the
// split array and the final output).
struct SubBuckets {
    const i64 *sub_starts;  // [G+1]
    const double2 *sub_y;   // [G] {ybase, yspan}
    __device__ __forceinline__ Bucket get(i64 g) const {
        Bucket k;
        k.in_base = sub_starts[g];
        k.m = sub_starts[g + 1] - k.in_base;
        k.out_base = k.in_base;
        const double2 y = sub_y[g];
        k.ybase = y.x;
        k.yspan = y.y;
        k.point = y.y < 0.0;
        return k;
    }
};

template <int NT>
__device__ __forceinline__ void block_scan_u32(u32 *a, int n, u32 *warp_tot) {
    // exclusive scan of a[0..n) in place, NT threads
    const int per = (n + NT - 1) / NT;
    const int j0 = threadIdx.x * per;
    u32 local = 0;
    for (int j = j0; j < j0 + per && j < n; ++j) local += a[j];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        u32 t = lane < NT / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        if (lane < NT / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    u32 run = (warp ? warp_tot[warp - 1] : 0) + incl - local;
    for (int j = j0; j < j0 + per && j < n; ++j) {
        u32 c = a[j];
        a[j] = run;
        run += c;
    }
    __syncthreads();
}

// The same scan over n words that each pack TWO u16 counters (slot 2j in the
// low half, 2j+1 in the high half): every half becomes its exclusive prefix
// (all sums stay below 2^15: n <= 12288 tuples per bucket).
template <int NT>
__device__ __forceinline__ void block_scan_u16x2(u32 *a, int n, u32 *warp_tot) {
    const int per = (n + NT - 1) / NT;
    const int j0 = threadIdx.x * per;
    u32 local = 0;
    for (int j = j0; j < j0 + per && j < n; ++j) {
        const u32 w = a[j];
        local += (w & 0xFFFFu) + (w >> 16);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        u32 t = lane < NT / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        if (lane < NT / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    u32 run = (warp ? warp_tot[warp - 1] : 0) + incl - local;
    for (int j = j0; j < j0 + per && j < n; ++j) {
        const u32 w = a[j];
        const u32 lo = w & 0xFFFFu, hi = w >> 16;
        a[j] = run | ((run + lo) << 16);
        run += lo + hi;
    }
    __syncthreads();
}

// Coarse bucket b -> F_b = ceil(m_b / SUB) slices of about SUB tuples.  With
// a fit sample the F_b - 1 split points are equi-depth sample quantiles of
// y, and every split value also gets its own "point" slice (y == v): a key
// repeated millions of times (Zipf) then lands alone in a point slice,
// which the sort recognises as constant and copies.  Slots per bucket:
// 2 F_b - 1 (many stay empty); without a sample, F_b uniform y-slices.
__device__ __forceinline__ i64 split_count(i64 m) {
    const i64 f = (m + SUB - 1) / SUB;
    return m == 0 ? 0 : (f < 1 ? 1 : (f > SPLIT_MAXF ? SPLIT_MAXF : f));
}

__global__ void k_split_plan(const i64 *bstart, const i64 *bend, int nb, int points, i64 *fcount) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
        if (b == nb) {
            fcount[b] = 0;
            continue;
        }
        const i64 f = split_count(bend[b] - bstart[b]);
        fcount[b] = points && f > 0 ? 2 * f - 1 : f;
    }
}

// split values of bucket b -> spv[fbase[b] .. fbase[b] + F_b - 1)
// bin of every sample key (the sample is sorted, so these are non-decreasing)
__global__ void k_sample_bins(LsjDev md, u32 *sbin) {
    md.m.fix();
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < md.nsample; i += (i64)gridDim.x * blockDim.x)
        sbin[i] = (u32)md.bin(md.sample[i]);
}

// sample index range [sr[b], se[b]) of every bin (bins are monotone over the
// sorted sample)
__global__ void k_split_ranges(LsjDev md, const u32 *sbin, int nb, i64 *sr, i64 *se) {
    md.m.fix();
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
        i64 lo = 0, hi = md.nsample;
        while (lo < hi) {
            i64 mid = (lo + hi) >> 1;
            if ((sbin ? (int)sbin[mid] : md.bin(md.sample[mid])) < b) lo = mid + 1; else hi = mid;
        }
        sr[b] = lo;
        hi = md.nsample;
        while (lo < hi) {
            i64 mid = (lo + hi) >> 1;
            if ((sbin ? (int)sbin[mid] : md.bin(md.sample[mid])) <= b) lo = mid + 1; else hi = mid;
        }
        se[b] = lo;
    }
}

// split KEYS at sample quantiles, one thread per slot g of the slot space
// (distinct keys always separate, even where the model's placement y is
// flat); too few sample keys: the quantiles repeat (empty slices), none:
// one slice for the bucket.  Bucket b's values: spv[fbase[b] + j - 1],
// j in [1, F_b).
__global__ void k_split_points(LsjDev md, const i64 *bstart, const i64 *bend, const i64 *fbase, int nb, const i64 *sr,
                               const i64 *se, u64 *spv) {
    md.m.fix();
    const i64 G = fbase[nb];
    for (i64 g = blockIdx.x * (i64)blockDim.x + threadIdx.x; g < G; g += (i64)gridDim.x * blockDim.x) {
        int lo = 0, hi = nb;  // bucket of slot g: last b with fbase[b] <= g
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (fbase[mid] <= g) lo = mid; else hi = mid;
        }
        const int b = lo;
        const i64 F = split_count(bend[b] - bstart[b]), j = g - fbase[b] + 1;
        if (F < 2 || j >= F) continue;
        const i64 sb = sr[b], ns = se[b] - sb;
        const i64 q = sb + (j * ns) / F;
        spv[g] = ns > 0 ? md.sample[q < se[b] ? q : se[b] - 1] : ~0ULL;
    }
}

__device__ __forceinline__ int y_slice(double y, double ybase, double scale, int F) {
    const double f = floor((y - ybase) * scale);
    return f < 0.0 ? 0 : (f >= (double)(F - 1) ? F - 1 : (int)f);
}

// point-slice mode: slot of key k among split keys v[0..K): 2i for keys in
// (v[i-1], v[i]), 2i+1 for k == v[i] (a repeated hot key gets a slice of
// its own), i = lower_bound(v, k):
// found through a radix table over the split keys (built per work
// item in shared memory): cells[c] = #{ i : cell(v[i]) < c } bounds the
// lower bound to [cells[c], cells[c+1]] (cell() monotone), so the search
// runs over a cell's few keys instead of all K.
constexpr int SPLIT_CELLS = 1024;
struct SplitTab {
    u64 v0;
    int sh;
};
__device__ __forceinline__ int split_cell(const SplitTab &t, u64 k) {
    if (k < t.v0) return 0;
    const u64 c = (k - t.v0) >> t.sh;
    return c >= (u64)SPLIT_CELLS ? SPLIT_CELLS - 1 : (int)c;
}
// all threads; v[0..K) staged and synced; returns the table parameters
__device__ SplitTab split_tab_build(const u64 *v, int K, u16 *cells) {
    SplitTab t;
    t.v0 = K ? v[0] : 0;
    const u64 span = K ? v[K - 1] - t.v0 : 0;
    int sh = 0;
    while (sh < 63 && (span >> sh) >= (u64)SPLIT_CELLS) ++sh;
    t.sh = sh;
    // value i on (c_{i-1}, c_i], c_{-1} = -1, c_K = SPLIT_CELLS
    for (int i = threadIdx.x; i <= K; i += blockDim.x) {
        const int lo = i == 0 ? 0 : split_cell(t, v[i - 1]) + 1;
        const int hi = i == K ? SPLIT_CELLS : split_cell(t, v[i]);
        for (int c = lo; c <= hi; ++c) cells[c] = (u16)i;
    }
    __syncthreads();
    return t;
}
__device__ __forceinline__ int point_slot_tab(const u64 *v, int K, const u16 *cells, const SplitTab &t, u64 k) {
    const int c = split_cell(t, k);
    int lo = cells[c], hi = cells[c + 1];  // lower bound in [lo, hi]
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (v[mid] < k) lo = mid + 1; else hi = mid;
    }
    return 2 * lo + ((lo < K && v[lo] == k) ? 1 : 0);
}

// Level 2 as a balanced, segmented partition.  Work item = a chunk of <=
// SPLIT_CH tuples of one coarse bucket (hot buckets span many chunks, so no
// CTA owns a whole hot-key bucket).  Pass 1 counts each chunk's slots in
// shared memory into a block-diagonal (slot x chunk) matrix laid out
// bucket-major, slot-major; one exclusive scan of it yields, for every
// (bucket, slot, chunk), the absolute output position (buckets are
// contiguous and in order); pass 2 re-walks the chunk and scatters through
// shared-memory cursors.  A chunk keeps <= 4095 write frontiers open.

struct SplitCtx {  // per-bucket layout shared by the split kernels
    const i64 *bstart;  // [nb] coarse bucket b = records [bstart[b], bend[b]) of the input
    const i64 *bend;    // (contiguous bins: bend = bstart + 1; one-pass regions leave gaps)
    const i64 *fbase;   // [nb+1] first slot of each bucket
    const i64 *cbase;   // [nb+1] first chunk of each bucket
    const i64 *mbase;   // [nb+1] first matrix entry of each bucket
    const u64 *spv;     // split keys (point mode), at fbase[b]
    int nb;
};

__global__ void k_chunk_plan(const i64 *bstart, const i64 *bend, const i64 *fbase, int nb, i64 *chunks, i64 *matc) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
        if (b == nb) {
            chunks[b] = matc[b] = 0;
            continue;
        }
        const i64 m = bend[b] - bstart[b];
        const i64 c = (m + SPLIT_CH - 1) / SPLIT_CH;
        chunks[b] = c;
        matc[b] = c * (fbase[b + 1] - fbase[b]);
    }
}

struct SplitItem {
    i64 b, c, chunks, a, e, g0;
    int F, K;
    double ybase, yspan, scale;
};

__device__ __forceinline__ SplitItem split_item(const LsjDev &md, const SplitCtx &cx, i64 q, bool points) {
    int lo = 0, hi = cx.nb;  // last bucket with cbase[b] <= q
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (cx.cbase[mid] <= q) lo = mid; else hi = mid;
    }
    SplitItem it;
    it.b = lo;
    it.c = q - cx.cbase[lo];
    it.chunks = cx.cbase[lo + 1] - cx.cbase[lo];
    const i64 a0 = cx.bstart[lo], e0 = cx.bend[lo];
    it.a = a0 + it.c * SPLIT_CH;
    it.e = min(it.a + (i64)SPLIT_CH, e0);
    it.g0 = cx.fbase[lo];
    it.F = (int)(cx.fbase[lo + 1] - it.g0);
    it.K = points ? (it.F - 1) / 2 : 0;
    it.ybase = i64_to_f64(md.pb[lo]) - 0.5;
    it.yspan = i64_to_f64(md.pb[lo + 1] - md.pb[lo]);
    if (!(it.yspan > 0.0)) it.yspan = 1.0;
    it.scale = (double)it.F / it.yspan;
    return it;
}

__device__ __forceinline__ int split_slot(const LsjDev &md, const SplitItem &it, const u64 *v, bool points, u64 k,
                                          const u16 *cells, const SplitTab &tab) {
    return points ? point_slot_tab(v, it.K, cells, tab, k) : y_slice(md.y(k), it.ybase, it.scale, it.F);
}

// pass 1: mat[mbase[b] + s * chunks_b + c] = tuples of chunk c in slot s
__global__ void __launch_bounds__(SPLIT_NT) k_split_count(LsjDev md, SplitCtx cx, const ulonglong2 *__restrict__ A,
                                                          const i64 *nitems, u32 *mat, SortCtl *ctl) {
    md.m.fix();
    __shared__ u32 h[2 * SPLIT_MAXF];
    __shared__ u64 v[SPLIT_MAXF];
    __shared__ u16 cells[SPLIT_CELLS + 1];
    __shared__ i64 s_q;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool points = md.sample != nullptr;
    const i64 total = *nitems;
    for (;;) {
        if (threadIdx.x == 0) s_q = (i64)atomicAdd(&ctl->next, 1ULL);
        __syncthreads();
        const i64 q = s_q;
        if (q >= total) break;
        const SplitItem it = split_item(md, cx, q, points);
        for (int j = threadIdx.x; j < it.F; j += SPLIT_NT) h[j] = 0;
        for (int j = threadIdx.x; j < it.K; j += SPLIT_NT) v[j] = cx.spv[it.g0 + j];
        __syncthreads();
        const SplitTab tab = points ? split_tab_build(v, it.K, cells) : SplitTab{0, 0};
        for (i64 base = it.a + (i64)warp * 32 * SPLIT_U; base < it.e; base += (i64)SPLIT_NT * SPLIT_U) {
            int s[SPLIT_U];
#pragma unroll
            for (int u = 0; u < SPLIT_U; ++u) {
                const i64 i = base + u * 32 + lane;
                s[u] = i < it.e ? split_slot(md, it, v, points, A[i].x, cells, tab) : -1;
            }
#pragma unroll
            for (int u = 0; u < SPLIT_U; ++u) {
                // one atomic for a warp on a single slot (runs of a hot key),
                // else one shared atomic per tuple (match.any is ~10x slower)
                const int s0 = __shfl_sync(0xffffffffu, s[u], 0);
                if (__all_sync(0xffffffffu, s[u] == s0)) {
                    if (lane == 0 && s0 >= 0) atomicAdd(h + s0, 32u);
                } else if (s[u] >= 0) {
                    atomicAdd(h + s[u], 1u);
                }
            }
        }
        __syncthreads();
        const i64 mb = cx.mbase[it.b];
        for (int j = threadIdx.x; j < it.F; j += SPLIT_NT) mat[mb + (i64)j * it.chunks + it.c] = h[j];
        __syncthreads();
    }
}

// slot bounds + placement ranges from the scanned matrix
__global__ void k_split_slots(LsjDev md, SplitCtx cx, const i64 *off, i64 n, i64 *sub_starts, double2 *sub_y) {
    md.m.fix();
    const bool points = md.sample != nullptr;
    const i64 G = cx.fbase[cx.nb];
    for (i64 g = blockIdx.x * (i64)blockDim.x + threadIdx.x; g <= G; g += (i64)gridDim.x * blockDim.x) {
        if (g == G) {
            sub_starts[g] = n;
            continue;
        }
        int lo = 0, hi = cx.nb;  // bucket of slot g
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (cx.fbase[mid] <= g) lo = mid; else hi = mid;
        }
        const i64 b = lo, j = g - cx.fbase[b], F = cx.fbase[b + 1] - cx.fbase[b];
        const i64 chunks = cx.cbase[b + 1] - cx.cbase[b];
        sub_starts[g] = off[cx.mbase[b] + j * chunks];
        const double ybase = i64_to_f64(md.pb[b]) - 0.5;
        double yspan = i64_to_f64(md.pb[b + 1] - md.pb[b]);
        if (!(yspan > 0.0)) yspan = 1.0;
        if (!points) {
            sub_y[g] = make_double2(ybase + (double)j * yspan / (double)F, yspan / (double)F);
        } else {
            const i64 K = (F - 1) / 2;
            const u64 *v = cx.spv + cx.fbase[b];
            // y is monotone in the key: the slice's placement range is the
            // y range of its bounding split keys
            if (j & 1) {  // point slot: every key equals v[(j-1)/2]; written to the
                          // output by the split scatter (span -1 marks it)
                sub_y[g] = make_double2(md.y(v[(j - 1) >> 1]), -1.0);
            } else {      // open interval between split keys
                const i64 q = j >> 1;
                const double l = q == 0 ? ybase : md.y(v[q - 1]);
                const double h = (q == K || v[q] == ~0ULL) ? ybase + yspan : md.y(v[q]);
                sub_y[g] = make_double2(l, h > l ? h - l : 0.0);
            }
        }
    }
}

// pass 2: scatter every chunk through shared-memory cursors
__global__ void __launch_bounds__(SPLIT_NT, LJ_SPLIT_MINB) k_split_scatter(LsjDev md, SplitCtx cx, const ulonglong2 *__restrict__ A,
                                                            const i64 *nitems, const i64 *__restrict__ off,
                                                            ulonglong2 *B, ulonglong2 *Out, SortCtl *ctl) {
    md.m.fix();
    __shared__ u32 cur[2 * SPLIT_MAXF];
    __shared__ u64 v[SPLIT_MAXF];
    __shared__ u16 cells[SPLIT_CELLS + 1];
    __shared__ i64 s_q;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool points = md.sample != nullptr;
    const i64 total = *nitems;
    for (;;) {
        if (threadIdx.x == 0) s_q = (i64)atomicAdd(&ctl->next, 1ULL);
        __syncthreads();
        const i64 q = s_q;
        if (q >= total) break;
        const SplitItem it = split_item(md, cx, q, points);
        // a0: the bucket's start in the OUTPUT (dense: the scanned matrix is
        // bucket-major, so its first entry is the tuples of all earlier buckets)
        const i64 mb = cx.mbase[it.b], a0 = off[mb];
        for (int j = threadIdx.x; j < it.F; j += SPLIT_NT) cur[j] = (u32)(off[mb + (i64)j * it.chunks + it.c] - a0);
        for (int j = threadIdx.x; j < it.K; j += SPLIT_NT) v[j] = cx.spv[it.g0 + j];
        __syncthreads();
        const SplitTab tab = points ? split_tab_build(v, it.K, cells) : SplitTab{0, 0};
        for (i64 base = it.a + (i64)warp * 32 * SPLIT_U; base < it.e; base += (i64)SPLIT_NT * SPLIT_U) {
            int s[SPLIT_U];
            ulonglong2 r[SPLIT_U];
            if ((lane & 7) == 0) {
                // the records of two steps ahead start their way into L2 (one
                // prefetch per 128-B line): more bytes in flight than the
                // registers hold
#pragma unroll
                for (int u = 0; u < SPLIT_U; ++u) {
                    const i64 ip = base + 2 * (i64)SPLIT_NT * SPLIT_U + u * 32 + lane;
                    if (ip < it.e) asm volatile("prefetch.global.L2 [%0];" ::"l"(A + ip));
                }
            }
#pragma unroll
            for (int u = 0; u < SPLIT_U; ++u) {
                const i64 i = base + u * 32 + lane;
                r[u] = i < it.e ? A[i] : make_ulonglong2(0, 0);
                s[u] = i < it.e ? split_slot(md, it, v, points, r[u].x, cells, tab) : -1;
            }
#pragma unroll
            for (int u = 0; u < SPLIT_U; ++u) {
                const int s0 = __shfl_sync(0xffffffffu, s[u], 0);
                if (__all_sync(0xffffffffu, s[u] == s0)) {
                    if (s0 >= 0) {
                        u32 at = 0;
                        if (lane == 0) at = atomicAdd(cur + s0, 32u);
                        // point slices (one key) are final: straight to the output
                        ulonglong2 *dst = (points && (s0 & 1)) ? Out : B;
                        dst[a0 + __shfl_sync(0xffffffffu, at, 0) + lane] = r[u];
                    }
                } else if (s[u] >= 0) {
                    ulonglong2 *dst = (points && (s[u] & 1)) ? Out : B;
                    dst[a0 + atomicAdd(cur + s[u], 1u)] = r[u];
                }
            }
        }
        __syncthreads();
    }
}

// Block-wide sort of the pairs (K[i], X[i]), i in [base, base+len), by key: a
// bitonic network in its "flip" form, whose comparators all put the minimum
// at the lower index, so positions >= len act as +inf and their comparators
// are skipped.
template <int NT>
__device__ void block_sort_pairs(u64 *K, u16 *X, int base, int len) {
    int w = 1;
    while (w < len) w <<= 1;
    for (int k = 2; k <= w; k <<= 1) {
        for (int j = k; j > 1; j >>= 1) {
            const bool flip = j == k;
            const int h = j >> 1;
            for (int t = threadIdx.x; t < (w >> 1); t += NT) {
                // t-th comparator of this stage: i in the lower half of its
                // j-block, partner mirrored (flip) or h apart
                const int i = (t / h) * j + (t % h);
                const int l = flip ? (i ^ (j - 1)) : (i + h);
                if (l < len) {
                    const u64 a = K[base + i], c = K[base + l];
                    if (a > c) {
                        K[base + i] = c;
                        K[base + l] = a;
                        const u16 x = X[base + i];
                        X[base + i] = X[base + l];
                        X[base + l] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// number of keys of the run KP[a, e) that sort before (k at placement p):
// smaller keys, and equal keys placed earlier
__device__ __forceinline__ int run_rank(const u64 *KP, int a, int e, int p, u64 k) {
    int r = 0;
    for (int q = a; q < e; ++q) {
        const u64 kq = KP[q];
        r += (kq < k || (kq == k && q < p)) ? 1 : 0;
    }
    return r;
}

// K8: one CTA per bucket (dynamic work counter), model-placed in shared
// memory.  Every thread OWNS E = CAPV / NT tuples of the bucket (tuple
// e * NT + tid) and keeps their keys and (slot, position) in registers:
//   1. load the keys (E loads in flight), slot = floor((y - ybase) * m /
//      yspan) in [0, m), count the slots;
//   2. exclusive scan of the counts;
//   3. claim a position in the slot's run (shared atomic), key -> KP[pos]:
//      keys in PLACEMENT order, misordered only inside a slot's run;
//   4. rank inside the run: runs of <= RUN_DIRECT keys by scanning the run
//      (one shared load per step); longer runs are first classified -- an
//      owner whose key differs from the run's first marks the run MIXED --
//      constant runs (one repeated key) keep their placement order, mixed
//      runs of <= RUN_SMALL are ranked by scanning, longer ones are queued
//      for a block-wide bitonic sort;
//   5. key -> KP[final] (the placement array is dead after the ranking),
//      tuple index -> IDX[final];
//   6. write-out in final order, coalesced: key from shared memory, payload
//      gathered from the bucket (L2-hot), with a sortedness check on the way
//      (a misordered bucket is re-sorted whole and rewritten: a safety net
//      that the monotone placement never needs).
// 14 B of shared memory per tuple.  Buckets above CAPV go to over_list
// (ctl->n_over); the "big" instance (one CTA per SM, CAPV = CAP_BIG) sorts
// that list and passes what exceeds it on.
constexpr int RUN_DIRECT = 8;

// Slot counters: one u32 per slot, or (LJ_SORT_SLOTS2) TWO placement slots
// per tuple packed as u16 halves of the same words -- half the collisions
// (runs of >= 2 keys hold 39 % of the tuples instead of 63 %) at the same
// shared memory, zeroing and scan cost.  A half holds a count, then a
// cursor, then its run's end (< 2^15) with the MIXED flag above it.
// Measured at C4: 7.24 vs 7.13 ms for both relations -- the shorter runs do
// not pay for the packing arithmetic -- so it is off by default.
#ifndef LJ_SORT_SLOTS2
#define LJ_SORT_SLOTS2 0
#endif
constexpr bool SLOTS2 = LJ_SORT_SLOTS2 != 0;
constexpr u32 SLOT_MIXED = SLOTS2 ? 0x8000u : 0x80000000u;
__device__ __forceinline__ void slot_count(u32 *cnt, int sl) {
    if (SLOTS2) atomicAdd(cnt + (sl >> 1), 1u << ((sl & 1) << 4));
    else atomicAdd(cnt + sl, 1u);
}
__device__ __forceinline__ u32 slot_claim(u32 *cnt, int sl) {
    if (!SLOTS2) return atomicAdd(cnt + sl, 1u);
    const int sh = (sl & 1) << 4;
    return (atomicAdd(cnt + (sl >> 1), 1u << sh) >> sh) & 0x7FFFu;
}
__device__ __forceinline__ u32 slot_word(const u32 *cnt, int sl) {  // run end | MIXED
    return SLOTS2 ? (cnt[sl >> 1] >> ((sl & 1) << 4)) & 0xFFFFu : cnt[sl];
}
__device__ __forceinline__ void slot_mark_mixed(u32 *cnt, int sl) {
    if (SLOTS2) atomicOr(cnt + (sl >> 1), SLOT_MIXED << ((sl & 1) << 4));
    else atomicOr(cnt + sl, SLOT_MIXED);
}

template <class Src, int NT, int CAPV, int CTAS>
__global__ void __launch_bounds__(NT, CTAS) k_lsj_sort(LsjDev md, Src src, const unsigned long long *nbuckets_dev,
                                                       const ulonglong2 *__restrict__ in, ulonglong2 *out,
                                                       SortCtl *ctl, i64 *over_list) {
    constexpr int E = CAPV / NT;
    static_assert(CAPV % NT == 0 && CAPV <= 65536, "tuples per thread / u16 indices");
    md.m.fix();
    const i64 nbuckets = (i64)*nbuckets_dev;
    extern __shared__ __align__(16) unsigned char smem[];
    u64 *KP = reinterpret_cast<u64 *>(smem);           // keys: placement order, then final order [CAPV]
    u32 *cnt = reinterpret_cast<u32 *>(KP + CAPV);       // slot counts -> cursors -> run ends [CAPV]
    u16 *IDX = reinterpret_cast<u16 *>(cnt + CAPV);      // tuple of every final position [CAPV]
    __shared__ u32 warp_tot[NT / 32];
    __shared__ i64 s_q[2];
    __shared__ int s_nruns;
    __shared__ int2 s_runs[MAX_RUNS];
    __shared__ u64 s_mm[2 * (NT / 32)];  // per-warp key min / max (flat-model buckets)
    constexpr u32 MIXED = SLOT_MIXED;
    static_assert(!SLOTS2 || CAPV < 32768, "u16 slot halves");
    const int tid = threadIdx.x;
    for (int j = tid; j < CAPV; j += NT) cnt[j] = 0;
    if (tid == 0) s_q[0] = (i64)atomicAdd(&ctl->next, 1ULL);
    __syncthreads();
    for (int par = 0;; par ^= 1) {
        const i64 b = s_q[par];
        if (b >= nbuckets) break;
        if (tid == 0) {
            // claim the next bucket now: its tuples stream into L2 (bulk
            // prefetch) while this one sorts
            const i64 nx = (i64)atomicAdd(&ctl->next, 1ULL);
            s_q[par ^ 1] = nx;
            s_nruns = 0;
            if (nx < nbuckets) {
                const Bucket nk = src.get(nx);
                if (!nk.point && nk.m > 1 && nk.m <= (i64)CAPV)
                    bulk_prefetch_l2(in + nk.in_base, (unsigned)(nk.m * sizeof(ulonglong2)));
            }
        }
        const Bucket bk = src.get(b);
        if (bk.m <= 1 || bk.point || bk.m > (i64)CAPV) {
            if (tid == 0 && !bk.point) {
                if (bk.m == 1) out[bk.out_base] = in[bk.in_base];
                if (bk.m > (i64)CAPV) {
                    over_list[atomicAdd(&ctl->n_over, 1ULL)] = b;
#ifdef LJ_SORT_DIAG
                    printf("over %d %lld %lld %f %f\n", CAPV, (long long)b, (long long)bk.m, bk.ybase, bk.yspan);
#endif
                }
            }
            __syncthreads();
            continue;
        }
        const int m = (int)bk.m;
        const ulonglong2 *src_rec = in + bk.in_base;
        const int ns = SLOTS2 ? 2 * m : m;  // placement slots
        const double scale = (double)ns / (bk.yspan > 0.0 ? bk.yspan : 1.0);
        // 1. keys, slots, slot counts
        u64 k[E];
        u32 sp[E];  // slot | position << 16
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = e * NT + tid;
            k[e] = i < m ? src_rec[i].x : 0;
        }
        // A bucket over which the model is FLAT (keys clamped to one leaf
        // bound: C4's S has 12 M such tuples) would put every key into one
        // slot and be bitonic-sorted whole: it is placed by linear
        // interpolation over its own key range instead (monotone in the key
        // like the model, so everything after is unchanged).
        const bool flat = !(bk.yspan > 0.0);
        u64 kmin = 0;
        double sc = scale;
        if (flat) {
            u64 kmax = 0;
            kmin = ~0ULL;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (e * NT + tid < m) {
                    kmin = k[e] < kmin ? k[e] : kmin;
                    kmax = k[e] > kmax ? k[e] : kmax;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const u64 a = __shfl_xor_sync(0xffffffffu, kmin, o), c = __shfl_xor_sync(0xffffffffu, kmax, o);
                kmin = a < kmin ? a : kmin;
                kmax = c > kmax ? c : kmax;
            }
            if ((tid & 31) == 0) {
                s_mm[2 * (tid >> 5)] = kmin;
                s_mm[2 * (tid >> 5) + 1] = kmax;
            }
            __syncthreads();
#pragma unroll 1
            for (int w = 0; w < NT / 32; ++w) {
                kmin = s_mm[2 * w] < kmin ? s_mm[2 * w] : kmin;
                kmax = s_mm[2 * w + 1] > kmax ? s_mm[2 * w + 1] : kmax;
            }
            sc = (double)ns / (u64_to_f64(kmax - kmin) + 1.0);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = e * NT + tid;
            if (i < m) {
                const double v = flat ? u64_to_f64(k[e] - kmin) : md.y(k[e]) - bk.ybase;
                const double f = floor(v * sc);
                const int sl = f < 0.0 ? 0 : (f >= (double)(ns - 1) ? ns - 1 : (int)f);
                sp[e] = (u32)sl;
                slot_count(cnt, sl);
            }
        }
        __syncthreads();
        // 2. run starts
        if (SLOTS2) block_scan_u16x2<NT>(cnt, m, warp_tot);
        else block_scan_u32<NT>(cnt, m, warp_tot);
        // 3. placement: afterwards cnt[s] = end of slot s's run = start of slot s+1's
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = e * NT + tid;
            if (i < m) {
                const u32 p = slot_claim(cnt, (int)sp[e]);
                KP[p] = k[e];
                sp[e] |= p << 16;
            }
        }
        __syncthreads();
        // 4. rank in the run -> final position (kept in sp's upper half)
        int need_long = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = e * NT + tid;
            if (i < m) {
                const int sl = (int)(sp[e] & 0xFFFFu), p = (int)(sp[e] >> 16);
                const int a = sl > 0 ? (int)(slot_word(cnt, sl - 1) & ~MIXED) : 0;
                const int en = (int)(slot_word(cnt, sl) & ~MIXED);
                if (en - a > RUN_DIRECT) {
                    need_long = 1;
                    if (k[e] != KP[a]) slot_mark_mixed(cnt, sl);
                } else if (en - a > 1) {
                    sp[e] = (u32)sl | ((u32)(a + run_rank(KP, a, en, p, k[e])) << 16);
                }
            }
        }
        if (__syncthreads_or(need_long)) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = e * NT + tid;
                if (i < m) {
                    const int sl = (int)(sp[e] & 0xFFFFu), p = (int)(sp[e] >> 16);
                    const u32 ce = slot_word(cnt, sl);
                    const int a = sl > 0 ? (int)(slot_word(cnt, sl - 1) & ~MIXED) : 0, en = (int)(ce & ~MIXED);
                    if (en - a > RUN_DIRECT && (ce & MIXED)) {
                        if (en - a <= RUN_SMALL) {
                            sp[e] = (u32)sl | ((u32)(a + run_rank(KP, a, en, p, k[e])) << 16);
                        } else if (p == a) {  // long mixed run: sorted block-wide below
                            const int q = atomicAdd(&s_nruns, 1);
                            if (q < MAX_RUNS) s_runs[q] = make_int2(a, en - a);
                        }
                    }
                }
            }
            __syncthreads();
        }
        // 5. final order (the ranking's reads of KP are done)
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = e * NT + tid;
            if (i < m) {
                const int f = (int)(sp[e] >> 16);
                KP[f] = k[e];
                IDX[f] = (u16)i;
            }
        }
        __syncthreads();
        const int nruns = s_nruns;
        if (nruns > MAX_RUNS) {
            block_sort_pairs<NT>(KP, IDX, 0, m);
        } else {
            for (int q = 0; q < nruns; ++q) block_sort_pairs<NT>(KP, IDX, s_runs[q].x, s_runs[q].y);
        }
        // 6. write out: key from smem, payload gathered from the bucket
        // (L2-hot); the slot counters are cleared for the next bucket
        for (int pass = 0;; ++pass) {
            int bad = 0;
            for (int i0 = tid; i0 < m; i0 += NT * SORT_U) {
                u64 kf[SORT_U], py[SORT_U];
#pragma unroll
                for (int u = 0; u < SORT_U; ++u) {
                    const int i = i0 + u * NT;
                    kf[u] = i < m ? KP[i] : 0;
                    py[u] = i < m ? __ldg(&src_rec[IDX[i]].y) : 0;
                    if (i + 1 < m && kf[u] > KP[i + 1]) bad = 1;
                }
#pragma unroll
                for (int u = 0; u < SORT_U; ++u) {
                    const int i = i0 + u * NT;
                    if (i < m) {
                        out[bk.out_base + i] = make_ulonglong2(kf[u], py[u]);
                        cnt[i] = 0;
                    }
                }
            }
            if (!__syncthreads_or(bad)) break;
            // safety net: the placement key is monotone, so a bucket is
            // never misordered here; if it is, sort it whole and rewrite
            block_sort_pairs<NT>(KP, IDX, 0, m);
            if (tid == 0 && pass == 0) atomicAdd(&ctl->n_fallback, 1ULL);
        }
    }
}

// The sub-buckets the main sort passed over (above CAP), by list index:
// the "big" sort instance (one CTA per SM, up to CAP_BIG tuples in shared
// memory) takes them from this view.
struct OverBuckets {
    const i64 *list;
    SubBuckets sub;
    __device__ __forceinline__ Bucket get(i64 q) const { return sub.get(list[q]); }
};

// The rare sub-buckets above CAP_BIG, device-driven (no host readback): one
// CTA per bucket sorts it in global memory -- chunks of HUGE_CH records
// sorted in shared memory (bitonic), then bottom-up merge passes (merge
// path: every thread finds its output range by a binary search over the
// two runs) ping-ponging between the split array and the output.
constexpr int HUGE_NT = 1024;
constexpr int HUGE_CH = 8192;  // 128 KB of records in shared memory

__device__ __forceinline__ bool rec_less(const ulonglong2 &a, const ulonglong2 &b) { return a.x < b.x; }

__device__ void huge_chunk_sort(ulonglong2 *sm, int len) {
    int w = 1;
    while (w < len) w <<= 1;
    for (int i = len + (int)threadIdx.x; i < w; i += HUGE_NT) sm[i] = make_ulonglong2(~0ULL, 0ULL);
    __syncthreads();
    for (int k = 2; k <= w; k <<= 1)
        for (int j = k; j > 1; j >>= 1) {
            const bool flip = j == k;
            const int h = j >> 1;
            for (int t = threadIdx.x; t < (w >> 1); t += HUGE_NT) {
                const int i = (t / h) * j + (t % h);
                const int l = flip ? (i ^ (j - 1)) : (i + h);
                const ulonglong2 x = sm[i], y = sm[l];
                if (rec_less(y, x)) {
                    sm[i] = y;
                    sm[l] = x;
                }
            }
            __syncthreads();
        }
}

// merge sorted A[0, na) and B[0, nb) into C: each thread its slice of the
// output (merge path)
__device__ void block_merge(const ulonglong2 *A, i64 na, const ulonglong2 *B, i64 nb, ulonglong2 *C) {
    const i64 tot = na + nb, per = (tot + HUGE_NT - 1) / HUGE_NT;
    const i64 d0 = min(tot, (i64)threadIdx.x * per), d1 = min(tot, d0 + per);
    if (d0 >= d1) return;
    // first diagonal split: i in [max(0, d0 - nb), min(d0, na)] with A[i-1] <= B[d0-i] < ...
    i64 lo = d0 > nb ? d0 - nb : 0, hi = d0 < na ? d0 : na;
    while (lo < hi) {
        const i64 i = (lo + hi) >> 1;
        if (A[i].x <= B[d0 - i - 1].x) lo = i + 1;
        else hi = i;
    }
    i64 i = lo, j = d0 - lo;
    for (i64 d = d0; d < d1; ++d) {
        if (j >= nb || (i < na && A[i].x <= B[j].x)) C[d] = A[i++];
        else C[d] = B[j++];
    }
}

// list[q] indexes the big instance's bucket space (OverBuckets): the big
// instance passed on its own bucket numbers
__global__ void __launch_bounds__(HUGE_NT, 1) k_lsj_huge(OverBuckets sub, const i64 *list,
                                                         const unsigned long long *nlist, ulonglong2 *B,
                                                         ulonglong2 *out) {
    extern __shared__ __align__(16) ulonglong2 hsm[];
    const i64 nh = (i64)*nlist;
    for (i64 q = blockIdx.x; q < nh; q += gridDim.x) {
        const Bucket bk = sub.get(list[q]);
        const i64 a = bk.in_base, len = bk.m;
        // sorted chunks -> out
        for (i64 c0 = 0; c0 < len; c0 += HUGE_CH) {
            const int cl = (int)min((i64)HUGE_CH, len - c0);
            for (int i = threadIdx.x; i < cl; i += HUGE_NT) hsm[i] = B[a + c0 + i];
            __syncthreads();
            huge_chunk_sort(hsm, cl);
            for (int i = threadIdx.x; i < cl; i += HUGE_NT) out[bk.out_base + c0 + i] = hsm[i];
            __syncthreads();
        }
        // merge passes: out -> B -> out ...
        ulonglong2 *src = out + bk.out_base, *dst = B + a;
        for (i64 wdt = HUGE_CH; wdt < len; wdt <<= 1) {
            for (i64 m0 = 0; m0 < len; m0 += 2 * wdt) {
                const i64 na = min(wdt, len - m0), nb = min(wdt, max((i64)0, len - m0 - wdt));
                block_merge(src + m0, na, src + m0 + na, nb, dst + m0);
            }
            __syncthreads();
            ulonglong2 *t = src;
            src = dst;
            dst = t;
        }
        if (src != out + bk.out_base)
            for (i64 i = threadIdx.x; i < len; i += HUGE_NT) out[bk.out_base + i] = src[i];
        __syncthreads();
    }
}

// SortCtl counters of both sort instances -> stats[4] (device): oversized
// sub-buckets (> CAP), fallbacks, sorted by the big instance, above CAP_BIG
__global__ void k_sort_stats(const SortCtl *c1, const SortCtl *c2, i64 *stats) {
    stats[0] = (i64)c1->n_over;
    stats[1] = (i64)(c1->n_fallback + c2->n_fallback);
    stats[2] = (i64)c1->n_over - (i64)c2->n_over;
    stats[3] = (i64)c2->n_over;
}

// reference bucket bounds at scale P of a sorted relation (for the
// reference's comparator / partition counters, lsj.py:250-286, 302-305)
__global__ void k_ref_bounds(RmiDev m, const ulonglong2 *sorted, i64 n, i64 P, i64 *bounds) {
    m.fix();
    for (i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x; c <= P; c += (i64)gridDim.x * blockDim.x) {
        i64 lo = 0, hi = n;  // first i with partition_index(key_i, P) >= c
        while (lo < hi) {
            i64 mid = (lo + hi) >> 1;
            if (scale_bucket(m.pos(u64_to_f64(sorted[mid].x)), P, m.n) < c) lo = mid + 1; else hi = mid;
        }
        bounds[c] = lo;
    }
}

// ------------------------------------------------------------------- join

// K9: see the file header.  mode 0: checksum; 1: per-S counts; 2: pairs.
// Exact R slice of every S tile: [lower_bound(first S key),
// upper_bound(last S key)) inside the R bucket range that R's model gives
// for them (lsj.py:346-356).  One thread per tile, all tiles at once, so
// the dependent probes of the searches overlap across the grid.
__global__ void k_join_bounds(LsjDev mr, const ulonglong2 *__restrict__ R, const i64 *__restrict__ rst,
                              const ulonglong2 *__restrict__ S, i64 ns, i64 ntiles, i64 *tb) {
    mr.m.fix();
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < ntiles; t += (i64)gridDim.x * blockDim.x) {
        const i64 a = t * JOIN_T, e = min(a + (i64)JOIN_T, ns);
        const u64 kf = S[a].x, kl = S[e - 1].x;
        const i64 wlo = rst[mr.bin(kf)], whi = rst[mr.bin(kl) + 1];
        i64 lo = wlo, hi = whi;
        while (lo < hi) {
            const i64 mid = (lo + hi) >> 1;
            if (R[mid].x < kf) lo = mid + 1; else hi = mid;
        }
        const i64 rlo = lo;
        hi = whi;
        while (lo < hi) {
            const i64 mid = (lo + hi) >> 1;
            if (R[mid].x <= kl) lo = mid + 1; else hi = mid;
        }
        tb[2 * t] = rlo;
        tb[2 * t + 1] = lo > rlo ? lo : rlo;
    }
}

// K9: per S tile of JOIN_T, the tile (keys + payloads) and its R slice keys
// staged in shared memory; each thread takes JOIN_PER consecutive S tuples:
// one lower bound in the slice for the first, then a forward merge walk.
// mode 0: checksum; mode 1: counts[ns]; mode 2: pairs at offsets[ns].
constexpr int JOIN_PER = JOIN_T / JOIN_NT;

__global__ void __launch_bounds__(JOIN_NT, LJ_JOIN_MINB) k_lsj_join(const ulonglong2 *__restrict__ R,
                                                      const ulonglong2 *__restrict__ S, i64 ns, const i64 *tb,
                                                      int mode, i64 *counts, const i64 *offsets, u64 *opr, u64 *ops,
                                                      u64 *out) {
    __shared__ u64 wk[WCAP + 1];
    __shared__ u64 sk[JOIN_T], sp[JOIN_T];
    u64 cnt = 0, sum = 0, x = 0;
    const i64 ntiles = (ns + JOIN_T - 1) / JOIN_T;
    // the next tile's R range is loaded one tile ahead (its latency would
    // otherwise open every tile), and its S tile and R range stream into L2
    // (bulk prefetch) while this tile merges
    i64 nlo = 0, nhi = 0;
    if (blockIdx.x < ntiles) {
        nlo = tb[2 * blockIdx.x];
        nhi = tb[2 * blockIdx.x + 1];
    }
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 a = tile * JOIN_T, e = min(a + (i64)JOIN_T, ns);
        const int ne = (int)(e - a);
        const i64 wlo = nlo, whi = nhi, w = whi - wlo;
        const i64 nt = tile + gridDim.x;
        if (nt < ntiles) {
            nlo = tb[2 * nt];
            nhi = tb[2 * nt + 1];
            if (threadIdx.x == 0) {
                const i64 na = nt * JOIN_T, nn = min((i64)JOIN_T, ns - na);
                bulk_prefetch_l2(S + na, (unsigned)(nn * sizeof(ulonglong2)));
            }
        }
        for (int j = threadIdx.x; j < ne; j += JOIN_NT) {
            const ulonglong2 v = S[a + j];
            sk[j] = v.x;
            sp[j] = v.y;
        }
        // The R slice goes through shared memory in chunks of WCAP keys (one
        // chunk for almost every tile; a sparse stretch of S -- the Zipf tail
        // of C4 -- can face a slice of 10^4+ keys).  Each thread owns JOIN_PER
        // consecutive (sorted) S keys and resolves, per chunk, those not
        // above the chunk's last key: their lower bound lies in the chunk.
        const int j0 = threadIdx.x * JOIN_PER;
        int un = 0;     // next unresolved key of this thread
        int pos = 0;    // lower bound of the previous key, chunk-relative
        for (i64 c0 = 0; c0 < w || (c0 == 0 && w == 0); c0 += WCAP) {
            const int cl = (int)min((i64)WCAP, w - c0);
            for (int j = threadIdx.x; j < cl; j += JOIN_NT) wk[j] = R[wlo + c0 + j].x;
            if (threadIdx.x == 0) wk[cl] = ~0ULL;  // sentinel above every key
            __syncthreads();
            const u64 clast = cl > 0 ? wk[cl - 1] : 0;
            const bool last_chunk = c0 + cl >= w;
            bool fresh = true;  // first key resolved in this chunk: binary search
            for (; un < JOIN_PER; ++un) {
                const int j = j0 + un;
                if (j >= ne) {
                    un = JOIN_PER;
                    break;
                }
                const u64 k = sk[j];
                if (!last_chunk && k > clast) break;  // lower bound in a later chunk
                if (fresh) {
                    int lo = 0, hi = cl;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (wk[mid] < k) lo = mid + 1; else hi = mid;
                    }
                    pos = lo;
                    fresh = false;
                } else {
                    while (wk[pos] < k) ++pos;  // S is sorted: lower bounds only grow
                }
                const i64 i = a + j;
                i64 c = 0, o = mode == 2 ? offsets[i] : 0;
                // equal run: from the staged keys (unique build keys: one
                // compare, one payload load), past the chunk from global
                int p2 = pos;
                if (p2 < cl && wk[p2] == k) {
                    const ulonglong2 *rr = R + wlo + c0;
                    const u64 spj = sp[j];
                    do {
                        const u64 pr = rr[p2].y;
                        if (mode == 0) {
                            const u64 v = pr + spj;
                            ++cnt;
                            sum += v;
                            x ^= v;
                        } else if (mode == 2) {
                            opr[o] = pr;
                            ops[o] = spj;
                            ++o;
                        }
                        ++c;
                        ++p2;
                    } while (p2 < cl && wk[p2] == k);
                    if (p2 == cl) {
                        for (i64 q = c0 + cl; q < w && R[wlo + q].x == k; ++q) {
                            const u64 pr = R[wlo + q].y;
                            if (mode == 0) {
                                const u64 v = pr + spj;
                                ++cnt;
                                sum += v;
                                x ^= v;
                            } else if (mode == 2) {
                                opr[o] = pr;
                                ops[o] = spj;
                                ++o;
                            }
                            ++c;
                        }
                    }
                }
                if (mode == 1) counts[i] = c;
            }
            __syncthreads();  // the chunk buffer is refilled next round
            if (w == 0) break;
        }
        if (threadIdx.x == 0 && nt < ntiles && nhi - nlo > 0 && nhi - nlo <= WCAP)
            bulk_prefetch_l2(R + nlo, (unsigned)((nhi - nlo) * sizeof(ulonglong2)));
    }
    if (mode == 0) reduce_checksum(cnt, sum, x, 0, out);
}

// ----------------------------------------------------------------- sample

// Stratified sample without replacement: one position per stratum
// [j*n/total, (j+1)*n/total), offset by a counter draw (results-neutral;
// the reference draws with numpy's Generator.choice, lsj.py:119-120).
// (stride: keys[i * stride], 2 for interleaved {key, payload} records)
__global__ void k_sample(const u64 *keys, i64 stride, i64 n, i64 total, u64 seed, u64 *out) {
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < total; j += (i64)gridDim.x * blockDim.x) {
        i64 lo = (i64)(((unsigned __int128)j * (u64)n) / (u64)total);
        i64 hi = (i64)(((unsigned __int128)(j + 1) * (u64)n) / (u64)total);
        i64 w = hi > lo ? hi - lo : 1;
        i64 p = lo + (i64)__umul64hi(mix64(seed ^ (u64)j), (u64)w);
        out[j] = keys[(p < n ? p : n - 1) * stride];
    }
}

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

// the big instance: one CTA per SM, 1024 threads, everything of up to
// CAP_BIG tuples in shared memory
constexpr int CAP_BIG = 12288;  // 12 tuples per thread, 168 KB

template <int CAPV>
static size_t sort_smem_bytes() {
    return (sizeof(u64) + sizeof(u32) + sizeof(u16)) * CAPV;
}

template <class Src, int NT, int CAPV, int CTAS>
static int launch_sort(const LsjDev &md, const Src &src, const unsigned long long *nb_dev, const ulonglong2 *in,
                       ulonglong2 *out, SortCtl *ctl, i64 *over, cudaStream_t st) {
    static unsigned long long attr = 0;  // one bit per device
    if (once_per_device(attr)) {
        LJ_CK(cudaFuncSetAttribute(k_lsj_sort<Src, NT, CAPV, CTAS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sort_smem_bytes<CAPV>()));
    }
    LJ_CK(cudaMemsetAsync(ctl, 0, sizeof(SortCtl), st));
    k_lsj_sort<Src, NT, CAPV, CTAS><<<sm_count() * CTAS, NT, sort_smem_bytes<CAPV>(), st>>>(md, src, nb_dev, in, out,
                                                                                          ctl, over);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

static size_t scan_i64_bytes(i64 items) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (const i64 *)nullptr, (i64 *)nullptr, (int64_t)items);
    return t;
}

}  // namespace lj

using namespace lj;

extern "C" {

size_t lj_lsj_sample_workspace_bytes(int64_t total) {
    size_t t = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t, (const u64 *)nullptr, (u64 *)nullptr, (int64_t)total);
    return al(sizeof(u64) * (size_t)total) + al(t);
}

int lj_lsj_sample(const uint64_t *keys, int64_t n, int64_t total, uint64_t seed, uint64_t *sample_sorted, void *ws,
                  size_t ws_bytes, void *stream) {
    return lj_lsj_sample_strided(keys, 1, n, total, seed, sample_sorted, ws, ws_bytes, stream);
}

int lj_lsj_sample_strided(const uint64_t *keys, int64_t stride, int64_t n, int64_t total, uint64_t seed,
                          uint64_t *sample_sorted, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(n >= 1 && total >= 1 && total <= n && stride >= 1, "need 1 <= total <= n, stride >= 1");
    if (ws_bytes < lj_lsj_sample_workspace_bytes(total)) {
        set_error("lj_lsj_sample: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    u64 *tmp = (u64 *)ws;
    char *cub_tmp = (char *)ws + al(sizeof(u64) * (size_t)total);
    size_t t = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t, (const u64 *)tmp, sample_sorted, (int64_t)total);
    k_sample<<<grid_for(total, 256, 8), 256, 0, st>>>(keys, stride, n, total, seed, tmp);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceRadixSort::SortKeys(cub_tmp, t, (const u64 *)tmp, sample_sorted, (int64_t)total, 0, 64, st));
    return LJ_OK;
}

size_t lj_lsj_bins_workspace_bytes(int64_t total) { return al(sizeof(i64) * (size_t)total); }

int lj_lsj_bins(const LjRmi *model, const uint64_t *sample_sorted, int64_t total, int64_t nbins, int64_t *pb,
                uint32_t *table, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n >= 1, "model is not fitted");
    LJ_REQUIRE(total >= 1 && nbins >= 1 && nbins <= PART2_MAXBINS, "need total >= 1 and 1 <= nbins <= 32768");
    if (ws_bytes < lj_lsj_bins_workspace_bytes(total)) {
        set_error("lj_lsj_bins: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    i64 *spos = (i64 *)ws;
    RmiDev m(*model);
    k_sample_pos<<<grid_for(total, 256, 8), 256, 0, st>>>(m, sample_sorted, total, spos);
    k_bin_bounds<<<(int)((nbins + 256) / 256), 256, 0, st>>>(spos, total, (int)nbins, model->n, pb);
    k_bin_table<<<grid_for(model->n, 256, 8), 256, 0, st>>>(pb, (int)nbins, model->n, table);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_lsj_bins_from_bounds(const int64_t *pb, int64_t nbins, int64_t trained_len, uint32_t *table, void *stream) {
    LJ_REQUIRE(nbins >= 1 && nbins <= PART2_MAXBINS && trained_len >= 1, "bad bins");
    k_bin_table<<<grid_for(trained_len, 256, 8), 256, 0, as_stream(stream)>>>(pb, (int)nbins, trained_len, table);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

// ---- the key-range bin structure on its own (tests: exactness against a
// plain search / the model's bins on arbitrary keys)
static __global__ void k_keybin_eval(KeyRangeBin kb, const u64 *keys, i64 nk, u32 *bins) {
    extern __shared__ __align__(16) u64 kb_s[];
    kb.stage(kb_s);
    __syncthreads();
    const KeyRangeBin f = kb.at(kb_s);
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nk; i += (i64)gridDim.x * blockDim.x)
        bins[i] = f.code(keys[i]);
}

static __global__ void k_copy_bounds(const u64 *bounds, int nb, u64 *lay) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += gridDim.x * blockDim.x)
        lay[4 + j] = j ? bounds[j] : 0;
}

static __global__ void k_read_bounds(const u64 *lay, int nb, u64 *bounds) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += gridDim.x * blockDim.x)
        bounds[j] = j ? lay[4 + j] : 0;
}

size_t lj_keybin_workspace_bytes(int64_t nbins) { return kb_bytes((int)nbins); }

int lj_keybin_eval(const uint64_t *bounds, int64_t nbins, const uint64_t *keys, int64_t nk, uint32_t *bins, void *ws,
                   size_t ws_bytes, void *stream) {
    LJ_REQUIRE(nbins >= 1 && nbins <= KB_MAXBINS, "need 1 <= nbins <= 2048");
    LJ_REQUIRE(ws_bytes >= kb_bytes((int)nbins), "workspace too small");
    cudaStream_t st = as_stream(stream);
    u64 *lay = (u64 *)ws;
    const int nb = (int)nbins;
    k_copy_bounds<<<(nb + 255) / 256, 256, 0, st>>>(bounds, nb, lay);
    k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
    LJ_CK_LAUNCH();
    if (nk > 0) {
        KeyRangeBin kb;
        kb.g = lay;
        kb.nb = nb;
        static unsigned long long attr = 0;  // one bit per device (the packed layout exceeds 48 KB)
        if (once_per_device(attr))
            LJ_CK(cudaFuncSetAttribute(k_keybin_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        k_keybin_eval<<<grid_for(nk, 256, 4), 256, kb_bytes(nb), st>>>(kb, keys, nk, bins);
        LJ_CK_LAUNCH();
    }
    return LJ_OK;
}

// ---- range shuffle of the distributed LSJ (dist.lsj_join): the shared
// model's bins are the destination ranks
size_t lj_lsj_shuffle_workspace_bytes(int64_t n, int64_t nbins) {
    return est_workspace_bytes((int)nbins) + part_align(sizeof(u16) * (size_t)(n < 0 ? 0 : n)) +
           al(kb_bytes((int)nbins));
}

static int shuffle_bins(const LjLsjModel *md, void *ws, size_t ws_bytes, int64_t n, KeyRangeBin &kb,
                        cudaStream_t st) {
    LJ_REQUIRE(md && md->pb && md->nbins >= 1 && md->nbins <= KB_MAXBINS, "model has no bins (or > 2048)");
    if (ws_bytes < lj_lsj_shuffle_workspace_bytes(n, md->nbins)) {
        set_error("lj_lsj_shuffle: workspace too small");
        return LJ_E_WORKSPACE;
    }
    const int nb = (int)md->nbins;
    u64 *lay = reinterpret_cast<u64 *>((char *)ws + ws_bytes - al(kb_bytes(nb)));
    lay = reinterpret_cast<u64 *>((uintptr_t)lay & ~(uintptr_t)255);
    kb.g = lay;
    kb.nb = nb;
    return LJ_OK;
}

int lj_lsj_shuffle_count(const LjLsjModel *md, const uint64_t *keys, const uint64_t *pay, int64_t n,
                         int64_t *counts, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
    KeyRangeBin kb;
    int rc = shuffle_bins(md, ws, ws_bytes, n, kb, st);
    if (rc) return rc;
    k_lsj_key_bounds<<<((int)md->nbins + 127) / 128, 128, 0, st>>>(make_lsj(*md), (u64 *)kb.g);
    k_keybin_build<<<1, 1024, 0, st>>>((u64 *)kb.g, (int)md->nbins);
    LJ_CK_LAUNCH();
    SoaSrc<KeyRangeBin> src{keys, pay, kb};
    return shuffle_count(src, n, (int)md->nbins, counts, ws, ws_bytes, st);
}

int lj_lsj_shuffle_scatter(const LjLsjModel *md, const uint64_t *keys, const uint64_t *pay, int64_t n,
                           const int64_t *bases, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
    KeyRangeBin kb;
    int rc = shuffle_bins(md, ws, ws_bytes, n, kb, st);
    if (rc) return rc;
    LJ_REQUIRE(((uintptr_t)keys & 15) == 0 && ((uintptr_t)pay & 15) == 0, "columns must be 16-B aligned");
    SoaSrc<KeyRangeBin> src{keys, pay, kb};
    return shuffle_scatter(src, n, (int)md->nbins, bases, ws, ws_bytes, st);
}

int lj_lsj_key_bounds(const LjLsjModel *md, uint64_t *bounds, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(md && md->pb && md->nbins >= 1 && md->nbins <= KB_MAXBINS, "model has no bins (or > 2048)");
    LJ_REQUIRE(ws_bytes >= kb_bytes((int)md->nbins), "workspace too small");
    cudaStream_t st = as_stream(stream);
    const int nb = (int)md->nbins;
    u64 *lay = (u64 *)ws;
    k_lsj_key_bounds<<<(nb + 127) / 128, 128, 0, st>>>(make_lsj(*md), lay);
    k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
    k_read_bounds<<<(nb + 255) / 256, 256, 0, st>>>(lay, nb, bounds);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

size_t lj_lsj_partition_workspace_bytes(int64_t n, int64_t nbins) {
    return part_workspace_bytes(n, (int)nbins) + al(kb_bytes((int)nbins));
}

int lj_lsj_partition(const LjLsjModel *md, const uint64_t *keys, const uint64_t *pay, int64_t n, uint64_t *pairs,
                     int64_t *starts, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(md && md->table && md->pb && md->nbins >= 1, "model has no bins");
    if (ws_bytes < lj_lsj_partition_workspace_bytes(n, md->nbins)) {
        set_error("lj_lsj_partition: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    const int nb = (int)md->nbins;
    const size_t pws = part_workspace_bytes(n, nb);
    static const bool model_bins = getenv("LJ_LSJ_MODEL_BINS") != nullptr;
    if (!model_bins && nb <= KB_MAXBINS) {
        // the model's bins as key ranges: no model evaluation per tuple
        u64 *lay = reinterpret_cast<u64 *>((char *)ws + pws);
        k_lsj_key_bounds<<<(nb + 127) / 128, 128, 0, st>>>(make_lsj(*md), lay);
        k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
        LJ_CK_LAUNCH();
        KeyRangeBin kb;
        kb.g = lay;
        kb.nb = nb;
        SoaSrc<KeyRangeBin> src{keys, pay, kb};
        return run_partition_fast(src, n, nb, reinterpret_cast<ulonglong2 *>(pairs), starts, ws, pws, st);
    }
    LsjBin f;
    f.d = make_lsj(*md);
    SoaSrc<LsjBin> src{keys, pay, f};
    return run_partition(src, n, nb, reinterpret_cast<ulonglong2 *>(pairs), starts, ws, pws, st);
}

// One pass into estimated-capacity regions (lj_part_est.cuh): no exact
// counting pass.  pairs: lj_lsj_partition_regions_capacity records; reg[2
// nbins + 2]: bin b = records [reg[b], reg[nbins + 1 + b]) of pairs (gaps
// between the bins).  An overflow of any region (practically never) makes
// the exact two-pass partition run instead, decided on the device.
int64_t lj_lsj_partition_regions_capacity(int64_t n, int64_t nbins) {
    const i64 c = est_capacity_regions(n, (int)nbins);
    return c > n ? c : n;
}

size_t lj_lsj_partition_regions_workspace_bytes(int64_t n, int64_t nbins) {
    (void)n;
    return est_exact_workspace_bytes((int)nbins) + al(kb_bytes((int)nbins));
}

int lj_lsj_partition_regions(const LjLsjModel *md, const uint64_t *keys, const uint64_t *pay, int64_t n,
                             uint64_t *pairs, int64_t *reg, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(md && md->table && md->pb && md->nbins >= 1 && md->nbins <= KB_MAXBINS, "model has no bins / > 2048 bins");
    LJ_REQUIRE(((uintptr_t)keys & 15) == 0 && ((uintptr_t)pay & 15) == 0 && n < (i64)0xFFFFFFFFLL,
               "columns must be 16-B aligned, n < 2^32");
    if (ws_bytes < lj_lsj_partition_regions_workspace_bytes(n, md->nbins)) {
        set_error("lj_lsj_partition_regions: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    const int nb = (int)md->nbins;
    const size_t pws = est_exact_workspace_bytes(nb);
    u64 *lay = reinterpret_cast<u64 *>((char *)ws + pws);
    k_lsj_key_bounds<<<(nb + 127) / 128, 128, 0, st>>>(make_lsj(*md), lay);
    k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
    LJ_CK_LAUNCH();
    KeyRangeBin kb;
    kb.g = lay;
    kb.nb = nb;
    SoaSrc<KeyRangeBin> src{keys, pay, kb};
    return run_partition_est_or_exact(src, n, nb, reinterpret_cast<ulonglong2 *>(pairs), reg, ws, pws, st);
}

// ... from interleaved 16-B records {key, payload} (the receive buffer of the
// distributed LSJ's range shuffle): read in place, no conversion to columns.
int lj_lsj_partition_regions_rec(const LjLsjModel *md, const uint64_t *records, int64_t n, uint64_t *pairs,
                                 int64_t *reg, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(md && md->table && md->pb && md->nbins >= 1 && md->nbins <= KB_MAXBINS, "model has no bins / > 2048 bins");
    LJ_REQUIRE(((uintptr_t)records & 15) == 0 && n < (i64)0xFFFFFFFFLL, "records must be 16-B aligned, n < 2^32");
    if (ws_bytes < lj_lsj_partition_regions_workspace_bytes(n, md->nbins)) {
        set_error("lj_lsj_partition_regions_rec: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    const int nb = (int)md->nbins;
    const size_t pws = est_exact_workspace_bytes(nb);
    u64 *lay = reinterpret_cast<u64 *>((char *)ws + pws);
    k_lsj_key_bounds<<<(nb + 127) / 128, 128, 0, st>>>(make_lsj(*md), lay);
    k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
    LJ_CK_LAUNCH();
    KeyRangeBin kb;
    kb.g = lay;
    kb.nb = nb;
    AosSrc<KeyRangeBin> src{records, kb};
    return run_partition_est_or_exact(src, n, nb, reinterpret_cast<ulonglong2 *>(pairs), reg, ws, pws, st);
}

static i64 max_subs(i64 n, i64 nbins) { return 2 * (n / SUB + nbins) + 2; }
static i64 max_mat(i64 n, i64 nbins) { return (i64)(2 * SPLIT_MAXF) * (n / SPLIT_CH + nbins + 1); }

static size_t mat_scan_bytes(i64 items) {
    size_t t = 0;
    cub::TransformInputIterator<i64, CastU32I64, const u32 *> it(nullptr, CastU32I64());
    cub::DeviceScan::ExclusiveSum(nullptr, t, it, (i64 *)nullptr, (int64_t)items);
    return t;
}

// Everything lives in the caller's workspace and every step is enqueued on
// the stream: the split's slot x chunk matrix is scanned at its bound (no
// readback of its size), the oversized sub-buckets go from the main sort to
// the big instance and then to k_lsj_huge through device-side lists.
size_t lj_lsj_sort_workspace_bytes(int64_t n, int64_t nbins) {
    const i64 G = max_subs(n, nbins), nbig = n / CAP + 2, M = max_mat(n, nbins);
    size_t sc = scan_i64_bytes(nbins + 1);
    const size_t ms = mat_scan_bytes(M);
    if (ms > sc) sc = ms;
    return 2 * al(sizeof(SortCtl)) + 2 * al(sizeof(i64) * (size_t)(nbins + 1)) +  // ctls, fcount, fbase
           4 * al(sizeof(i64) * (size_t)(nbins + 1)) +                           // chunks, cbase, matc, mbase
           al(sizeof(u32) * (size_t)M) + al(sizeof(i64) * (size_t)M) +            // slot x chunk matrix, offsets
           al(sizeof(ulonglong2) * (size_t)n) +                                  // split array
           al(sizeof(i64) * (size_t)(G + 1)) + al(sizeof(double2) * (size_t)G) +  // sub starts, y ranges
           al(sizeof(double) * (size_t)G) +                                      // split values
           2 * al(sizeof(i64) * (size_t)nbig) +                                  // over / huge lists
           al(sc);
}

__global__ void k_set_last(const i64 *fbase, int nb, i64 n, i64 *sub_starts) { sub_starts[fbase[nb]] = n; }

// dense bucket starts of the sorted output: the scanned matrix's first entry
// of every bucket (empty trailing buckets: n)
__global__ void k_dense_starts(const i64 *mbase, const i64 *off, int nb, i64 n, i64 *dstarts) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x)
        dstarts[b] = (b < nb && mbase[b] < mbase[nb]) ? off[mbase[b]] : n;
}

static int lsj_sort_impl(const LjLsjModel *md, const uint64_t *pairs_in, uint64_t *pairs_out, int64_t n,
                         const int64_t *bstart, const int64_t *bend, int64_t *dense_starts, void *ws, size_t ws_bytes,
                         int64_t *stats, void *stream);

int lj_lsj_sort(const LjLsjModel *md, const uint64_t *pairs_in, uint64_t *pairs_out, int64_t n,
                const int64_t *starts, void *ws, size_t ws_bytes, int64_t *stats, void *stream) {
    return lsj_sort_impl(md, pairs_in, pairs_out, n, starts, starts + 1, nullptr, ws, ws_bytes, stats, stream);
}

int lj_lsj_sort_regions(const LjLsjModel *md, const uint64_t *pairs_in, uint64_t *pairs_out, int64_t n,
                        const int64_t *reg, int64_t *starts_out, void *ws, size_t ws_bytes, int64_t *stats,
                        void *stream) {
    LJ_REQUIRE(md && md->nbins >= 1 && reg && starts_out, "null regions / starts");
    return lsj_sort_impl(md, pairs_in, pairs_out, n, reg, reg + md->nbins + 1, starts_out, ws, ws_bytes, stats,
                         stream);
}

static int lsj_sort_impl(const LjLsjModel *md, const uint64_t *pairs_in, uint64_t *pairs_out, int64_t n,
                         const int64_t *bstart, const int64_t *bend, int64_t *dense_starts, void *ws, size_t ws_bytes,
                         int64_t *stats, void *stream) {
    LJ_REQUIRE(md && md->table && md->pb && md->nbins >= 1, "model has no bins");
    if (ws_bytes < lj_lsj_sort_workspace_bytes(n, md->nbins)) {
        set_error("lj_lsj_sort: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
        if (stats) LJ_CK(cudaMemsetAsync(stats, 0, 4 * sizeof(i64), st));
        if (dense_starts) LJ_CK(cudaMemsetAsync(dense_starts, 0, sizeof(i64) * (size_t)(md->nbins + 1), st));
        return LJ_OK;
    }
    const i64 nb = md->nbins, G = max_subs(n, nb);
    char *p = (char *)ws;
    auto take = [&](size_t bytes) {
        char *r = p;
        p += al(bytes);
        return r;
    };
    SortCtl *ctl = (SortCtl *)take(sizeof(SortCtl));
    SortCtl *ctl2 = (SortCtl *)take(sizeof(SortCtl));
    i64 *fcount = (i64 *)take(sizeof(i64) * (size_t)(nb + 1));
    i64 *fbase = (i64 *)take(sizeof(i64) * (size_t)(nb + 1));
    i64 *chunks = (i64 *)take(sizeof(i64) * (size_t)(nb + 1));
    i64 *cbase = (i64 *)take(sizeof(i64) * (size_t)(nb + 1));
    i64 *matc = (i64 *)take(sizeof(i64) * (size_t)(nb + 1));
    i64 *mbase = (i64 *)take(sizeof(i64) * (size_t)(nb + 1));
    const i64 Mcap = max_mat(n, nb);
    u32 *mat = (u32 *)take(sizeof(u32) * (size_t)Mcap);
    i64 *moff = (i64 *)take(sizeof(i64) * (size_t)Mcap);
    ulonglong2 *B = (ulonglong2 *)take(sizeof(ulonglong2) * (size_t)n);
    i64 *sub_starts = (i64 *)take(sizeof(i64) * (size_t)(G + 1));
    double2 *sub_y = (double2 *)take(sizeof(double2) * (size_t)G);
    u64 *spv = (u64 *)take(sizeof(u64) * (size_t)G);
    const i64 nbig_cap = n / CAP + 2;
    i64 *overlist = (i64 *)take(sizeof(i64) * (size_t)nbig_cap);
    i64 *hugelist = (i64 *)take(sizeof(i64) * (size_t)nbig_cap);
    char *cub_tmp = p;

    const LsjDev dev = make_lsj(*md);
    const ulonglong2 *A = reinterpret_cast<const ulonglong2 *>(pairs_in);
    ulonglong2 *out = reinterpret_cast<ulonglong2 *>(pairs_out);
    // level 2: slices of ~SUB tuples per coarse bucket (segmented, chunked)
    const int points = dev.sample != nullptr && dev.nsample > 0;
    k_split_plan<<<(int)((nb + 256) / 256), 256, 0, st>>>(bstart, bend, (int)nb, points, fcount);
    LJ_CK_LAUNCH();
    size_t t = scan_i64_bytes(nb + 1);
    LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, t, fcount, fbase, (int64_t)(nb + 1), st));
    if (points) {
        // the bins' sample ranges go through chunks / matc (free until
        // k_chunk_plan); sample bins evaluated inside the searches
        k_split_ranges<<<(int)((nb + 63) / 64), 64, 0, st>>>(dev, nullptr, (int)nb, chunks, matc);
        k_split_points<<<grid_for(max_subs(n, nb), 256, 8), 256, 0, st>>>(dev, bstart, bend, fbase, (int)nb, chunks,
                                                                         matc, spv);
        LJ_CK_LAUNCH();
    }
    k_chunk_plan<<<(int)((nb + 256) / 256), 256, 0, st>>>(bstart, bend, fbase, (int)nb, chunks, matc);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, t, chunks, cbase, (int64_t)(nb + 1), st));
    LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, t, matc, mbase, (int64_t)(nb + 1), st));
    const SplitCtx cx{bstart, bend, fbase, cbase, mbase, spv, (int)nb};
    LJ_CK(cudaMemsetAsync(ctl, 0, sizeof(SortCtl), st));
    k_split_count<<<sm_count() * 2, SPLIT_NT, 0, st>>>(dev, cx, A, cbase + nb, mat, ctl);
    LJ_CK_LAUNCH();
    {
        // the matrix holds mbase[nb] <= Mcap entries: scanning the bound is
        // exact for every used entry (the tail is never read)
        size_t tm = mat_scan_bytes(Mcap);
        cub::TransformInputIterator<i64, CastU32I64, const u32 *> it(mat, CastU32I64());
        LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, tm, it, moff, (int64_t)Mcap, st));
    }
    k_split_slots<<<grid_for(G + 1, 256, 8), 256, 0, st>>>(dev, cx, moff, n, sub_starts, sub_y);
    if (dense_starts) k_dense_starts<<<(int)((nb + 256) / 256), 256, 0, st>>>(mbase, moff, (int)nb, n, dense_starts);
    LJ_CK_LAUNCH();
    LJ_CK(cudaMemsetAsync(ctl, 0, sizeof(SortCtl), st));
    k_split_scatter<<<sm_count() * 2, SPLIT_NT, 0, st>>>(dev, cx, A, cbase + nb, moff, B, out, ctl);
    LJ_CK_LAUNCH();
    // K8 over the sub-buckets, B -> out (G = fbase[nb] read on device)
    SubBuckets sb{sub_starts, sub_y};
    int rc = launch_sort<SubBuckets, SORT_NT, CAP, SORT_CTAS>(
        dev, sb, reinterpret_cast<const unsigned long long *>(fbase + nb), B, out, ctl, overlist, st);
    if (rc) return rc;
    // the big instance over the oversized list (count on device)
    OverBuckets ob{overlist, sb};
    rc = launch_sort<OverBuckets, 1024, CAP_BIG, 1>(dev, ob, &ctl->n_over, B, out, ctl2, hugelist, st);
    if (rc) return rc;
    // above CAP_BIG: chunk sort + merge passes in global memory
    static unsigned long long hattr = 0;  // one bit per device
    if (once_per_device(hattr)) {
        LJ_CK(cudaFuncSetAttribute(k_lsj_huge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(HUGE_CH * sizeof(ulonglong2))));
    }
    k_lsj_huge<<<sm_count(), HUGE_NT, HUGE_CH * sizeof(ulonglong2), st>>>(ob, hugelist, &ctl2->n_over, B, out);
    LJ_CK_LAUNCH();
    if (stats) {
        k_sort_stats<<<1, 1, 0, st>>>(ctl, ctl2, stats);
        LJ_CK_LAUNCH();
    }
    return LJ_OK;
}

int lj_lsj_ref_bounds(const LjRmi *model, const uint64_t *sorted_pairs, int64_t n, int64_t P, int64_t *bounds,
                      void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n >= 1 && P >= 1, "model is not fitted / P < 1");
    k_ref_bounds<<<grid_for(P + 1, 256, 8), 256, 0, as_stream(stream)>>>(
        RmiDev(*model), reinterpret_cast<const ulonglong2 *>(sorted_pairs), n, P, bounds);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

size_t lj_lsj_join_workspace_bytes(int64_t ns) {
    return sizeof(i64) * 2 * (size_t)((ns + JOIN_T - 1) / JOIN_T + 1);
}

int lj_lsj_join(const LjLsjModel *model_r, const uint64_t *r_pairs, int64_t nr, const int64_t *r_starts,
                const uint64_t *s_pairs, int64_t ns, int mode, int64_t *counts, const int64_t *offsets,
                uint64_t *out_pr, uint64_t *out_ps, uint64_t *out, int accumulate, void *ws, size_t ws_bytes,
                void *stream) {
    LJ_REQUIRE(model_r && model_r->table && model_r->pb, "R model has no bins");
    LJ_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0, 1 or 2");
    cudaStream_t st = as_stream(stream);
    if (mode == 0 && !accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nr == 0 || ns == 0) {
        if (mode == 1 && ns > 0) LJ_CK(cudaMemsetAsync(counts, 0, sizeof(i64) * (size_t)ns, st));
        return LJ_OK;
    }
    if (ws_bytes < lj_lsj_join_workspace_bytes(ns)) {
        set_error("lj_lsj_join: workspace too small");
        return LJ_E_WORKSPACE;
    }
    const i64 ntiles = (ns + JOIN_T - 1) / JOIN_T;
    i64 *tb = (i64 *)ws;
    const ulonglong2 *R = reinterpret_cast<const ulonglong2 *>(r_pairs);
    const ulonglong2 *S = reinterpret_cast<const ulonglong2 *>(s_pairs);
    k_join_bounds<<<grid_for(ntiles, 128, 16), 128, 0, st>>>(make_lsj(*model_r), R, r_starts, S, ns, ntiles, tb);
    LJ_CK_LAUNCH();
    // one wave of resident CTAs (the tile loop strides by the grid)
    int per_sm = 0;
    LJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lsj_join, JOIN_NT, 0));
    const i64 wave = (i64)sm_count() * (per_sm > 0 ? per_sm : 1);
    const unsigned g = (unsigned)(ntiles < wave ? ntiles : wave);
    k_lsj_join<<<g, JOIN_NT, 0, st>>>(R, S, ns, tb, mode, counts, offsets, out_pr, out_ps, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

}  // extern "C"

// ------------------------------------------------------ one-call LSJ

namespace lj {

// {min, max} of the keys (unsigned), one block: the two-key "sample" of a
// relation too small for sample_rate (lsj.py zero-sample fallback)
__global__ void k_minmax2(const u64 *keys, i64 stride, i64 n, u64 *out) {
    __shared__ u64 smin[1024], smax[1024];
    u64 lo = ~0ULL, hi = 0;
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
        const u64 k = keys[i * stride];
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    }
    smin[threadIdx.x] = lo;
    smax[threadIdx.x] = hi;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            smin[threadIdx.x] = smin[threadIdx.x + o] < smin[threadIdx.x] ? smin[threadIdx.x + o] : smin[threadIdx.x];
            smax[threadIdx.x] = smax[threadIdx.x + o] > smax[threadIdx.x] ? smax[threadIdx.x + o] : smax[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = smin[0];
        out[1] = smax[0];
    }
}

// per-relation layout of lj_lsj_run's workspace
struct LsjRunRel {
    i64 n, total, tl, fanout, nbins;
};

static LsjRunRel run_rel(i64 n, double rate) {
    LsjRunRel r;
    r.n = n;
    r.total = (i64)nearbyint(rate * (double)n);  // Python round(): half to even
    r.tl = r.total > 0 ? r.total : 2;
    r.fanout = r.total > 0 ? std::min<i64>(1000, std::max<i64>(1, r.total / 8)) : 1;
    r.nbins = std::max<i64>(1, std::min<i64>(2048, (n + 8191) / 8192));  // lsj.default_bins
    return r;
}

// bytes that stay live until the join (model, bins, partitioned and sorted pairs)
static size_t run_keep_bytes(const LsjRunRel &r) {
    return al(sizeof(u64) * (size_t)r.tl) + al(sizeof(double) * 2) + al(sizeof(LjLeaf) * (size_t)r.fanout) +
           al(sizeof(i64) * 2 * (size_t)r.fanout) + al(sizeof(i64) * (size_t)(r.nbins + 1)) +
           al(sizeof(u32) * (size_t)r.tl) + al(sizeof(ulonglong2) * (size_t)r.n) +
           al(sizeof(i64) * (size_t)(r.nbins + 1)) + al(sizeof(i64) * (size_t)(2 * r.nbins + 2));
}

// the partition buffer both relations go through, one after the other:
// one-pass regions (gaps between the bins) for the larger relation
static size_t run_part_bytes(const LsjRunRel &a, const LsjRunRel &b) {
    const i64 ca = lj_lsj_partition_regions_capacity(a.n, a.nbins), cb = lj_lsj_partition_regions_capacity(b.n, b.nbins);
    return al(sizeof(ulonglong2) * (size_t)std::max(ca, cb));
}

// scratch of the sample / fit / bins steps alone (S's run on a side stream
// while R is partitioned and sorted, so they need their own)
static size_t run_smpl_scratch_bytes(const LsjRunRel &r) {
    size_t s = lj_lsj_sample_workspace_bytes(std::max<i64>(r.total, 1));
    s = std::max(s, lj_rmi_fit_workspace_bytes(r.tl, r.fanout));
    s = std::max(s, lj_lsj_bins_workspace_bytes(r.tl));
    return al(s);
}

// A side stream and fork / join events per (host thread, device): S's model
// steps are a chain of small kernels that leave the GPU mostly idle, so they
// run beside R's partition and sort.  Event record / wait on the caller's
// stream keeps the whole call asynchronous and capturable (the side stream
// joins the capture through the fork event and leaves it at the join event).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream *side_stream() {
    thread_local SideStream tab[64];
    int dev = 0;
    cudaGetDevice(&dev);
    SideStream &t = tab[dev & 63];
    if (!t.s) {
        if (cudaStreamCreateWithFlags(&t.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&t.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&t.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            t.s = nullptr;
            return nullptr;  // no side stream: everything on the caller's stream
        }
    }
    return &t;
}

static size_t run_scratch_bytes(const LsjRunRel &r) {
    size_t s = lj_lsj_sample_workspace_bytes(std::max<i64>(r.total, 1));
    s = std::max(s, lj_rmi_fit_workspace_bytes(r.tl, r.fanout));
    s = std::max(s, lj_lsj_bins_workspace_bytes(r.tl));
    s = std::max(s, lj_lsj_partition_workspace_bytes(r.n, r.nbins));
    s = std::max(s, lj_lsj_partition_regions_workspace_bytes(r.n, r.nbins));
    s = std::max(s, lj_lsj_sort_workspace_bytes(r.n, r.nbins));
    return al(s);
}

}  // namespace lj

extern "C" {

size_t lj_lsj_run_workspace_bytes(int64_t nr, int64_t ns, double sample_rate) {
    const LsjRunRel a = run_rel(nr, sample_rate), b = run_rel(ns, sample_rate);
    return run_keep_bytes(a) + run_keep_bytes(b) + run_part_bytes(a, b) +
           std::max(run_scratch_bytes(a), run_scratch_bytes(b)) + run_smpl_scratch_bytes(b) +
           al(lj_lsj_join_workspace_bytes(ns)) + 1024;
}

// records = true: rk / sk point at n interleaved {key, payload} records (rp / sp unused)
static int lsj_run_impl(bool records, const uint64_t *rk, const uint64_t *rp, int64_t nr, const uint64_t *sk,
                        const uint64_t *sp, int64_t ns, double sample_rate, uint64_t seed, uint64_t *out, void *ws,
                        size_t ws_bytes, void *stream) {
    LJ_REQUIRE(sample_rate > 0.0 && sample_rate <= 1.0, "sample_rate must be in (0, 1]");
    LJ_REQUIRE(nr >= 0 && ns >= 0, "sizes must be >= 0");
    cudaStream_t st = as_stream(stream);
    LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nr == 0 || ns == 0) return LJ_OK;
    if (ws_bytes < lj_lsj_run_workspace_bytes(nr, ns, sample_rate)) {
        set_error("lj_lsj_run: workspace too small");
        return LJ_E_WORKSPACE;
    }
    char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    auto take = [&](size_t bytes) {
        char *r = p;
        p += al(bytes);
        return r;
    };
    const LsjRunRel rel[2] = {run_rel(nr, sample_rate), run_rel(ns, sample_rate)};
    const uint64_t *keys[2] = {rk, sk}, *pays[2] = {rp, sp};
    const u64 seeds[2] = {seed, seed ^ 0x5DEECE66DULL};  // lsj.py:388-391: S's model seed
    LjRmi rmi[2];
    LjLsjModel md[2];
    u64 *sbuf[2];
    i64 *reg[2];
    double *root[2];
    LjLeaf *leaves[2];
    i64 *err[2], *pb[2], *starts[2];
    u32 *table[2];
    ulonglong2 *sorted[2];
    for (int x = 0; x < 2; ++x) {
        const LsjRunRel &r = rel[x];
        sbuf[x] = (u64 *)take(sizeof(u64) * (size_t)r.tl);
        root[x] = (double *)take(sizeof(double) * 2);
        leaves[x] = (LjLeaf *)take(sizeof(LjLeaf) * (size_t)r.fanout);
        err[x] = (i64 *)take(sizeof(i64) * 2 * (size_t)r.fanout);
        pb[x] = (i64 *)take(sizeof(i64) * (size_t)(r.nbins + 1));
        table[x] = (u32 *)take(sizeof(u32) * (size_t)r.tl);
        sorted[x] = (ulonglong2 *)take(sizeof(ulonglong2) * (size_t)r.n);
        starts[x] = (i64 *)take(sizeof(i64) * (size_t)(r.nbins + 1));
        reg[x] = (i64 *)take(sizeof(i64) * (size_t)(2 * r.nbins + 2));
        // the root stays on the device (root_dev): nothing is read back
        rmi[x] = LjRmi{0.0, 0.0, r.fanout, r.tl, leaves[x], err[x], root[x]};
        md[x] = LjLsjModel{rmi[x], r.nbins, pb[x], table[x], r.total > 0 ? sbuf[x] : nullptr, r.total > 0 ? r.tl : 0};
    }
    u64 *pairs = (u64 *)take(run_part_bytes(rel[0], rel[1]));
    char *scratch = p;
    const size_t sb = std::max(run_scratch_bytes(rel[0]), run_scratch_bytes(rel[1]));
    p += sb;
    char *join_ws = take(lj_lsj_join_workspace_bytes(ns));
    const size_t ssb = run_smpl_scratch_bytes(rel[1]);
    char *smpl_scratch = take(ssb);
    // smpl: stratified sample (or {min, max}), RMI fit, equi-depth bins
    auto smpl = [&](int x, char *scr, size_t scr_bytes, void *strm) -> int {
        const LsjRunRel &r = rel[x];
        int rc;
        if (r.total > 0) {
            rc = lj_lsj_sample_strided(keys[x], records ? 2 : 1, r.n, r.total, seeds[x], sbuf[x], scr, scr_bytes, strm);
            if (rc) return rc;
        } else {
            k_minmax2<<<1, 1024, 0, as_stream(strm)>>>(keys[x], records ? 2 : 1, r.n, sbuf[x]);
            LJ_CK_LAUNCH();
        }
        rc = lj_rmi_fit(sbuf[x], r.tl, r.fanout, root[x], leaves[x], err[x], scr, scr_bytes, strm);
        if (rc) return rc;
        return lj_lsj_bins(&rmi[x], sbuf[x], r.tl, r.nbins, pb[x], table[x], scr, scr_bytes, strm);
    };
    // S's model on the side stream, beside R's partition and sort
    static const bool one_stream = getenv("LJ_LSJ_ONE_STREAM") != nullptr;
    SideStream *side = one_stream ? nullptr : side_stream();
    if (side) {
        LJ_CK(cudaEventRecord(side->fork, st));
        LJ_CK(cudaStreamWaitEvent(side->s, side->fork, 0));
        const int rc = smpl(1, smpl_scratch, ssb, side->s);
        // (join the side stream even on an error: a capture must not be left forked)
        LJ_CK(cudaEventRecord(side->join, side->s));
        if (rc) {
            cudaStreamWaitEvent(st, side->join, 0);
            return rc;
        }
    }
    for (int x = 0; x < 2; ++x) {
        const LsjRunRel &r = rel[x];
        int rc;
        if (x == 0 || !side) {
            rc = smpl(x, scratch, sb, stream);
            if (rc) return rc;
        } else {
            LJ_CK(cudaStreamWaitEvent(st, side->join, 0));
        }
        // part + sort (K6/K7, split, K8): one-pass regions when the columns
        // allow the bulk-copy ring, else the exact partition
        if (records) {
            rc = lj_lsj_partition_regions_rec(&md[x], keys[x], r.n, pairs, reg[x], scratch, sb, stream);
            if (rc) return rc;
            rc = lj_lsj_sort_regions(&md[x], pairs, reinterpret_cast<u64 *>(sorted[x]), r.n, reg[x], starts[x], scratch,
                                     sb, nullptr, stream);
        } else if (r.nbins <= KB_MAXBINS && ((uintptr_t)keys[x] & 15) == 0 && ((uintptr_t)pays[x] & 15) == 0 &&
                   r.n < (i64)0xFFFFFFFFLL) {
            rc = lj_lsj_partition_regions(&md[x], keys[x], pays[x], r.n, pairs, reg[x], scratch, sb, stream);
            if (rc) return rc;
            rc = lj_lsj_sort_regions(&md[x], pairs, reinterpret_cast<u64 *>(sorted[x]), r.n, reg[x], starts[x], scratch,
                                     sb, nullptr, stream);
        } else {
            rc = lj_lsj_partition(&md[x], keys[x], pays[x], r.n, pairs, starts[x], scratch, sb, stream);
            if (rc) return rc;
            rc = lj_lsj_sort(&md[x], pairs, reinterpret_cast<u64 *>(sorted[x]), r.n, starts[x], scratch, sb, nullptr,
                             stream);
        }
        if (rc) return rc;
    }
    // join (K9): S's tiles against R's windows through R's model
    return lj_lsj_join(&md[0], reinterpret_cast<const u64 *>(sorted[0]), nr, starts[0],
                       reinterpret_cast<const u64 *>(sorted[1]), ns, 0, nullptr, nullptr, nullptr, nullptr, out, 0,
                       join_ws, lj_lsj_join_workspace_bytes(ns), stream);
}

int lj_lsj_run(const uint64_t *rk, const uint64_t *rp, int64_t nr, const uint64_t *sk, const uint64_t *sp, int64_t ns,
               double sample_rate, uint64_t seed, uint64_t *out, void *ws, size_t ws_bytes, void *stream) {
    return lsj_run_impl(false, rk, rp, nr, sk, sp, ns, sample_rate, seed, out, ws, ws_bytes, stream);
}

int lj_lsj_run_rec(const uint64_t *r_records, int64_t nr, const uint64_t *s_records, int64_t ns, double sample_rate,
                   uint64_t seed, uint64_t *out, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE((((uintptr_t)r_records | (uintptr_t)s_records) & 15) == 0 && nr < (i64)0xFFFFFFFFLL &&
                   ns < (i64)0xFFFFFFFFLL,
               "records must be 16-B aligned, fewer than 2^32 - 1 per relation");
    return lsj_run_impl(true, r_records, nullptr, nr, s_records, nullptr, ns, sample_rate, seed, out, ws, ws_bytes,
                        stream);
}

}  // extern "C"
