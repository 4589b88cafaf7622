// lj_grmi.cu -- Gapped-RMI index build (K11), the fused INLJ probe (K1),
// per-probe search/materialisation kernels and the Request-Buffer analogue
// (K4, leaf bucketing).  Reference: gapped.py:20-338, buffers.py:73-150.
//
// Layout in HBM: one 16-B slot per gapped position, {gkey, gpayload}
// interleaved, so the slot that ends a search also carries its payload in
// the same 32-B sector; gap slots copy the nearest real key to their left
// and hold payload 0 (gapped.py:245-255).  The occupancy bitmap is packed
// 32 slots per word and is only read when some real payload is 0.
#include <cub/cub.cuh>

#include <cstdio>
#include <vector>

#include "lj_common.cuh"
#include "lj_part.cuh"
#include "lj_keybin.cuh"
#include "lj_part_est.cuh"
#include "lj_pipe.cuh"
#include "lj_probe_count.h"

namespace lj {

struct MaxOpG {
    __device__ __forceinline__ i64 operator()(const i64 &a, const i64 &b) const {
        return a > b ? a : b;
    }
};

struct GrmiDev {
    RmiDev model;
    i64 n, L;
    const u64 *slots;
    const u32 *bitmap;
    int payload_nonzero;
    SlotMap slot_of;
    __host__ explicit GrmiDev(const LjGrmi &g)
        : model(g.model), n(g.n), L(g.L), slots(g.slots), bitmap(g.bitmap),
          payload_nonzero(g.payload_nonzero), slot_of(g.n, g.L) {}

    __device__ __forceinline__ u64 key(i64 i) const { return ldg(slots + 2 * i); }
    __device__ __forceinline__ i64 predict_slot(u64 k) const {
        return slot_of(model.pos(u64_to_f64(k)));
    }
    __device__ __forceinline__ bool real(i64 i, u64 pay) const {
        if (payload_nonzero) return pay != 0;
        return (__ldg(bitmap + (i >> 5)) >> (i & 31)) & 1u;
    }

    // first real slot >= i, or L (bitmap words: 32 slots per load)
    __device__ __forceinline__ i64 next_real(i64 i) const {
        if (i >= L) return L;
        i64 w = i >> 5;
        const i64 nw = (L + 31) >> 5;
        u32 v = __ldg(bitmap + w) & (0xffffffffu << (i & 31));
        while (v == 0) {
            if (++w >= nw) return L;
            v = __ldg(bitmap + w);
        }
        const i64 r = (w << 5) + __ffs((int)v) - 1;
        return r < L ? r : L;
    }
    // last real slot <= i, or -1
    __device__ __forceinline__ i64 prev_real(i64 i) const {
        i64 w = i >> 5;
        u32 v = __ldg(bitmap + w) & (0xffffffffu >> (31 - (i & 31)));
        while (v == 0) {
            if (--w < 0) return -1;
            v = __ldg(bitmap + w);
        }
        return (w << 5) + 31 - __clz((int)v);
    }
    // The real entries of the equal-key run that contains slot s (gapped.py:
    // 163-203), folded into the checksum of t = payload + ps.  Gap slots copy
    // the real key to their left (k_grmi_fill), so the key changes only at
    // real slots and the walk visits real slots only, whatever the run length.
    __device__ __forceinline__ void gather_run(i64 s, u64 k, u64 ps, u64 &cnt, u64 &sum, u64 &x) const {
        i64 r = prev_real(s);
        if (r < 0) r = next_real(s);  // s before the first entry: its copies
        for (;;) {                    // equal real keys to the left (duplicates)
            const i64 q = r > 0 ? prev_real(r - 1) : -1;
            if (q < 0 || key(q) != k) break;
            r = q;
        }
        for (; r < L; r = next_real(r + 1)) {
            const ulonglong2 e = ldg2(slots + 2 * r);
            if (e.x != k) break;
            const u64 t = e.y + ps;
            ++cnt;
            sum += t;
            x ^= t;
        }
    }

    // gapped.py:86-160 -- exponential search from `start`, one lane per
    // probe; returns any slot of the equal-key run or -1 and counts probes
    // exactly as the reference does.
    __device__ __forceinline__ i64 search(i64 start, u64 k, i64 &probes) const {
        probes = 1;
        u64 v = key(start);
        if (v == k) return start;
        i64 lo, hi;
        if (v < k) {
            i64 prev = start, step = 1;
            for (;;) {
                i64 idx = start + step;
                if (idx >= L) { lo = prev + 1; hi = L; break; }
                ++probes;
                u64 w = key(idx);
                if (w < k) { prev = idx; step <<= 1; }
                else if (w == k) return idx;
                else { lo = prev + 1; hi = idx; break; }
            }
        } else {
            i64 prev = start, step = 1;
            for (;;) {
                i64 idx = start - step;
                if (idx < 0) { lo = 0; hi = prev; break; }
                ++probes;
                u64 w = key(idx);
                if (w > k) { prev = idx; step <<= 1; }
                else if (w == k) return idx;
                else { lo = idx + 1; hi = prev; break; }
            }
        }
        while (lo < hi) {
            i64 mid = (lo + hi) >> 1;
            ++probes;
            if (key(mid) < k) lo = mid + 1; else hi = mid;
        }
        if (lo < L) {
            ++probes;
            if (key(lo) == k) return lo;
        }
        return -1;
    }
};

// ------------------------------------------------------------ build (K11)

// target_i - i, target_i = rint(pos_i / n * L) (gapped.py:238-240)
__global__ void k_grmi_targets(RmiDev r, const u64 *sk, i64 n, i64 L, i64 *d) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        i64 pos = r.pos(u64_to_f64(sk[i]));
        double t = rint(__dmul_rn(__ddiv_rn(i64_to_f64(pos), i64_to_f64(n)), i64_to_f64(L)));
        d[i] = f64_to_i64(t) - i;
    }
}

// slot_i = min(cummax_i + i, L - n + i) (gapped.py:241-243); scatter
__global__ void k_grmi_place(const i64 *cm, const u64 *sk, const u64 *sp, i64 n, i64 L, u64 *slots,
                             u32 *bitmap, int *nonzero) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        i64 s = cm[i] + i, cap = L - n + i;
        s = s < cap ? s : cap;
        u64 pay = sp[i];
        slots[2 * s] = sk[i];
        slots[2 * s + 1] = pay;
        atomicOr(bitmap + (s >> 5), 1u << (s & 31));
        if (pay == 0) *nonzero = 0;
    }
}

__global__ void k_grmi_fill_src(const u32 *bitmap, i64 L, i64 *f) {
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < L; j += (i64)gridDim.x * blockDim.x)
        f[j] = ((bitmap[j >> 5] >> (j & 31)) & 1u) ? j : -1;
}

// gap fill with the nearest real key to the left; slots before the first
// entry copy it (gapped.py:250-252)
__global__ void k_grmi_fill(const u32 *bitmap, const i64 *f, const i64 *cm, i64 n, i64 L, u64 *slots) {
    i64 first = cm[0] < L - n ? cm[0] : L - n;  // slot of entry 0
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < L; j += (i64)gridDim.x * blockDim.x) {
        if ((bitmap[j >> 5] >> (j & 31)) & 1u) continue;
        i64 src = f[j] < 0 ? first : f[j];
        slots[2 * j] = slots[2 * src];
    }
}

// ------------------------------------------------------------ probe (K1)

// Fused per-probe join: predict (gapped.py:258-261), exponential search
// (:86-160), equal-run scan and real-entry gather (:163-203), reduced to
// the checksum of t = R.payload + S.payload.  One lane per probe; the S
// stream is read once with evict-first loads.
// S as two columns (a Relation) or as interleaved records (bucketed S)
struct SoaIn {
    const u64 *__restrict__ keys;
    const u64 *__restrict__ pay;
    __device__ __forceinline__ void get(i64 t, u64 &k, u64 &p) const {
        k = ld_stream(keys + t);
        p = ld_stream(pay + t);
    }
};
struct AosIn {
    const ulonglong2 *__restrict__ rec;
    __device__ __forceinline__ void get(i64 t, u64 &k, u64 &p) const {
        ulonglong2 e = __ldcs(rec + t);
        k = e.x;
        p = e.y;
    }
};

template <int NT, class In>
__global__ void __launch_bounds__(NT) k_grmi_probe(GrmiDev g, In in, i64 nk, u64 *out) {
    u64 cnt = 0, sum = 0, x = 0, steps = 0;
    for (i64 t = blockIdx.x * (i64)NT + threadIdx.x; t < nk; t += (i64)gridDim.x * NT) {
        u64 k, ps;
        in.get(t, k, ps);
        i64 probes;
        const i64 s = g.search(g.predict_slot(k), k, probes);
        steps += (u64)probes;
        if (s >= 0) g.gather_run(s, k, ps, cnt, sum, x);
    }
    reduce_checksum(cnt, sum, x, steps, out);
}

// K1 over the overflow area of K4's regions: records [reg[nwin], +reg[2nwin+1])
__global__ void __launch_bounds__(256) k_grmi_probe_overflow(GrmiDev g, const ulonglong2 *__restrict__ rec,
                                                            const i64 *reg, int nwin, u64 *out) {
    const i64 base = reg[nwin], n = reg[2 * nwin + 1];
    u64 cnt = 0, sum = 0, x = 0, steps = 0;
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < n; t += (i64)gridDim.x * blockDim.x) {
        const ulonglong2 r = __ldcs(rec + base + t);
        i64 probes;
        const i64 s = g.search(g.predict_slot(r.x), r.x, probes);
        steps += (u64)probes;
        if (s >= 0) g.gather_run(s, r.x, r.y, cnt, sum, x);
    }
    reduce_checksum(cnt, sum, x, steps, out);
}

// ---------------------------------------------- staged probe (K1 over K4)
//
// K4 groups S by KEY-RANGE window: window w holds the probes k with
// W[w] < k <= W[w+1], W[w] = the gapped array's key at slot w * 2^shift.
// Gapped keys are sorted, so such a key's lower bound lb (first slot with a
// key >= k) lies in [w * 2^shift, (w+1) * 2^shift]: a window's lookups never
// leave its slot range, whatever the model's error.
//
// A CTA takes a piece of the grouped probes; for each window segment of the
// piece it stages in shared memory the REAL entries of the window's slot
// range: keys ck[] and slot offsets cp[] (compacted through the occupancy
// bitmap, with a sentinel entry at n_c), a 2^STAGE_TB-entry radix table over
// the staged key range (T[p] = first entry whose key prefix >= p) and the
// RMI leaves the range routes to.  Gap slots copy the real key to their left
// (k_grmi_fill), so the gapped array's equal-key runs are described by the
// real entries alone: with i the first staged entry >= k and j the first > k,
//   lb = cp[i]   (slots before it in range copy keys <= W[w] < k; slot 0
//                 when the range starts at slot 0: slots before the first
//                 entry copy it),
//   re = cp[j]   (first slot with a key > k; past the range: bitmap walk),
// the matches are entries i..j-1, and the reference's probe count
// (gapped.py:86-160) follows from the predicted slot, lb and re alone
// (ref_probe_count).  Per probe: model evaluation (leaf from shared memory),
// one table pair plus a fixed-trip branch-free binary search, one payload
// load per match.

constexpr int STAGE_NT = 1024;
#ifndef LJ_STAGE_PIECE
#define LJ_STAGE_PIECE 65536
#endif
constexpr int STAGE_PIECE = LJ_STAGE_PIECE;  // probes per work item (C2 step 6.41 / 6.20 / 6.19 ms at 2^15 / 2^16 / 2^17)
constexpr i64 STAGE_MIN = 2048;         // windows with fewer probes: global search
constexpr int STAGE_U = 2;              // probes in flight per thread
constexpr int STAGE_TB = 13;            // radix-table bits
constexpr int STAGE_TBINS = 1 << STAGE_TB;
constexpr int STAGE_MAX_SHIFT = 14;     // staged range <= 2^14 + 1 slots
constexpr int STAGE_SPAN = (1 << STAGE_MAX_SHIFT) + 1;
constexpr int STAGE_LEAVES = 1024;      // RMI leaves cached per window
// fixed shared-memory layout (bytes), sized for the largest window
constexpr int SO_CK = 0;                                                  // u64 [SPAN + 1]
constexpr int SO_CP = (SO_CK + 8 * (STAGE_SPAN + 1) + 15) & ~15;          // u16 [SPAN + 1]
constexpr int SO_T = (SO_CP + 2 * (STAGE_SPAN + 1) + 15) & ~15;           // u16 [TBINS + 1]
constexpr int SO_WB = (SO_T + 2 * (STAGE_TBINS + 1) + 15) & ~15;          // u32 [SPAN / 32 + 2]
constexpr int SO_LC = (SO_WB + 4 * (STAGE_SPAN / 32 + 2) + 15) & ~15;     // LjLeaf [LEAVES]
constexpr int SO_END = SO_LC + 32 * STAGE_LEAVES;

struct Acc4 {
    u64 c, s, x, st;
};

// one probe entirely in global memory (the reference's search, gapped.py:86-160)
__device__ __noinline__ Acc4 probe_global(const GrmiDev &g, i64 start, u64 k, u64 ps) {
    Acc4 a{0, 0, 0, 0};
    i64 probes;
    const i64 s = g.search(start, k, probes);
    if (s >= 0) g.gather_run(s, k, ps, a.c, a.s, a.x);
    a.st = (u64)probes;
    return a;
}

static size_t staged_smem_bytes(int) { return SO_END; }

// exclusive scan of one value per thread over the block; returns the prefix,
// *total gets the sum (all threads).  wsum: NT/32 + 1 words of shared memory.
template <int NT>
__device__ __forceinline__ u32 block_exclusive_scan(u32 v, u32 *wsum, u32 *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const u32 w = lane < NT / 32 ? wsum[lane] : 0;
        u32 wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(0xffffffffu, wi, d);
            if (lane >= d) wi += y;
        }
        if (lane < NT / 32) wsum[lane] = wi - w;
        if (lane == 31) wsum[NT / 32] = wi;
    }
    __syncthreads();
    const u32 r = wsum[warp] + inc - v;
    *total = wsum[NT / 32];
    return r;
}

// ---- staging of window [slo, shi) into (ck, cp, T, lc) -- shared memory in
// the probe, global memory when building the staging image.  Every thread
// of the CTA calls it.
struct StageOut {
    int n_c, lc_lo, lc_n;
};
struct StageHdr {  // 32 B per window in front of the image
    int n_c, lc_lo, lc_n, smax;
    i64 f0, pad;
};
__host__ __device__ inline size_t stage_hdr_bytes(int nwin) { return ((size_t)nwin * sizeof(StageHdr) + 255) & ~(size_t)255; }

__device__ StageOut stage_window(const GrmiDev &g, i64 slo, i64 shi, int span, u64 *ck, u16 *cp, u16 *T, u32 *wb,
                                 LjLeaf *lc, u32 *s_wsum, int *ps_max, i64 *ps_f0) {
    const int tid = threadIdx.x;
    int &s_max = *ps_max;
    i64 &s_f0 = *ps_f0;
    const i64 w0 = slo >> 5;
    const int bo = (int)(slo & 31);  // staged slot i is bit i + bo of the range's words
    const int nbw = (span + bo + 31) >> 5;
    auto word = [&](int j) -> u32 {  // bitmap word j, bits outside [slo, shi) cleared
        u32 v = __ldg(g.bitmap + w0 + j);
        if (j == 0) v &= 0xffffffffu << bo;
        const int top = span + bo - (j << 5);
        if (top < 32) v &= (1u << top) - 1u;
        return v;
    };
    u32 nc;
    {
        const int j0 = 2 * tid;  // nbw <= 2 * STAGE_NT words: two per thread
        const u32 c0 = j0 < nbw ? __popc(word(j0)) : 0, c1 = j0 + 1 < nbw ? __popc(word(j0 + 1)) : 0;
        const u32 pre = block_exclusive_scan<STAGE_NT>(c0 + c1, s_wsum, &nc);
        if (j0 < nbw) wb[j0] = pre;
        if (j0 + 1 < nbw) wb[j0 + 1] = pre + c0;
    }
    if (tid == 0) s_max = 0;
    __syncthreads();
    for (int i = tid; i < span; i += STAGE_NT) {
        const int b = i + bo;
        const u32 v = word(b >> 5);
        if ((v >> (b & 31)) & 1u) {
            const u32 idx = wb[b >> 5] + __popc(v & ((1u << (b & 31)) - 1u));
            ck[idx] = ldg(g.slots + 2 * (slo + i));
            cp[idx] = (u16)i;
        }
    }
    const int n_c = (int)nc;
    if (tid == 0) {
        ck[n_c] = ~0ULL;  // sentinel: larger than every key (keys < 2^64 - 1)
        cp[n_c] = (u16)span;
        // window 0 with no entry: every slot copies entry 0 (gapped.py:250-252)
        s_f0 = (slo == 0 && n_c == 0) ? g.next_real(shi) : -1;
    }
    __syncthreads();
    const u64 kmin = n_c ? ck[0] : 0, kmax = n_c ? ck[n_c - 1] : 0;
    const u64 krange = kmax - kmin;
    const int sh = krange == 0 ? 0 : max(0, 64 - __clzll((long long)krange) - STAGE_TB);
    for (int i = tid; i < n_c; i += STAGE_NT) {
        const int p = (int)((ck[i] - kmin) >> sh);
        const int pp = i == 0 ? -1 : (int)((ck[i - 1] - kmin) >> sh);
        for (int q = pp + 1; q <= p; ++q) T[q] = (u16)i;
    }
    for (int q = (n_c ? (int)(krange >> sh) + 1 : 0) + tid; q <= STAGE_TBINS; q += STAGE_NT) T[q] = (u16)n_c;
    // leaves the staged keys route to (+ a margin); probes routed elsewhere
    // read their leaf from global memory
    int lc_lo = 0, lc_n = 0;
    if (n_c) {
        const i64 l0 = max((i64)0, g.model.route(u64_to_f64(kmin)) - 8);
        const i64 l1 = min(g.model.m - 1, g.model.route(u64_to_f64(kmax)) + 8);
        lc_lo = (int)l0;
        lc_n = (int)min(l1 - l0 + 1, (i64)STAGE_LEAVES);
        for (int l = tid; l < lc_n; l += STAGE_NT) lc[l] = load_leaf(g.model.leaves, l0 + l);
    }
    __syncthreads();
    {
        int mb = 0;
        for (int q = tid; q < STAGE_TBINS; q += STAGE_NT) mb = max(mb, (int)T[q + 1] - (int)T[q]);
        mb = __reduce_max_sync(0xffffffffu, mb);
        if ((tid & 31) == 0 && mb) atomicMax(&s_max, mb);
    }
    __syncthreads();
    return StageOut{n_c, lc_lo, lc_n};
}

// staging image of every window (built once per index): header + the
// shared-memory layout of each window
__global__ void __launch_bounds__(STAGE_NT, 1) k_grmi_stage_image(GrmiDev g, int nwin, int shift, unsigned char *img) {
    __shared__ u32 s_wsum[STAGE_NT / 32 + 1];
    __shared__ int s_max;
    __shared__ i64 s_f0;
    const int w = blockIdx.x;
    const int span_max = (1 << shift) + 1;
    const i64 slo = (i64)w << shift, shi = min(g.L, slo + span_max);
    unsigned char *base = img + stage_hdr_bytes(nwin) + (size_t)w * SO_END;
    const StageOut so = stage_window(g, slo, shi, (int)(shi - slo), reinterpret_cast<u64 *>(base + SO_CK),
                                     reinterpret_cast<u16 *>(base + SO_CP), reinterpret_cast<u16 *>(base + SO_T),
                                     reinterpret_cast<u32 *>(base + SO_WB), reinterpret_cast<LjLeaf *>(base + SO_LC),
                                     s_wsum, &s_max, &s_f0);
    if (threadIdx.x == 0) {
        StageHdr h;
        h.n_c = so.n_c;
        h.lc_lo = so.lc_lo;
        h.lc_n = so.lc_n;
        h.smax = s_max;
        h.f0 = s_f0;
        h.pad = 0;
        reinterpret_cast<StageHdr *>(img)[w] = h;
    }
}

// COUNT: also reproduce the reference's probe counter (search_steps,
// gapped.py:86-160): the model's predicted slot of every probe and the
// closed-form count from (predicted slot, lower bound, run end).  The staged
// search itself never needs the prediction -- the window's radix table
// finds the lower bound -- so without the counter the model evaluation goes
// too (out[3] stays 0).
template <bool COUNT>
__global__ void __launch_bounds__(STAGE_NT, 1) k_grmi_probe_staged(GrmiDev g, const ulonglong2 *__restrict__ rec,
                                                                   const i64 *__restrict__ reg, int nwin, int shift,
                                                                   unsigned long long *work,
                                                                   u64 *out, u64 *trace, i64 *dbg,
                                                                   const unsigned char *__restrict__ img) {
    extern __shared__ __align__(16) unsigned char smem[];
    u64 *ck = reinterpret_cast<u64 *>(smem + SO_CK);    // real keys of the staged range (+ sentinel)
    u16 *cp = reinterpret_cast<u16 *>(smem + SO_CP);    // their slot offsets (+ sentinel: span)
    u16 *T = reinterpret_cast<u16 *>(smem + SO_T);      // radix table over ck
    u32 *wb = reinterpret_cast<u32 *>(smem + SO_WB);    // bitmap-word prefix counts
    LjLeaf *lc = reinterpret_cast<LjLeaf *>(smem + SO_LC);  // cached RMI leaves
    __shared__ i64 s_piece, s_f0;
    __shared__ int s_max;
    __shared__ u32 s_wsum[STAGE_NT / 32 + 1];
    __shared__ u32 s_small[2048 / 32];  // windows with < STAGE_MIN probes: global search
    __shared__ StageHdr s_hdr;
    __shared__ __align__(8) uint64_t s_bar;
    unsigned s_phase = 0;
    const int tid = threadIdx.x;
    for (int j = tid; j < 2048 / 32; j += STAGE_NT) s_small[j] = 0;
    if (img && tid == 0) {
        mbar_init(&s_bar, 1);
        mbar_init_fence();
    }
    __syncthreads();
    // regions: window w's records are [reg[w], rend[w]); reg[nwin] = end of
    // the regions (the overflow area, probed separately, starts there)
    const i64 *rend = reg + nwin + 1;
    const i64 nk = reg[nwin];
    for (int w = tid; w < nwin; w += STAGE_NT)
        if (rend[w] - reg[w] < STAGE_MIN) atomicOr(&s_small[w >> 5], 1u << (w & 31));
    const int span_max = (1 << shift) + 1;
    u64 cnt = 0, sum = 0, x = 0, steps = 0;
    for (;;) {
        if (tid == 0) s_piece = (i64)atomicAdd(work, 1ULL);
        __syncthreads();
        const i64 p0 = s_piece * STAGE_PIECE;
        __syncthreads();
        if (p0 >= nk) break;
        const i64 p1 = min(p0 + STAGE_PIECE, nk);
        u64 t_begin = 0, t_stage = 0, t_mark = 0;
        if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        int nstaged = 0;
        int wlo = 0, whi = nwin;  // first window overlapping p0
        while (whi - wlo > 1) {
            const int mid = (wlo + whi) >> 1;
            if (reg[mid] <= p0) wlo = mid; else whi = mid;
        }
        bool any_small = false;
        for (int w = wlo; w < nwin && reg[w] < p1; ++w) {
            const i64 a = max(p0, reg[w]), e = min(p1, rend[w]);
            if (e <= a) continue;
            if ((s_small[w >> 5] >> (w & 31)) & 1u) {
                any_small = true;
                continue;
            }
            ++nstaged;
            if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_mark));
            // ---- stage the real entries of [slo, shi), the radix table, the leaves
            const i64 slo = (i64)w << shift;
            const i64 shi = min(g.L, slo + span_max);
            const int span = (int)(shi - slo);
            int n_c, lc_lo, lc_n;
            if (img) {
                // precomputed staging image of window w: four bulk copies
                if (tid == 0) {
                    const StageHdr h = reinterpret_cast<const StageHdr *>(img)[w];
                    s_hdr = h;
                    s_f0 = h.f0;
                    s_max = h.smax;
                    const unsigned bk = ((unsigned)(h.n_c + 1) * 8u + 15u) & ~15u;
                    const unsigned bp = ((unsigned)(h.n_c + 1) * 2u + 15u) & ~15u;
                    const unsigned bt = ((unsigned)(STAGE_TBINS + 1) * 2u + 15u) & ~15u;
                    const unsigned bl = (unsigned)h.lc_n * 32u;
                    const unsigned char *src = img + stage_hdr_bytes(nwin) + (size_t)w * SO_END;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive_expect_tx(&s_bar, bk + bp + bt + bl);
                    bulk_g2s(smem + SO_CK, src + SO_CK, bk, &s_bar);
                    bulk_g2s(smem + SO_CP, src + SO_CP, bp, &s_bar);
                    bulk_g2s(smem + SO_T, src + SO_T, bt, &s_bar);
                    if (bl) bulk_g2s(smem + SO_LC, src + SO_LC, bl, &s_bar);
                }
                __syncthreads();
                mbar_wait(&s_bar, s_phase);
                s_phase ^= 1u;
                n_c = s_hdr.n_c;
                lc_lo = s_hdr.lc_lo;
                lc_n = s_hdr.lc_n;
            } else {
                const StageOut so = stage_window(g, slo, shi, span, ck, cp, T, wb, lc, s_wsum, &s_max, &s_f0);
                n_c = so.n_c;
                lc_lo = so.lc_lo;
                lc_n = so.lc_n;
            }
            const u64 kmin = n_c ? ck[0] : 0, kmax = n_c ? ck[n_c - 1] : 0;
            const u64 krange = kmax - kmin;
            const int sh = krange == 0 ? 0 : max(0, 64 - __clzll((long long)krange) - STAGE_TB);
            const int iters = 32 - __clz(s_max);  // lower-bound steps for the largest bucket
            if (trace && tid == 0) {
                u64 t_now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
                t_stage += t_now - t_mark;
            }
            const int lim = (int)(g.L - slo), zero = -(int)slo;  // L < 2^30 on this path
            const bool hi_open = shi < g.L;
            const int m1 = (int)g.model.m - 1, Lm1 = (int)g.L - 1;
            const ulonglong2 *wrec = rec + a;
            const u64 *wpay = g.slots + 2 * slo + 1;  // payload of staged slot i: wpay[2 * i]
            const int ne = (int)(e - a);
            // ---- probes: STAGE_U per thread per step, phase by phase
            for (int t0 = tid; t0 < ne; t0 += STAGE_NT * STAGE_U) {
                u64 k[STAGE_U], ps[STAGE_U];
                int start[STAGE_U], lo[STAGE_U];
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {
                    const int t = t0 + u * STAGE_NT;
                    const ulonglong2 r = t < ne ? __ldcs(wrec + t) : make_ulonglong2(kmin, 0);
                    k[u] = r.x;
                    ps[u] = r.y;
                    // the records of two steps ahead start their way into L2
                    const int tp = t + 2 * STAGE_NT * STAGE_U;
                    if (tp < ne) asm volatile("prefetch.global.L2 [%0];" ::"l"(wrec + tp));
                }
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {
                    if (!COUNT) {
                        start[u] = 0;
                        continue;
                    }
                    // models.py:112-124 + gapped.py:258-261, the leaf from smem
                    // the same operations as RmiDev::pos + SlotMap in 32-bit
                    // integers (n <= L < 2^30 on this path; saturating
                    // conversions clamp exactly like the 64-bit forms)
                    const double xf = u64_to_f64(k[u]);
                    const double rr = __dadd_rn(__dmul_rn(g.model.rs, xf), g.model.ri);
                    const int lr = min(max(__double2int_rd(rr), 0), m1);
                    const int l = lr - lc_lo;
                    const LjLeaf lf = ((unsigned)l < (unsigned)lc_n) ? lc[l] : load_leaf(g.model.leaves, lr);
                    const double raw = __dadd_rn(__dmul_rn(lf.slope, xf), lf.icpt);
                    const int clo = (int)lf.clamp_lo, chi = (int)lf.clamp_hi;
                    const int pos = (raw >= -9223372036854775808.0 && raw < 9223372036854775808.0)
                                        ? min(max(__double2int_rn(raw), clo), chi)
                                        : clo;
                    const double z = __dmul_rn((double)pos, g.slot_of.c);
                    const double fr = __dadd_rn(z, -floor(z));
                    const int slot = fabs(__dadd_rn(fr, -0.5)) > g.slot_of.g ? min(max(__double2int_rn(z), 0), Lm1)
                                                                            : (int)grmi_slot_of_pos(pos, g.n, g.L);
                    start[u] = slot - (int)slo;
                }
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {  // first entry of k's table bucket
                    const u64 d = k[u] - kmin;
                    lo[u] = k[u] < kmin ? 0 : T[(int)((d < krange ? d : krange) >> sh)];
                }
                // lower bound by binary lifting: the answer is at most
                // s_max < 2^iters entries past the bucket start, and every
                // entry past the bucket (or the sentinel at n_c) is >= k
                for (int st = iters > 0 ? 1 << (iters - 1) : 0; st > 0; st >>= 1) {
#pragma unroll
                    for (int u = 0; u < STAGE_U; ++u)
                        if (ck[min(lo[u] + st - 1, n_c)] < k[u]) lo[u] += st;
                }
                // first match of every probe and its payload, all in flight at once
                bool m0[STAGE_U];
                u64 pay0[STAGE_U];
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {
                    m0[u] = ck[lo[u]] == k[u];
                    pay0[u] = m0[u] ? ldg(wpay + 2 * cp[lo[u]]) : 0;
                }
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {
                    if (t0 + u * STAGE_NT >= ne) continue;
                    const int il = lo[u];
                    if (il == n_c && hi_open) {
                        // no staged entry >= k: window 0 before the first entry
                        // (its slots copy entry 0 and k <= entry 0), else a guard
                        const i64 f0 = s_f0;
                        if (f0 < 0 || f0 >= g.L) {
                            const Acc4 ac = probe_global(g, start[u] + slo, k[u], ps[u]);
                            cnt += ac.c;
                            sum += ac.s;
                            x ^= ac.x;
                            steps += ac.st;
                            continue;
                        }
                        i64 ja = f0;  // k == entry 0: entry 0 and its duplicates
                        for (;; ++ja) {
                            ja = g.next_real(ja);
                            if (ja >= g.L) break;
                            const ulonglong2 ev = ldg2(g.slots + 2 * ja);
                            if (ev.x != k[u]) break;
                            const u64 t2 = ev.y + ps[u];
                            ++cnt;
                            sum += t2;
                            x ^= t2;
                        }
                        const int re0 = ja == f0 ? 0 : (int)ja;  // absent (k < entry 0): [0, 0)
                        if (COUNT) steps += (u64)ref_probe_count(start[u], 0, re0, lim, zero);
                        continue;
                    }
                    int iu = il;
                    const u64 cnt_before = cnt;
                    if (m0[u]) {
                        const u64 tt = pay0[u] + ps[u];
                        ++cnt;
                        sum += tt;
                        x ^= tt;
                        for (iu = il + 1; ck[iu] == k[u]; ++iu) {  // duplicate keys in R
                            const u64 t2 = ldg(wpay + 2 * cp[iu]) + ps[u];
                            ++cnt;
                            sum += t2;
                            x ^= t2;
                        }
                    }
                    const int lb = (il == 0 && slo == 0) ? 0 : (int)cp[il];
                    int re = cp[iu];
                    if (iu == n_c && iu > il && hi_open) {  // the run goes on past the staged range
                        i64 ja = shi;
                        for (;; ++ja) {
                            ja = g.next_real(ja);
                            if (ja >= g.L) break;
                            const ulonglong2 ev = ldg2(g.slots + 2 * ja);
                            if (ev.x != k[u]) break;
                            const u64 t2 = ev.y + ps[u];
                            ++cnt;
                            sum += t2;
                            x ^= t2;
                        }
                        re = (int)(ja - slo);
                    }
                    if (COUNT) steps += (u64)ref_probe_count(start[u], lb, re, lim, zero);
                    if (dbg) {
                        i64 *dp = dbg + 4 * (a + t0 + u * STAGE_NT);
                        dp[0] = lb + slo;
                        dp[1] = re + slo;
                        dp[2] = (i64)(cnt - cnt_before);
                        dp[3] = (i64)k[u];
                    }
                }
            }
            __syncthreads();
        }
        if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_mark));
        if (any_small) {  // block-uniform: every thread walked the same windows
            for (i64 t = p0 + tid; t < p1; t += STAGE_NT) {
                int lo = wlo, hi = nwin;  // window of probe t
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (__ldg(reg + mid) <= t) lo = mid; else hi = mid;
                }
                if (t >= rend[lo] || !((s_small[lo >> 5] >> (lo & 31)) & 1u)) continue;  // a gap / staged window
                const ulonglong2 r = __ldcs(rec + t);
                const Acc4 ac = probe_global(g, g.predict_slot(r.x), r.x, r.y);
                cnt += ac.c;
                sum += ac.s;
                x ^= ac.x;
                steps += ac.st;
            }
        }
        if (trace) {
            __syncthreads();
            if (tid == 0) {
                u64 t_end, smid;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
                asm volatile("{ .reg .u32 r; mov.u32 r, %%smid; cvt.u64.u32 %0, r; }" : "=l"(smid));
                u64 *tr = trace + 8 * (p0 / STAGE_PIECE);
                tr[0] = t_begin;
                tr[1] = t_end;
                tr[2] = smid;
                tr[3] = (u64)nstaged;
                tr[4] = (u64)any_small;
                tr[5] = (u64)wlo;
                tr[6] = t_stage;
                tr[7] = t_end - t_mark;
            }
        }
    }
    reduce_checksum(cnt, sum, x, steps, out);
}

__global__ void k_grmi_predict_slots(GrmiDev g, const u64 *keys, i64 nk, i64 *out) {
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < nk; t += (i64)gridDim.x * blockDim.x)
        out[t] = g.predict_slot(keys[t]);
}

__global__ void k_grmi_search(GrmiDev g, const i64 *slots0, const u64 *keys, i64 nk, i64 *out_slot,
                              i64 *out_probes) {
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < nk; t += (i64)gridDim.x * blockDim.x) {
        i64 probes;
        i64 start = slots0[t];
        start = start < 0 ? 0 : (start >= g.L ? g.L - 1 : start);
        out_slot[t] = g.search(start, keys[t], probes);
        out_probes[t] = probes;
    }
}

// gapped.py:163-185 (+ the search): leftmost slot and real-entry count
__global__ void k_grmi_count(GrmiDev g, const i64 *slots0, const u64 *keys, i64 nk, i64 *lefts, i64 *counts,
                             i64 *probes_out) {
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < nk; t += (i64)gridDim.x * blockDim.x) {
        u64 k = keys[t];
        i64 probes;
        i64 start = slots0 ? clip_i64(slots0[t], 0, g.L - 1) : g.predict_slot(k);
        i64 s = g.search(start, k, probes);
        if (probes_out) probes_out[t] = probes;
        i64 c = 0;
        if (s >= 0) {
            while (s > 0 && g.key(s - 1) == k) --s;
            for (i64 i = s; i < g.L; ++i) {
                ulonglong2 e = ldg2(g.slots + 2 * i);
                if (e.x != k) break;
                c += g.real(i, e.y) ? 1 : 0;
            }
        }
        lefts[t] = s;
        counts[t] = c;
    }
}

// gapped.py:188-203
__global__ void k_grmi_collect(GrmiDev g, const u64 *keys, i64 nk, const i64 *lefts, const i64 *offsets,
                               u64 *out_pay, i64 *out_src) {
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < nk; t += (i64)gridDim.x * blockDim.x) {
        i64 s = lefts[t];
        if (s < 0) continue;
        u64 k = keys[t];
        i64 o = offsets[t];
        for (i64 i = s; i < g.L; ++i) {
            ulonglong2 e = ldg2(g.slots + 2 * i);
            if (e.x != k) break;
            if (!g.real(i, e.y)) continue;
            out_pay[o] = e.y;
            out_src[o] = t;
            ++o;
        }
    }
}

// ------------------------------------------------------- leaf bucket (K4)

// Bin = KEY-RANGE window of 2^wshift gapped slots: the w with
// wk[w] < k <= wk[w+1], wk[w] = gapped key at slot w << wshift (wk[0] = -inf,
// wk[nwin] = +inf).  A key's lower bound then lies inside its window's slot
// range, whatever the model's error (see the staged probe).  The window is
// the one of the model's PREDICTED slot (gapped.py:258-261), corrected by
// the neighbouring window keys held in shared memory (0-1 steps for all but
// the model's worst misses).  A branch-free search over the window keys
// alone measured 2x slower (shared-memory bank conflicts, 11 dependent
// steps).  A leaf-based grouping is useless on skewed keys: the linear root
// routes most lognormal keys to a handful of huge leaves.  <= 2048 windows
// (256 KB of index each at C2).
struct SlotBin {
    RmiDev m;
    SlotMap slot_of;
    int wshift, nwin;
    const u64 *wk;
    int shift = 0;  // code = window
    __host__ __device__ int smem_words() const { return nwin; }
    __device__ void stage(u64 *dst) const {
        for (int i = threadIdx.x; i < nwin; i += blockDim.x) dst[i] = wk[i];
    }
    __device__ __forceinline__ SlotBin at(u64 *tab) const {
        SlotBin c = *this;
        c.wk = tab;
        return c;
    }
    __device__ __forceinline__ u32 code(u64 k) const {
        int w = (int)(slot_of(m.pos(u64_to_f64(k))) >> wshift);
        const u64 a = w > 0 ? wk[w] : 0, b = w + 1 < nwin ? wk[w + 1] : ~0ULL;
        if (w > 0 && a >= k) {
            --w;
            while (w > 0 && wk[w] >= k) --w;
        } else if (w + 1 < nwin && b < k) {
            ++w;
            while (w + 1 < nwin && wk[w + 1] < k) ++w;
        }
        return (u32)w;
    }
};

__global__ void k_window_keys(const u64 *slots, int nwin, int wshift, u64 *wk) {
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += gridDim.x * blockDim.x)
        wk[w] = slots[2 * ((i64)w << wshift)];
}

// key-range boundaries of the windows: B[j] = wk[j] + 1 (gapped keys are
// never the reserved maximum key)
__global__ void k_window_bounds(const u64 *wk, int nwin, u64 *lay) {
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += gridDim.x * blockDim.x)
        lay[4 + w] = w ? wk[w] + 1 : 0;
}

static int slot_window_shift(i64 L) {
    int s = 0;
    // <= 2048 windows: blocks x bins open write lines (~148 x 2048 x 128 B)
    // stay L2-resident during the scatter, so records leave L2 as full lines
    while (((L + ((i64)1 << s) - 1) >> s) > 2048) ++s;
    return s;
}

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

// the staged probe handles this index (window fits shared memory, 32-bit
// relative slot arithmetic); otherwise K4 keeps the exact, gap-free layout
static bool staged_ok(const LjGrmi *idx) {
    const int shift = slot_window_shift(idx->L);
    return shift <= STAGE_MAX_SHIFT && staged_smem_bytes(shift) <= 220 * 1024 && idx->bitmap != nullptr &&
           idx->L < ((int64_t)1 << 30) && lj_leaf_bucket_bins(idx->L) <= 2 * PART2_NT;
}

__global__ void k_starts_to_reg(int nwin, i64 *reg) {
    // reg[0..nwin] already holds the exact bin starts
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= nwin; w += gridDim.x * blockDim.x) {
        if (w < nwin) reg[nwin + 1 + w] = reg[w + 1];
        else reg[2 * nwin + 1] = 0;
    }
}

static size_t scan_i64_bytes(i64 n) {
    size_t t = 0;
    cub::DeviceScan::InclusiveScan((void *)nullptr, t, (i64 *)nullptr, (i64 *)nullptr, MaxOpG(), (int64_t)n);
    return t;
}

}  // namespace lj

using namespace lj;

extern "C" {

size_t lj_grmi_build_workspace_bytes(int64_t n, int64_t L) {
    size_t a = scan_i64_bytes(n), b = scan_i64_bytes(L);
    return al(sizeof(i64) * (size_t)n) + al(sizeof(i64) * (size_t)L) + al(a > b ? a : b);
}

int lj_grmi_build(const LjRmi *model, const uint64_t *sk, const uint64_t *sp, int64_t n, int64_t L,
                  uint64_t *slots, uint32_t *bitmap, int32_t *payload_nonzero_dev, void *ws,
                  size_t ws_bytes, void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n == n, "model must be fitted on the n sorted keys");
    LJ_REQUIRE(n >= 1 && L >= n, "need n >= 1 and L >= n");
    if (ws_bytes < lj_grmi_build_workspace_bytes(n, L)) {
        set_error("lj_grmi_build: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    char *p = (char *)ws;
    i64 *cm = (i64 *)p;
    p += al(sizeof(i64) * (size_t)n);
    i64 *f = (i64 *)p;
    p += al(sizeof(i64) * (size_t)L);
    size_t sb = scan_i64_bytes(n > L ? n : L);
    int one = 1;
    LJ_CK(cudaMemsetAsync(slots, 0, sizeof(u64) * 2 * (size_t)L, st));
    LJ_CK(cudaMemsetAsync(bitmap, 0, sizeof(u32) * (size_t)((L + 31) / 32), st));
    LJ_CK(cudaMemcpyAsync(payload_nonzero_dev, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    k_grmi_targets<<<grid_for(n, 256, 8), 256, 0, st>>>(RmiDev(*model), sk, n, L, cm);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceScan::InclusiveScan(p, sb, cm, cm, MaxOpG(), (int64_t)n, st));
    k_grmi_place<<<grid_for(n, 256, 8), 256, 0, st>>>(cm, sk, sp, n, L, slots, bitmap, payload_nonzero_dev);
    k_grmi_fill_src<<<grid_for(L, 256, 8), 256, 0, st>>>(bitmap, L, f);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceScan::InclusiveScan(p, sb, f, f, MaxOpG(), (int64_t)L, st));
    k_grmi_fill<<<grid_for(L, 256, 8), 256, 0, st>>>(bitmap, f, cm, n, L, slots);
    LJ_CK_LAUNCH();
    // the host copy of `one` must outlive the async copy
    LJ_CK(cudaStreamSynchronize(st));
    return LJ_OK;
}

int lj_grmi_predict_slots(const LjGrmi *idx, const uint64_t *keys, int64_t nk, int64_t *out, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    if (nk <= 0) return LJ_OK;
    k_grmi_predict_slots<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(GrmiDev(*idx), keys, nk, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_grmi_search(const LjGrmi *idx, const int64_t *slots0, const uint64_t *keys, int64_t nk,
                   int64_t *out_slot, int64_t *out_probes, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    if (nk <= 0) return LJ_OK;
    k_grmi_search<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(GrmiDev(*idx), slots0, keys, nk,
                                                                        out_slot, out_probes);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_grmi_probe(const LjGrmi *idx, const uint64_t *s_keys, const uint64_t *s_pay, int64_t nk,
                  uint64_t *out, int accumulate, void *stream) {
    LJ_REQUIRE(idx != nullptr, "null index");
    cudaStream_t st = as_stream(stream);
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nk <= 0 || idx->n == 0) return LJ_OK;
    constexpr int NT = 256;
    k_grmi_probe<NT, SoaIn><<<grid_for(nk, NT, 8), NT, 0, st>>>(GrmiDev(*idx), SoaIn{s_keys, s_pay}, nk, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

static int probe_bucketed(const LjGrmi *idx, const uint64_t *s_pairs, const int64_t *reg, void *ws,
                          const unsigned char *img, uint64_t *out, int accumulate, void *stream);

size_t lj_grmi_stage_image_bytes(const LjGrmi *idx) {
    if (!idx || idx->n == 0 || !staged_ok(idx)) return 0;
    const int nwin = lj_leaf_bucket_bins(idx->L);
    return stage_hdr_bytes(nwin) + (size_t)nwin * SO_END;
}

int lj_grmi_stage_image_build(const LjGrmi *idx, void *img, size_t bytes, void *stream) {
    LJ_REQUIRE(idx != nullptr && img != nullptr, "null index or image");
    const size_t need = lj_grmi_stage_image_bytes(idx);
    LJ_REQUIRE(need > 0, "this index is not probed through staged windows");
    if (bytes < need) {
        set_error("lj_grmi_stage_image_build: buffer too small");
        return LJ_E_WORKSPACE;
    }
    const int nwin = lj_leaf_bucket_bins(idx->L);
    k_grmi_stage_image<<<nwin, STAGE_NT, 0, as_stream(stream)>>>(GrmiDev(*idx), nwin, slot_window_shift(idx->L),
                                                                 (unsigned char *)img);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_grmi_probe_bucketed(const LjGrmi *idx, const uint64_t *s_pairs, const int64_t *reg, void *ws, uint64_t *out,
                           int accumulate, void *stream) {
    return probe_bucketed(idx, s_pairs, reg, ws, nullptr, out, accumulate, stream);
}

int lj_grmi_probe_bucketed_img(const LjGrmi *idx, const uint64_t *s_pairs, const int64_t *reg, void *ws,
                               const void *img, uint64_t *out, int accumulate, void *stream) {
    return probe_bucketed(idx, s_pairs, reg, ws, (const unsigned char *)img, out, accumulate, stream);
}

static int probe_bucketed(const LjGrmi *idx, const uint64_t *s_pairs, const int64_t *reg, void *ws,
                          const unsigned char *img, uint64_t *out, int accumulate, void *stream) {
    LJ_REQUIRE(idx != nullptr, "null index");
    cudaStream_t st = as_stream(stream);
    // accumulate: bit 0 = add to out instead of overwriting it; bit 1
    // (LJ_PROBE_NO_STEPS) = skip the reference's probe counter
    const bool count_steps = !(accumulate & 2);
    accumulate &= 1;
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (idx->n == 0) return LJ_OK;
    const int shift = slot_window_shift(idx->L);
    const int nwin = lj_leaf_bucket_bins(idx->L);
    const GrmiDev gd(*idx);
    // overflow records of the one-pass bucketing: plain K1
    k_grmi_probe_overflow<<<sm_count() * 8, 256, 0, st>>>(gd, reinterpret_cast<const ulonglong2 *>(s_pairs), reg, nwin,
                                                          out);
    LJ_CK_LAUNCH();
    const size_t sm = staged_smem_bytes(shift);
    if (!staged_ok(idx)) {
        // window too large to stage: plain K1 over the records (K4 used the
        // exact, gap-free layout for such an index)
        int64_t nk = 0;
        LJ_CK(cudaMemcpyAsync(&nk, reg + nwin, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaStreamSynchronize(st));
        return lj_grmi_probe_pairs(idx, s_pairs, nk, out, 1, stream);
    }
    static unsigned long long attr = 0;  // one bit per device
    if (once_per_device(attr)) {
        LJ_CK(cudaFuncSetAttribute(k_grmi_probe_staged<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   220 * 1024));
        LJ_CK(cudaFuncSetAttribute(k_grmi_probe_staged<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   220 * 1024));
    }
    unsigned long long *work = reinterpret_cast<unsigned long long *>(ws);
    LJ_CK(cudaMemsetAsync(work, 0, sizeof(unsigned long long), st));
    // LJ_STAGE_TRACE=<file>: per-piece timing records (diagnostics only)
    static const char *trace_path = getenv("LJ_STAGE_TRACE");
    u64 *trace = nullptr;
    int64_t nk = 0;  // diagnostics only: region span for the trace buffers
    if (trace_path || getenv("LJ_STAGE_DEBUG")) {
        LJ_CK(cudaMemcpyAsync(&nk, reg + nwin, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaStreamSynchronize(st));
    }
    const size_t npieces = (size_t)((nk + STAGE_PIECE - 1) / STAGE_PIECE);
    if (trace_path) LJ_CK(cudaMalloc(&trace, npieces * 8 * sizeof(u64)));
    // LJ_STAGE_DEBUG=<file>: per-probe (lb, re, matches, key) of staged probes (diagnostics only)
    static const char *dbg_path = getenv("LJ_STAGE_DEBUG");
    i64 *dbg = nullptr;
    if (dbg_path) {
        LJ_CK(cudaMalloc(&dbg, (size_t)nk * 4 * sizeof(i64)));
        LJ_CK(cudaMemsetAsync(dbg, 0xff, (size_t)nk * 4 * sizeof(i64), st));
    }
    if (count_steps)
        k_grmi_probe_staged<true><<<sm_count(), STAGE_NT, sm, st>>>(gd, reinterpret_cast<const ulonglong2 *>(s_pairs),
                                                                    reg, nwin, shift, work, out, trace, dbg, img);
    else
        k_grmi_probe_staged<false><<<sm_count(), STAGE_NT, sm, st>>>(gd, reinterpret_cast<const ulonglong2 *>(s_pairs),
                                                                     reg, nwin, shift, work, out, trace, dbg, img);
    LJ_CK_LAUNCH();
    if (dbg) {
        std::vector<i64> h((size_t)nk * 4);
        LJ_CK(cudaMemcpyAsync(h.data(), dbg, h.size() * sizeof(i64), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaStreamSynchronize(st));
        LJ_CK(cudaFree(dbg));
        if (FILE *f = fopen(dbg_path, "wb")) {
            fwrite(h.data(), sizeof(i64), h.size(), f);
            fclose(f);
        }
    }
    if (trace) {
        std::vector<u64> h(npieces * 8);
        LJ_CK(cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(u64), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaStreamSynchronize(st));
        LJ_CK(cudaFree(trace));
        if (FILE *f = fopen(trace_path, "wb")) {
            fwrite(h.data(), sizeof(u64), h.size(), f);
            fclose(f);
        }
    }
    return LJ_OK;
}

int lj_grmi_probe_pairs(const LjGrmi *idx, const uint64_t *s_pairs, int64_t nk, uint64_t *out, int accumulate,
                        void *stream) {
    LJ_REQUIRE(idx != nullptr, "null index");
    cudaStream_t st = as_stream(stream);
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nk <= 0 || idx->n == 0) return LJ_OK;
    constexpr int NT = 256;
    k_grmi_probe<NT, AosIn><<<grid_for(nk, NT, 8), NT, 0, st>>>(
        GrmiDev(*idx), AosIn{reinterpret_cast<const ulonglong2 *>(s_pairs)}, nk, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_grmi_count(const LjGrmi *idx, const int64_t *slots0, const uint64_t *keys, int64_t nk, int64_t *lefts,
                  int64_t *counts, int64_t *probes, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    if (nk <= 0) return LJ_OK;
    k_grmi_count<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(GrmiDev(*idx), slots0, keys, nk,
                                                                       lefts, counts, probes);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_grmi_collect(const LjGrmi *idx, const uint64_t *keys, int64_t nk, const int64_t *lefts,
                    const int64_t *offsets, uint64_t *out_pay, int64_t *out_src, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    if (nk <= 0) return LJ_OK;
    k_grmi_collect<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(GrmiDev(*idx), keys, nk, lefts,
                                                                         offsets, out_pay, out_src);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_leaf_bucket_bins(int64_t L) {
    if (L < 1) return 0;
    int sh = slot_window_shift(L);
    return (int)((L + ((i64)1 << sh) - 1) >> sh);
}

int lj_leaf_bucket_regions(int64_t L) { return 2 * lj_leaf_bucket_bins(L) + 2; }

int64_t lj_leaf_bucket_capacity(int64_t nk, int64_t L) {
    return est_capacity(nk < 0 ? 0 : nk, lj_leaf_bucket_bins(L));
}

size_t lj_leaf_bucket_workspace_bytes(int64_t nk, int64_t L) {
    const int nwin = lj_leaf_bucket_bins(L);
    const size_t a = part_workspace_bytes(nk, nwin), b = est_workspace_bytes(nwin);
    return (a > b ? a : b) + al(sizeof(u64) * (size_t)nwin) + al(kb_bytes(nwin));
}

int lj_leaf_bucket(const LjGrmi *idx, const uint64_t *keys, const uint64_t *pay, int64_t nk, uint64_t *pairs_out,
                   int64_t *reg_out, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1 && idx->L >= 1, "index is empty");
    if (ws_bytes < lj_leaf_bucket_workspace_bytes(nk, idx->L)) {
        set_error("lj_leaf_bucket: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    const int nwin = lj_leaf_bucket_bins(idx->L);
    const size_t a = part_workspace_bytes(nk, nwin), b = est_workspace_bytes(nwin);
    const size_t pws = a > b ? a : b;
    SlotBin f;
    f.m = RmiDev(idx->model);
    f.slot_of = SlotMap(idx->n, idx->L);
    f.wshift = slot_window_shift(idx->L);
    f.nwin = nwin;
    f.wk = reinterpret_cast<const u64 *>((char *)ws + pws);
    k_window_keys<<<(nwin + 255) / 256, 256, 0, st>>>(idx->slots, nwin, f.wshift, (u64 *)f.wk);
    LJ_CK_LAUNCH();
    SoaSrc<SlotBin> src{keys, pay, f};
    static const bool exact_only = getenv("LJ_K4_EXACT") != nullptr;
    static const bool model_bins = getenv("LJ_K4_MODEL_BINS") != nullptr;
    if (staged_ok(idx) && src.aligned16() && !exact_only) {
        // one pass into estimated-capacity regions (+ overflow), the layout
        // the staged probe reads
        if (!model_bins && nwin <= KB_MAXBINS) {
            // window = #{ j >= 1 : wk[j] < k } = #{ j : wk[j] + 1 <= k }:
            // the same bins without a model evaluation per tuple
            u64 *lay = reinterpret_cast<u64 *>((char *)ws + pws + al(sizeof(u64) * (size_t)nwin));
            k_window_bounds<<<(nwin + 255) / 256, 256, 0, st>>>(f.wk, nwin, lay);
            k_keybin_build<<<1, 1024, 0, st>>>(lay, nwin);
            LJ_CK_LAUNCH();
            KeyRangeBin kb;
            kb.g = lay;
            kb.nb = nwin;
            SoaSrc<KeyRangeBin> ksrc{keys, pay, kb};
            return run_partition_est(ksrc, nk, nwin, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out, ws, pws, st);
        }
        return run_partition_est(src, nk, nwin, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out, ws, pws, st);
    }
    const int rc = run_partition(src, nk, nwin, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out, ws, pws, st);
    if (rc) return rc;
    k_starts_to_reg<<<(nwin + 256) / 256, 256, 0, st>>>(nwin, reg_out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

}  // extern "C"
