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

// ---------------------------------------------- staged probe (K1 over K4)
//
// After K4 every window of 2^shift predicted slots has its probes stored
// contiguously.  A CTA takes a piece of that array; for each window segment
// of the piece it stages in shared memory the window's gapped KEYS (+ a halo
// of STAGE_H slots each side), the matching occupancy-bitmap words, and a
// 2^STAGE_TB-entry radix table over the staged key range (T[p] = first
// staged slot whose key prefix >= p).  Per probe:
//   * lower bound lb of the key: one table pair + a branch-free binary search
//     whose trip count is fixed per window (the largest table bucket), so a
//     warp never waits for its slowest lane;
//   * run [lb, re) of equal keys and its real entries from shared memory;
//     payloads (for the checksum) from global memory, normally one per hit;
//   * the reference's probe count (gapped.py:86-160) computed from
//     (start, lb, re) alone (ref_probe_count), so results and counters are
//     exactly those of the exponential search from the predicted slot.
// A lower bound or run that is not provably inside the staged range is
// redone in global memory from scratch (probe_global).

constexpr int STAGE_NT = 1024;
constexpr int STAGE_H = 2048;           // halo slots on each side
constexpr i64 STAGE_PIECE = 65536;      // probes per work item
constexpr i64 STAGE_MIN = 2048;         // smaller window segments: global search
constexpr int STAGE_U = 2;              // probes in flight per thread
constexpr int STAGE_TB = 12;            // radix-table bits
constexpr int STAGE_TBINS = 1 << STAGE_TB;
constexpr int STAGE_MAX_SHIFT = 15;     // span < 2^16 (u16 table entries)

// one probe entirely in global memory (the reference's search, gapped.py:86-160)
__device__ __noinline__ void probe_global(const GrmiDev &g, i64 start, u64 k, u64 ps, u64 &cnt, u64 &sum,
                                          u64 &x, u64 &steps) {
    i64 probes;
    const i64 s = g.search(start, k, probes);
    if (s >= 0) g.gather_run(s, k, ps, cnt, sum, x);
    steps += (u64)probes;
}

static size_t staged_smem_bytes(int shift) {
    const size_t span = ((size_t)1 << shift) + 2 * STAGE_H;
    return sizeof(u64) * span + sizeof(u32) * (span / 32 + 2) + sizeof(u16) * (STAGE_TBINS + 2) +
           sizeof(u16) * (span / 32 + 2);
}

// first set bit at staged slot >= j (bit of slot i is bm bit i + bo), or
// span; nz[w] = first nonzero bitmap word >= w (0xffff: none), so long gap
// runs cost no more than short ones
__device__ __forceinline__ int next_real(const u32 *bm, const u16 *nz, int nbw, int bo, int j, int span) {
    const int b = j + bo;
    int wi = b >> 5;
    u32 wv = bm[wi] & (0xffffffffu << (b & 31));
    if (wv == 0) {
        wi = wi + 1 < nbw ? (int)nz[wi + 1] : nbw;
        if (wi >= nbw) return span;
        wv = bm[wi];
    }
    return min(span, (wi << 5) + __ffs((int)wv) - 1 - bo);
}

__global__ void __launch_bounds__(STAGE_NT, 1) k_grmi_probe_staged(GrmiDev g, const ulonglong2 *__restrict__ rec,
                                                                   i64 nk, const i64 *__restrict__ wstarts,
                                                                   int nwin, int shift, unsigned long long *work,
                                                                   u64 *out, u64 *trace) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int span_max = (1 << shift) + 2 * STAGE_H;
    u64 *sk = reinterpret_cast<u64 *>(smem);
    u32 *bm = reinterpret_cast<u32 *>(sk + span_max);
    u16 *T = reinterpret_cast<u16 *>(bm + span_max / 32 + 2);
    u16 *nz = T + STAGE_TBINS + 2;
    __shared__ i64 s_piece;
    __shared__ int s_max;
    __shared__ unsigned s_esc, s_iters;
    __shared__ u32 s_small[2048 / 32];  // windows with < STAGE_MIN probes: global search
    const int tid = threadIdx.x;
    for (int j = tid; j < 2048 / 32; j += STAGE_NT) s_small[j] = 0;
    __syncthreads();
    for (int w = tid; w < nwin; w += STAGE_NT)
        if (wstarts[w + 1] - wstarts[w] < STAGE_MIN) atomicOr(&s_small[w >> 5], 1u << (w & 31));
    u64 cnt = 0, sum = 0, x = 0, steps = 0;
    for (;;) {
        if (tid == 0) s_piece = (i64)atomicAdd(work, 1ULL);
        __syncthreads();
        const i64 p0 = s_piece * STAGE_PIECE;
        __syncthreads();
        if (p0 >= nk) break;
        const i64 p1 = min(p0 + STAGE_PIECE, nk);
        u64 t_begin = 0;
        if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        int nstaged = 0;
        if (tid == 0) s_esc = s_iters = 0;
        int wlo = 0, whi = nwin;  // first window overlapping p0
        while (whi - wlo > 1) {
            const int mid = (wlo + whi) >> 1;
            if (wstarts[mid] <= p0) wlo = mid; else whi = mid;
        }
        bool any_small = false;
        for (int w = wlo; w < nwin && wstarts[w] < p1; ++w) {
            const i64 a = max(p0, wstarts[w]), e = min(p1, wstarts[w + 1]);
            if (e <= a) continue;
            if ((s_small[w >> 5] >> (w & 31)) & 1u) {
                any_small = true;
                continue;
            }
            ++nstaged;
            // ---- stage keys, bitmap words and the radix table of the window
            const i64 slo = max((i64)0, ((i64)w << shift) - STAGE_H);
            const i64 shi = min(g.L, (((i64)w + 1) << shift) + STAGE_H);
            const int span = (int)(shi - slo);
            for (int i = tid; i < span; i += STAGE_NT) sk[i] = ldg(g.slots + 2 * (slo + i));
            const i64 w0 = slo >> 5;
            const int nbw = (int)(((shi - 1) >> 5) - w0 + 1);
            for (int j = tid; j < nbw; j += STAGE_NT) bm[j] = __ldg(g.bitmap + w0 + j);
            if (tid == 0) s_max = 0;
            __syncthreads();
            const u64 kmin = sk[0], kmax = sk[span - 1];
            const u64 krange = kmax - kmin;
            const int sh = krange == 0 ? 0 : max(0, 64 - __clzll((long long)krange) - STAGE_TB);
            for (int i = tid; i < span; i += STAGE_NT) {
                const int p = (int)((sk[i] - kmin) >> sh);
                const int pp = i == 0 ? -1 : (int)((sk[i - 1] - kmin) >> sh);
                for (int q = pp + 1; q <= p; ++q) T[q] = (u16)i;
            }
            for (int q = (int)(krange >> sh) + 1 + tid; q <= STAGE_TBINS; q += STAGE_NT) T[q] = (u16)span;
            for (int j = tid; j < nbw; j += STAGE_NT) nz[j] = bm[j] ? (u16)j : (u16)0xffff;
            __syncthreads();
            // suffix minimum of nz (doubling); nbw <= 2 * STAGE_NT
            for (int off = 1; off < nbw; off <<= 1) {
                u16 v[2];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int j = tid + r * STAGE_NT;
                    v[r] = j < nbw ? (j + off < nbw ? min(nz[j], nz[j + off]) : nz[j]) : (u16)0;
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (tid + r * STAGE_NT < nbw) nz[tid + r * STAGE_NT] = v[r];
                __syncthreads();
            }
            {
                int mb = 0;
                for (int q = tid; q < STAGE_TBINS; q += STAGE_NT) mb = max(mb, (int)T[q + 1] - (int)T[q]);
                mb = __reduce_max_sync(0xffffffffu, mb);
                if ((tid & 31) == 0 && mb) atomicMax(&s_max, mb);
            }
            __syncthreads();
            const int iters = 32 - __clz(s_max);
            if (trace && tid == 0) s_iters = max(s_iters, (unsigned)s_max);
            const int bo = (int)(slo & 31);
            const int lim = (int)min(g.L - slo, (i64)1 << 30);
            const int zero = -(int)min(slo, (i64)1 << 30);
            const bool lo_open = slo > 0, hi_open = shi < g.L;
            // ---- probes: STAGE_U per thread per step, phase by phase
            for (i64 t0 = a + tid; t0 < e; t0 += (i64)STAGE_NT * STAGE_U) {
                u64 k[STAGE_U], ps[STAGE_U];
                int start[STAGE_U], lo[STAGE_U], len[STAGE_U];
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {
                    const i64 t = t0 + (i64)u * STAGE_NT;
                    const ulonglong2 r = t < e ? __ldcs(rec + t) : make_ulonglong2(kmin, 0);
                    k[u] = r.x;
                    ps[u] = r.y;
                }
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) start[u] = (int)(g.predict_slot(k[u]) - slo);
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {
                    if (k[u] < kmin) { lo[u] = 0; len[u] = 0; }
                    else if (k[u] > kmax) { lo[u] = span; len[u] = 0; }
                    else {
                        const int p = (int)((k[u] - kmin) >> sh);
                        lo[u] = T[p];
                        len[u] = (int)T[p + 1] - lo[u];
                    }
                }
                for (int it = 0; it < iters; ++it) {
#pragma unroll
                    for (int u = 0; u < STAGE_U; ++u) {
                        const int half = len[u] >> 1;
                        const bool less = sk[min(lo[u] + half, span - 1)] < k[u];
                        if (len[u] > 0) {
                            lo[u] = less ? lo[u] + half + 1 : lo[u];
                            len[u] = less ? len[u] - half - 1 : half;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < STAGE_U; ++u) {
                    if (t0 + (i64)u * STAGE_NT >= e) continue;
                    const int lb = lo[u];
                    bool ok = (lb > 0 || !lo_open) && (lb < span || !hi_open);
                    int re = lb;
                    u64 c = 0, sm = 0, xx = 0;
                    if (ok && lb < span && sk[lb] == k[u]) {
                        // gap slots copy the real key to their left, so the
                        // key changes only at real slots: walk the real
                        // slots of the run through the bitmap
                        int j = lb;
                        for (;;) {
                            j = next_real(bm, nz, nbw, bo, j, span);
                            if (j >= span) {
                                re = span;
                                if (hi_open) {  // the run goes on past the staged range
                                    i64 ja = shi;
                                    for (;; ++ja) {
                                        ja = g.next_real(ja);
                                        if (ja >= g.L) break;
                                        const ulonglong2 ev = ldg2(g.slots + 2 * ja);
                                        if (ev.x != k[u]) break;
                                        const u64 tt = ev.y + ps[u];
                                        ++c;
                                        sm += tt;
                                        xx ^= tt;
                                    }
                                    re = (int)min(ja - slo, (i64)1 << 30);
                                }
                                break;
                            }
                            if (sk[j] != k[u]) {
                                re = j;
                                break;
                            }
                            const u64 tt = ldg(g.slots + 2 * (slo + j) + 1) + ps[u];
                            ++c;
                            sm += tt;
                            xx ^= tt;
                            ++j;
                        }
                    }
                    if (!ok) {
                        if (trace) atomicAdd(&s_esc, 1u);
                        probe_global(g, start[u] + slo, k[u], ps[u], cnt, sum, x, steps);
                        continue;
                    }
                    steps += (u64)ref_probe_count(start[u], lb, re, lim, zero);
                    cnt += c;
                    sum += sm;
                    x ^= xx;
                }
            }
            __syncthreads();
        }
        if (any_small) {  // block-uniform: every thread walked the same windows
            for (i64 t = p0 + tid; t < p1; t += STAGE_NT) {
                const ulonglong2 r = __ldcs(rec + t);
                const i64 start = g.predict_slot(r.x);
                const int w = (int)(start >> shift);
                if ((s_small[w >> 5] >> (w & 31)) & 1u) probe_global(g, start, r.x, r.y, cnt, sum, x, steps);
            }
        }
        if (trace) {
            __syncthreads();
            if (tid == 0) {
                u64 t_end, smid;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
                asm volatile("{ .reg .u32 r; mov.u32 r, %%smid; cvt.u64.u32 %0, r; }" : "=l"(smid));
                u64 *tr = trace + 6 * (p0 / STAGE_PIECE);
                tr[0] = t_begin;
                tr[1] = t_end;
                tr[2] = smid;
                tr[3] = (u64)nstaged;
                tr[4] = (u64)any_small | ((u64)s_iters << 8);
                tr[5] = (u64)wlo | ((u64)s_esc << 16);
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

// Bin = window of 2^shift gapped slots around the PREDICTED slot of the key
// (gapped.py:258-261).  A leaf-based grouping is useless on skewed keys:
// the linear root routes most lognormal keys to a handful of huge leaves.
// Predicted-slot windows (<= 2048 bins, e.g. 16384 slots = 256 KB at C2) make
// every warp's searches after bucketing stay inside one L1/L2-resident
// stretch of the index, so each index sector comes from DRAM ~once.
struct SlotBin {
    RmiDev m;
    SlotMap slot_of;
    int shift;
    __device__ __forceinline__ void prepare() const {}
    __device__ __forceinline__ int operator()(u64 k) const {
        return (int)(slot_of(m.pos(u64_to_f64(k))) >> shift);
    }
};

static int slot_window_shift(i64 L) {
    int s = 0;
    // <= 2048 windows: blocks x bins open write lines (~148 x 2048 x 128 B)
    // stay L2-resident during the scatter, so records leave L2 as full lines
    while (((L + ((i64)1 << s) - 1) >> s) > 2048) ++s;
    return s;
}

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

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

int lj_grmi_probe_bucketed(const LjGrmi *idx, const uint64_t *s_pairs, int64_t nk, const int64_t *wstarts,
                           void *ws, uint64_t *out, int accumulate, void *stream) {
    LJ_REQUIRE(idx != nullptr, "null index");
    cudaStream_t st = as_stream(stream);
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nk <= 0 || idx->n == 0) return LJ_OK;
    const int shift = slot_window_shift(idx->L);
    const int nwin = lj_leaf_bucket_bins(idx->L);
    const size_t sm = staged_smem_bytes(shift);
    if (shift > STAGE_MAX_SHIFT || sm > 200 * 1024 || idx->bitmap == nullptr) {
        // window too large to stage: plain K1 over the grouped records
        return lj_grmi_probe_pairs(idx, s_pairs, nk, out, 1, stream);
    }
    static bool attr = false;
    if (!attr) {
        LJ_CK(cudaFuncSetAttribute(k_grmi_probe_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    unsigned long long *work = reinterpret_cast<unsigned long long *>(ws);
    LJ_CK(cudaMemsetAsync(work, 0, sizeof(unsigned long long), st));
    // LJ_STAGE_TRACE=<file>: per-piece timing records (diagnostics only)
    static const char *trace_path = getenv("LJ_STAGE_TRACE");
    u64 *trace = nullptr;
    const size_t npieces = (size_t)((nk + STAGE_PIECE - 1) / STAGE_PIECE);
    if (trace_path) LJ_CK(cudaMalloc(&trace, npieces * 6 * sizeof(u64)));
    k_grmi_probe_staged<<<sm_count(), STAGE_NT, sm, st>>>(GrmiDev(*idx), reinterpret_cast<const ulonglong2 *>(s_pairs),
                                                          nk, wstarts, nwin, shift, work, out, trace);
    LJ_CK_LAUNCH();
    if (trace) {
        std::vector<u64> h(npieces * 6);
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

size_t lj_leaf_bucket_workspace_bytes(int64_t nk, int64_t L) {
    return part_workspace_bytes(nk, lj_leaf_bucket_bins(L));
}

int lj_leaf_bucket(const LjGrmi *idx, const uint64_t *keys, const uint64_t *pay, int64_t nk, uint64_t *pairs_out,
                   int64_t *starts_out, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1 && idx->L >= 1, "index is empty");
    SlotBin f;
    f.m = RmiDev(idx->model);
    f.slot_of = SlotMap(idx->n, idx->L);
    f.shift = slot_window_shift(idx->L);
    SoaSrc<SlotBin> src{keys, pay, f};
    return run_partition(src, nk, lj_leaf_bucket_bins(idx->L), reinterpret_cast<ulonglong2 *>(pairs_out),
                         starts_out, ws, ws_bytes, as_stream(stream));
}

}  // extern "C"
