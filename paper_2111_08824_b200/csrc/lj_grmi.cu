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

#include "lj_common.cuh"
#include "lj_part.cuh"

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
    __host__ explicit GrmiDev(const LjGrmi &g)
        : model(g.model), n(g.n), L(g.L), slots(g.slots), bitmap(g.bitmap),
          payload_nonzero(g.payload_nonzero) {}

    __device__ __forceinline__ u64 key(i64 i) const { return ldg(slots + 2 * i); }
    __device__ __forceinline__ i64 predict_slot(u64 k) const {
        return grmi_slot_of_pos(model.pos(u64_to_f64(k)), n, L);
    }
    __device__ __forceinline__ bool real(i64 i, u64 pay) const {
        if (payload_nonzero) return pay != 0;
        return (__ldg(bitmap + (i >> 5)) >> (i & 31)) & 1u;
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
        i64 s = g.search(g.predict_slot(k), k, probes);
        steps += (u64)probes;
        if (s < 0) continue;
        while (s > 0 && g.key(s - 1) == k) --s;  // leftmost slot of the run is real
        for (; s < g.L; ++s) {
            ulonglong2 e = ldg2(g.slots + 2 * s);
            if (e.x != k) break;
            if (!g.real(s, e.y)) continue;
            u64 v = e.y + ps;
            ++cnt;
            sum += v;
            x ^= v;
        }
    }
    reduce_checksum(cnt, sum, x, steps, out);
}

// K1 v2: the same per-probe semantics as k_grmi_probe, restructured so a
// warp never waits for its slowest search.  Every lane runs the reference's
// search (gapped.py:86-160) as a state machine that issues exactly ONE
// dependent load per loop iteration (leaf record, or one gapped slot); a
// lane whose probe finishes pops the next probe from a per-warp queue in
// shared memory, which the warp refills with coalesced, evict-first loads of
// S.  Work per warp therefore tracks the MEAN search length, not the max,
// and every iteration keeps 32 independent loads in flight per warp.
enum : int { PH_IDLE = 0, PH_LEAF, PH_FIRST, PH_RIGHT, PH_LEFT, PH_BIN, PH_VERIFY, PH_WL, PH_SCAN };

template <int NT>
__global__ void __launch_bounds__(NT) k_grmi_probe_sm(GrmiDev g, const u64 *__restrict__ skeys,
                                                      const u64 *__restrict__ spay, i64 nk, u64 *out) {
    constexpr int QN = 64;  // probes queued per warp
    __shared__ ulonglong2 q[NT / 32][QN];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const i64 L = g.L;
    i64 next = ((i64)blockIdx.x * (NT / 32) + w) * 32;
    const i64 wstride = (i64)gridDim.x * NT;
    unsigned qh = 0, qt = 0;
    int ph = PH_IDLE;
    u64 k = 0, ps = 0;
    i64 start = 0, step = 0, lo = 0, hi = 0, cur = 0;  // lo doubles as the reference's `prev`
    unsigned probes = 0;
    u64 cnt = 0, sum = 0, x = 0, steps = 0;
    for (;;) {
        if (qt - qh <= (unsigned)(QN - 32) && next < nk) {  // warp-uniform refill
            i64 i = next + lane;
            if (i < nk) q[w][(qt + lane) & (QN - 1)] = make_ulonglong2(ld_stream(skeys + i), ld_stream(spay + i));
            qt += (unsigned)min((i64)32, nk - next);
            next += wstride;
            __syncwarp();
        }
        const unsigned idle = __ballot_sync(0xffffffffu, ph == PH_IDLE);
        const unsigned avail = qt - qh;
        if (ph == PH_IDLE) {
            unsigned r = __popc(idle & lt);
            if (r < avail) {
                ulonglong2 e = q[w][(qh + r) & (QN - 1)];
                k = e.x;
                ps = e.y;
                ph = PH_LEAF;
            }
        }
        qh += min((unsigned)__popc(idle), avail);
        __syncwarp();
        if (__ballot_sync(0xffffffffu, ph != PH_IDLE) == 0 && qh == qt && next >= nk) break;
        if (ph == PH_LEAF) {
            // models.py:112-124 + gapped.py:258-261 (one leaf-record load)
            double xf = u64_to_f64(k);
            LjLeaf lf = load_leaf(g.model.leaves, g.model.route(xf));
            start = grmi_slot_of_pos(rmi_leaf_pos(lf, xf), g.n, L);
            cur = start;
            ph = PH_FIRST;
            continue;
        }
        if (ph == PH_IDLE) continue;
        const ulonglong2 e = ldg2(g.slots + 2 * cur);
        bool found = false, bsetup = false;
        switch (ph) {
            case PH_FIRST:
                probes = 1;
                if (e.x == k) {
                    found = true;
                } else if (e.x < k) {
                    lo = start;  // prev
                    step = 1;
                    if (start + 1 >= L) { lo = start + 1; hi = L; bsetup = true; }
                    else { cur = start + 1; ph = PH_RIGHT; }
                } else {
                    lo = start;  // prev
                    step = 1;
                    if (start - 1 < 0) { lo = 0; hi = start; bsetup = true; }
                    else { cur = start - 1; ph = PH_LEFT; }
                }
                break;
            case PH_RIGHT:
                ++probes;
                if (e.x < k) {
                    lo = cur;
                    step <<= 1;
                    if (start + step >= L) { lo = lo + 1; hi = L; bsetup = true; }
                    else cur = start + step;
                } else if (e.x == k) {
                    found = true;
                } else {
                    lo = lo + 1;
                    hi = cur;
                    bsetup = true;
                }
                break;
            case PH_LEFT:
                ++probes;
                if (e.x > k) {
                    lo = cur;
                    step <<= 1;
                    if (start - step < 0) { hi = lo; lo = 0; bsetup = true; }
                    else cur = start - step;
                } else if (e.x == k) {
                    found = true;
                } else {
                    hi = lo;
                    lo = cur + 1;
                    bsetup = true;
                }
                break;
            case PH_BIN:
                ++probes;
                if (e.x < k) lo = cur + 1; else hi = cur;
                bsetup = true;
                break;
            case PH_VERIFY:
                ++probes;
                if (e.x == k) found = true;
                else { steps += probes; ph = PH_IDLE; }
                break;
            case PH_WL:  // walk to the leftmost slot of the equal run
                if (e.x == k && cur > 0) --cur;
                else { cur = e.x == k ? cur : cur + 1; ph = PH_SCAN; }
                break;
            case PH_SCAN:  // gather the real entries of the run
                if (e.x != k) {
                    ph = PH_IDLE;
                } else {
                    if (g.real(cur, e.y)) {
                        u64 v = e.y + ps;
                        ++cnt;
                        sum += v;
                        x ^= v;
                    }
                    if (++cur >= L) ph = PH_IDLE;
                }
                break;
        }
        if (bsetup) {
            if (lo < hi) { cur = (lo + hi) >> 1; ph = PH_BIN; }
            else if (lo < L) { cur = lo; ph = PH_VERIFY; }
            else { steps += probes; ph = PH_IDLE; }
        }
        if (found) {
            steps += probes;
            if (cur > 0) { --cur; ph = PH_WL; }
            else ph = PH_SCAN;
        }
    }
    reduce_checksum(cnt, sum, x, steps, out);
}

// ---------------------------------------------- staged probe (K1 over K4)
//
// After K4 every window of 2^shift predicted slots has its probes stored
// contiguously.  A CTA takes a piece of that array; for each window segment
// of the piece it stages the window's gapped KEYS (+ a halo of STAGE_H slots
// each side) in shared memory and runs the reference's exponential search
// (gapped.py:86-160, identical probe counting) there.  A search or run scan
// that leaves the staged range is redone in global memory from scratch, so
// results and probe counts never depend on the staging.  Payloads (needed
// for occupancy and the checksum) are read from global memory, 1-2 per hit.

constexpr int STAGE_NT = 1024;
constexpr int STAGE_H = 2048;           // halo slots on each side
constexpr i64 STAGE_PIECE = 65536;      // probes per work item
constexpr i64 STAGE_MIN = 2048;         // smaller window segments: global search
constexpr int STAGE_U = 2;              // probes in flight per thread

// exponential search over any key accessor; kf(i, ok) clears ok when slot i
// is not available (then the result is meaningless and the caller redoes it)
template <class KeyF>
__device__ __forceinline__ i64 exp_search_with(const KeyF &kf, i64 L, i64 start, u64 k, i64 &probes, bool &ok) {
    probes = 1;
    u64 v = kf(start, ok);
    if (v == k) return start;
    i64 lo, hi;
    if (v < k) {
        i64 prev = start, step = 1;
        for (;;) {
            i64 idx = start + step;
            if (idx >= L) { lo = prev + 1; hi = L; break; }
            ++probes;
            u64 w = kf(idx, ok);
            if (!ok) return -1;
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
            u64 w = kf(idx, ok);
            if (!ok) return -1;
            if (w > k) { prev = idx; step <<= 1; }
            else if (w == k) return idx;
            else { lo = idx + 1; hi = prev; break; }
        }
    }
    while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        ++probes;
        if (kf(mid, ok) < k) lo = mid + 1; else hi = mid;
        if (!ok) return -1;
    }
    if (lo < L) {
        ++probes;
        if (kf(lo, ok) == k) return lo;
    }
    return -1;
}

// The reference's probe count (gapped.py:86-160) of an exponential search
// from `start`, computed without touching memory from the key's position in
// the sorted gapped array: slots [lb, re) hold the key, slots < lb are
// smaller, slots >= re larger.  Every comparison the reference makes is
// decided by where its index falls relative to lb and re.
__device__ __forceinline__ i64 ref_probe_count(i64 start, i64 lb, i64 re, i64 L) {
    i64 probes = 1;
    if (start >= lb && start < re) return 1;
    i64 lo, hi;
    if (start < lb) {
        i64 prev = start, step = 1;
        for (;;) {
            const i64 idx = start + step;
            if (idx >= L) { lo = prev + 1; hi = L; break; }
            ++probes;
            if (idx < lb) { prev = idx; step <<= 1; }
            else if (idx < re) return probes;
            else { lo = prev + 1; hi = idx; break; }
        }
    } else {
        i64 prev = start, step = 1;
        for (;;) {
            const i64 idx = start - step;
            if (idx < 0) { lo = 0; hi = prev; break; }
            ++probes;
            if (idx >= re) { prev = idx; step <<= 1; }
            else if (idx >= lb) return probes;
            else { lo = idx + 1; hi = prev; break; }
        }
    }
    while (lo < hi) {
        const i64 mid = (lo + hi) >> 1;
        ++probes;
        if (mid < lb) lo = mid + 1; else hi = mid;
    }
    if (lo < L) ++probes;
    return probes;
}

struct StagedKeys {
    const u64 *sk;
    i64 lo, hi;
    __device__ __forceinline__ u64 operator()(i64 i, bool &ok) const {
        if (i < lo || i >= hi) {
            ok = false;
            return 0;
        }
        return sk[i - lo];
    }
};

// one probe against the index: staged search + run scan, global redo on escape
__device__ __forceinline__ void probe_one(const GrmiDev &g, const StagedKeys &st, u64 k, u64 ps, u64 &cnt, u64 &sum,
                                          u64 &x, u64 &steps) {
    const i64 start = g.predict_slot(k);
    i64 probes;
    bool ok = true;
    i64 s = exp_search_with(st, g.L, start, k, probes, ok);
    u64 c = 0, sm = 0, xx = 0;
    if (ok && s >= 0) {
        while (s > 0) {
            const u64 v = st(s - 1, ok);
            if (!ok || v != k) break;
            --s;
        }
        for (i64 i = s; ok && i < g.L; ++i) {
            const u64 v = st(i, ok);
            if (!ok || v != k) break;
            const u64 pay = ldg(g.slots + 2 * i + 1);
            if (!g.real(i, pay)) continue;
            const u64 t = pay + ps;
            ++c;
            sm += t;
            xx ^= t;
        }
    }
    if (!ok) {  // left the staged range: the plain global-memory probe
        c = sm = xx = 0;
        s = g.search(start, k, probes);
        if (s >= 0) {
            while (s > 0 && g.key(s - 1) == k) --s;
            for (; s < g.L; ++s) {
                const ulonglong2 e = ldg2(g.slots + 2 * s);
                if (e.x != k) break;
                if (!g.real(s, e.y)) continue;
                const u64 t = e.y + ps;
                ++c;
                sm += t;
                xx ^= t;
            }
        }
    }
    steps += (u64)probes;
    cnt += c;
    sum += sm;
    x ^= xx;
}

__global__ void __launch_bounds__(STAGE_NT, 1) k_grmi_probe_staged(GrmiDev g, const ulonglong2 *__restrict__ rec,
                                                                   i64 nk, const i64 *__restrict__ wstarts,
                                                                   int nwin, int shift, unsigned long long *work,
                                                                   u64 *out) {
    extern __shared__ u64 sk[];
    __shared__ i64 s_piece;
    const i64 wsz = (i64)1 << shift;
    u64 cnt = 0, sum = 0, x = 0, steps = 0;
    const StagedKeys none{sk, 0, 0};
    for (;;) {
        if (threadIdx.x == 0) s_piece = (i64)atomicAdd(work, 1ULL);
        __syncthreads();
        const i64 p0 = s_piece * STAGE_PIECE;
        __syncthreads();
        if (p0 >= nk) break;
        const i64 p1 = min(p0 + STAGE_PIECE, nk);
        // first window overlapping p0
        int lo = 0, hi = nwin;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (wstarts[mid] <= p0) lo = mid; else hi = mid;
        }
        for (int w = lo; w < nwin && wstarts[w] < p1; ++w) {
            const i64 a = max(p0, wstarts[w]), e = min(p1, wstarts[w + 1]);
            if (e <= a) continue;
            if (e - a >= STAGE_MIN) {
                const i64 slo = max((i64)0, ((i64)w << shift) - STAGE_H);
                const i64 shi = min(g.L, (((i64)w + 1) << shift) + STAGE_H);
                for (i64 i = threadIdx.x; i < shi - slo; i += STAGE_NT) sk[i] = ldg(g.slots + 2 * (slo + i));
                __syncthreads();
                const StagedKeys st{sk, slo, shi};
                // STAGE_U probes per thread per step, each phase issued for
                // all of them before the next: the global loads (probe
                // record, leaf record, payloads) of different probes overlap
                for (i64 t0 = a + threadIdx.x; t0 < e; t0 += (i64)STAGE_NT * STAGE_U) {
                    u64 k[STAGE_U], ps[STAGE_U];
                    i64 start[STAGE_U], s[STAGE_U], probes[STAGE_U];
                    bool ok[STAGE_U];
#pragma unroll
                    for (int u = 0; u < STAGE_U; ++u) {
                        const i64 t = t0 + (i64)u * STAGE_NT;
                        ulonglong2 r = t < e ? __ldcs(rec + t) : make_ulonglong2(0, 0);
                        k[u] = r.x;
                        ps[u] = r.y;
                    }
#pragma unroll
                    for (int u = 0; u < STAGE_U; ++u) start[u] = g.predict_slot(k[u]);
                    // lower bound in the staged keys: a branch-free binary
                    // search whose trip count is the same for every lane
                    const i64 span = shi - slo;
#pragma unroll
                    for (int u = 0; u < STAGE_U; ++u) {
                        i64 base = 0, len = span;
                        while (len > 1) {
                            const i64 half = len >> 1;
                            base = sk[base + half - 1] < k[u] ? base + half : base;
                            len -= half;
                        }
                        s[u] = slo + base + ((span > 0 && sk[base] < k[u]) ? 1 : 0);  // first slot >= key
                        // the lower bound is exact only strictly inside the staged range
                        ok[u] = (s[u] > slo || slo == 0) && (s[u] < shi || shi == g.L);
                    }
                    // payload of the first slot of the run (a one-slot run is the common case)
                    u64 pay[STAGE_U];
#pragma unroll
                    for (int u = 0; u < STAGE_U; ++u)
                        pay[u] = (ok[u] && s[u] < g.L && sk[s[u] - slo] == k[u]) ? ldg(g.slots + 2 * s[u] + 1) : 0;
#pragma unroll
                    for (int u = 0; u < STAGE_U; ++u) {
                        if (t0 + (i64)u * STAGE_NT >= e) continue;
                        u64 c = 0, sm = 0, xx = 0;
                        i64 re = s[u];
                        if (ok[u]) {
                            for (; re < g.L; ++re) {
                                if (re >= shi) { ok[u] = false; break; }
                                if (sk[re - slo] != k[u]) break;
                                const u64 py = re == s[u] ? pay[u] : ldg(g.slots + 2 * re + 1);
                                if (!g.real(re, py)) continue;
                                const u64 tt = py + ps[u];
                                ++c;
                                sm += tt;
                                xx ^= tt;
                            }
                        }
                        if (!ok[u]) {  // outside the staged range: the global-memory probe
                            probe_one(g, StagedKeys{sk, 0, 0}, k[u], ps[u], cnt, sum, x, steps);
                            continue;
                        }
                        probes[u] = ref_probe_count(start[u], s[u], re, g.L);
                        steps += (u64)probes[u];
                        cnt += c;
                        sum += sm;
                        x ^= xx;
                    }
                }
                __syncthreads();
            } else {
                for (i64 t = a + threadIdx.x; t < e; t += STAGE_NT) {
                    const ulonglong2 r = __ldcs(rec + t);
                    probe_one(g, none, r.x, r.y, cnt, sum, x, steps);
                }
            }
        }
    }
    (void)wsz;
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
    i64 n, L;
    int shift;
    __device__ __forceinline__ void prepare() const {}
    __device__ __forceinline__ int operator()(u64 k) const {
        return (int)(grmi_slot_of_pos(m.pos(u64_to_f64(k)), n, L) >> shift);
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
    static const int sm_variant = getenv("LJ_K1_SM") ? atoi(getenv("LJ_K1_SM")) : 0;
    if (sm_variant) {
        k_grmi_probe_sm<NT><<<grid_for(nk, NT, 6), NT, 0, st>>>(GrmiDev(*idx), s_keys, s_pay, nk, out);
    } else {
        k_grmi_probe<NT, SoaIn><<<grid_for(nk, NT, 8), NT, 0, st>>>(GrmiDev(*idx), SoaIn{s_keys, s_pay}, nk, out);
    }
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
    const size_t sm = sizeof(u64) * (size_t)(((i64)1 << shift) + 2 * STAGE_H);
    if (sm > 200 * 1024) {  // window too large to stage: plain K1 over the grouped records
        return lj_grmi_probe_pairs(idx, s_pairs, nk, out, 1, stream);
    }
    static bool attr = false;
    if (!attr) {
        LJ_CK(cudaFuncSetAttribute(k_grmi_probe_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    unsigned long long *work = reinterpret_cast<unsigned long long *>(ws);
    LJ_CK(cudaMemsetAsync(work, 0, sizeof(unsigned long long), st));
    k_grmi_probe_staged<<<sm_count(), STAGE_NT, sm, st>>>(GrmiDev(*idx), reinterpret_cast<const ulonglong2 *>(s_pairs),
                                                          nk, wstarts, nwin, shift, work, out);
    LJ_CK_LAUNCH();
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
    f.n = idx->n;
    f.L = idx->L;
    f.shift = slot_window_shift(idx->L);
    SoaSrc<SlotBin> src{keys, pay, f};
    return run_partition(src, nk, lj_leaf_bucket_bins(idx->L), reinterpret_cast<ulonglong2 *>(pairs_out),
                         starts_out, ws, ws_bytes, as_stream(stream));
}

}  // extern "C"
