// lj_lsj.cu -- learned sort-join (LSJ) on the GPU.  Reference: lsj.py:95-405.
//
//   smpl  K10 on a stratified 1% sample (lj_lsj_sample + lj_rmi_fit)
//   part  K6 histogram + K7 scatter of (key, payload) into Pf = P*F fine
//         CDF buckets (warp-aggregated atomics; 16-B interleaved output)
//   sort  K8 per fine bucket in shared memory: MODEL-PLACED counting sort
//         by the predicted position (the RMI is monotone, so ordering by
//         predicted position is consistent with key order and only runs of
//         equal predicted position remain unsorted), then insertion sort of
//         those runs; long runs go to a bitonic pass (k_sort_runs);
//         buckets larger than shared memory take the same model placement
//         through global memory (k_over_*); runs of one repeated key are
//         left as they are.
//   join  K9 per S tile of 1024 sorted tuples: the R window is found
//         through R's model (chunked_join's [f_R, l_R], lsj.py:343-346, at
//         the fine scale), staged in shared memory and merge-searched;
//         emits the checksum (or counts / pairs when materialising).
//
// Fine scale: the reference sorts P = effective_fanout buckets; Pf = P*F
// nests exactly inside them (floor(pos*P*F/n)/F == floor(pos*P/n)), so the
// coarse bucket bounds the reference reports are every F-th fine bound.
#include <cub/cub.cuh>

#include <vector>

#include "lj_common.cuh"

namespace lj {

constexpr int PART_NT = 256;
constexpr int SORT_NT = 512;
constexpr int CAP = 4096;     // largest bucket sorted in shared memory
constexpr int NBMAX = 2048;   // predicted-position bins per bucket
constexpr int RUN_SMALL = 32; // runs up to this length: insertion sort
constexpr int JOIN_T = 1024;  // S tile of the join
constexpr int JOIN_NT = 256;
constexpr int WCAP = 4096;    // R window keys staged in shared memory

// exact floor(x / d) for 0 <= x < 2^63, d >= 1: float reciprocal + fix-up
__device__ __forceinline__ i64 fdiv(i64 x, i64 d, double rd) {
    i64 q = (i64)__dmul_rn(i64_to_f64(x), rd);
    i64 r = x - q * d;
    while (r < 0) { --q; r += d; }
    while (r >= d) { ++q; r -= d; }
    return q;
}

struct Bin {
    RmiDev m;
    i64 nbins;
    double rn;  // 1.0 / m.n
    __device__ __forceinline__ i64 pos(const LjLeaf *lv, u64 k) const {
        double x = u64_to_f64(k);
        return rmi_leaf_pos(lv[m.route(x)], x);
    }
    // models.py:297 partition_index at scale nbins, exact
    __device__ __forceinline__ i64 of_pos(i64 p) const {
        return clip_i64(fdiv(p * nbins, m.n, rn), 0, nbins - 1);
    }
};

// Stage the leaf table in shared memory when it fits (LSJ sample models
// have <= 1000 leaves = 32 KB); otherwise read it through L1.
__device__ __forceinline__ const LjLeaf *stage_leaves(const RmiDev &m, LjLeaf *sl, bool stage) {
    if (!stage) return m.leaves;
    for (i64 i = threadIdx.x; i < m.m; i += blockDim.x) sl[i] = m.leaves[i];
    __syncthreads();
    return sl;
}

// ----------------------------------------------------------------- part

__global__ void __launch_bounds__(PART_NT) k_part_hist(Bin bn, const u64 *__restrict__ keys, i64 n, u32 *hist,
                                                       int stage) {
    extern __shared__ LjLeaf s_leaves[];
    const LjLeaf *lv = stage_leaves(bn.m, s_leaves, stage);
    const int lane = threadIdx.x & 31;
    const i64 stride = (i64)gridDim.x * PART_NT;
    for (i64 base = blockIdx.x * (i64)PART_NT + threadIdx.x - lane; base < n; base += stride) {
        i64 i = base + lane;
        long long b = -1;
        if (i < n) b = bn.of_pos(bn.pos(lv, ld_stream(keys + i)));
        unsigned peers = __match_any_sync(0xffffffffu, b);
        if (b >= 0 && lane == __ffs(peers) - 1) atomicAdd(hist + b, (u32)__popc(peers));
    }
}

__global__ void __launch_bounds__(PART_NT) k_part_scatter(Bin bn, const u64 *__restrict__ keys,
                                                          const u64 *__restrict__ pay, i64 n,
                                                          unsigned long long *cursor, ulonglong2 *out, int stage) {
    extern __shared__ LjLeaf s_leaves[];
    const LjLeaf *lv = stage_leaves(bn.m, s_leaves, stage);
    const int lane = threadIdx.x & 31;
    const i64 stride = (i64)gridDim.x * PART_NT;
    for (i64 base = blockIdx.x * (i64)PART_NT + threadIdx.x - lane; base < n; base += stride) {
        i64 i = base + lane;
        long long b = -1;
        u64 k = 0, p = 0;
        if (i < n) {
            k = ld_stream(keys + i);
            p = ld_stream(pay + i);
            b = bn.of_pos(bn.pos(lv, k));
        }
        unsigned peers = __match_any_sync(0xffffffffu, b);
        int leader = __ffs(peers) - 1;
        unsigned long long at = 0;
        if (b >= 0 && lane == leader) at = atomicAdd(cursor + b, (unsigned long long)__popc(peers));
        at = __shfl_sync(0xffffffffu, at, leader);
        if (b >= 0) out[at + __popc(peers & ((1u << lane) - 1u))] = make_ulonglong2(k, p);
    }
}

struct CastI64 {
    __host__ __device__ __forceinline__ i64 operator()(const u32 &v) const { return (i64)v; }
};

// ----------------------------------------------------------------- sort

struct SortCtl {
    unsigned long long next;   // work counter over buckets
    unsigned long long n_over; // buckets larger than CAP
    unsigned long long n_med;  // runs of RUN_SMALL < len <= CAP
    unsigned long long n_huge; // non-constant runs > CAP
    unsigned long long next_run;
};

// first predicted position of fine bucket b: ceil(b*n / nbins)
__device__ __forceinline__ i64 pos_lo_of(i64 b, i64 n, i64 nbins) { return (b * n + nbins - 1) / nbins; }

__device__ __forceinline__ void insertion_sort_idx(u16 *idx, int len, const ulonglong2 *A) {
    for (int i = 1; i < len; ++i) {
        u16 v = idx[i];
        u64 kv = A[v].x;
        int j = i - 1;
        while (j >= 0 && A[idx[j]].x > kv) {
            idx[j + 1] = idx[j];
            --j;
        }
        idx[j + 1] = v;
    }
}

// Block-wide exclusive scan of cnt[0..nb) into st[] (and cu[] = st[]).
__device__ __forceinline__ void block_exclusive_scan(const u32 *cnt, u32 *st, u32 *cu, int nb, u32 *warp_tot) {
    const int per = (nb + SORT_NT - 1) / SORT_NT;
    const int j0 = threadIdx.x * per;
    u32 local = 0;
    for (int j = j0; j < j0 + per && j < nb; ++j) local += cnt[j];
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
        u32 t = lane < SORT_NT / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        if (lane < SORT_NT / 32) warp_tot[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    u32 run = (warp ? warp_tot[warp - 1] : 0) + incl - local;
    for (int j = j0; j < j0 + per && j < nb; ++j) {
        st[j] = run;
        cu[j] = run;
        run += cnt[j];
    }
    __syncthreads();
}

// K8: one CTA per fine bucket (dynamic work counter).  Model-placed
// counting sort in shared memory, then fix-up of equal-position runs.
__global__ void __launch_bounds__(SORT_NT, 2) k_sort_buckets(Bin bn, ulonglong2 *pairs, const i64 *starts,
                                                             SortCtl *ctl, i64 *over_list, i64 *med_list) {
    extern __shared__ __align__(16) unsigned char smem[];
    ulonglong2 *A = reinterpret_cast<ulonglong2 *>(smem);
    u16 *rel = reinterpret_cast<u16 *>(A + CAP);
    u16 *idx = rel + CAP;
    u32 *cnt = reinterpret_cast<u32 *>(idx + CAP);
    u32 *st = cnt + NBMAX;
    u32 *cu = st + NBMAX;
    __shared__ u32 warp_tot[SORT_NT / 32];
    __shared__ i64 s_b;
    const i64 n = bn.m.n, nbins = bn.nbins;
    for (;;) {
        if (threadIdx.x == 0) s_b = (i64)atomicAdd(&ctl->next, 1ULL);
        __syncthreads();
        const i64 b = s_b;
        __syncthreads();
        if (b >= nbins) break;
        const i64 a = starts[b], m = starts[b + 1] - a;
        if (m <= 1) continue;
        const i64 plo = pos_lo_of(b, n, nbins);
        const int nb = (int)(pos_lo_of(b + 1, n, nbins) - plo);
        if (m > CAP || nb > NBMAX || nb < 1) {
            if (threadIdx.x == 0) over_list[atomicAdd(&ctl->n_over, 1ULL)] = b;
            continue;
        }
        for (int j = threadIdx.x; j < nb; j += SORT_NT) cnt[j] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += SORT_NT) {
            ulonglong2 v = pairs[a + i];
            A[i] = v;
            i64 r = bn.pos(bn.m.leaves, v.x) - plo;
            r = r < 0 ? 0 : (r >= nb ? nb - 1 : r);
            rel[i] = (u16)r;
            atomicAdd(cnt + r, 1u);
        }
        __syncthreads();
        block_exclusive_scan(cnt, st, cu, nb, warp_tot);
        for (int i = threadIdx.x; i < m; i += SORT_NT) idx[atomicAdd(cu + rel[i], 1u)] = (u16)i;
        __syncthreads();
        for (int j = threadIdx.x; j < nb; j += SORT_NT) {
            int len = (int)cnt[j];
            if (len < 2) continue;
            if (len <= RUN_SMALL) {
                insertion_sort_idx(idx + st[j], len, A);
            } else {
                unsigned long long q = atomicAdd(&ctl->n_med, 1ULL);
                med_list[2 * q] = a + st[j];
                med_list[2 * q + 1] = len;
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += SORT_NT) pairs[a + i] = A[idx[i]];
        __syncthreads();
    }
}

// Bitonic sort (by key) of runs RUN_SMALL < len <= CAP listed as
// (start, len) pairs, one CTA per run, padded with the sentinel key.
__global__ void __launch_bounds__(SORT_NT) k_sort_runs(ulonglong2 *pairs, const i64 *list, SortCtl *ctl) {
    extern __shared__ __align__(16) unsigned char smem[];
    ulonglong2 *A = reinterpret_cast<ulonglong2 *>(smem);
    __shared__ i64 s_r;
    const unsigned long long nruns = ctl->n_med;
    for (;;) {
        if (threadIdx.x == 0) s_r = (i64)atomicAdd(&ctl->next_run, 1ULL);
        __syncthreads();
        const i64 r = s_r;
        __syncthreads();
        if ((unsigned long long)r >= nruns) break;
        const i64 a = list[2 * r];
        const int len = (int)list[2 * r + 1];
        int w = 1;
        while (w < len) w <<= 1;
        for (int i = threadIdx.x; i < w; i += SORT_NT)
            A[i] = i < len ? pairs[a + i] : make_ulonglong2(~0ULL, 0ULL);
        __syncthreads();
        for (int k = 2; k <= w; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < w; i += SORT_NT) {
                    int l = i ^ j;
                    if (l > i) {
                        ulonglong2 x = A[i], y = A[l];
                        bool up = (i & k) == 0;
                        if ((x.x > y.x) == up) {
                            A[i] = y;
                            A[l] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int i = threadIdx.x; i < len; i += SORT_NT) pairs[a + i] = A[i];
        __syncthreads();
    }
}

// ------------------------------------------- oversized buckets (global)
//
// Flattened over the oversized buckets: element t belongs to oversized
// bucket k with ooff[k] <= t < ooff[k+1]; its bin is k*NBMAX + (pos - plo).

__device__ __forceinline__ int find_seg(const i64 *off, int nseg, i64 t) {
    int lo = 0, hi = nseg;  // last k with off[k] <= t
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (off[mid] <= t) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void k_over_hist(Bin bn, const ulonglong2 *pairs, const i64 *obkt, const i64 *obeg, const i64 *ooff,
                            int nseg, i64 total, u32 *hist, unsigned long long *bmin, unsigned long long *bmax) {
    const int lane = threadIdx.x & 31;
    const i64 stride = (i64)gridDim.x * blockDim.x;
    for (i64 base = blockIdx.x * (i64)blockDim.x + threadIdx.x - lane; base < total; base += stride) {
        i64 t = base + lane;
        long long bin = -1;
        u64 k = 0;
        if (t < total) {
            int s = find_seg(ooff, nseg, t);
            k = pairs[obeg[s] + (t - ooff[s])].x;
            i64 plo = pos_lo_of(obkt[s], bn.m.n, bn.nbins);
            i64 r = bn.pos(bn.m.leaves, k) - plo;
            r = r < 0 ? 0 : (r >= NBMAX ? NBMAX - 1 : r);
            bin = (long long)s * NBMAX + r;
        }
        unsigned peers = __match_any_sync(0xffffffffu, bin);
        int leader = __ffs(peers) - 1;
        u64 lk = __shfl_sync(0xffffffffu, k, leader);
        if (bin >= 0) {
            if (lane == leader) atomicAdd(hist + bin, (u32)__popc(peers));
            if (lane == leader || k != lk) {
                atomicMin(bmin + bin, (unsigned long long)k);
                atomicMax(bmax + bin, (unsigned long long)k);
            }
        }
    }
}

__global__ void k_over_scatter(Bin bn, const ulonglong2 *pairs, const i64 *obkt, const i64 *obeg, const i64 *ooff,
                               int nseg, i64 total, unsigned long long *cursor, ulonglong2 *tmp) {
    const int lane = threadIdx.x & 31;
    const i64 stride = (i64)gridDim.x * blockDim.x;
    for (i64 base = blockIdx.x * (i64)blockDim.x + threadIdx.x - lane; base < total; base += stride) {
        i64 t = base + lane;
        long long bin = -1;
        ulonglong2 v = make_ulonglong2(0, 0);
        if (t < total) {
            int s = find_seg(ooff, nseg, t);
            v = pairs[obeg[s] + (t - ooff[s])];
            i64 plo = pos_lo_of(obkt[s], bn.m.n, bn.nbins);
            i64 r = bn.pos(bn.m.leaves, v.x) - plo;
            r = r < 0 ? 0 : (r >= NBMAX ? NBMAX - 1 : r);
            bin = (long long)s * NBMAX + r;
        }
        unsigned peers = __match_any_sync(0xffffffffu, bin);
        int leader = __ffs(peers) - 1;
        unsigned long long at = 0;
        if (bin >= 0 && lane == leader) at = atomicAdd(cursor + bin, (unsigned long long)__popc(peers));
        at = __shfl_sync(0xffffffffu, at, leader);
        if (bin >= 0) tmp[at + __popc(peers & ((1u << lane) - 1u))] = v;
    }
}

__global__ void k_over_copyback(const ulonglong2 *tmp, const i64 *obeg, const i64 *ooff, int nseg, i64 total,
                                ulonglong2 *pairs) {
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < total; t += (i64)gridDim.x * blockDim.x) {
        int s = find_seg(ooff, nseg, t);
        pairs[obeg[s] + (t - ooff[s])] = tmp[t];
    }
}

// runs of equal predicted position inside oversized buckets
__global__ void k_over_runs(ulonglong2 *pairs, const i64 *obeg, const i64 *ooff, const i64 *bst, i64 nbin_total,
                            const unsigned long long *bmin, const unsigned long long *bmax, SortCtl *ctl,
                            i64 *med_list, i64 *huge_list) {
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < nbin_total; j += (i64)gridDim.x * blockDim.x) {
        i64 len = bst[j + 1] - bst[j];
        if (len < 2 || bmin[j] == bmax[j]) continue;  // empty, single or one repeated key
        int s = (int)(j / NBMAX);
        i64 a = obeg[s] + (bst[j] - ooff[s]);
        if (len <= RUN_SMALL) {
            for (i64 i = 1; i < len; ++i) {  // insertion sort in place (global)
                ulonglong2 v = pairs[a + i];
                i64 q = i - 1;
                while (q >= 0 && pairs[a + q].x > v.x) {
                    pairs[a + q + 1] = pairs[a + q];
                    --q;
                }
                pairs[a + q + 1] = v;
            }
        } else if (len <= CAP) {
            unsigned long long q = atomicAdd(&ctl->n_med, 1ULL);
            med_list[2 * q] = a;
            med_list[2 * q + 1] = len;
        } else {
            unsigned long long q = atomicAdd(&ctl->n_huge, 1ULL);
            huge_list[2 * q] = a;
            huge_list[2 * q + 1] = len;
        }
    }
}

__global__ void k_deinterleave(const ulonglong2 *p, i64 n, u64 *k, u64 *v) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        ulonglong2 e = p[i];
        k[i] = e.x;
        v[i] = e.y;
    }
}

__global__ void k_interleave(const u64 *k, const u64 *v, i64 n, ulonglong2 *p) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        p[i] = make_ulonglong2(k[i], v[i]);
}

// ----------------------------------------------------------------- join

// K9: per S tile, the R window [starts_r[f], starts_r[l+1]) of the tile's
// first/last key through R's model (lsj.py:343-367); staged in shared
// memory when it fits; lower-bound + equal-run scan per S tuple.
// mode 0: checksum into out[4]; 1: per-S match counts; 2: emit pairs.
__global__ void __launch_bounds__(JOIN_NT) k_lsj_join(Bin br, const ulonglong2 *__restrict__ R, i64 nr,
                                                      const i64 *__restrict__ rst, const ulonglong2 *__restrict__ S,
                                                      i64 ns, int mode, i64 *counts, const i64 *offsets, u64 *opr,
                                                      u64 *ops, u64 *out) {
    __shared__ u64 wk[WCAP];
    u64 cnt = 0, sum = 0, x = 0;
    const i64 ntiles = (ns + JOIN_T - 1) / JOIN_T;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 a = tile * JOIN_T, e = min(a + (i64)JOIN_T, ns);
        const u64 kf = S[a].x, kl = S[e - 1].x;
        const i64 f = br.of_pos(br.pos(br.m.leaves, kf)), l = br.of_pos(br.pos(br.m.leaves, kl));
        const i64 wlo = rst[f], whi = rst[l + 1], w = whi - wlo;
        const bool staged = w <= WCAP;
        if (staged)
            for (i64 j = threadIdx.x; j < w; j += JOIN_NT) wk[j] = R[wlo + j].x;
        __syncthreads();
        for (i64 i = a + threadIdx.x; i < e; i += JOIN_NT) {
            ulonglong2 sv = S[i];
            i64 lo, hi;
            if (staged) {
                lo = 0;
                hi = w;
                while (lo < hi) {
                    i64 mid = (lo + hi) >> 1;
                    if (wk[mid] < sv.x) lo = mid + 1; else hi = mid;
                }
                lo += wlo;
            } else {
                lo = wlo;
                hi = whi;
                while (lo < hi) {
                    i64 mid = (lo + hi) >> 1;
                    if (R[mid].x < sv.x) lo = mid + 1; else hi = mid;
                }
            }
            i64 c = 0;
            i64 o = mode == 2 ? offsets[i] : 0;
            for (i64 j = lo; j < whi; ++j) {
                ulonglong2 rv = R[j];
                if (rv.x != sv.x) break;
                if (mode == 0) {
                    u64 v = rv.y + sv.y;
                    ++cnt;
                    sum += v;
                    x ^= v;
                } else if (mode == 2) {
                    opr[o] = rv.y;
                    ops[o] = sv.y;
                    ++o;
                }
                ++c;
            }
            if (mode == 1) counts[i] = c;
        }
        __syncthreads();
    }
    if (mode == 0) reduce_checksum(cnt, sum, x, 0, out);
}

// ----------------------------------------------------------------- sample

// Stratified sample without replacement: one position per stratum
// [j*n/total, (j+1)*n/total), offset by a counter draw (results-neutral;
// the reference draws with numpy's Generator.choice, lsj.py:119-120).
__global__ void k_sample(const u64 *keys, i64 n, i64 total, u64 seed, u64 *out) {
    for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < total; j += (i64)gridDim.x * blockDim.x) {
        i64 lo = (i64)(((unsigned __int128)j * (u64)n) / (u64)total);
        i64 hi = (i64)(((unsigned __int128)(j + 1) * (u64)n) / (u64)total);
        i64 w = hi > lo ? hi - lo : 1;
        i64 p = lo + (i64)__umul64hi(mix64(seed ^ (u64)j), (u64)w);
        out[j] = keys[p < n ? p : n - 1];
    }
}

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

static Bin make_bin(const LjRmi &m, i64 nbins) {
    Bin b;
    b.m = RmiDev(m);
    b.nbins = nbins;
    b.rn = 1.0 / (double)m.n;
    return b;
}

static size_t scan_bytes(i64 nitems) {
    size_t t = 0;
    cub::TransformInputIterator<i64, CastI64, const u32 *> it(nullptr, CastI64());
    cub::DeviceScan::ExclusiveSum(nullptr, t, it, (i64 *)nullptr, (int64_t)nitems);
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
    LJ_REQUIRE(n >= 1 && total >= 1 && total <= n, "need 1 <= total <= n");
    if (ws_bytes < lj_lsj_sample_workspace_bytes(total)) {
        set_error("lj_lsj_sample: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    u64 *tmp = (u64 *)ws;
    char *cub_tmp = (char *)ws + al(sizeof(u64) * (size_t)total);
    size_t t = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t, (const u64 *)tmp, sample_sorted, (int64_t)total);
    k_sample<<<grid_for(total, 256, 8), 256, 0, st>>>(keys, n, total, seed, tmp);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceRadixSort::SortKeys(cub_tmp, t, (const u64 *)tmp, sample_sorted, (int64_t)total, 0, 64, st));
    return LJ_OK;
}

size_t lj_lsj_partition_workspace_bytes(int64_t n, int64_t nbins) {
    (void)n;
    return al(sizeof(u32) * (size_t)(nbins + 1)) + al(scan_bytes(nbins + 1));
}

int lj_lsj_partition(const LjRmi *model, const uint64_t *keys, const uint64_t *pay, int64_t n, int64_t nbins,
                     uint64_t *pairs, int64_t *starts, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n >= 1, "model is not fitted");
    LJ_REQUIRE(n >= 0 && nbins >= 1, "need n >= 0 and nbins >= 1");
    LJ_REQUIRE(n < (int64_t)0xFFFFFFFFLL, "per-bucket counters are 32-bit");
    if (ws_bytes < lj_lsj_partition_workspace_bytes(n, nbins)) {
        set_error("lj_lsj_partition: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    u32 *hist = (u32 *)ws;
    char *cub_tmp = (char *)ws + al(sizeof(u32) * (size_t)(nbins + 1));
    LJ_CK(cudaMemsetAsync(hist, 0, sizeof(u32) * (size_t)(nbins + 1), st));
    Bin bn = make_bin(*model, nbins);
    int stage = model->m <= 2048;
    size_t sm = stage ? sizeof(LjLeaf) * (size_t)model->m : 0;
    if (n > 0) {
        k_part_hist<<<grid_for(n, PART_NT, 8), PART_NT, sm, st>>>(bn, keys, n, hist, stage);
        LJ_CK_LAUNCH();
    }
    size_t t = scan_bytes(nbins + 1);
    cub::TransformInputIterator<i64, CastI64, const u32 *> it(hist, CastI64());
    LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, t, it, starts, (int64_t)(nbins + 1), st));
    if (n > 0) {
        // the exclusive starts double as the scatter cursors (rebuilt below)
        k_part_scatter<<<grid_for(n, PART_NT, 8), PART_NT, sm, st>>>(
            bn, keys, pay, n, reinterpret_cast<unsigned long long *>(starts), reinterpret_cast<ulonglong2 *>(pairs),
            stage);
        LJ_CK_LAUNCH();
        // starts[b] now holds the end of bucket b == start of b+1: rescan
        LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, t, it, starts, (int64_t)(nbins + 1), st));
    }
    return LJ_OK;
}

static void sort_ws_parts(void *ws, i64 n, SortCtl **ctl, i64 **over, i64 **med) {
    char *p = (char *)ws;
    *ctl = (SortCtl *)p;
    p += al(sizeof(SortCtl));
    *over = (i64 *)p;
    p += al(sizeof(i64) * (size_t)(n / CAP + 2));
    *med = (i64 *)p;
}

size_t lj_lsj_sort_workspace_bytes(int64_t n, int64_t nbins) {
    (void)nbins;
    return al(sizeof(SortCtl)) + al(sizeof(i64) * (size_t)(n / CAP + 2)) +
           al(sizeof(i64) * 2 * (size_t)(n / (RUN_SMALL + 1) + 2));
}

int lj_lsj_sort_buckets(const LjRmi *model, uint64_t *pairs, int64_t n, int64_t nbins, const int64_t *starts,
                        void *ws, size_t ws_bytes, int64_t *stats_host, void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && model->n >= 1, "model is not fitted");
    if (ws_bytes < lj_lsj_sort_workspace_bytes(n, nbins)) {
        set_error("lj_lsj_sort_buckets: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    SortCtl *ctl;
    i64 *over, *med;
    sort_ws_parts(ws, n, &ctl, &over, &med);
    LJ_CK(cudaMemsetAsync(ctl, 0, sizeof(SortCtl), st));
    if (n >= 2) {
        size_t sm = sizeof(ulonglong2) * CAP + 2 * sizeof(u16) * CAP + 3 * sizeof(u32) * NBMAX;
        static bool attr = false;
        if (!attr) {
            LJ_CK(cudaFuncSetAttribute(k_sort_buckets, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            LJ_CK(cudaFuncSetAttribute(k_sort_runs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(ulonglong2) * CAP)));
            attr = true;
        }
        unsigned g = (unsigned)(sm_count() * 2);
        k_sort_buckets<<<g, SORT_NT, sm, st>>>(make_bin(*model, nbins), reinterpret_cast<ulonglong2 *>(pairs),
                                                starts, ctl, over, med);
        LJ_CK_LAUNCH();
    }
    SortCtl h;
    LJ_CK(cudaMemcpyAsync(&h, ctl, sizeof(SortCtl), cudaMemcpyDeviceToHost, st));
    LJ_CK(cudaStreamSynchronize(st));
    stats_host[0] = (int64_t)h.n_over;
    stats_host[1] = (int64_t)h.n_med;
    return LJ_OK;
}

int lj_lsj_oversized_list_host(void *sort_ws, int64_t n, int64_t count, int64_t *buckets_host) {
    SortCtl *ctl;
    i64 *over, *med;
    sort_ws_parts(sort_ws, n, &ctl, &over, &med);
    LJ_CK(cudaMemcpy(buckets_host, over, sizeof(i64) * (size_t)count, cudaMemcpyDeviceToHost));
    return LJ_OK;
}

size_t lj_lsj_sort_oversized_workspace_bytes(int64_t nseg, int64_t total) {
    i64 nbin = nseg * NBMAX;
    size_t t = scan_bytes(nbin + 1), r = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, r, (const u64 *)nullptr, (u64 *)nullptr, (const u64 *)nullptr,
                                    (u64 *)nullptr, (int64_t)total);
    return al(sizeof(i64) * 3 * (size_t)(nseg + 1)) + al(sizeof(u32) * (size_t)(nbin + 1)) +
           al(sizeof(i64) * (size_t)(nbin + 1)) + 2 * al(sizeof(u64) * (size_t)(nbin + 1)) +
           al(sizeof(ulonglong2) * (size_t)total) + 4 * al(sizeof(u64) * (size_t)total) + al(t > r ? t : r) +
           al(sizeof(i64) * 2 * (size_t)(total / CAP + 2));
}

// Model placement of the buckets that did not fit in shared memory, through
// global memory: histogram of predicted positions (with per-position key
// min/max), scan, scatter, copy back; then the equal-position runs are fixed
// (insertion sort; medium runs join the bitonic list; runs of one repeated
// key are left alone; longer mixed runs -- rare -- are radix sorted here).
// seg_*_host: bucket id and [begin, end) of each oversized bucket.
int lj_lsj_sort_oversized(const LjRmi *model, uint64_t *pairs, int64_t n, int64_t nbins,
                          const int64_t *seg_bucket_host, const int64_t *seg_begin_host,
                          const int64_t *seg_end_host, int64_t nseg, void *sort_ws, void *ws, size_t ws_bytes,
                          int64_t *stats_host, void *stream) {
    LJ_REQUIRE(model && model->m >= 1 && nseg >= 1, "no oversized buckets");
    cudaStream_t st = as_stream(stream);
    std::vector<i64> hb(3 * (size_t)(nseg + 1));
    i64 total = 0;
    for (i64 s = 0; s < nseg; ++s) {
        hb[s] = seg_bucket_host[s];
        hb[(nseg + 1) + s] = seg_begin_host[s];
        hb[2 * (nseg + 1) + s] = total;
        total += seg_end_host[s] - seg_begin_host[s];
    }
    hb[2 * (nseg + 1) + nseg] = total;
    if (ws_bytes < lj_lsj_sort_oversized_workspace_bytes(nseg, total)) {
        set_error("lj_lsj_sort_oversized: workspace too small");
        return LJ_E_WORKSPACE;
    }
    const i64 nbin = nseg * NBMAX;
    char *p = (char *)ws;
    i64 *dseg = (i64 *)p;
    p += al(sizeof(i64) * 3 * (size_t)(nseg + 1));
    u32 *hist = (u32 *)p;
    p += al(sizeof(u32) * (size_t)(nbin + 1));
    i64 *bst = (i64 *)p;
    p += al(sizeof(i64) * (size_t)(nbin + 1));
    unsigned long long *bmin = (unsigned long long *)p;
    p += al(sizeof(u64) * (size_t)(nbin + 1));
    unsigned long long *bmax = (unsigned long long *)p;
    p += al(sizeof(u64) * (size_t)(nbin + 1));
    ulonglong2 *tmp = (ulonglong2 *)p;
    p += al(sizeof(ulonglong2) * (size_t)total);
    u64 *k1 = (u64 *)p;
    p += al(sizeof(u64) * (size_t)total);
    u64 *v1 = (u64 *)p;
    p += al(sizeof(u64) * (size_t)total);
    u64 *k2 = (u64 *)p;
    p += al(sizeof(u64) * (size_t)total);
    u64 *v2 = (u64 *)p;
    p += al(sizeof(u64) * (size_t)total);
    char *cub_tmp = p;
    size_t t = scan_bytes(nbin + 1), rsz = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, rsz, (const u64 *)nullptr, (u64 *)nullptr, (const u64 *)nullptr,
                                    (u64 *)nullptr, (int64_t)total);
    p += al(t > rsz ? t : rsz);
    i64 *huge = (i64 *)p;
    LJ_CK(cudaMemcpyAsync(dseg, hb.data(), sizeof(i64) * hb.size(), cudaMemcpyHostToDevice, st));
    const i64 *obkt = dseg, *obeg = dseg + (nseg + 1), *ooff = dseg + 2 * (nseg + 1);
    LJ_CK(cudaMemsetAsync(hist, 0, sizeof(u32) * (size_t)(nbin + 1), st));
    LJ_CK(cudaMemsetAsync(bmin, 0xFF, sizeof(u64) * (size_t)(nbin + 1), st));
    LJ_CK(cudaMemsetAsync(bmax, 0, sizeof(u64) * (size_t)(nbin + 1), st));
    Bin bn = make_bin(*model, nbins);
    ulonglong2 *pp = reinterpret_cast<ulonglong2 *>(pairs);
    k_over_hist<<<grid_for(total, 256, 8), 256, 0, st>>>(bn, pp, obkt, obeg, ooff, (int)nseg, total, hist, bmin,
                                                          bmax);
    LJ_CK_LAUNCH();
    cub::TransformInputIterator<i64, CastI64, const u32 *> it(hist, CastI64());
    LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, t, it, bst, (int64_t)(nbin + 1), st));
    // bst doubles as the scatter cursor, then is rebuilt by a second scan
    k_over_scatter<<<grid_for(total, 256, 8), 256, 0, st>>>(bn, pp, obkt, obeg, ooff, (int)nseg, total,
                                                             reinterpret_cast<unsigned long long *>(bst), tmp);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, t, it, bst, (int64_t)(nbin + 1), st));
    k_over_copyback<<<grid_for(total, 256, 8), 256, 0, st>>>(tmp, obeg, ooff, (int)nseg, total, pp);
    LJ_CK_LAUNCH();
    SortCtl *ctl;
    i64 *over, *med;
    sort_ws_parts(sort_ws, n, &ctl, &over, &med);
    k_over_runs<<<grid_for(nbin, 256, 8), 256, 0, st>>>(pp, obeg, ooff, bst, nbin, bmin, bmax, ctl, med, huge);
    LJ_CK_LAUNCH();
    SortCtl h;
    LJ_CK(cudaMemcpyAsync(&h, ctl, sizeof(SortCtl), cudaMemcpyDeviceToHost, st));
    LJ_CK(cudaStreamSynchronize(st));
    stats_host[0] = (int64_t)h.n_huge;
    stats_host[1] = (int64_t)h.n_med;
    if (h.n_huge) {
        std::vector<i64> hh(2 * (size_t)h.n_huge);
        LJ_CK(cudaMemcpy(hh.data(), huge, sizeof(i64) * hh.size(), cudaMemcpyDeviceToHost));
        for (unsigned long long r = 0; r < h.n_huge; ++r) {
            i64 a = hh[2 * r], len = hh[2 * r + 1];
            k_deinterleave<<<grid_for(len, 256, 8), 256, 0, st>>>(pp + a, len, k1, v1);
            size_t tt = rsz;
            LJ_CK(cub::DeviceRadixSort::SortPairs(cub_tmp, tt, k1, k2, v1, v2, (int64_t)len, 0, 64, st));
            k_interleave<<<grid_for(len, 256, 8), 256, 0, st>>>(k2, v2, len, pp + a);
            LJ_CK_LAUNCH();
        }
    }
    return LJ_OK;
}

// Bitonic pass over every medium run listed in the sort workspace.
int lj_lsj_sort_runs(uint64_t *pairs, int64_t n, void *sort_ws, void *stream) {
    SortCtl *ctl;
    i64 *over, *med;
    sort_ws_parts(sort_ws, n, &ctl, &over, &med);
    k_sort_runs<<<sm_count() * 2, SORT_NT, sizeof(ulonglong2) * CAP, as_stream(stream)>>>(
        reinterpret_cast<ulonglong2 *>(pairs), med, ctl);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_lsj_join(const LjRmi *model_r, const uint64_t *r_pairs, int64_t nr, int64_t r_nbins, const int64_t *r_starts,
                const uint64_t *s_pairs, int64_t ns, int mode, int64_t *counts, const int64_t *offsets,
                uint64_t *out_pr, uint64_t *out_ps, uint64_t *out, int accumulate, void *stream) {
    LJ_REQUIRE(model_r && model_r->m >= 1 && model_r->n >= 1, "R model is not fitted");
    LJ_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0, 1 or 2");
    cudaStream_t st = as_stream(stream);
    if (mode == 0 && !accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nr == 0 || ns == 0) {
        if (mode == 1 && ns > 0) LJ_CK(cudaMemsetAsync(counts, 0, sizeof(i64) * (size_t)ns, st));
        return LJ_OK;
    }
    i64 ntiles = (ns + JOIN_T - 1) / JOIN_T;
    unsigned g = (unsigned)(ntiles < (i64)sm_count() * 8 ? ntiles : (i64)sm_count() * 8);
    k_lsj_join<<<g, JOIN_NT, 0, st>>>(make_bin(*model_r, r_nbins), reinterpret_cast<const ulonglong2 *>(r_pairs), nr,
                                      r_starts, reinterpret_cast<const ulonglong2 *>(s_pairs), ns, mode, counts, offsets,
                                      out_pr, out_ps, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

}  // extern "C"
