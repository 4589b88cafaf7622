// lj_spline.cu -- RadixSpline evaluation, the spline-keyed chained hash
// build and the fused probe (K5).  Reference: models.py:150-299,
// learned_hash.py:17-101.
//
// Layout in HBM: entries {key, payload} interleaved 16 B, grouped by
// bucket in insertion order (the reference's stable argsort,
// learned_hash.py:60); chain offsets `starts` in 32-bit words.  When the
// table length P is a multiple of n (the default table_factor 4.0 gives
// P = 4n), partition_index is exactly pos * (P/n) -- injective, with every
// non-multiple bucket empty -- so starts is indexed by pos and holds n+1
// words instead of P+1 (16 B/key smaller, results identical).
#include <cub/cub.cuh>

#include "lj_common.cuh"
#include "lj_keybin.cuh"
#include "lj_part.cuh"
#include "lj_part_est.cuh"

namespace lj {

// lj_hash_staged.cu
size_t hash_staged_meta_bytes(int nb);
int hash_windows(const LjSpline &model, const u64 *lay, int nb, u64 kmin, void *meta_ws, cudaStream_t st);
int hash_probe_staged(const LjSplineHash &idx, const ulonglong2 *rec, const i64 *reg, int nb, const void *meta_ws,
                      unsigned long long *ctr, u64 *out, cudaStream_t st);

struct HashDev {
    SplineDev model;
    i64 n, P, stride;
    const u64 *entries;
    const u32 *starts;
    bool direct;  // P == stride * trained_len: bucket / stride == pos, no division
    __host__ explicit HashDev(const LjSplineHash &h)
        : model(h.model), n(h.n), P(h.table_len), stride(h.stride), entries(h.entries), starts(h.starts),
          direct(h.model.n > 0 && h.table_len == h.stride * h.model.n) {}
    template <class L = LdNc>
    __device__ __forceinline__ i64 slot_of(u64 k, const L &ld = L()) const {
        // models.py:297 clip(pos*P // n, 0, P-1) / stride; pos is in [0, n)
        const i64 p = model.pos(k, ld);
        return direct ? p : scale_bucket(p, P, model.n) / stride;
    }
};

__global__ void k_spline_predict(SplineDev m, const u64 *keys, i64 nk, i64 *pos, i64 *lo, i64 *hi) {
    i64 last = m.n - 1;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nk; i += (i64)gridDim.x * blockDim.x) {
        i64 p = m.pos(keys[i]);
        if (pos) pos[i] = p;
        if (lo) lo[i] = clip_i64(p - m.max_error, 0, last);
        if (hi) hi[i] = clip_i64(p + m.max_error, 0, last);
    }
}

__global__ void k_spline_partition(SplineDev m, const u64 *keys, i64 nk, i64 P, i64 *out) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nk; i += (i64)gridDim.x * blockDim.x)
        out[i] = scale_bucket(m.pos(keys[i]), P, m.n);
}

// build: (bucket/stride, original index) pairs for a stable sort
__global__ void k_hash_bucket_of(SplineDev m, const u64 *keys, i64 n, i64 P, i64 stride, u64 *bk, u64 *idx) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        bk[i] = (u64)(scale_bucket(m.pos(keys[i]), P, m.n) / stride);
        idx[i] = (u64)i;
    }
}

__global__ void k_hash_gather(const u64 *order, const u64 *keys, const u64 *pay, i64 n, u64 *entries) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        u64 j = order[i];
        entries[2 * i] = keys[j];
        entries[2 * i + 1] = pay[j];
    }
}

// starts[b] = first sorted position with bucket >= b, for b in [0, nb]
__global__ void k_hash_starts(const u64 *sorted_b, i64 n, i64 nb, u32 *starts) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i <= n; i += (i64)gridDim.x * blockDim.x) {
        i64 prev = i == 0 ? -1 : (i64)sorted_b[i - 1];
        i64 cur = i == n ? nb : (i64)sorted_b[i];
        for (i64 b = prev + 1; b <= cur; ++b) starts[b] = (u32)i;
    }
}

// K5: learned_hash.py:81-96 fused with the checksum.  One lane per probe:
// spline position (radix table + bounded search over spline points, both
// L2-resident), bucket, chain offsets, chain scan.
// Each thread carries U independent probes through the same stages so their
// dependent load chains overlap (the chain is latency-bound: radix/aux ->
// sub-table -> spline points -> chain offsets -> entries).  Chain offsets
// and entries are random, touched once: they are read evict-first so they do
// not push the (L2-resident) spline structures out of L2.
struct HashSoa {
    const u64 *__restrict__ keys;
    const u64 *__restrict__ pay;
    __device__ __forceinline__ void get(i64 t, u64 &k, u64 &p) const {
        k = ld_stream(keys + t);
        p = ld_stream(pay + t);
    }
};
struct HashAos {  // records grouped by predicted position (lj_spline_hash_bucket)
    const ulonglong2 *__restrict__ rec;
    __device__ __forceinline__ void get(i64 t, u64 &k, u64 &p) const {
        const ulonglong2 e = __ldcs(rec + t);
        k = e.x;
        p = e.y;
    }
};

// GROUPED: the probes arrive grouped by predicted position, so consecutive
// probes reuse chain offsets and entries -> cached loads; otherwise they are
// touched once -> evict-first loads.
template <int NT, int U, class In, bool GROUPED>
__global__ void __launch_bounds__(NT) k_hash_probe(HashDev h, In in, i64 nk, u64 *out) {
    u64 cnt = 0, sum = 0, x = 0;
    const i64 stride = (i64)gridDim.x * NT;
    for (i64 t0 = blockIdx.x * (i64)NT + threadIdx.x; t0 < nk; t0 += stride * U) {
        u64 k[U], ps[U];
        i64 b[U];
        u32 a[U], e[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const i64 t = t0 + u * stride;
            k[u] = ps[u] = 0;
            if (t < nk) in.get(t, k[u], ps[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) b[u] = t0 + u * stride < nk ? h.slot_of(k[u]) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = b[u] >= 0 ? (GROUPED ? __ldg(h.starts + b[u]) : __ldcs(h.starts + b[u])) : 0;
            e[u] = b[u] >= 0 ? (GROUPED ? __ldg(h.starts + b[u] + 1) : __ldcs(h.starts + b[u] + 1)) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            for (u32 i = a[u]; i < e[u]; ++i) {
                const ulonglong2 *ep = reinterpret_cast<const ulonglong2 *>(h.entries) + i;
                ulonglong2 en = GROUPED ? __ldg(ep) : __ldcs(ep);
                if (en.x != k[u]) continue;
                u64 v = en.y + ps[u];
                ++cnt;
                sum += v;
                x ^= v;
            }
        }
    }
    reduce_checksum(cnt, sum, x, 0, out);
}

// Grouped probe with ordered dynamic dispatch: each CTA takes the next
// chunk of CH records from a global counter, so all SMs work on a sliding
// stretch of ~(CTAs x CH) records -- a few windows, whose chain offsets and
// entries stay in L2 (a grid-stride loop lets CTAs drift apart over
// thousands of iterations and spread the working set over the table).
// Records span [0, reg[nb] + reg[2 nb + 1]) (est regions + overflow); gap
// records carry the reserved key ~0 (never a build key) and are skipped.
template <int NT, int U, int R>
__global__ void __launch_bounds__(NT) k_hash_probe_chunks(HashDev h, const ulonglong2 *__restrict__ rec,
                                                          const i64 *reg, int nb, unsigned long long *ctr, u64 *out) {
    constexpr i64 CH = (i64)NT * U * R;
    __shared__ i64 s_c;
    u64 cnt = 0, sum = 0, x = 0;
    const LdKeep keep = LdKeep::make();
    const i64 nk = reg[nb] + reg[2 * nb + 1];
    for (;;) {
        if (threadIdx.x == 0) s_c = (i64)atomicAdd(ctr, 1ULL) * CH;
        __syncthreads();
        const i64 c0 = s_c;
        __syncthreads();
        if (c0 >= nk) break;
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
            const i64 t0 = c0 + (i64)r * NT * U + threadIdx.x;
            u64 k[U], ps[U];
            i64 b[U];
            u32 a[U], e[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const i64 t = t0 + u * NT;
                k[u] = ps[u] = 0;
                if (t < nk) {
                    const ulonglong2 v = __ldcs(rec + t);
                    k[u] = v.x;
                    ps[u] = v.y;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) b[u] = (t0 + u * NT < nk && k[u] != ~0ULL) ? h.slot_of(k[u], keep) : -1;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                a[u] = b[u] >= 0 ? __ldg(h.starts + b[u]) : 0;
                e[u] = b[u] >= 0 ? __ldg(h.starts + b[u] + 1) : 0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                for (u32 i = a[u]; i < e[u]; ++i) {
                    const ulonglong2 en = __ldg(reinterpret_cast<const ulonglong2 *>(h.entries) + i);
                    if (en.x != k[u]) continue;
                    const u64 v = en.y + ps[u];
                    ++cnt;
                    sum += v;
                    x ^= v;
                }
            }
        }
    }
    reduce_checksum(cnt, sum, x, 0, out);
}

__global__ void k_hash_count(HashDev h, const u64 *keys, i64 nk, i64 *counts) {
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < nk; t += (i64)gridDim.x * blockDim.x) {
        u64 k = keys[t];
        i64 b = h.slot_of(k);
        i64 c = 0;
        for (u32 i = h.starts[b]; i < h.starts[b + 1]; ++i) c += h.entries[2 * (i64)i] == k;
        counts[t] = c;
    }
}

__global__ void k_hash_collect(HashDev h, const u64 *keys, i64 nk, const i64 *offsets, u64 *out_pay,
                               i64 *out_src) {
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < nk; t += (i64)gridDim.x * blockDim.x) {
        u64 k = keys[t];
        i64 b = h.slot_of(k);
        i64 o = offsets[t];
        for (u32 i = h.starts[b]; i < h.starts[b + 1]; ++i) {
            if (h.entries[2 * (i64)i] != k) continue;
            out_pay[o] = h.entries[2 * (i64)i + 1];
            out_src[o] = t;
            ++o;
        }
    }
}

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

static int end_bit_for(u64 maxv) {
    int b = 0;
    while (b < 64 && (maxv >> b)) ++b;
    return b < 1 ? 1 : b;
}

}  // namespace lj

using namespace lj;

extern "C" {

int lj_spline_predict(const LjSpline *model, const uint64_t *keys, int64_t nk, int64_t *pos, int64_t *lo,
                      int64_t *hi, void *stream) {
    LJ_REQUIRE(model && model->npts >= 1 && model->n >= 1, "model is not fitted");
    if (nk <= 0) return LJ_OK;
    k_spline_predict<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(SplineDev(*model), keys, nk,
                                                                           pos, lo, hi);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_spline_partition_index(const LjSpline *model, const uint64_t *keys, int64_t nk, int64_t P,
                              int64_t *out, void *stream) {
    LJ_REQUIRE(model && model->npts >= 1 && model->n >= 1, "model is not fitted");
    LJ_REQUIRE(P >= 1, "num_partitions must be >= 1");
    if (nk <= 0) return LJ_OK;
    k_spline_partition<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(SplineDev(*model), keys, nk,
                                                                             P, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

size_t lj_spline_hash_build_workspace_bytes(int64_t n, int64_t P) {
    (void)P;
    size_t t = 0;
    cub::DeviceRadixSort::SortPairs((void *)nullptr, t, (const u64 *)nullptr, (u64 *)nullptr,
                                    (const u64 *)nullptr, (u64 *)nullptr, (int64_t)n, 0, 64);
    return 4 * al(sizeof(u64) * (size_t)n) + al(t);
}

int lj_spline_hash_build(const LjSpline *model, const uint64_t *keys, const uint64_t *pay, int64_t n,
                         int64_t P, uint64_t *entries, uint32_t *starts, void *ws, size_t ws_bytes,
                         void *stream) {
    LJ_REQUIRE(model && model->npts >= 1 && model->n >= 1, "model is not fitted");
    LJ_REQUIRE(n >= 1 && P >= 1, "need n >= 1 and P >= 1");
    LJ_REQUIRE(n < (int64_t)0xFFFFFFFFLL, "chain offsets are 32-bit: n must be < 2^32");
    if (ws_bytes < lj_spline_hash_build_workspace_bytes(n, P)) {
        set_error("lj_spline_hash_build: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    i64 stride = (P % n == 0) ? P / n : 1;
    i64 nb = P / stride;
    char *p = (char *)ws;
    u64 *bk = (u64 *)p; p += al(sizeof(u64) * (size_t)n);
    u64 *idx = (u64 *)p; p += al(sizeof(u64) * (size_t)n);
    u64 *bk2 = (u64 *)p; p += al(sizeof(u64) * (size_t)n);
    u64 *idx2 = (u64 *)p; p += al(sizeof(u64) * (size_t)n);
    k_hash_bucket_of<<<grid_for(n, 256, 8), 256, 0, st>>>(SplineDev(*model), keys, n, P, stride, bk, idx);
    LJ_CK_LAUNCH();
    int eb = end_bit_for((u64)nb);
    size_t t = 0;
    LJ_CK(cub::DeviceRadixSort::SortPairs((void *)nullptr, t, bk, bk2, idx, idx2, (int64_t)n, 0, eb, st));
    // radix sort is stable: chains keep insertion order (learned_hash.py:60)
    LJ_CK(cub::DeviceRadixSort::SortPairs(p, t, bk, bk2, idx, idx2, (int64_t)n, 0, eb, st));
    k_hash_gather<<<grid_for(n, 256, 8), 256, 0, st>>>(idx2, keys, pay, n, entries);
    k_hash_starts<<<grid_for(n + 1, 256, 8), 256, 0, st>>>(bk2, n, nb, starts);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_spline_hash_probe(const LjSplineHash *idx, const uint64_t *s_keys, const uint64_t *s_pay,
                         int64_t nk, uint64_t *out, int accumulate, void *stream) {
    LJ_REQUIRE(idx != nullptr, "null index");
    cudaStream_t st = as_stream(stream);
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nk <= 0 || idx->n == 0) return LJ_OK;
    constexpr int NT = 256;
    // 4 probes in flight per thread (measured: 125 ms vs 154 ms with 1 at C3)
    // (L2 evict_last on the spline + evict_first on the chains measured
    // 173 ms vs 118 ms at C3: plain loads)
    k_hash_probe<NT, 4, HashSoa, false><<<grid_for((nk + 3) / 4, NT, 8), NT, 0, st>>>(
        HashDev(*idx), HashSoa{s_keys, s_pay}, nk, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

// est-region gaps [rend[b], rstart[b+1]) get the reserved key ~0 (skipped
// by the probe)
__global__ void k_fill_gaps(const i64 *reg, int nb, ulonglong2 *out) {
    const int b = blockIdx.x;
    const i64 lo = reg[nb + 1 + b], hi = reg[b + 1];
    for (i64 i = lo + threadIdx.x; i < hi; i += blockDim.x) out[i] = make_ulonglong2(~0ULL, 0ULL);
}

// Request-Buffer analogue for the learned hash: group S by a window of
// APPROXIMATE position (<= 2048 windows): the rank of the first spline point
// of the key's (sub-)radix bucket -- two or three L2-resident loads, no
// search and no division.  Grouping only buys locality (the probe computes
// the exact bucket), and that rank is within one bucket's span of the
// key's position, so a window's chains stay in one small stretch of the
// table.  (The exact spline evaluation here cost 50 ms at C3.)
// PosBin with the last two loads folded into precomputed tables: the window
// of the first spline point of k's (sub-)radix bucket, per radix bucket
// (wrad) and per sub-table entry (wsub) -- the same bin for every key, one
// dependent load fewer (aux -> window instead of aux -> sub -> ranks).
struct WinBin : NoTable {
    const u64 *aux;
    const u16 *wrad, *wsub;
    u64 kshift;
    u64 rmax;
    int shift = 0;
    __device__ __forceinline__ u32 code(u64 k) const {
        const u64 raw = kshift >= 64 ? 0 : (k >> kshift);
        const u64 ax = (aux && raw <= rmax) ? ldg(aux + raw) : 0;
        if (ax & 0xFF) {
            const int bits = (int)(ax & 0xFF);
            const u64 q = (k >> (kshift - (u64)bits)) & ((1ULL << bits) - 1ULL);
            return __ldg(wsub + (ax >> 8) + q);
        }
        return __ldg(wrad + (raw > rmax ? rmax : raw));
    }
    __device__ __forceinline__ WinBin at(u64 *) const { return *this; }
};

__device__ __forceinline__ u16 win_of_point(const SplineDev &m, i64 lo, i64 nb, double rn) {
    lo = lo < 0 ? 0 : (lo > m.K - 1 ? m.K - 1 : lo);
    const i64 b = (i64)(__ldg(m.ranks + lo) * rn);
    return (u16)(b < 0 ? 0 : (b >= nb ? nb - 1 : b));
}

__global__ void k_win_tables(SplineDev m, i64 nb, double rn, u16 *wrad, i64 nrad, u16 *wsub, i64 nsub) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nrad + nsub; i += (i64)gridDim.x * blockDim.x) {
        if (i < nrad) wrad[i] = win_of_point(m, (i64)__ldg(m.radix + i), nb, rn);
        else wsub[i - nrad] = win_of_point(m, (i64)__ldg(m.sub + (i - nrad)), nb, rn);
    }
}

struct PosBin : NoTable {
    SplineDev m;
    i64 nb, n;
    double rn;
    int shift = 0;
    __device__ __forceinline__ u32 code(u64 k) const {
        const double r = __ldg(m.ranks + m.bucket_first_point(k));
        const i64 b = (i64)(r * rn);
        return (u32)(b < 0 ? 0 : (b >= nb ? nb - 1 : b));
    }
    __device__ __forceinline__ PosBin at(u64 *) const { return *this; }
};

static int hash_bins(i64 n) {
    const char *e = getenv("LJ_HASH_BINS");  // diagnostic: window count of the grouping
    const int want = e ? atoi(e) : 512;
    const int nb = want < 1 ? 1 : (want > 2048 ? 2048 : want);
    return (int)(n < nb ? (n < 1 ? 1 : n) : nb);
}

size_t lj_spline_hash_bucket_workspace_bytes(int64_t nk, int64_t n) {
    return part_workspace_bytes(nk, hash_bins(n)) + kb_bytes(hash_bins(n)) + 256;
}

// equi-depth key windows over the build side: B[j] = key of entry j*n/nb
// (entries are grouped by predicted position, monotone in the key; the
// layout build takes a running maximum)
__global__ void k_hash_window_bounds(const u64 *entries, i64 n, int nb, u64 *lay) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += gridDim.x * blockDim.x)
        lay[4 + j] = j ? entries[2 * (i64)(((unsigned __int128)j * (u64)n) / (u64)nb)] : 0;
}

int lj_spline_hash_bucket(const LjSplineHash *idx, const uint64_t *keys, const uint64_t *pay, int64_t nk,
                          uint64_t *pairs_out, int64_t *starts_out, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    LJ_REQUIRE(ws_bytes >= lj_spline_hash_bucket_workspace_bytes(nk, idx->n), "workspace too small");
    static const bool pos_bins = getenv("LJ_HASH_POS_BINS") != nullptr;
    if (!pos_bins) {
        // KEY windows, evaluated in shared memory (lj_keybin.cuh)
        const int nb = hash_bins(idx->n);
        const size_t pws = part_workspace_bytes(nk, nb);
        u64 *lay = reinterpret_cast<u64 *>(((uintptr_t)ws + pws + 255) & ~(uintptr_t)255);
        cudaStream_t st = as_stream(stream);
        k_hash_window_bounds<<<(nb + 255) / 256, 256, 0, st>>>(idx->entries, idx->n, nb, lay);
        k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
        LJ_CK_LAUNCH();
        KeyRangeBin kb;
        kb.g = lay;
        kb.nb = nb;
        SoaSrc<KeyRangeBin> src{keys, pay, kb};
        return run_partition_fast(src, nk, nb, reinterpret_cast<ulonglong2 *>(pairs_out), starts_out, ws, pws, st);
    }
    PosBin f;
    f.m = SplineDev(idx->model);
    f.nb = hash_bins(idx->model.n);
    f.n = idx->model.n;
    f.rn = (double)f.nb / (double)idx->model.n;
    SoaSrc<PosBin> src{keys, pay, f};
    return run_partition(src, nk, (int)f.nb, reinterpret_cast<ulonglong2 *>(pairs_out), starts_out, ws, ws_bytes,
                         as_stream(stream));
}

int lj_spline_hash_probe_grouped(const LjSplineHash *idx, const uint64_t *s_pairs, int64_t nk, uint64_t *out,
                                 int accumulate, void *stream) {
    LJ_REQUIRE(idx != nullptr, "null index");
    cudaStream_t st = as_stream(stream);
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (nk <= 0 || idx->n == 0) return LJ_OK;
    constexpr int NT = 256;
    k_hash_probe<NT, 4, HashAos, true><<<grid_for((nk + 3) / 4, NT, 8), NT, 0, st>>>(
        HashDev(*idx), HashAos{reinterpret_cast<const ulonglong2 *>(s_pairs)}, nk, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int64_t lj_spline_hash_bucket_bins(int64_t n) { return hash_bins(n); }

int64_t lj_spline_hash_bucket_capacity(int64_t nk, int64_t n) { return est_capacity(nk < 0 ? 0 : nk, hash_bins(n)); }

// window tables of the grouping (WinBin): u16 per radix bucket and per
// sub-table entry
static size_t win_tables_bytes(const LjSpline &m) {
    if (m.npts <= 1 || m.radix_bits > 24) return 0;
    return part_align(sizeof(u16) * ((size_t)1 << m.radix_bits)) + part_align(sizeof(u16) * (size_t)(m.nsub + 1));
}

size_t lj_spline_hash_bucket_est_workspace_bytes(const LjSplineHash *idx, int64_t nk) {
    if (!idx) return 0;
    const int nb = hash_bins(idx->model.n);
    return est_workspace_bytes(nb) + part_align(sizeof(u16) * (size_t)(nk < 0 ? 0 : nk)) + win_tables_bytes(idx->model) +
           kb_bytes(nb) + 256 + part_align(hash_staged_meta_bytes(nb)) + 256;
}

// exact regions in lj_leaf_bucket's layout: ends = next starts, no overflow
__global__ void k_exact_regions(int nb, i64 *reg) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
        if (b < nb) reg[nb + 1 + b] = reg[b + 1];
        else reg[2 * nb + 1] = 0;
    }
}

int lj_spline_hash_bucket_est(const LjSplineHash *idx, const uint64_t *keys, const uint64_t *pay, int64_t nk,
                              uint64_t *pairs_out, int64_t *reg_out, void *ws, size_t ws_bytes, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    LJ_REQUIRE(((uintptr_t)keys & 15) == 0 && ((uintptr_t)pay & 15) == 0, "key/payload columns must be 16-B aligned");
    cudaStream_t st = as_stream(stream);
    PosBin f;
    f.m = SplineDev(idx->model);
    f.nb = hash_bins(idx->model.n);
    f.n = idx->model.n;
    f.rn = (double)f.nb / (double)idx->model.n;
    SoaSrc<PosBin> src{keys, pay, f};
    static const bool keybin = getenv("LJ_HASH_KEYBIN") != nullptr;
    static const bool nostage = getenv("LJ_HASH_NOSTAGE") != nullptr;
    if (idx->slots && !nostage) {
        // the staged probe's grouping: equi-depth KEY windows over the build
        // side (lj_keybin.cuh, evaluated in shared memory) + every window's
        // staging metadata for k_hash_probe_staged
        const int nb = (int)f.nb;
        const size_t eb = est_workspace_bytes(nb);
        LJ_REQUIRE(ws_bytes >= eb + kb_bytes(nb) + 512 + hash_staged_meta_bytes(nb), "workspace too small");
        u64 *lay = reinterpret_cast<u64 *>(((uintptr_t)ws + eb + 255) & ~(uintptr_t)255);
        void *meta = reinterpret_cast<void *>(((uintptr_t)lay + kb_bytes(nb) + 255) & ~(uintptr_t)255);
        k_hash_window_bounds<<<(nb + 255) / 256, 256, 0, st>>>(idx->entries, idx->n, nb, lay);
        k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
        LJ_CK_LAUNCH();
        KeyRangeBin kb;
        kb.g = lay;
        kb.nb = nb;
        SoaSrc<KeyRangeBin> ksrc{keys, pay, kb};
        int rc = run_partition_est(ksrc, nk, nb, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out, ws, eb, st);
        if (rc) return rc;
        // (the staged probe reads only the filled part [reg[w], reg[nb + 1 + w]) of
        // every region: the gaps behind the fills need no reserved-key records)
        return hash_windows(idx->model, lay, nb, 0, meta, st);
    }
    if (keybin) {
        // equi-depth KEY windows over the build side, evaluated in shared
        // memory (lj_keybin.cuh): no per-tuple global load
        const int nb = (int)f.nb;
        const size_t eb = est_workspace_bytes(nb);
        LJ_REQUIRE(ws_bytes >= eb + kb_bytes(nb) + 256, "workspace too small");
        u64 *lay = reinterpret_cast<u64 *>(((uintptr_t)ws + eb + 255) & ~(uintptr_t)255);
        k_hash_window_bounds<<<(nb + 255) / 256, 256, 0, st>>>(idx->entries, idx->n, nb, lay);
        k_keybin_build<<<1, 1024, 0, st>>>(lay, nb);
        LJ_CK_LAUNCH();
        KeyRangeBin kb;
        kb.g = lay;
        kb.nb = nb;
        SoaSrc<KeyRangeBin> ksrc{keys, pay, kb};
        static const bool direct = getenv("LJ_HASH_DIRECT") != nullptr;
        const int rc = direct ? run_partition_direct(ksrc, nk, nb, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out,
                                                     ws, eb, st)
                              : run_partition_est(ksrc, nk, nb, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out,
                                                  ws, eb, st);
        if (rc) return rc;
        k_fill_gaps<<<(unsigned)nb, 256, 0, st>>>(reg_out, nb, reinterpret_cast<ulonglong2 *>(pairs_out));
        LJ_CK_LAUNCH();
        return LJ_OK;
    }
    const size_t wtb = win_tables_bytes(idx->model);
    static const bool no_win = getenv("LJ_HASH_POSBIN") != nullptr;
    if (!no_win && wtb && idx->model.aux && ws_bytes >= est_workspace_bytes((int)f.nb) + wtb) {
        // one pass with the window tables (last bytes of the workspace)
        const size_t nrad = (size_t)1 << idx->model.radix_bits;
        u16 *wrad = reinterpret_cast<u16 *>((char *)ws + ws_bytes - wtb);
        u16 *wsub = reinterpret_cast<u16 *>((char *)wrad + part_align(sizeof(u16) * nrad));
        k_win_tables<<<grid_for((i64)nrad + idx->model.nsub, 256, 4), 256, 0, st>>>(
            f.m, f.nb, f.rn, wrad, (i64)nrad, wsub, idx->model.nsub);
        LJ_CK_LAUNCH();
        WinBin wb;
        wb.aux = idx->model.aux;
        wb.wrad = wrad;
        wb.wsub = wsub;
        wb.kshift = idx->model.shift;
        wb.rmax = nrad - 1;
        SoaSrc<WinBin> wsrc{keys, pay, wb};
        static const bool direct = getenv("LJ_HASH_DIRECT") != nullptr;
        const int rc = direct ? run_partition_direct(wsrc, nk, (int)f.nb, reinterpret_cast<ulonglong2 *>(pairs_out),
                                                     reg_out, ws, ws_bytes - wtb, st)
                              : run_partition_est(wsrc, nk, (int)f.nb, reinterpret_cast<ulonglong2 *>(pairs_out),
                                                  reg_out, ws, ws_bytes - wtb, st);
        if (rc) return rc;
        k_fill_gaps<<<(unsigned)f.nb, 256, 0, st>>>(reg_out, (int)f.nb, reinterpret_cast<ulonglong2 *>(pairs_out));
        LJ_CK_LAUNCH();
        return LJ_OK;
    }
    // LJ_HASH_EXACT=1: a counting pass stores every probe's window (u16)
    // and the claims scatter streams them (no gaps, no overflow); measured
    // 42.4 ms vs 37.7 ms for the one-pass default at C3 (the counting pass
    // pays the spline-table loads once more)
    static const bool exact = getenv("LJ_HASH_EXACT") != nullptr;
    const size_t eb = est_workspace_bytes((int)f.nb);
    if (exact && ws_bytes >= eb + part_align(sizeof(u16) * (size_t)nk) && nk < (i64)0xFFFFFFFFLL) {
        const int rc = run_partition_claims(src, nk, (int)f.nb, 1, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out,
                                            ws, ws_bytes, st, reinterpret_cast<u16 *>((char *)ws + eb));
        if (rc) return rc;
        k_exact_regions<<<((int)f.nb + 256) / 256, 256, 0, st>>>((int)f.nb, reg_out);
        LJ_CK_LAUNCH();
        return LJ_OK;
    }
    const int rc = run_partition_est(src, nk, (int)f.nb, reinterpret_cast<ulonglong2 *>(pairs_out), reg_out, ws,
                                     ws_bytes, st);
    if (rc) return rc;
    k_fill_gaps<<<(unsigned)f.nb, 256, 0, st>>>(reg_out, (int)f.nb, reinterpret_cast<ulonglong2 *>(pairs_out));
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_spline_hash_probe_regions(const LjSplineHash *idx, const uint64_t *s_pairs, const int64_t *reg, int64_t nbins,
                                 void *ws, size_t ws_bytes, uint64_t *out, int accumulate, void *stream) {
    LJ_REQUIRE(idx != nullptr && reg != nullptr, "null index or regions");
    LJ_REQUIRE(ws != nullptr && ws_bytes >= 8, "workspace too small");
    cudaStream_t st = as_stream(stream);
    if (!accumulate) LJ_CK(cudaMemsetAsync(out, 0, 4 * sizeof(u64), st));
    if (idx->n == 0) return LJ_OK;
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(ws);
    LJ_CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    constexpr int NT = 256;
    // measured at C3 (ms): U=4 x 3 CTAs/SM 37.5, U=4 x 4 32.4, U=2 x 6 30.0, U=8 38.4
    static const int per_sm = getenv("LJ_HASH_CTAS") ? atoi(getenv("LJ_HASH_CTAS")) : 6;
    static const int u = getenv("LJ_HASH_U") ? atoi(getenv("LJ_HASH_U")) : 2;
    const ulonglong2 *rec = reinterpret_cast<const ulonglong2 *>(s_pairs);
    static const bool nostage = getenv("LJ_HASH_NOSTAGE") != nullptr;
    if (idx->slots && !nostage) {
        // k_hash_probe_staged over the windows lj_spline_hash_bucket_est
        // left (its staging metadata sits behind the key-range bin layout)
        const int nb = (int)nbins;
        const size_t eb = est_workspace_bytes(nb);
        LJ_REQUIRE(ws_bytes >= eb + kb_bytes(nb) + 512 + hash_staged_meta_bytes(nb), "workspace too small");
        const uintptr_t lay = ((uintptr_t)ws + eb + 255) & ~(uintptr_t)255;
        const void *meta = reinterpret_cast<const void *>((lay + kb_bytes(nb) + 255) & ~(uintptr_t)255);
        return hash_probe_staged(*idx, rec, reg, nb, meta, ctr, out, st);
    }
    const HashDev hd(*idx);
    if (u == 2)
        k_hash_probe_chunks<NT, 2, 16><<<sm_count() * per_sm, NT, 0, st>>>(hd, rec, reg, (int)nbins, ctr, out);
    else if (u == 8)
        k_hash_probe_chunks<NT, 8, 4><<<sm_count() * per_sm, NT, 0, st>>>(hd, rec, reg, (int)nbins, ctr, out);
    else
        k_hash_probe_chunks<NT, 4, 8><<<sm_count() * per_sm, NT, 0, st>>>(hd, rec, reg, (int)nbins, ctr, out);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_spline_hash_count(const LjSplineHash *idx, const uint64_t *keys, int64_t nk, int64_t *counts,
                         void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    if (nk <= 0) return LJ_OK;
    k_hash_count<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(HashDev(*idx), keys, nk, counts);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

int lj_spline_hash_collect(const LjSplineHash *idx, const uint64_t *keys, int64_t nk, const int64_t *offsets,
                           uint64_t *out_pay, int64_t *out_src, void *stream) {
    LJ_REQUIRE(idx && idx->n >= 1, "index is empty");
    if (nk <= 0) return LJ_OK;
    k_hash_collect<<<grid_for(nk, 256, 8), 256, 0, as_stream(stream)>>>(HashDev(*idx), keys, nk, offsets,
                                                                         out_pay, out_src);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

}  // extern "C"
