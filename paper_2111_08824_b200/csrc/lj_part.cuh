// lj_part.cuh -- partition (key, payload) tuples into <= 32768 bins with
// shared-memory privatised counters: no per-tuple global atomics.
//
// Global-atomic histograms over 10^5 random bins run at ~60 G atomics/s on
// B200 (measured, profiles/), far below HBM speed.  Here every block owns a
// fixed contiguous chunk of the input; pass 1 counts its chunk into a
// shared-memory histogram and stores it as one column of a bins x blocks
// matrix; an exclusive scan of the matrix (bin-major) gives every block its
// private write offset per bin; pass 2 recomputes the bins of the same
// chunk and scatters with shared-memory cursors.  Output is interleaved
// 16-B (key, payload) records; bins are contiguous; order inside a bin is
// unspecified.  Every tuple takes one shared-memory atomic (ATOMS, ~5-7 per
// clock per SM even with a quarter of the keys in one bin); warp-level
// aggregation with match.any measured ~10x slower (tools/micro/match_atoms).
#pragma once

#include <cub/cub.cuh>

#include "lj_common.cuh"
#include "lj_pipe.cuh"

namespace lj {

constexpr int PART2_NT = 1024;
constexpr int PART2_U = 4;  // tuple groups in flight per warp step
constexpr int PART2_MAXBINS = 32768;

struct PartPlan {
    int nbins;
    int blocks;
    int groups;  // cursor copies per block (rows of 32 tuples: copy = row % groups)
    int hc;      // histogram copies per block in pass 1 (multiple of groups)
    i64 chunk;   // tuples per block (multiple of 32)
};

// Hot bins (skewed keys: a quarter of C2's probes fall in one window) make
// every warp of a block hit the same shared-memory counter; spreading rows
// of 32 tuples over several counter copies divides that serialisation.
// Pass 2 keeps only `groups` cursor copies: each copy is its own output
// segment, and blocks x bins x groups open write lines must stay in L2.
inline PartPlan part_plan(i64 n, int nbins) {
    PartPlan p;
    p.nbins = nbins;
    p.groups = 1;
    p.hc = p.groups;
    while (p.hc * 2 * nbins * 4 <= 64 * 1024 && p.hc < 8) p.hc *= 2;
    // one block per SM: blocks x bins open write lines (148 x 2048 x 128 B
    // = 39 MB) stay inside L2, so records leave L2 as whole lines
    p.blocks = sm_count();
    i64 c = (n + p.blocks - 1) / p.blocks;
    c = (c + 31) / 32 * 32;
    p.chunk = c < 32 ? 32 : c;
    return p;
}

// A tuple source: bin_of(i) reads only what the bin needs; load(i, k, p)
// reads the tuple and returns its bin.
template <class BinF>
struct SoaSrc {
    const u64 *__restrict__ keys;
    const u64 *__restrict__ pay;
    BinF f;
    __host__ bool aligned16() const {
        return ((uintptr_t)keys & 15) == 0 && ((uintptr_t)pay & 15) == 0;
    }
    __device__ __forceinline__ void prepare() const { f.prepare(); }
    __device__ __forceinline__ int bin_of(i64 i) const { return f(ld_stream(keys + i)); }
    __device__ __forceinline__ int load(i64 i, u64 &k, u64 &p) const {
        k = ld_stream(keys + i);
        p = ld_stream(pay + i);
        return f(k);
    }
};

// pass 1: per-block histogram -> mat[bin * blocks + block]
// histogram copies -> mat[((bin * blocks + block) * groups + g], g = copy % groups
__device__ __forceinline__ void hist_store(const u32 *h, int nbins, int hc, int groups, u32 *mat) {
    for (int j = threadIdx.x; j < nbins; j += PART2_NT)
        for (int g = 0; g < groups; ++g) {
            u32 v = 0;
            for (int c = g; c < hc; c += groups) v += h[c * nbins + j];
            mat[((i64)j * gridDim.x + blockIdx.x) * groups + g] = v;
        }
}

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_hist(Src f, i64 n, i64 chunk, int nbins, int hc, int groups,
                                                       u32 *mat) {
    extern __shared__ u32 h[];
    for (int j = threadIdx.x; j < nbins * hc; j += PART2_NT) h[j] = 0;
    f.prepare();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    // each warp takes PART2_U groups of 32 consecutive tuples per step: the
    // U dependent chains (key -> model -> bin) overlap in flight
    for (i64 base = lo + (i64)warp * 32 * PART2_U; base < hi; base += (i64)PART2_NT * PART2_U) {
        int b[PART2_U];
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            const i64 i = base + u * 32 + lane;
            b[u] = i < hi ? f.bin_of(i) : -1;
        }
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            const int c = (int)(((base + u * 32 - lo) >> 5) % hc);
            if (b[u] >= 0) atomicAdd(h + c * nbins + b[u], 1u);
        }
    }
    __syncthreads();
    hist_store(h, nbins, hc, groups, mat);
}

// pass 2: scatter the same chunk through shared-memory cursors
__device__ __forceinline__ void cursor_load(u32 *cur, int nbins, int groups, const i64 *off) {
    for (int j = threadIdx.x; j < nbins; j += PART2_NT)
        for (int g = 0; g < groups; ++g) cur[g * nbins + j] = (u32)off[((i64)j * gridDim.x + blockIdx.x) * groups + g];
}

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_scatter(Src f, i64 n, i64 chunk, int nbins, int groups,
                                                          const i64 *__restrict__ off, ulonglong2 *out) {
    extern __shared__ u32 cur[];
    cursor_load(cur, nbins, groups, off);
    f.prepare();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    for (i64 base = lo + (i64)warp * 32 * PART2_U; base < hi; base += (i64)PART2_NT * PART2_U) {
        int b[PART2_U];
        u64 k[PART2_U], p[PART2_U];
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            const i64 i = base + u * 32 + lane;
            k[u] = p[u] = 0;
            b[u] = i < hi ? f.load(i, k[u], p[u]) : -1;
        }
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            const int g = (int)(((base + u * 32 - lo) >> 5) % groups);
            if (b[u] >= 0) out[atomicAdd(cur + g * nbins + b[u], 1u)] = make_ulonglong2(k[u], p[u]);
        }
    }
}


// ---- bulk-copy pipelined variants (SoA sources with 16-B aligned columns)
//
// Same chunks, same counts and the same scatter as above, but each CTA
// streams its chunk through a ring of `nst` shared-memory tiles filled by
// cp.async.bulk, so the key -> model -> bin chain never waits on HBM.

constexpr int PT_TILE_H = PART2_NT * 4;  // keys per histogram tile (32 KB)
constexpr int PT_TILE_S = PART2_NT * 2;  // records per scatter tile (32 KB)
constexpr int PT_MAXST = 6;

template <class Src>
__device__ __forceinline__ void pt_issue(const Src &f, bool with_pay, int tile_n, u64 *ring, uint64_t *bars, int nst,
                                         i64 lo, i64 hi, int t) {
    const int s = t % nst;
    const i64 base = lo + (i64)t * tile_n;
    const int cnt = (int)min((i64)tile_n, hi - base);
    const unsigned bytes = (unsigned)(cnt * 8) & ~15u;
    u64 *dst = ring + (size_t)s * tile_n * (with_pay ? 2 : 1);
    if (bytes) {
        mbar_arrive_expect_tx(&bars[s], with_pay ? 2 * bytes : bytes);
        bulk_g2s(dst, f.keys + base, bytes, &bars[s]);
        if (with_pay) bulk_g2s(dst + tile_n, f.pay + base, bytes, &bars[s]);
    } else {
        mbar_arrive(&bars[s]);
    }
}

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_hist_tma(Src f, i64 n, i64 chunk, int nbins, int hc, int groups,
                                                           int nst, u32 *mat, u16 *bins) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int U = PT_TILE_H / PART2_NT;
    u32 *h = reinterpret_cast<u32 *>(smem);
    u64 *ring = reinterpret_cast<u64 *>(smem + ((nbins * hc * 4 + 127) & ~127));
    __shared__ __align__(8) uint64_t bars[PT_MAXST];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < nbins * hc; j += PART2_NT) h[j] = 0;
    f.prepare();
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    const int ntiles = hi > lo ? (int)((hi - lo + PT_TILE_H - 1) / PT_TILE_H) : 0;
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) mbar_init(&bars[s], 1);
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
        for (int t = 0; t < min(nst - 1, ntiles); ++t) pt_issue(f, false, PT_TILE_H, ring, bars, nst, lo, hi, t);
    for (int t = 0; t < ntiles; ++t) {
        const int s = t % nst;
        if (tid == 0 && t + nst - 1 < ntiles) pt_issue(f, false, PT_TILE_H, ring, bars, nst, lo, hi, t + nst - 1);
        mbar_wait(&bars[s], (unsigned)(t / nst) & 1u);
        const i64 base = lo + (i64)t * PT_TILE_H;
        const int cnt = (int)min((i64)PT_TILE_H, hi - base), nb = cnt & ~1;
        const u64 *ks = ring + (size_t)s * PT_TILE_H;
        int b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = (warp * U + u) * 32 + lane;
            b[u] = j < cnt ? f.f(j < nb ? ks[j] : ld_stream(f.keys + base + j)) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = (t * (PT_TILE_H / 32) + warp * U + u) % hc;
            if (b[u] >= 0) {
                atomicAdd(h + c * nbins + b[u], 1u);
                bins[base + (warp * U + u) * 32 + lane] = (u16)b[u];
            }
        }
        __syncthreads();
    }
    __syncthreads();
    hist_store(h, nbins, hc, groups, mat);
}

// Pass 2 with the bins pass 1 stored (no model evaluation), tile-sorted.
// Scattering single 16-B records leaves ~300K partially written segment
// frontiers open in L2 at once; lines get evicted half-written and come
// back as read-modify-write traffic (profiles/: 1.4x DRAM bytes).  Here each
// tile of PT_TILE_S records is counting-sorted by bin in shared memory and
// written bin run by bin run, so every (block, bin) segment grows by whole
// runs of consecutive 16-B records per tile.
constexpr int PT_TILE_S2 = 4096;
constexpr size_t PT_STAGE_S = (size_t)PT_TILE_S2 * (8 + 8 + 2);
constexpr int PT_S2_U = PT_TILE_S2 / PART2_NT;

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_scatter_tma(Src f, const u16 *__restrict__ bins, i64 n, i64 chunk,
                                                              int nbins, int nst, const i64 *__restrict__ off,
                                                              ulonglong2 *out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int nb4 = (nbins + 31) & ~31;
    u32 *cur = reinterpret_cast<u32 *>(smem);  // block's next free output position per bin
    u32 *thist = cur + nb4;                      // this tile's count per bin
    u32 *tstart = thist + nb4;                   // this tile's run start per bin
    u32 *gbase = tstart + nb4;                   // global position of the run
    u16 *perm = reinterpret_cast<u16 *>(gbase + nb4);
    unsigned char *ring = reinterpret_cast<unsigned char *>(perm) + ((PT_TILE_S2 * 2 + 127) & ~127);
    __shared__ __align__(8) uint64_t full[PT_MAXST];
    __shared__ u32 wsum[PART2_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < nbins; j += PART2_NT) {
        cur[j] = (u32)off[(i64)j * gridDim.x + blockIdx.x];
        thist[j] = 0;
    }
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    const int ntiles = hi > lo ? (int)((hi - lo + PT_TILE_S2 - 1) / PT_TILE_S2) : 0;
    auto issue = [&](int t) {
        const int s = t % nst;
        const i64 base = lo + (i64)t * PT_TILE_S2;
        const int cnt = (int)min((i64)PT_TILE_S2, hi - base);
        const unsigned b8 = (unsigned)(cnt * 8) & ~15u, b2 = (unsigned)(cnt * 2) & ~15u;
        unsigned char *st = ring + (size_t)s * PT_STAGE_S;
        if (b8 + b2) {
            mbar_arrive_expect_tx(&full[s], 2 * b8 + b2);
            if (b8) {
                bulk_g2s(st, f.keys + base, b8, &full[s]);
                bulk_g2s(st + PT_TILE_S2 * 8, f.pay + base, b8, &full[s]);
            }
            if (b2) bulk_g2s(st + PT_TILE_S2 * 16, bins + base, b2, &full[s]);
        } else {
            mbar_arrive(&full[s]);
        }
    };
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
        mbar_init_fence();
        for (int t = 0; t < min(nst - 1, ntiles); ++t) issue(t);
    }
    __syncthreads();
    for (int t = 0; t < ntiles; ++t) {
        const int s = t % nst;
        if (tid == 0 && t + nst - 1 < ntiles) issue(t + nst - 1);  // stage consumed in round t-1
        mbar_wait(&full[s], (unsigned)(t / nst) & 1u);
        const i64 base = lo + (i64)t * PT_TILE_S2;
        const int cnt = (int)min((i64)PT_TILE_S2, hi - base), nb = cnt & ~1, nb2 = cnt & ~7;
        const unsigned char *st = ring + (size_t)s * PT_STAGE_S;
        const u64 *ks = reinterpret_cast<const u64 *>(st), *ps = ks + PT_TILE_S2;
        const u16 *bs = reinterpret_cast<const u16 *>(st + PT_TILE_S2 * 16);
        // (1) rank of each record inside its bin's run of this tile
        int bj[PT_S2_U], rj[PT_S2_U];
#pragma unroll
        for (int u = 0; u < PT_S2_U; ++u) {
            const int j = u * PART2_NT + tid;
            bj[u] = j < cnt ? (j < nb2 ? bs[j] : bins[base + j]) : -1;
            rj[u] = bj[u] >= 0 ? (int)atomicAdd(thist + bj[u], 1u) : 0;
        }
        __syncthreads();
        // (2) exclusive scan of the tile histogram -> run starts; reserve the
        // runs in the block's segments
        {
            constexpr int PER = 2;  // nbins <= PER * PART2_NT handled here
            u32 v[PER], tot = 0;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int j = tid * PER + q;
                v[q] = j < nbins ? thist[j] : 0;
                tot += v[q];
            }
            u32 inc = tot;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += y;
            }
            if (lane == 31) wsum[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                u32 w = wsum[lane], wi = w;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const u32 y = __shfl_up_sync(0xffffffffu, wi, d);
                    if (lane >= d) wi += y;
                }
                wsum[lane] = wi - w;
            }
            __syncthreads();
            u32 run = wsum[warp] + inc - tot;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int j = tid * PER + q;
                if (j < nbins) {
                    tstart[j] = run;
                    gbase[j] = cur[j];
                    cur[j] += v[q];
                    thist[j] = 0;
                }
                run += v[q];
            }
        }
        __syncthreads();
        // (3) tile permutation sorted by bin
#pragma unroll
        for (int u = 0; u < PT_S2_U; ++u)
            if (bj[u] >= 0) perm[tstart[bj[u]] + rj[u]] = (u16)(u * PART2_NT + tid);
        __syncthreads();
        // (4) write bin runs: consecutive threads -> consecutive addresses
#pragma unroll
        for (int u = 0; u < PT_S2_U; ++u) {
            const int i = u * PART2_NT + tid;
            if (i < cnt) {
                const int j = perm[i];
                const int b = j < nb2 ? bs[j] : bins[base + j];
                const u64 k = j < nb ? ks[j] : ld_stream(f.keys + base + j);
                const u64 p = j < nb ? ps[j] : ld_stream(f.pay + base + j);
                out[gbase[b] + (u32)i - tstart[b]] = make_ulonglong2(k, p);
            }
        }
        __syncthreads();
    }
}

inline size_t pt_scatter_fixed_bytes(int nbins) {
    const size_t nb4 = (size_t)((nbins + 31) & ~31);
    return 4 * nb4 * sizeof(u32) + (((size_t)PT_TILE_S2 * 2 + 127) & ~(size_t)127);
}

// bin starts[j] = off[j * cols] (first column's offset), starts[nbins] = n
static __global__ void k_bin_starts(const i64 *off, int nbins, int cols, i64 n, i64 *starts) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= nbins; j += gridDim.x * blockDim.x)
        starts[j] = j < nbins ? off[(i64)j * cols] : n;
}

struct CastU32I64 {
    __host__ __device__ __forceinline__ i64 operator()(const u32 &v) const { return (i64)v; }
};

inline size_t part_align(size_t v) { return (v + 255) & ~(size_t)255; }

inline size_t part_scan_bytes(i64 items) {
    size_t t = 0;
    cub::TransformInputIterator<i64, CastU32I64, const u32 *> it(nullptr, CastU32I64());
    cub::DeviceScan::ExclusiveSum(nullptr, t, it, (i64 *)nullptr, (int64_t)items);
    return t;
}

inline size_t part_workspace_bytes(i64 n, int nbins) {
    PartPlan p = part_plan(n, nbins);
    i64 items = (i64)nbins * p.blocks * p.groups;
    return part_align(sizeof(u32) * (size_t)items) + part_align(sizeof(i64) * (size_t)items) +
           part_align(part_scan_bytes(items)) + part_align(sizeof(u16) * (size_t)n);
}

// Full partition of the n tuples of `f`: out[n] records grouped by bin,
// starts[nbins+1].
template <class Src>
int run_partition(const Src &f, i64 n, int nbins, ulonglong2 *out, i64 *starts, void *ws, size_t ws_bytes,
                  cudaStream_t st) {
    if (nbins < 1 || nbins > PART2_MAXBINS) {
        set_error("partition: nbins must be in [1, 32768]");
        return LJ_E_INVALID;
    }
    if (n >= (i64)0xFFFFFFFFLL) {
        set_error("partition: cursors are 32-bit");
        return LJ_E_INVALID;
    }
    if (ws_bytes < part_workspace_bytes(n, nbins)) {
        set_error("partition: workspace too small");
        return LJ_E_WORKSPACE;
    }
    PartPlan p = part_plan(n, nbins);
    i64 items = (i64)nbins * p.blocks * p.groups;
    char *q = (char *)ws;
    u32 *mat = (u32 *)q;
    q += part_align(sizeof(u32) * (size_t)items);
    i64 *off = (i64 *)q;
    q += part_align(sizeof(i64) * (size_t)items);
    u16 *bins = (u16 *)q;  // pass-1 bins for the pipelined pass 2
    q += part_align(sizeof(u16) * (size_t)n);
    const size_t sm_h = sizeof(u32) * (size_t)nbins * p.hc, sm_s = sizeof(u32) * (size_t)nbins * p.groups;
    static bool attr_set = false;
    constexpr int kSmemMax = 220 * 1024;
    if (!attr_set) {
        LJ_CK(cudaFuncSetAttribute(k_bin_hist<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
        LJ_CK(cudaFuncSetAttribute(k_bin_scatter<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
        LJ_CK(cudaFuncSetAttribute(k_bin_hist_tma<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
        LJ_CK(cudaFuncSetAttribute(k_bin_scatter_tma<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
        attr_set = true;
    }
    // bulk-copy ring: 16-B aligned columns, >= 2 stages next to the counters
    static const bool no_tma = getenv("LJ_PART_NO_TMA") != nullptr;
    const size_t cnt_h = (sm_h + 127) & ~(size_t)127, cnt_s = pt_scatter_fixed_bytes(nbins);
    const size_t st_h = sizeof(u64) * PT_TILE_H, st_s = PT_STAGE_S;
    const int nst_h = cnt_h < (size_t)kSmemMax ? (int)min((size_t)PT_MAXST, (kSmemMax - cnt_h) / st_h) : 0;
    const int nst_s = cnt_s < (size_t)kSmemMax ? (int)min((size_t)PT_MAXST, (kSmemMax - cnt_s) / st_s) : 0;
    const bool tma = !no_tma && f.aligned16() && nst_h >= 2 && nst_s >= 2 && nbins <= 2 * PART2_NT && p.groups == 1;
    if (n > 0 && tma) {
        k_bin_hist_tma<Src><<<p.blocks, PART2_NT, cnt_h + nst_h * st_h, st>>>(f, n, p.chunk, nbins, p.hc, p.groups,
                                                                                nst_h, mat, bins);
        LJ_CK_LAUNCH();
    } else if (n > 0) {
        k_bin_hist<Src><<<p.blocks, PART2_NT, sm_h, st>>>(f, n, p.chunk, nbins, p.hc, p.groups, mat);
        LJ_CK_LAUNCH();
    } else {
        LJ_CK(cudaMemsetAsync(mat, 0, sizeof(u32) * (size_t)items, st));
    }
    size_t t = part_scan_bytes(items);
    cub::TransformInputIterator<i64, CastU32I64, const u32 *> it(mat, CastU32I64());
    LJ_CK(cub::DeviceScan::ExclusiveSum(q, t, it, off, (int64_t)items, st));
    k_bin_starts<<<(nbins + 256) / 256, 256, 0, st>>>(off, nbins, p.blocks * p.groups, n, starts);
    LJ_CK_LAUNCH();
    if (n > 0 && tma) {
        k_bin_scatter_tma<Src><<<p.blocks, PART2_NT, cnt_s + nst_s * st_s, st>>>(f, bins, n, p.chunk, nbins, nst_s,
                                                                                  off, out);
        LJ_CK_LAUNCH();
    } else if (n > 0) {
        k_bin_scatter<Src><<<p.blocks, PART2_NT, sm_s, st>>>(f, n, p.chunk, nbins, p.groups, off, out);
        LJ_CK_LAUNCH();
    }
    return LJ_OK;
}

}  // namespace lj
