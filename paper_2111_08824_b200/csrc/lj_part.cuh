// lj_part.cuh -- partition (key, payload) tuples into <= 32768 bins with
// shared-memory privatised counters: no per-tuple global atomics.
//
// Every block owns a fixed contiguous chunk of the input.  Pass 1 evaluates
// the bin function once per tuple, counts the chunk into a shared-memory
// histogram stored as one column of a bins x blocks matrix, and keeps the
// tuple's bin (u16); an exclusive scan of the matrix (bin-major) gives every
// block its private write offset per bin; pass 2 scatters the chunk by the
// stored bins.  Output is interleaved 16-B (key, payload) records, bins
// contiguous, order inside a bin unspecified.
//
// Measured design points (B200, profiles/, tools/micro/):
//  * one shared atomic per tuple (ATOMS: 5-7 tuples/clk/SM even with a
//    quarter of the keys in one bin); warp aggregation with match.any is
//    ~10x slower;
//  * hot bins: pass 1 spreads rows of 32 tuples over `hc` counter copies;
//  * both passes stream their chunk through a ring of shared-memory tiles
//    filled by cp.async.bulk (TMA 1-D) on an mbarrier per stage;
//  * pass 2 counting-sorts each 4096-tuple tile by bin in shared memory and
//    writes whole bin runs: scattering single records left ~300K partially
//    written segment frontiers in L2 and cost 1.4x the DRAM bytes.
#pragma once

#include <cub/cub.cuh>

#include "lj_common.cuh"
#include "lj_pipe.cuh"

namespace lj {

constexpr int PART2_NT = 1024;
constexpr int PART2_U = 4;  // tuple groups in flight per warp step (fallback kernels)
constexpr int PART2_MAXBINS = 32768;

struct PartPlan {
    int nbins;
    int blocks;
    int hc;     // histogram copies per block in pass 1
    i64 chunk;  // tuples per block (multiple of 32)
};

inline PartPlan part_plan(i64 n, int nbins) {
    PartPlan p;
    p.nbins = nbins;
    p.hc = 1;
    while (p.hc * 2 * nbins * 4 <= 64 * 1024 && p.hc < 8) p.hc *= 2;
    p.blocks = sm_count();  // one 1024-thread block per SM
    i64 c = (n + p.blocks - 1) / p.blocks;
    c = (c + 31) / 32 * 32;
    p.chunk = c < 32 ? 32 : c;
    return p;
}

// A tuple source over two key / payload columns.  BinF provides
// `u32 code(u64 key)` and `int shift` (bin = code >> shift), plus
// `smem_words()` / `stage(u64 *)` / `at(u64 *)`: a table of that many words
// the block copies into shared memory once and `code` then reads there.
struct NoTable {
    __host__ __device__ int smem_words() const { return 0; }
    __device__ void stage(u64 *) const {}
};
template <class BinF>
struct SoaSrc {
    static constexpr bool AOS = false;
    const u64 *__restrict__ keys;
    const u64 *__restrict__ pay;
    BinF f;
    __host__ bool aligned16() const {
        return ((uintptr_t)keys & 15) == 0 && ((uintptr_t)pay & 15) == 0;
    }
    __device__ __forceinline__ u32 code(u64 k) const { return f.code(k); }
    __device__ __forceinline__ const u64 *key_ptr(i64 i) const { return keys + i; }
    __device__ __forceinline__ const u64 *pay_ptr(i64 i) const { return pay + i; }
};

// The same relation as interleaved 16-B records {key, payload} (what the
// range shuffle of the distributed LSJ delivers): the claims scatter and its
// sample read them in place -- no conversion back to columns.
template <class BinF>
struct AosSrc {
    static constexpr bool AOS = true;
    const u64 *__restrict__ rec;
    BinF f;
    __host__ bool aligned16() const { return ((uintptr_t)rec & 15) == 0; }
    __device__ __forceinline__ u32 code(u64 k) const { return f.code(k); }
    __device__ __forceinline__ const u64 *key_ptr(i64 i) const { return rec + 2 * i; }
    __device__ __forceinline__ const u64 *pay_ptr(i64 i) const { return rec + 2 * i + 1; }
};

// histogram copies -> mat[bin * blocks + block]
__device__ __forceinline__ void hist_store(const u32 *h, int nbins, int hc, u32 *mat) {
    for (int j = threadIdx.x; j < nbins; j += PART2_NT) {
        u32 v = 0;
        for (int c = 0; c < hc; ++c) v += h[c * nbins + j];
        mat[(i64)j * gridDim.x + blockIdx.x] = v;
    }
}

// ---- fallback kernels (unaligned columns, > 2048 bins): plain loads

// shared-memory layout: [table words][counters ...], table first (8-B aligned)
__host__ __device__ inline size_t pt_table_bytes(int words) { return ((size_t)words * 8 + 127) & ~(size_t)127; }

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_hist(Src f0, i64 n, i64 chunk, int nbins, int hc, u32 *mat) {
    extern __shared__ __align__(128) unsigned char smem_h[];
    u64 *tab = reinterpret_cast<u64 *>(smem_h);
    u32 *h = reinterpret_cast<u32 *>(smem_h + pt_table_bytes(f0.f.smem_words()));
    f0.f.stage(tab);
    Src f = f0;
    f.f = f0.f.at(tab);
    for (int j = threadIdx.x; j < nbins * hc; j += PART2_NT) h[j] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, shift = f.f.shift;
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    for (i64 base = lo + (i64)warp * 32 * PART2_U; base < hi; base += (i64)PART2_NT * PART2_U) {
        int b[PART2_U];
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            const i64 i = base + u * 32 + lane;
            b[u] = i < hi ? (int)(f.code(ld_stream(f.keys + i)) >> shift) : -1;
        }
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            const int c = (int)(((base + u * 32 - lo) >> 5) % hc);
            if (b[u] >= 0) atomicAdd(h + c * nbins + b[u], 1u);
        }
    }
    __syncthreads();
    hist_store(h, nbins, hc, mat);
}

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_scatter(Src f0, i64 n, i64 chunk, int nbins,
                                                          const i64 *__restrict__ off, ulonglong2 *out) {
    extern __shared__ __align__(128) unsigned char smem_c[];
    u64 *tab = reinterpret_cast<u64 *>(smem_c);
    u32 *cur = reinterpret_cast<u32 *>(smem_c + pt_table_bytes(f0.f.smem_words()));
    f0.f.stage(tab);
    Src f = f0;
    f.f = f0.f.at(tab);
    for (int j = threadIdx.x; j < nbins; j += PART2_NT) cur[j] = (u32)off[(i64)j * gridDim.x + blockIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, shift = f.f.shift;
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    for (i64 base = lo + (i64)warp * 32 * PART2_U; base < hi; base += (i64)PART2_NT * PART2_U) {
        u32 c[PART2_U];
        u64 k[PART2_U], p[PART2_U];
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            const i64 i = base + u * 32 + lane;
            k[u] = i < hi ? ld_stream(f.keys + i) : 0;
            p[u] = i < hi ? ld_stream(f.pay + i) : 0;
            c[u] = i < hi ? f.code(k[u]) : 0;
        }
#pragma unroll
        for (int u = 0; u < PART2_U; ++u) {
            if (base + u * 32 + lane >= hi) continue;
            out[atomicAdd(cur + (c[u] >> shift), 1u)] = make_ulonglong2(k[u], p[u]);
        }
    }
}

// ---- bulk-copy pipelined kernels (16-B aligned columns)

constexpr int PT_TILE_H = PART2_NT * 4;  // keys per histogram tile (32 KB)
constexpr int PT_TILE_S = 4096;          // tuples per sorted scatter tile (longer bin runs beat deeper rings)
constexpr size_t PT_STAGE_H = sizeof(u64) * PT_TILE_H;
constexpr size_t PT_STAGE_S = (size_t)PT_TILE_S * (8 + 8 + 2);
constexpr int PT_MAXST = 6;
constexpr int PT_SMEM_MAX = 226 * 1024;  // + < 1 KB static, within the 227 KB opt-in

// Pass 1, warp-specialised: the last warp issues the bulk copies, the other
// 31 consume rows of 32 keys round-robin and release a stage on its `empty`
// barrier, so no warp ever waits for another at a block barrier (the bin
// function is a chain of dependent loads; a per-tile __syncthreads made
// every tile as slow as its slowest row).
constexpr int PT_H_CONS = PART2_NT / 32 - 1;

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_hist_tma(Src f0, i64 n, i64 chunk, int nbins, int hc, int nst,
                                                           u32 *mat, u16 *bins) {
    extern __shared__ __align__(128) unsigned char smem_t[];
    u64 *tab = reinterpret_cast<u64 *>(smem_t);
    unsigned char *smem = smem_t + pt_table_bytes(f0.f.smem_words());
    f0.f.stage(tab);
    Src f = f0;
    f.f = f0.f.at(tab);
    u32 *h = reinterpret_cast<u32 *>(smem);
    u64 *ring = reinterpret_cast<u64 *>(smem + ((nbins * hc * 4 + 127) & ~127));
    __shared__ __align__(8) uint64_t full[PT_MAXST], empty[PT_MAXST];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, shift = f.f.shift;
    for (int j = tid; j < nbins * hc; j += PART2_NT) h[j] = 0;
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    const int ntiles = hi > lo ? (int)((hi - lo + PT_TILE_H - 1) / PT_TILE_H) : 0;
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], PT_H_CONS);
        }
        mbar_init_fence();
    }
    __syncthreads();
    if (warp == PT_H_CONS) {  // producer
        if (lane == 0)
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % nst;
                if (t >= nst) mbar_wait(&empty[s], (unsigned)(t / nst - 1) & 1u);
                const i64 base = lo + (i64)t * PT_TILE_H;
                const unsigned b8 = (unsigned)(min((i64)PT_TILE_H, hi - base) * 8) & ~15u;
                if (b8) {
                    mbar_arrive_expect_tx(&full[s], b8);
                    bulk_g2s(ring + (size_t)s * PT_TILE_H, f.keys + base, b8, &full[s]);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
    } else {
        u32 *hw = h + (warp % hc) * nbins;  // this warp's histogram copy
        constexpr int U = 4;
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % nst;
            mbar_wait(&full[s], (unsigned)(t / nst) & 1u);
            const i64 base = lo + (i64)t * PT_TILE_H;
            const int cnt = (int)min((i64)PT_TILE_H, hi - base), nb = cnt & ~1;
            const u64 *ks = ring + (size_t)s * PT_TILE_H;
            for (int r0 = warp; r0 < PT_TILE_H / 32; r0 += U * PT_H_CONS) {
                u32 c[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = (r0 + u * PT_H_CONS) * 32 + lane;
                    c[u] = (j < cnt) ? f.code(j < nb ? ks[j] : ld_stream(f.keys + base + j)) : 0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = (r0 + u * PT_H_CONS) * 32 + lane;
                    if (j < cnt) {
                        const u32 b = c[u] >> shift;
                        atomicAdd(hw + b, 1u);
                        bins[base + j] = (u16)b;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    __syncthreads();
    hist_store(h, nbins, hc, mat);
}

template <class Src>
__global__ void __launch_bounds__(PART2_NT) k_bin_scatter_tma(Src f, const u16 *__restrict__ bins, i64 n, i64 chunk,
                                                              int nbins, int nst, const i64 *__restrict__ off,
                                                              ulonglong2 *out) {
    constexpr int U = PT_TILE_S / PART2_NT;
    extern __shared__ __align__(128) unsigned char smem[];
    const int nb4 = (nbins + 31) & ~31;
    u32 *cur = reinterpret_cast<u32 *>(smem);  // block's next free output position per bin
    u32 *thist = cur + nb4;                      // this tile's count per bin
    u32 *tstart = thist + nb4;                   // this tile's run start per bin
    u32 *gbase = tstart + nb4;                   // output position of the run
    u16 *perm = reinterpret_cast<u16 *>(gbase + nb4);
    unsigned char *ring = reinterpret_cast<unsigned char *>(perm) + ((PT_TILE_S * 2 + 127) & ~127);
    __shared__ __align__(8) uint64_t full[PT_MAXST];
    __shared__ u32 wsum[PART2_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < nbins; j += PART2_NT) {
        cur[j] = (u32)off[(i64)j * gridDim.x + blockIdx.x];
        thist[j] = 0;
    }
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    const int ntiles = hi > lo ? (int)((hi - lo + PT_TILE_S - 1) / PT_TILE_S) : 0;
    auto issue = [&](int t) {
        const int s = t % nst;
        const i64 base = lo + (i64)t * PT_TILE_S;
        const int cnt = (int)min((i64)PT_TILE_S, hi - base);
        const unsigned b8 = (unsigned)(cnt * 8) & ~15u, b2 = (unsigned)(cnt * 2) & ~15u;
        unsigned char *st = ring + (size_t)s * PT_STAGE_S;
        if (b8 + b2) {
            mbar_arrive_expect_tx(&full[s], 2 * b8 + b2);
            if (b8) {
                bulk_g2s(st, f.keys + base, b8, &full[s]);
                bulk_g2s(st + PT_TILE_S * 8, f.pay + base, b8, &full[s]);
            }
            if (b2) bulk_g2s(st + PT_TILE_S * 16, bins + base, b2, &full[s]);
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
    // Four barriers per tile (no barrier after the writes): the stage of
    // tile t-1 is refilled once every warp has passed the first barrier of
    // tile t.
    for (int t = 0; t < ntiles; ++t) {
        const int s = t % nst;
        mbar_wait(&full[s], (unsigned)(t / nst) & 1u);
        const i64 base = lo + (i64)t * PT_TILE_S;
        const int cnt = (int)min((i64)PT_TILE_S, hi - base), nb = cnt & ~1, nb8 = cnt & ~7;
        const unsigned char *st = ring + (size_t)s * PT_STAGE_S;
        const u64 *ks = reinterpret_cast<const u64 *>(st), *ps = ks + PT_TILE_S;
        const u16 *bs = reinterpret_cast<const u16 *>(st + PT_TILE_S * 16);
        // (1) rank of each tuple inside its bin's run of this tile
        int bj[U], rj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = u * PART2_NT + tid;
            bj[u] = j < cnt ? (int)(j < nb8 ? bs[j] : bins[base + j]) : -1;
            rj[u] = bj[u] >= 0 ? (int)atomicAdd(thist + bj[u], 1u) : 0;
        }
        __syncthreads();
        if (tid == 0 && t + nst - 1 < ntiles) issue(t + nst - 1);  // stage of tile t-1
        // (2) exclusive scan of the tile histogram (nbins <= 2 * PART2_NT)
        // -> run starts; reserve the runs in the block's segments
        {
            u32 v0 = 2 * tid < nbins ? thist[2 * tid] : 0, v1 = 2 * tid + 1 < nbins ? thist[2 * tid + 1] : 0;
            const u32 tot = v0 + v1;
            u32 inc = tot;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += y;
            }
            if (lane == 31) wsum[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                const u32 w = wsum[lane];
                u32 wi = w;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const u32 y = __shfl_up_sync(0xffffffffu, wi, d);
                    if (lane >= d) wi += y;
                }
                wsum[lane] = wi - w;
            }
            __syncthreads();
            const u32 r0 = wsum[warp] + inc - tot;
            if (2 * tid < nbins) {
                tstart[2 * tid] = r0;
                gbase[2 * tid] = cur[2 * tid];
                cur[2 * tid] += v0;
                thist[2 * tid] = 0;
            }
            if (2 * tid + 1 < nbins) {
                tstart[2 * tid + 1] = r0 + v0;
                gbase[2 * tid + 1] = cur[2 * tid + 1];
                cur[2 * tid + 1] += v1;
                thist[2 * tid + 1] = 0;
            }
        }
        __syncthreads();
        // (3) tile permutation sorted by bin
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (bj[u] >= 0) perm[tstart[bj[u]] + rj[u]] = (u16)(u * PART2_NT + tid);
        __syncthreads();
        // (4) write bin runs: consecutive threads -> consecutive addresses
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = u * PART2_NT + tid;
            if (i < cnt) {
                const int j = perm[i];
                const int b = j < nb8 ? bs[j] : bins[base + j];
                const u64 k = j < nb ? ks[j] : ld_stream(f.keys + base + j);
                const u64 p = j < nb ? ps[j] : ld_stream(f.pay + base + j);
                const u32 at = gbase[b] + (u32)i - tstart[b];
                out[at] = make_ulonglong2(k, p);
            }
        }
    }
}

inline size_t pt_scatter_fixed_bytes(int nbins) {
    const size_t nb4 = (size_t)((nbins + 31) & ~31);
    return 4 * nb4 * sizeof(u32) + (((size_t)PT_TILE_S * 2 + 127) & ~(size_t)127);
}

// bin starts[j] = off[j * blocks] (first block's offset), starts[nbins] = n
static __global__ void k_bin_starts(const i64 *off, int nbins, int blocks, i64 n, i64 *starts) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= nbins; j += gridDim.x * blockDim.x)
        starts[j] = j < nbins ? off[(i64)j * blocks] : n;
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
    i64 items = (i64)nbins * p.blocks;
    return part_align(sizeof(u32) * (size_t)items) + part_align(sizeof(i64) * (size_t)items) +
           part_align(sizeof(u16) * (size_t)n) + part_align(part_scan_bytes(items));
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
    if (f.f.shift < 0 || f.f.shift > 31) {
        set_error("partition: bad bin shift");
        return LJ_E_INVALID;
    }
    if (ws_bytes < part_workspace_bytes(n, nbins)) {
        set_error("partition: workspace too small");
        return LJ_E_WORKSPACE;
    }
    PartPlan p = part_plan(n, nbins);
    i64 items = (i64)nbins * p.blocks;
    char *q = (char *)ws;
    u32 *mat = (u32 *)q;
    q += part_align(sizeof(u32) * (size_t)items);
    i64 *off = (i64 *)q;
    q += part_align(sizeof(i64) * (size_t)items);
    u16 *bins = (u16 *)q;  // pass-1 bins for the pipelined pass 2
    q += part_align(sizeof(u16) * (size_t)n);
    const size_t sm_h = sizeof(u32) * (size_t)nbins * p.hc, sm_s = sizeof(u32) * (size_t)nbins;
    static unsigned long long attr_set = 0;  // one bit per device
    if (once_per_device(attr_set)) {
        LJ_CK(cudaFuncSetAttribute(k_bin_hist<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM_MAX));
        LJ_CK(cudaFuncSetAttribute(k_bin_scatter<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM_MAX));
        LJ_CK(cudaFuncSetAttribute(k_bin_hist_tma<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM_MAX));
        LJ_CK(cudaFuncSetAttribute(k_bin_scatter_tma<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM_MAX));
    }
    // bulk-copy rings: 16-B aligned columns, >= 2 stages next to the counters
    static const bool no_tma = getenv("LJ_PART_NO_TMA") != nullptr;
    const size_t tb = pt_table_bytes(f.f.smem_words());
    const size_t fix_h = tb + ((sm_h + 127) & ~(size_t)127), fix_s = pt_scatter_fixed_bytes(nbins);
    const int nst_h = fix_h < (size_t)PT_SMEM_MAX ? (int)min((size_t)PT_MAXST, (PT_SMEM_MAX - fix_h) / PT_STAGE_H) : 0;
    const int nst_s = fix_s < (size_t)PT_SMEM_MAX ? (int)min((size_t)PT_MAXST, (PT_SMEM_MAX - fix_s) / PT_STAGE_S) : 0;
    const bool tma = !no_tma && f.aligned16() && nst_h >= 2 && nst_s >= 2 && nbins <= 2 * PART2_NT;
    if (n > 0 && tma) {
        k_bin_hist_tma<Src><<<p.blocks, PART2_NT, fix_h + nst_h * PT_STAGE_H, st>>>(f, n, p.chunk, nbins, p.hc, nst_h,
                                                                                     mat, bins);
        LJ_CK_LAUNCH();
    } else if (n > 0) {
        k_bin_hist<Src><<<p.blocks, PART2_NT, tb + sm_h, st>>>(f, n, p.chunk, nbins, p.hc, mat);
        LJ_CK_LAUNCH();
    } else {
        LJ_CK(cudaMemsetAsync(mat, 0, sizeof(u32) * (size_t)items, st));
    }
    size_t t = part_scan_bytes(items);
    cub::TransformInputIterator<i64, CastU32I64, const u32 *> it(mat, CastU32I64());
    LJ_CK(cub::DeviceScan::ExclusiveSum(q, t, it, off, (int64_t)items, st));
    k_bin_starts<<<(nbins + 256) / 256, 256, 0, st>>>(off, nbins, p.blocks, n, starts);
    LJ_CK_LAUNCH();
    if (n > 0 && tma) {
        k_bin_scatter_tma<Src><<<p.blocks, PART2_NT, fix_s + nst_s * PT_STAGE_S, st>>>(f, bins, n, p.chunk, nbins,
                                                                                        nst_s, off, out);
        LJ_CK_LAUNCH();
    } else if (n > 0) {
        k_bin_scatter<Src><<<p.blocks, PART2_NT, tb + sm_s, st>>>(f, n, p.chunk, nbins, off, out);
        LJ_CK_LAUNCH();
    }
    return LJ_OK;
}

}  // namespace lj
