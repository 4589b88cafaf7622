// lj_part_est.cuh -- ONE-pass partition into estimated-capacity regions.
//
// The exact two-pass partition (lj_part.cuh) reads the keys twice and
// evaluates the bin function in its own latency-bound pass.  When the
// consumer can live with (a) gaps after each bin and (b) a small unsorted
// overflow area, one pass suffices: a strided 1/EST_STRIDE sample of the
// keys estimates every bin's count, each bin gets a region of
// cap = est * (1 + 1/16) + EST_PAD records (exclusive scan -> rstart), and
// the pass streams the tuples (TMA ring), evaluates the bin, counting-sorts
// each tile by bin in shared memory and claims every bin run of the tile
// with ONE global atomic on the bin's cursor; a run that does not fit goes
// to the overflow area behind the regions.  Output layout (records):
//   [rstart[b], rend[b])  bin b, rend[b] = rstart[b] + min(fill, cap)
//   [rstart[nb], rstart[nb] + overflow)  records of any bin
// reg[] = {rstart[0..nb], rend[0..nb), overflow count}.
#pragma once

#include <cub/cub.cuh>

#include "lj_part.cuh"

namespace lj {

constexpr int EST_STRIDE = 16;
constexpr int EST_STRIDE_MAX = 64;
// The sample is every stride-th block of 32 tuples.  Above 2^30 tuples one
// block in 64 keeps >= 8192 sampled tuples per bin at 2048 bins (C4's count
// at 2^28 and stride 16), so the regions' 1/16 slack stays > 8 sigma of the
// estimate; C3's 2 * 10^9 probes: sample pass 0.57 -> 0.15 ms.
inline int est_stride(i64 n) { return n >= ((i64)1 << 30) ? EST_STRIDE_MAX : EST_STRIDE; }
constexpr i64 EST_PAD = 4096;
constexpr int EST_TILE = 4096;
constexpr size_t EST_STAGE = (size_t)EST_TILE * 16;

// shared memory of the claims scatter beside the bin table and the ring:
// tile histogram, run starts (u32), region starts, output deltas (i64),
// the tile permutation (u32)
inline size_t est_fix_bytes(size_t nb4) {
    return 2 * nb4 * sizeof(u32) + (nb4 + 32) * sizeof(i64) + nb4 * sizeof(i64) + (size_t)EST_TILE * 4;
}

// capacity of the output (records) for n tuples in nb bins: regions + overflow
// (the estimates sum to at most n + 32 * stride: the last sampled block; 17/16 of that + the per-bin pads)
inline i64 est_capacity_regions(i64 n, int nb) {
    return n + n / 16 + (i64)nb * (EST_PAD + EST_STRIDE_MAX + 1) + 34 * EST_STRIDE_MAX + 64;
}
inline i64 est_capacity(i64 n, int nb) { return est_capacity_regions(n, nb) + n; }
// ... est_capacity_regions: without the overflow area (run_partition_est_or_exact drops overflowing records)

// per-bin counts of every `stride`-th tuple (stride 1: the exact histogram)
template <class Src>
__global__ void __launch_bounds__(256) k_est_sample(Src f0, i64 n, int nbins, int stride, u32 *est, u16 *codes,
                                                    const unsigned long long *run_if = nullptr) {
    if (run_if && *run_if == 0) return;  // a fallback pass that is not needed
    extern __shared__ __align__(128) unsigned char smem_e[];
    u64 *tab = reinterpret_cast<u64 *>(smem_e);
    u32 *h = reinterpret_cast<u32 *>(smem_e + pt_table_bytes(f0.f.smem_words()));
    f0.f.stage(tab);
    Src f = f0;
    f.f = f0.f.at(tab);
    for (int j = threadIdx.x; j < nbins; j += blockDim.x) h[j] = 0;
    __syncthreads();
    const int shift = f.f.shift;
    // the sample is every stride-th block of 32 consecutive tuples (a warp
    // reads whole sectors; a strided single-key sample wasted 3/4 of every
    // 32-B sector it fetched); stride 1 visits every tuple
    const i64 lane = threadIdx.x & 31;
    const i64 ngrp = ((i64)gridDim.x * blockDim.x) >> 5, bs = 32 * (i64)stride;
    i64 blk = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    for (; (blk + 3 * ngrp) * bs < n; blk += 4 * ngrp) {  // four independent loads in flight
        u64 k[4];
        i64 i[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            i[u] = (blk + u * ngrp) * bs + lane;
            k[u] = i[u] < n ? ld_stream(f.key_ptr(i[u])) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i[u] >= n) continue;
            const u32 b = f.code(k[u]) >> shift;
            atomicAdd(h + b, 1u);
            if (codes) codes[i[u]] = (u16)b;  // stride 1 only
        }
    }
    for (; blk * bs < n; blk += ngrp) {
        const i64 i = blk * bs + lane;
        if (i >= n) continue;
        const u32 b = f.code(ld_stream(f.key_ptr(i))) >> shift;
        atomicAdd(h + b, 1u);
        if (codes) codes[i] = (u16)b;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nbins; j += blockDim.x)
        if (h[j]) atomicAdd(est + j, h[j]);
}

// region capacity per bin: the exact count, or the sample estimate with
// slack (est * 17/16 + pad)
static __global__ void k_est_caps(const u32 *est, int nbins, int exact, i64 *cap, int tight = 0,
                                  int stride = EST_STRIDE) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nbins; b += gridDim.x * blockDim.x) {
        if (b == nbins) {
            cap[b] = 0;
            continue;
        }
        if (exact) {
            cap[b] = (i64)est[b];
            continue;
        }
        const i64 e = (i64)est[b] * stride;
        cap[b] = tight ? e : e + e / 16 + EST_PAD + stride;  // tight (LJ_EST_TIGHT): tests force overflow
    }
}

// STORED: the bins were written by the exact counting pass (u16 per tuple)
// and arrive through the ring with the tuples (no bin evaluation, no table)
// PEER: regions are exact and rstart[b] is the ABSOLUTE record index (address
// / 16) of bin b's region -- possibly in another GPU's memory (NVLink P2P
// stores through a symmetric-memory pointer) -- so out is null and there
// is no overflow check.
template <class Src, bool STORED, bool PEER = false>
__global__ void __launch_bounds__(PART2_NT, 1) k_bin_scatter_est(Src f0, i64 n, i64 chunk, int nbins, int nst,
                                                              const i64 *__restrict__ rstart, u32 *gcur,
                                                              unsigned long long *ovf, ulonglong2 *out,
                                                              const u16 *__restrict__ codes,
                                                              const unsigned long long *run_if = nullptr,
                                                              int drop = 0) {
    if (run_if && *run_if == 0) return;  // a fallback pass that is not needed
    constexpr int U = EST_TILE / PART2_NT;
    constexpr size_t STAGE = EST_STAGE + (STORED ? EST_TILE * 2 : 0);
    extern __shared__ __align__(128) unsigned char smem_s[];
    u64 *tab = reinterpret_cast<u64 *>(smem_s);
    unsigned char *smem = smem_s + (STORED ? 0 : pt_table_bytes(f0.f.smem_words()));
    if (!STORED) f0.f.stage(tab);
    Src f = f0;
    if (!STORED) f.f = f0.f.at(tab);
    const int nb4 = (nbins + 31) & ~31;
    u32 *thist = reinterpret_cast<u32 *>(smem);  // this tile's count per bin
    u32 *tstart = thist + nb4;                   // this tile's run start per bin
    i64 *srst = reinterpret_cast<i64 *>(tstart + nb4);  // region starts [nbins + 1]
    // output position of the tile-sorted tuple i of bin b = dlt[b] + i
    // (region start + claimed position of the run - the run's start in the tile)
    i64 *dlt = srst + nb4 + 32;
    // tile permutation sorted by bin: tile index | bin << 16
    u32 *perm = reinterpret_cast<u32 *>(dlt + nb4);
    unsigned char *ring = reinterpret_cast<unsigned char *>(perm) + EST_TILE * 4;
    __shared__ __align__(8) uint64_t full[PT_MAXST];
    __shared__ u32 wsum[PART2_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, shift = f.f.shift;
    for (int j = tid; j < nbins; j += PART2_NT) thist[j] = 0;
    for (int j = tid; j <= nbins; j += PART2_NT) srst[j] = rstart[j];
    // The tiles cover [0, n_main): whole 16-B units of every column (chunks are
    // multiples of 32 tuples), so a tile never has a tail outside its ring
    // stage; the last n - n_main < 8 tuples are placed one by one by a single
    // thread below.
    // (interleaved records: every record is a 16-B unit of its own)
    constexpr bool AOS = Src::AOS;
    const i64 n_main = STORED ? (n & ~(i64)7) : (AOS ? n : (n & ~(i64)1));
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n_main);
    const int ntiles = hi > lo ? (int)((hi - lo + EST_TILE - 1) / EST_TILE) : 0;
    auto issue = [&](int t, int s) {
        const i64 base = lo + (i64)t * EST_TILE;
        const int cnt = (int)min((i64)EST_TILE, hi - base);
        const unsigned b8 = AOS ? (unsigned)(cnt * 8) : ((unsigned)(cnt * 8) & ~15u);
        const unsigned b2 = STORED ? ((unsigned)(cnt * 2) & ~15u) : 0u;
        unsigned char *st = ring + (size_t)s * STAGE;
        if (b8 + b2) {
            mbar_arrive_expect_tx(&full[s], 2 * b8 + b2);
            if (b8) {
                if constexpr (AOS) {
                    bulk_g2s(st, f.key_ptr(base), 2 * b8, &full[s]);
                } else {
                    bulk_g2s(st, f.key_ptr(base), b8, &full[s]);
                    bulk_g2s(st + EST_TILE * 8, f.pay_ptr(base), b8, &full[s]);
                }
            }
            if (b2) bulk_g2s(st + EST_TILE * 16, codes + base, b2, &full[s]);
        } else {
            mbar_arrive(&full[s]);
        }
    };
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
        mbar_init_fence();
        for (int t = 0; t < min(nst - 1, ntiles); ++t) issue(t, t);
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) {
        for (i64 i = n_main; i < n; ++i) {
            const u64 k = *f.key_ptr(i), p = *f.pay_ptr(i);
            const int b = STORED ? (int)codes[i] : (int)(f.code(k) >> shift);
            i64 dst = rstart[b] + (i64)atomicAdd(gcur + b, 1u);
            if (!PEER && !STORED && dst >= rstart[b + 1]) {
                const i64 q = (i64)atomicAdd(ovf, 1ULL);
                if (drop) continue;
                dst = rstart[nbins] + q;
            }
            ulonglong2 *o = PEER ? reinterpret_cast<ulonglong2 *>((uintptr_t)dst << 4) : out + dst;
            *o = make_ulonglong2(k, p);
        }
    }
    // Four barriers per tile.  The next tile's binning (1) may start while
    // slower warps still write this tile's runs (4): (1) writes only the
    // tile histogram, which (4) does not read.  The run claims (global
    // atomics) are issued before the scan and their results are used only
    // after it, so their latency overlaps the scan.
    int s = 0;           // ring stage of tile t
    unsigned phase = 0;  // its mbarrier phase
    int sn = nst - 1;    // stage refilled during tile t (tile t + nst - 1)
    for (int t = 0; t < ntiles; ++t) {
        mbar_wait(&full[s], phase);
        const i64 base = lo + (i64)t * EST_TILE;
        const int cnt = (int)min((i64)EST_TILE, hi - base);
        const unsigned char *st = ring + (size_t)s * STAGE;
        const u64 *ks = reinterpret_cast<const u64 *>(st), *ps = ks + EST_TILE;
        const u16 *cs = reinterpret_cast<const u16 *>(st + EST_TILE * 16);
        // (1) bin of every tuple and its rank in the tile's run
        int bj[U], rj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = u * PART2_NT + tid;
            if (STORED) bj[u] = j < cnt ? (int)cs[j] : -1;
            else bj[u] = j < cnt ? (int)(f.code(AOS ? ks[2 * j] : ks[j]) >> shift) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) rj[u] = bj[u] >= 0 ? (int)atomicAdd(thist + bj[u], 1u) : 0;
        __syncthreads();
        // every warp is past tile t-1's writes: its stage may be refilled
        if (tid == 0 && t + nst - 1 < ntiles) issue(t + nst - 1, sn);
        // (2) claim every run in its bin (one global atomic each), then the
        // exclusive scan of the tile histogram -> run starts
        const u32 v0 = 2 * tid < nbins ? thist[2 * tid] : 0, v1 = 2 * tid + 1 < nbins ? thist[2 * tid + 1] : 0;
        const u32 g0 = v0 ? atomicAdd(gcur + 2 * tid, v0) : 0;
        const u32 g1 = v1 ? atomicAdd(gcur + 2 * tid + 1, v1) : 0;
        u32 r0;
        {
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
            r0 = wsum[warp] + inc - tot;
            if (2 * tid < nbins) {
                tstart[2 * tid] = r0;
                thist[2 * tid] = 0;
            }
            if (2 * tid + 1 < nbins) {
                tstart[2 * tid + 1] = r0 + v0;
                thist[2 * tid + 1] = 0;
            }
        }
        __syncthreads();
        // (3) tile permutation sorted by bin; the claims land
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (bj[u] >= 0) perm[tstart[bj[u]] + rj[u]] = (u32)(u * PART2_NT + tid) | ((u32)bj[u] << 16);
        if (v0) dlt[2 * tid] = srst[2 * tid] + (i64)g0 - (i64)r0;
        if (v1) dlt[2 * tid + 1] = srst[2 * tid + 1] + (i64)g1 - (i64)(r0 + v0);
        __syncthreads();
        // (4) write bin runs into their regions (overflow behind the regions)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = u * PART2_NT + tid;
            if (i < cnt) {
                const u32 pj = perm[i];
                const int j = (int)(pj & 0xFFFFu), b = (int)(pj >> 16);
                u64 k, p;
                if constexpr (AOS) {
                    const ulonglong2 r = reinterpret_cast<const ulonglong2 *>(st)[j];
                    k = r.x;
                    p = r.y;
                } else {
                    k = ks[j];
                    p = ps[j];
                }
                i64 dst = dlt[b] + i;
                if (!PEER && !STORED && dst >= srst[b + 1]) {
                    // past the bin's region: the overflow area behind the regions
                    // -- or only counted (drop: the consumer redoes the partition
                    // exactly when the count is not zero, so the area need not exist)
                    const i64 q = (i64)atomicAdd(ovf, 1ULL);
                    if (drop) continue;
                    dst = srst[nbins] + q;
                }
                ulonglong2 *o = PEER ? reinterpret_cast<ulonglong2 *>((uintptr_t)dst << 4) : out + dst;
                *o = make_ulonglong2(k, p);
            }
        }
        if (++s == nst) {
            s = 0;
            phase ^= 1u;
        }
        if (++sn == nst) sn = 0;
    }
}

// Direct claims scatter: the same regions, claims and overflow as
// k_bin_scatter_est, without the in-tile permutation.  Each tuple keeps its
// (bin, rank in the tile's run) in registers; after one claim per (tile,
// bin) every thread stores its own tuples straight to base[bin] + rank.  A
// warp's stores scatter over ~32 runs, but every run is one contiguous
// piece of its bin's shared frontier, so L2 assembles whole lines before
// they are written back.  Per tuple: 2 sequential + 2 random shared-memory
// accesses (the permuting scatter needs ~11) and 2 barriers per tile.
// DT tuples per tile, DNT threads, 2 CTAs per SM (their barriers overlap).
constexpr int DNT = 512;
constexpr int DTILE = 2048;
template <class Src>
__global__ void __launch_bounds__(DNT, 2) k_scatter_direct(Src f0, i64 n, i64 chunk, int nbins, int nst,
                                                           const i64 *__restrict__ rstart, u32 *gcur,
                                                           unsigned long long *ovf, ulonglong2 *out) {
    constexpr int U = DTILE / DNT;
    constexpr size_t STAGE = (size_t)DTILE * 16;
    extern __shared__ __align__(128) unsigned char smem_d[];
    u64 *tab = reinterpret_cast<u64 *>(smem_d);
    unsigned char *smem = smem_d + pt_table_bytes(f0.f.smem_words());
    f0.f.stage(tab);
    Src f = f0;
    f.f = f0.f.at(tab);
    const int nb4 = (nbins + 31) & ~31;
    u32 *thist = reinterpret_cast<u32 *>(smem);                // this tile's count per bin
    i64 *base = reinterpret_cast<i64 *>(thist + nb4);          // this tile's run start per bin (records)
    i64 *lim = base + nb4;                                     // region end per bin
    unsigned char *ring = reinterpret_cast<unsigned char *>(lim + nb4);
    __shared__ __align__(8) uint64_t full[PT_MAXST];
    const int tid = threadIdx.x, shift = f.f.shift;
    for (int j = tid; j < nbins; j += DNT) {
        thist[j] = 0;
        lim[j] = rstart[j + 1];
    }
    const i64 ovf0 = rstart[nbins];
    const i64 lo = blockIdx.x * chunk, hi = min(lo + chunk, n);
    const int ntiles = hi > lo ? (int)((hi - lo + DTILE - 1) / DTILE) : 0;
    auto issue = [&](int t) {
        const int s = t % nst;
        const i64 b0 = lo + (i64)t * DTILE;
        const int cnt = (int)min((i64)DTILE, hi - b0);
        const unsigned b8 = (unsigned)(cnt * 8) & ~15u;
        unsigned char *st = ring + (size_t)s * STAGE;
        if (b8) {
            mbar_arrive_expect_tx(&full[s], 2 * b8);
            bulk_g2s(st, f.keys + b0, b8, &full[s]);
            bulk_g2s(st + DTILE * 8, f.pay + b0, b8, &full[s]);
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
        mbar_wait(&full[s], (unsigned)(t / nst) & 1u);
        const i64 b0 = lo + (i64)t * DTILE;
        const int cnt = (int)min((i64)DTILE, hi - b0), nb2 = cnt & ~1;
        const unsigned char *st = ring + (size_t)s * STAGE;
        const u64 *ks = reinterpret_cast<const u64 *>(st), *ps = ks + DTILE;
        // (1) bin + rank in the tile's run
        int bj[U];
        u32 rj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = u * DNT + tid;
            bj[u] = j < cnt ? (int)(f.code(j < nb2 ? ks[j] : ld_stream(f.keys + b0 + j)) >> shift) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) rj[u] = bj[u] >= 0 ? atomicAdd(thist + bj[u], 1u) : 0u;
        __syncthreads();
        // every thread is past tile t-1's stores: its stage may be refilled
        if (tid == 0 && t + nst - 1 < ntiles) issue(t + nst - 1);
        // (2) one claim per nonempty (tile, bin)
        for (int b = tid; b < nbins; b += DNT) {
            const u32 c = thist[b];
            if (c) {
                base[b] = rstart[b] + (i64)atomicAdd(gcur + b, c);
                thist[b] = 0;
            }
        }
        __syncthreads();
        // (3) every tuple to its run (overflow behind the regions)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (bj[u] < 0) continue;
            const int j = u * DNT + tid;
            const u64 k = j < nb2 ? ks[j] : ld_stream(f.keys + b0 + j);
            const u64 p = j < nb2 ? ps[j] : ld_stream(f.pay + b0 + j);
            i64 dst = base[bj[u]] + (i64)rj[u];
            if (dst >= lim[bj[u]]) dst = ovf0 + (i64)atomicAdd(ovf, 1ULL);
            out[dst] = make_ulonglong2(k, p);
        }
    }
}

static __global__ void k_est_regions(const i64 *rstart, const u32 *gcur, const unsigned long long *ovf, int nbins,
                              i64 *reg) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nbins; b += gridDim.x * blockDim.x) {
        reg[b] = rstart[b];
        if (b < nbins) reg[nbins + 1 + b] = rstart[b] + min((i64)gcur[b], rstart[b + 1] - rstart[b]);
        else reg[2 * nbins + 1] = (i64)*ovf;
    }
}

inline size_t est_workspace_bytes(int nbins) {  // (+ part_align(2 n) for stored bins)
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (i64 *)nullptr, (i64 *)nullptr, (int64_t)(nbins + 1));
    return part_align(sizeof(u32) * (size_t)nbins) * 2 + part_align(sizeof(i64) * (size_t)(nbins + 1)) * 2 +
           part_align(sizeof(unsigned long long)) + part_align(t);
}

// Partition of the n tuples of `f` into regions claimed run by run with
// one global atomic per (tile, bin), so the open write frontiers are one
// per bin, shared by all CTAs (per-CTA bin segments leave blocks x bins
// half-written lines in L2; measured +22 % DRAM writes and reads).
//   exact = 0: one pass; a 1/EST_STRIDE sample sizes the regions
//              (est_capacity records, gaps, overflow), reg as above.
//   exact = 1: an exact counting pass sizes them: out[n] grouped by bin,
//              contiguous, reg[0..nbins] = bin starts (no overflow).
template <class Src>
int run_partition_claims(const Src &f, i64 n, int nbins, int exact, ulonglong2 *out, i64 *reg, void *ws,
                         size_t ws_bytes, cudaStream_t st, u16 *codes = nullptr,
                         const unsigned long long *run_if = nullptr, int drop_overflow = 0) {
    if (nbins < 1 || nbins > 2 * PART2_NT) {
        set_error("partition_est: nbins must be in [1, 2048]");
        return LJ_E_INVALID;
    }
    if (ws_bytes < est_workspace_bytes(nbins)) {
        set_error("partition_est: workspace too small");
        return LJ_E_WORKSPACE;
    }
    char *q = (char *)ws;
    u32 *est = (u32 *)q;
    q += part_align(sizeof(u32) * (size_t)nbins);
    u32 *gcur = (u32 *)q;
    q += part_align(sizeof(u32) * (size_t)nbins);
    i64 *cap = (i64 *)q;
    q += part_align(sizeof(i64) * (size_t)(nbins + 1));
    i64 *rstart = exact ? reg : (i64 *)q;
    q += part_align(sizeof(i64) * (size_t)(nbins + 1));
    unsigned long long *ovf = (unsigned long long *)q;
    q += part_align(sizeof(unsigned long long));
    LJ_CK(cudaMemsetAsync(est, 0, sizeof(u32) * (size_t)nbins, st));
    LJ_CK(cudaMemsetAsync(gcur, 0, sizeof(u32) * (size_t)nbins, st));
    LJ_CK(cudaMemsetAsync(ovf, 0, sizeof(unsigned long long), st));
    const size_t tb = pt_table_bytes(f.f.smem_words());
    static unsigned long long attr = 0;  // one bit per device
    if (once_per_device(attr)) {
        LJ_CK(cudaFuncSetAttribute(k_bin_scatter_est<Src, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   PT_SMEM_MAX));
        LJ_CK(cudaFuncSetAttribute(k_bin_scatter_est<Src, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   PT_SMEM_MAX));
        LJ_CK(cudaFuncSetAttribute(k_est_sample<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM_MAX));
    }
    const int stride = exact ? 1 : est_stride(n);
    const bool stored = exact && codes != nullptr && nbins <= 65536;
    if (n > 0) {
        k_est_sample<Src><<<grid_for((n + stride - 1) / stride, 256, 4), 256, tb + sizeof(u32) * nbins, st>>>(
            f, n, nbins, stride, est, stored ? codes : nullptr, run_if);
        LJ_CK_LAUNCH();
    }
    k_est_caps<<<(nbins + 256) / 256, 256, 0, st>>>(est, nbins, exact, cap, getenv("LJ_EST_TIGHT") != nullptr, stride);
    LJ_CK_LAUNCH();
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, cap, rstart, (int64_t)(nbins + 1));
    LJ_CK(cub::DeviceScan::ExclusiveSum(q, t, cap, rstart, (int64_t)(nbins + 1), st));
    if (n > 0) {
        const PartPlan p = part_plan(n, nbins);
        const size_t nb4 = (size_t)((nbins + 31) & ~31);
        const size_t fix = (stored ? 0 : tb) + est_fix_bytes(nb4);
        const size_t stage = EST_STAGE + (stored ? EST_TILE * 2 : 0);
        const int nst = fix < (size_t)PT_SMEM_MAX ? (int)min((size_t)PT_MAXST, (PT_SMEM_MAX - fix) / stage) : 0;
        if (nst < 2) {
            set_error("partition_est: shared memory too small for the ring");
            return LJ_E_INVALID;
        }
        if (stored)
            k_bin_scatter_est<Src, true><<<p.blocks, PART2_NT, fix + nst * stage, st>>>(
                f, n, p.chunk, nbins, nst, rstart, gcur, ovf, out, codes, run_if);
        else
            k_bin_scatter_est<Src, false><<<p.blocks, PART2_NT, fix + nst * stage, st>>>(
                f, n, p.chunk, nbins, nst, rstart, gcur, ovf, out, nullptr, run_if, drop_overflow);
        LJ_CK_LAUNCH();
    }
    if (!exact) {
        k_est_regions<<<(nbins + 256) / 256, 256, 0, st>>>(rstart, gcur, ovf, nbins, reg);
        LJ_CK_LAUNCH();
    }
    return LJ_OK;
}

// ---- the range shuffle of the distributed LSJ, fused with its partition:
// (1) exact per-destination counts, every tuple's destination stored (u16);
// (2) the claims scatter with the destinations' region bases (absolute
// record indices) -- each source owns its region in every destination, so
// no cross-GPU atomics.  ws: est_workspace_bytes(nbins) + 2 n bytes.
template <class Src>
int shuffle_count(const Src &f, i64 n, int nbins, i64 *counts, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (nbins < 1 || nbins > 2 * PART2_NT) {
        set_error("shuffle: 1 <= destinations <= 2048");
        return LJ_E_INVALID;
    }
    const size_t eb = est_workspace_bytes(nbins);
    if (ws_bytes < eb + part_align(sizeof(u16) * (size_t)n)) {
        set_error("shuffle: workspace too small");
        return LJ_E_WORKSPACE;
    }
    u32 *est = (u32 *)ws;
    u16 *codes = reinterpret_cast<u16 *>((char *)ws + eb);
    LJ_CK(cudaMemsetAsync(est, 0, sizeof(u32) * (size_t)nbins, st));
    const size_t tb = pt_table_bytes(f.f.smem_words());
    static unsigned long long attr = 0;  // one bit per device
    if (once_per_device(attr)) {
        LJ_CK(cudaFuncSetAttribute(k_est_sample<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM_MAX));
        LJ_CK(cudaFuncSetAttribute(k_bin_scatter_est<Src, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   PT_SMEM_MAX));
    }
    if (n > 0) {
        k_est_sample<Src><<<grid_for(n, 256, 4), 256, tb + sizeof(u32) * nbins, st>>>(f, n, nbins, 1, est, codes);
        LJ_CK_LAUNCH();
    }
    k_est_caps<<<(nbins + 256) / 256, 256, 0, st>>>(est, nbins, 1, counts);  // counts[b] = est[b], counts[nbins] = 0
    LJ_CK_LAUNCH();
    return LJ_OK;
}

template <class Src>
int shuffle_scatter(const Src &f, i64 n, int nbins, const i64 *bases, void *ws, size_t ws_bytes, cudaStream_t st) {
    const size_t eb = est_workspace_bytes(nbins);
    if (ws_bytes < eb + part_align(sizeof(u16) * (size_t)n)) {
        set_error("shuffle: workspace too small");
        return LJ_E_WORKSPACE;
    }
    if (n <= 0) return LJ_OK;
    char *q = (char *)ws;
    q += part_align(sizeof(u32) * (size_t)nbins);
    u32 *gcur = (u32 *)q;
    q += part_align(sizeof(u32) * (size_t)nbins);
    q += 2 * part_align(sizeof(i64) * (size_t)(nbins + 1));
    unsigned long long *ovf = (unsigned long long *)q;
    const u16 *codes = reinterpret_cast<const u16 *>((char *)ws + eb);
    LJ_CK(cudaMemsetAsync(gcur, 0, sizeof(u32) * (size_t)nbins, st));
    const PartPlan p = part_plan(n, nbins);
    const size_t nb4 = (size_t)((nbins + 31) & ~31);
    const size_t fix = est_fix_bytes(nb4);
    const size_t stage = EST_STAGE + EST_TILE * 2;
    const int nst = (int)min((size_t)PT_MAXST, (PT_SMEM_MAX - fix) / stage);
    k_bin_scatter_est<Src, true, true><<<p.blocks, PART2_NT, fix + nst * stage, st>>>(
        f, n, p.chunk, nbins, nst, bases, gcur, ovf, nullptr, codes);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

// One pass into estimated-capacity regions (est_capacity records);
// reg[2*nbins+2] as described above.
template <class Src>
int run_partition_est(const Src &f, i64 n, int nbins, ulonglong2 *out, i64 *reg, void *ws, size_t ws_bytes,
                      cudaStream_t st) {
    return run_partition_claims(f, n, nbins, 0, out, reg, ws, ws_bytes, st);
}

// a fallback partition ran (*cond != 0): its contiguous bins as regions
static __global__ void k_cond_regions(unsigned long long *cond, const i64 *starts, int nbins, i64 *reg) {
    const bool ran = *cond != 0;
    __syncthreads();
    if (!ran) return;
    for (int b = threadIdx.x; b <= nbins; b += blockDim.x) {
        reg[b] = starts[b];
        if (b < nbins) reg[nbins + 1 + b] = starts[b + 1];
    }
    if (threadIdx.x == 0) reg[2 * nbins + 1] = 0;
}

inline size_t est_exact_workspace_bytes(int nbins) {
    return est_workspace_bytes(nbins) + part_align(sizeof(i64) * (size_t)(nbins + 1));
}

// One pass into estimated-capacity regions with NO overflow area for the
// consumer: if any record overflowed (practically never: the slack is many
// standard deviations of the sample estimate), the exact two-pass partition
// runs over the same output instead.  Its kernels are always enqueued and
// return at once when the overflow count is zero, so the decision stays on
// the device (no readback).  reg as run_partition_est, reg[2 nbins + 1] = 0;
// out: est_capacity_regions records (overflowing records are only counted).
template <class Src>
int run_partition_est_or_exact(const Src &f, i64 n, int nbins, ulonglong2 *out, i64 *reg, void *ws, size_t ws_bytes,
                               cudaStream_t st) {
    if (ws_bytes < est_exact_workspace_bytes(nbins)) {
        set_error("partition_est: workspace too small");
        return LJ_E_WORKSPACE;
    }
    const size_t eb = est_workspace_bytes(nbins);
    i64 *starts = reinterpret_cast<i64 *>((char *)ws + eb);
    int rc = run_partition_claims(f, n, nbins, 0, out, reg, ws, eb, st, nullptr, nullptr, 1);
    if (rc) return rc;
    unsigned long long *cond = reinterpret_cast<unsigned long long *>(reg + 2 * nbins + 1);
    rc = run_partition_claims(f, n, nbins, 1, out, starts, ws, eb, st, nullptr, cond);
    if (rc) return rc;
    k_cond_regions<<<1, 1024, 0, st>>>(cond, starts, nbins, reg);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

// The same one-pass regions through the direct claims scatter
// (k_scatter_direct: 2 CTAs per SM, no in-tile permutation).
template <class Src>
int run_partition_direct(const Src &f, i64 n, int nbins, ulonglong2 *out, i64 *reg, void *ws, size_t ws_bytes,
                         cudaStream_t st) {
    if (nbins < 1 || nbins > 4096) {
        set_error("partition_direct: nbins must be in [1, 4096]");
        return LJ_E_INVALID;
    }
    if (ws_bytes < est_workspace_bytes(nbins)) {
        set_error("partition_direct: workspace too small");
        return LJ_E_WORKSPACE;
    }
    char *q = (char *)ws;
    u32 *est = (u32 *)q;
    q += part_align(sizeof(u32) * (size_t)nbins);
    u32 *gcur = (u32 *)q;
    q += part_align(sizeof(u32) * (size_t)nbins);
    i64 *cap = (i64 *)q;
    q += part_align(sizeof(i64) * (size_t)(nbins + 1));
    i64 *rstart = (i64 *)q;
    q += part_align(sizeof(i64) * (size_t)(nbins + 1));
    unsigned long long *ovf = (unsigned long long *)q;
    q += part_align(sizeof(unsigned long long));
    LJ_CK(cudaMemsetAsync(est, 0, sizeof(u32) * (size_t)nbins, st));
    LJ_CK(cudaMemsetAsync(gcur, 0, sizeof(u32) * (size_t)nbins, st));
    LJ_CK(cudaMemsetAsync(ovf, 0, sizeof(unsigned long long), st));
    const size_t tb = pt_table_bytes(f.f.smem_words());
    const size_t nb4 = (size_t)((nbins + 31) & ~31);
    const size_t fix = tb + nb4 * (sizeof(u32) + 2 * sizeof(i64));
    const size_t stage = (size_t)DTILE * 16;
    const int nst = (int)min((size_t)4, ((size_t)(113 * 1024) - fix) / stage);  // two CTAs per SM
    if (nst < 2) {
        set_error("partition_direct: shared memory too small for the ring");
        return LJ_E_INVALID;
    }
    static unsigned long long attr = 0;  // one bit per device
    if (once_per_device(attr)) {
        LJ_CK(cudaFuncSetAttribute(k_scatter_direct<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(fix + nst * stage)));
        LJ_CK(cudaFuncSetAttribute(k_est_sample<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM_MAX));
    }
    if (n > 0) {
        k_est_sample<Src><<<grid_for((n + EST_STRIDE - 1) / EST_STRIDE, 256, 4), 256, tb + sizeof(u32) * nbins,
                            st>>>(f, n, nbins, EST_STRIDE, est, nullptr);
        LJ_CK_LAUNCH();
    }
    k_est_caps<<<(nbins + 256) / 256, 256, 0, st>>>(est, nbins, 0, cap);
    LJ_CK_LAUNCH();
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, cap, rstart, (int64_t)(nbins + 1));
    LJ_CK(cub::DeviceScan::ExclusiveSum(q, t, cap, rstart, (int64_t)(nbins + 1), st));
    if (n > 0) {
        const int blocks = 2 * sm_count();
        i64 c = (n + blocks - 1) / blocks;
        c = (c + 31) / 32 * 32;
        k_scatter_direct<Src><<<blocks, DNT, fix + nst * stage, st>>>(f, n, c < 32 ? 32 : c, nbins, nst, rstart, gcur,
                                                                      ovf, out);
        LJ_CK_LAUNCH();
    }
    k_est_regions<<<(nbins + 256) / 256, 256, 0, st>>>(rstart, gcur, ovf, nbins, reg);
    LJ_CK_LAUNCH();
    return LJ_OK;
}

// Exact partition: out[n] grouped by bin, starts[nbins+1].  Bulk-copy
// ring + shared frontiers when the columns are 16-B aligned and nbins <=
// 2048, else the per-CTA-segment two-pass partition (lj_part.cuh).
template <class Src>
int run_partition_fast(const Src &f, i64 n, int nbins, ulonglong2 *out, i64 *starts, void *ws, size_t ws_bytes,
                       cudaStream_t st) {
    static const bool legacy = getenv("LJ_PART_SEGMENTS") != nullptr;
    static const bool recompute = getenv("LJ_PART_RECOMPUTE") != nullptr;
    if (!legacy && f.aligned16() && nbins <= 2 * PART2_NT && n < (i64)0xFFFFFFFFLL) {
        // the counting pass stores every tuple's bin (u16) when the workspace
        // has room; the scatter then streams bins instead of evaluating them
        const size_t eb = est_workspace_bytes(nbins);
        u16 *codes = (!recompute && ws_bytes >= eb + part_align(sizeof(u16) * (size_t)n))
                         ? reinterpret_cast<u16 *>((char *)ws + eb)
                         : nullptr;
        return run_partition_claims(f, n, nbins, 1, out, starts, ws, ws_bytes, st, codes);
    }
    return run_partition(f, n, nbins, out, starts, ws, ws_bytes, st);
}

}  // namespace lj
