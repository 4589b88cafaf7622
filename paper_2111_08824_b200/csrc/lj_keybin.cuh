// lj_keybin.cuh -- exact key-range bin function evaluated in shared memory.
//
// Every bin function the partition passes use is monotone in the key, so it
// is a key-range function: bin(k) = #{ j in [1, nb) : B[j] <= k } for
// non-decreasing boundary keys B.  K4's windows are key ranges by
// definition (B[j] = gapped key at slot j*2^shift, plus one); LSJ's
// equi-depth bins over the model's predicted positions are key ranges
// because pos() is monotone (B[j] = the first key whose predicted position
// reaches pb[j], found once per call by a 64-step search over the key
// domain).  Evaluating the model per tuple costs a dependent leaf load from
// L2 (plus, for LSJ, a bin-table load); this structure needs none: a radix
// table over a monotone image t(k) of the key -- the key itself or a
// log-like image (the key's float bit pattern: bit length, then the bits
// below the leading one) for skewed keys, whichever leaves fewer boundaries
// per cell -- narrows the
// boundary range to a few entries, and a short binary search over the
// boundaries (both staged in shared memory, <= 32 KB) finishes it.
//
// Exactness: with cell() monotone, every boundary in a cell before k's is
// < k and every boundary in a cell after k's is > k, so bin(k) lies in
// [cells[c], cells[c+1]] (cells[c] = #{ j : cell(B[j]) < c }) and the
// search over that range returns exactly #{ j : B[j] <= k }.
//
// Crowded cells (clustered keys put a cluster's boundaries into one cell)
// get a second level: up to kb_nsub(nb) of them carry a sub-table of
// KB_SUBN sub-cells spanning just their own boundaries' image range [base,
// base + (KB_SUBN << sh)), with the same exactness argument one level down
// (sub-cell monotone in the image, clamped at both ends).
//
// Layout (u64 words, global and shared alike):
//   [0] t0 (image of B[1])   [1] shift | log << 8   [2] nb   [3] sub-tables used
//   [4 + j]  B[j], j in [1, nb)   (word 4 unused)
//   sets of > 1024 boundaries:   u16 cells[KB_CELLS + 1]
//   sets of <= 1024 boundaries (with sub-tables), packed so the lookup is
//   one load per level:
//     u32 cell32[KB_CELLS]        lo | (hi - lo) << 12 | sub-table << 24 (0xFF = none)
//     {u64 base, u64 shift} shdr[nsub]
//     u32 sub32[nsub][KB_SUBN]    lo | hi << 16 of every sub-cell
#pragma once

#include "lj_part.cuh"

namespace lj {

constexpr int KB_CELLS = 8192;
constexpr int KB_MAXBINS = 2048;
constexpr int KB_SUBN = 64;

// sub-tables: only next to small boundary sets (the partition kernels keep
// two ring stages beside the staged table)
__host__ __device__ inline int kb_nsub(int nb) { return nb <= 1024 ? 64 : 0; }
__host__ __device__ inline int kb_cells_words() { return (KB_CELLS + 1 + 3) / 4; }
__host__ __device__ inline int kb_words(int nb) {
    const int ns = kb_nsub(nb);
    return 4 + ((nb + 3) & ~3) + (ns ? KB_CELLS / 2 + 2 * ns + ns * KB_SUBN / 2 : kb_cells_words());
}
inline size_t kb_bytes(int nb) { return (size_t)kb_words(nb) * 8; }

// Monotone log-like image: the bit pattern of the key converted to float
// with truncation -- the exponent (bit length), then the 23 bits below the
// leading one; one conversion instruction.  a <= b  =>  kb_lg(a) <= kb_lg(b)
// (truncation is monotone, and non-negative floats order like their bits).
__device__ __forceinline__ u64 kb_lg(u64 k) { return (u64)__float_as_uint(__ull2float_rz(k)); }

__device__ __forceinline__ u64 kb_image(u64 k, int lg) { return lg ? kb_lg(k) : k; }

__device__ __forceinline__ u32 kb_cell(u64 t, u64 t0, int shift) {
    if (t < t0) return 0;
    const u64 c = (t - t0) >> shift;
    return c >= (u64)KB_CELLS ? (u32)(KB_CELLS - 1) : (u32)c;
}

struct KeyRangeBin {
    const u64 *g;  // layout (global before staging, shared after)
    int nb;
    int shift = 0;  // code -> bin shift of the partition passes (code == bin)
    // header words, cached in registers by at() (read from the global layout,
    // so no barrier is needed before them)
    u64 t0 = 0;
    u32 ctl = 0;
    __host__ __device__ int smem_words() const { return kb_words(nb); }
    __device__ void stage(u64 *dst) const {
        const int w = kb_words(nb);
        for (int i = threadIdx.x; i < w; i += blockDim.x) dst[i] = g[i];
    }
    __device__ __forceinline__ KeyRangeBin at(u64 *tab) const {
        KeyRangeBin c = *this;
        c.t0 = g[0];
        c.ctl = (u32)g[1];
        c.g = tab;
        return c;
    }
    // only on the copy at() returns
    __device__ __forceinline__ u32 code(u64 k) const {
        const u64 *B = g + 4;
        const u64 *cw = g + 4 + ((nb + 3) & ~3);
        const u64 t = kb_image(k, (int)(ctl >> 8) & 1);
        const u32 c = kb_cell(t, t0, (int)(ctl & 63));
        int lo, hi;
        const int ns = kb_nsub(nb);
        if (ns) {
            // packed: one load per level
            const u32 e = reinterpret_cast<const u32 *>(cw)[c];
            lo = (int)(e & 0xFFFu);
            hi = lo + (int)((e >> 12) & 0xFFFu);
            const u32 q = e >> 24;
            if (q != 0xFFu) {
                const ulonglong2 h = reinterpret_cast<const ulonglong2 *>(cw + KB_CELLS / 2)[q];  // {base, shift}
                const u64 d = t > h.x ? (t - h.x) >> h.y : 0;
                const u32 sc = d >= (u64)KB_SUBN ? (u32)(KB_SUBN - 1) : (u32)d;
                const u32 p = reinterpret_cast<const u32 *>(cw + KB_CELLS / 2 + 2 * ns)[q * KB_SUBN + sc];
                lo = (int)(p & 0xFFFFu);
                hi = (int)(p >> 16);
            }
        } else {
            const u16 *cells = reinterpret_cast<const u16 *>(cw);
            lo = cells[c];
            hi = cells[c + 1];
        }
        // two unconditional, branch-free steps settle every range of <= 3
        // boundaries (a step on lo == hi is a no-op: B[lo] <= k there, B[0] =
        // 0), so consecutive evaluations overlap; longer ranges finish in the loop
        if (ctl & 0x10000u) {  // dense boundary sets only (most cells non-empty ranges)
#pragma unroll
            for (int it = 0; it < 2; ++it) {
                const int mid = (lo + hi + 1) >> 1;
                const bool ge = B[mid] <= k;
                lo = ge ? mid : lo;
                hi = ge ? hi : mid - 1;
            }
        }
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (B[mid] <= k) lo = mid;
            else hi = mid - 1;
        }
        return (u32)lo;
    }
};

// One block of 1024 threads: header + cells from the boundaries already in
// lay[4 + j], j in [1, nb).  Both images are tried; the one whose fullest
// cell holds fewer boundaries wins (ties: the key itself).
static __global__ void __launch_bounds__(1024) k_keybin_build(u64 *lay, int nb) {
    __shared__ u32 worst[2];
    __shared__ u64 s_t0[2];
    __shared__ int s_shift[2];
    __shared__ u64 pm[KB_MAXBINS];
    __shared__ u16 cand[KB_CELLS + 1];
    u64 *B = lay + 4;
    const int tid = threadIdx.x;
    // the boundaries must be non-decreasing: a running maximum (a no-op
    // for the monotone bin functions; it keeps the structure sound for any
    // input)
    for (int j = tid; j < nb; j += blockDim.x) pm[j] = j ? B[j] : 0;
    __syncthreads();
    for (int d = 1; d < nb; d <<= 1) {
        u64 v[2];
        for (int r = 0; r < 2; ++r) {
            const int j = tid + r * (int)blockDim.x;
            v[r] = (j < nb && j >= d && pm[j - d] > pm[j]) ? pm[j - d] : (j < nb ? pm[j] : 0);
        }
        __syncthreads();
        for (int r = 0; r < 2; ++r) {
            const int j = tid + r * (int)blockDim.x;
            if (j < nb) pm[j] = v[r];
        }
        __syncthreads();
    }
    for (int j = tid; j < nb; j += blockDim.x) B[j] = pm[j];
    __syncthreads();
    if (tid < 2) {
        worst[tid] = 0;
        u64 t0 = 0, t1 = 0;
        if (nb >= 2) {
            t0 = kb_image(pm[1], tid);
            t1 = kb_image(pm[nb - 1], tid);
        }
        int s = 0;
        while (s < 63 && ((t1 - t0) >> s) >= (u64)KB_CELLS) ++s;
        s_t0[tid] = t0;
        s_shift[tid] = s;
    }
    __syncthreads();
    // cells[c] = #{ j in [1, nb) : c_j < c } with c_j = cell(B[j])
    // (non-decreasing in j): value j on (c_j, c_{j+1}], c_0 = -1,
    // c_nb = KB_CELLS -- one thread per boundary fills its range
    auto cellj = [&](int m, int j) -> int {
        if (j <= 0) return -1;
        if (j >= nb) return KB_CELLS;
        return (int)kb_cell(kb_image(pm[j], m), s_t0[m], s_shift[m]);
    };
    auto fill = [&](int m) {
        for (int j = tid; j < nb; j += blockDim.x) {
            const int lo = cellj(m, j) + 1, hi = cellj(m, j + 1);
            for (int c = lo; c <= hi; ++c) cand[c] = (u16)j;
        }
        __syncthreads();
    };
    for (int m = 1; m >= 0; --m) {  // mode 0 last: it stays in cand unless mode 1 wins
        fill(m);
        u32 w = 0;
        for (int c = tid; c < KB_CELLS; c += blockDim.x) {
            const u32 d = (u32)cand[c + 1] - (u32)cand[c];
            w = d > w ? d : w;
        }
        atomicMax(&worst[m], w);
        __syncthreads();
    }
    const int m = worst[1] < worst[0] ? 1 : 0;
    if (m == 1) fill(1);
    u64 *cw = lay + 4 + ((nb + 3) & ~3);
    __shared__ int s_nsub;
    const int ns = kb_nsub(nb);
    if (!ns) {
        u16 *cells = reinterpret_cast<u16 *>(cw);
        for (int c = tid; c <= KB_CELLS; c += blockDim.x) cells[c] = cand[c];
    }
    if (tid == 0) {
        lay[0] = s_t0[m];
        // bit 16: the search starts with two unconditional steps (sets with a
        // boundary for at least every eighth cell)
        lay[1] = (u64)s_shift[m] | ((u64)m << 8) | ((u64)(nb * 8 >= KB_CELLS ? 1 : 0) << 16);
        lay[2] = (u64)nb;
        s_nsub = 0;
    }
    __syncthreads();
    if (ns) {
        // second level for the crowded cells (> 2 boundaries), first come
        // first served up to the budget (any choice is exact)
        u32 *cell32 = reinterpret_cast<u32 *>(cw);
        u64 *shdr = cw + KB_CELLS / 2;
        u32 *sub32 = reinterpret_cast<u32 *>(shdr + 2 * ns);
        const u64 t0 = s_t0[m];
        const int sh0 = s_shift[m];
        for (int c = tid; c < KB_CELLS; c += blockDim.x) {
            int q = 0xFF;
            if ((int)cand[c + 1] - (int)cand[c] > 2) {
                const int got = atomicAdd(&s_nsub, 1);
                if (got < ns) q = got;
            }
            cell32[c] = (u32)cand[c] | ((u32)(cand[c + 1] - cand[c]) << 12) | ((u32)q << 24);
            if (q == 0xFF) continue;
            const int a = cand[c], e = cand[c + 1];  // boundaries j in (a, e] lie in cell c
            const u64 b = kb_image(pm[a + 1], m), last = kb_image(pm[e], m);
            int sh = 0;
            while (sh < 63 && ((last - b) >> sh) >= (u64)KB_SUBN) ++sh;
            shdr[2 * q] = b;
            shdr[2 * q + 1] = (u64)sh;
            u32 *st = sub32 + q * KB_SUBN;
            // s_sc = a + #{ j in (a, e] : subcell(B[j]) < sc }: the search in
            // sub-cell sc runs over (s_sc, s_{sc+1}] like the cells above;
            // st[sc] = s_sc | s_{sc+1} << 16
            int j = a + 1;
            u32 prev = 0;
            for (int sc = 0; sc <= KB_SUBN; ++sc) {
                while (j <= e) {
                    const u64 tj = kb_image(pm[j], m);
                    const u64 d = tj > b ? (tj - b) >> sh : 0;
                    const int scj = d >= (u64)KB_SUBN ? KB_SUBN - 1 : (int)d;
                    if (scj < sc) ++j;
                    else break;
                }
                const u32 cur = (u32)(sc == KB_SUBN ? e : j - 1);
                if (sc > 0) st[sc - 1] = prev | (cur << 16);
                prev = cur;
            }
        }
        (void)t0;
        (void)sh0;
    }
    __syncthreads();
    if (tid == 0) lay[3] = (u64)(s_nsub < ns ? s_nsub : ns);
}

}  // namespace lj
