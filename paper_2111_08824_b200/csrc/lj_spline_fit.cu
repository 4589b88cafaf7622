// lj_spline_fit.cu -- RadixSpline greedy-corridor fit on the GPU
// (models.py:171-219 `RadixSplineIndex.fit` / `_greedy_corridor`).
//
// The corridor is sequential by definition: whether point i becomes a knot
// depends on the corridor left by the previous knot.  But the corridor's
// state right after a knot j is emitted is a function of j alone (base =
// point j, slope window from point j+1), so two runs that emit the same
// knot are identical from then on.  The fit therefore runs in three steps:
//   1. every chunk of L unique points runs the greedy speculatively, as if
//      its first point were a knot (chunk 0's run is the true one);
//   2. every chunk c >= 1 re-runs from the speculative end state of chunk
//      c-1 until it emits a knot its own speculative run also emitted
//      ("convergence", typically within a knot or two); the knots before
//      that point replace the speculative prefix;
//   3. one thread walks the chunks in order: a chunk whose predecessor did
//      not converge is re-run from the true state (rare: the chunk must be
//      shorter than the distance to convergence).
// Knots are then spliced with one scan.  Every operation is the reference's
// float64 operation in its order (u64 -> f64 round-to-nearest, (y + e) - b,
// no contraction), so the knots equal lj_spline_fit_host's -- and the
// reference's -- bit for bit (tests/test_gpu_parity.py).
#include <cub/cub.cuh>

#include <vector>

#include "lj_common.cuh"

namespace lj {

constexpr i64 FIT_CHUNK = 32768;  // unique points per speculative run

struct Corr {
    double bx, by, hi, lo;
};

struct FitPts {
    const u64 *keys;   // sorted keys
    const i64 *uidx;   // first index of every unique key
    double err;
    __device__ __forceinline__ double x(i64 i) const { return u64_to_f64(keys[uidx[i]]); }
    __device__ __forceinline__ double y(i64 i) const { return i64_to_f64(uidx[i]); }
    // models.py:200-217 for point i inside the corridor (no knot)
    __device__ __forceinline__ void step_in(Corr &c, i64 i) const {
        const double xi = x(i), yi = y(i), dx = __dsub_rn(xi, c.bx);
        const double u = __ddiv_rn(__dsub_rn(__dadd_rn(yi, err), c.by), dx);
        const double l = __ddiv_rn(__dsub_rn(__dsub_rn(yi, err), c.by), dx);
        if (u < c.hi) c.hi = u;
        if (l > c.lo) c.lo = l;
    }
    // processes point i: true (and the corridor restarted at i - 1) when
    // point i leaves the corridor, i.e. knot i - 1 is emitted
    __device__ __forceinline__ bool step(Corr &c, i64 i) const {
        const double xi = x(i), yi = y(i);
        const double slope = __ddiv_rn(__dsub_rn(yi, c.by), __dsub_rn(xi, c.bx));
        if (slope > c.hi || slope < c.lo) {
            c.bx = x(i - 1);
            c.by = y(i - 1);
            const double dx = __dsub_rn(xi, c.bx);
            c.hi = __ddiv_rn(__dsub_rn(__dadd_rn(yi, err), c.by), dx);
            c.lo = __ddiv_rn(__dsub_rn(__dsub_rn(yi, err), c.by), dx);
            return true;
        }
        step_in(c, i);
        return false;
    }
};

// unique-key starts: flag[i] = keys[i] != keys[i-1]
__global__ void k_fit_flags(const u64 *keys, i64 n, unsigned char *flag) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// step 1: speculative run of every chunk
__global__ void k_fit_spec(FitPts P, i64 s, i64 nch, u32 *spk, i64 *spn, Corr *spend) {
    for (i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x; c < nch; c += (i64)gridDim.x * blockDim.x) {
        const i64 a = c * FIT_CHUNK, e = min(a + FIT_CHUNK, s);
        u32 *out = spk + a;
        i64 n = 0;
        out[n++] = (u32)a;  // assumed (chunk 0: the reference's first knot)
        Corr cr;
        cr.bx = P.x(a);
        cr.by = P.y(a);
        cr.hi = INFINITY;
        cr.lo = -INFINITY;
        for (i64 i = a + 1; i < e; ++i)
            if (P.step(cr, i)) out[n++] = (u32)(i - 1);
        spn[c] = n;
        spend[c] = cr;
    }
}

// re-run of chunk c from corridor `cr`; cond knots before convergence into
// cdk; returns the position in c's speculative list where they converge,
// or -1 (then *end = the corridor after the chunk)
__device__ i64 fit_rerun(const FitPts &P, i64 s, i64 c, Corr cr, const u32 *spk, const i64 *spn, u32 *cdk,
                         i64 *cdn, Corr *end) {
    const i64 a = c * FIT_CHUNK, e = min(a + FIT_CHUNK, s);
    const u32 *sp = spk + a;
    const i64 ns = spn[c];
    i64 p = 0, n = 0;
    for (i64 i = a; i < e; ++i) {
        if (!P.step(cr, i)) continue;
        const u32 j = (u32)(i - 1);
        while (p < ns && sp[p] < j) ++p;
        if (p < ns && sp[p] == j) {
            *cdn = n;
            return p;
        }
        cdk[a + n++] = j;
    }
    *cdn = n;
    *end = cr;
    return -1;
}

// step 2: every chunk c >= 1 from the speculative end state of chunk c-1
__global__ void k_fit_conv(FitPts P, i64 s, i64 nch, const u32 *spk, const i64 *spn, const Corr *spend, u32 *cdk,
                           i64 *cdn, i64 *cvg, Corr *cdend) {
    for (i64 c = 1 + blockIdx.x * (i64)blockDim.x + threadIdx.x; c < nch; c += (i64)gridDim.x * blockDim.x)
        cvg[c] = fit_rerun(P, s, c, spend[c - 1], spk, spn, cdk, cdn + c, cdend + c);
}

// step 3: the true chain (one thread); then knots per chunk
__global__ void k_fit_chain(FitPts P, i64 s, i64 nch, const u32 *spk, const i64 *spn, const Corr *spend, u32 *cdk,
                            i64 *cdn, i64 *cvg, Corr *cdend, i64 *cnt, unsigned long long *reruns) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    bool valid = true;  // the corridor entering chunk c is spend[c-1]
    Corr truth = spend[0];
    cnt[0] = spn[0];
    for (i64 c = 1; c < nch; ++c) {
        if (!valid) {
            cvg[c] = fit_rerun(P, s, c, truth, spk, spn, cdk, cdn + c, cdend + c);
            ++*reruns;
        }
        if (cvg[c] >= 0) {
            truth = spend[c];
            valid = true;
            cnt[c] = cdn[c] + spn[c] - cvg[c];
        } else {
            truth = cdend[c];
            valid = false;
            cnt[c] = cdn[c];
        }
    }
}

__global__ void k_fit_emit(const u64 *keys, const i64 *uidx, i64 s, i64 nch, const u32 *spk, const i64 *spn,
                           const u32 *cdk, const i64 *cdn, const i64 *cvg, const i64 *off, u64 *kout, i64 *rout) {
    for (i64 c = blockIdx.x; c < nch; c += gridDim.x) {
        const i64 a = c * FIT_CHUNK, o = off[c];
        const i64 nc = c == 0 ? 0 : cdn[c];
        const i64 p0 = c == 0 ? 0 : cvg[c];
        const i64 nsp = p0 >= 0 ? spn[c] - p0 : 0;
        for (i64 t = threadIdx.x; t < nc + nsp; t += blockDim.x) {
            const u32 j = t < nc ? cdk[a + t] : spk[a + p0 + (t - nc)];
            kout[o + t] = keys[uidx[j]];
            rout[o + t] = uidx[j];
        }
    }
}

__global__ void k_fit_all(const u64 *keys, const i64 *uidx, i64 s, u64 *kout, i64 *rout) {
    for (i64 t = threadIdx.x; t < s; t += blockDim.x) {
        kout[t] = keys[uidx[t]];
        rout[t] = uidx[t];
    }
}

// radix_table[p] = first knot whose key prefix >= p, p in [0, 2^r]
__global__ void k_fit_radix(const u64 *kk, i64 k, u64 shift, i64 np1, i64 *radix) {
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < np1; p += (i64)gridDim.x * blockDim.x) {
        i64 lo = 0, hi = k;
        while (lo < hi) {
            const i64 mid = (lo + hi) >> 1;
            if ((i64)(kk[mid] >> shift) < p) lo = mid + 1; else hi = mid;
        }
        radix[p] = lo;
    }
}

static size_t fal(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace lj

using namespace lj;

extern "C" {

size_t lj_spline_fit_workspace_bytes(int64_t n) {
    const i64 nch = (n + FIT_CHUNK - 1) / FIT_CHUNK + 1;
    size_t t1 = 0, t2 = 0;
    cub::DeviceSelect::Flagged(nullptr, t1, (cub::CountingInputIterator<i64>)0, (const unsigned char *)nullptr,
                               (i64 *)nullptr, (i64 *)nullptr, (int64_t)n);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, (const i64 *)nullptr, (i64 *)nullptr, (int64_t)nch);
    return fal(n) + fal(8 * (size_t)n) + 2 * fal(4 * (size_t)n) + 5 * fal(8 * (size_t)nch) +
           2 * fal(sizeof(Corr) * (size_t)nch) + fal(64) + fal(t1 > t2 ? t1 : t2);
}

int lj_spline_fit(const uint64_t *keys, int64_t n, int64_t max_error, int64_t radix_bits, uint64_t *knot_keys,
                  int64_t *knot_ranks, int64_t *radix_out, int64_t *npts_out, uint64_t *shift_out, void *ws,
                  size_t ws_bytes, void *stream) {
    LJ_REQUIRE(n >= 1 && max_error >= 1 && radix_bits >= 1 && radix_bits <= 30, "bad spline parameters");
    LJ_REQUIRE(n < ((int64_t)1 << 32), "the GPU fit indexes points with 32 bits: n < 2^32");
    if (ws_bytes < lj_spline_fit_workspace_bytes(n)) {
        set_error("lj_spline_fit: workspace too small");
        return LJ_E_WORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    const i64 nch_max = (n + FIT_CHUNK - 1) / FIT_CHUNK + 1;
    char *q = (char *)ws;
    auto take = [&](size_t b) {
        char *r = q;
        q += fal(b);
        return r;
    };
    unsigned char *flag = (unsigned char *)take(n);
    i64 *uidx = (i64 *)take(8 * (size_t)n);
    u32 *spk = (u32 *)take(4 * (size_t)n);
    u32 *cdk = (u32 *)take(4 * (size_t)n);
    i64 *spn = (i64 *)take(8 * (size_t)nch_max);
    i64 *cdn = (i64 *)take(8 * (size_t)nch_max);
    i64 *cvg = (i64 *)take(8 * (size_t)nch_max);
    i64 *cnt = (i64 *)take(8 * (size_t)nch_max);
    i64 *off = (i64 *)take(8 * (size_t)nch_max);
    Corr *spend = (Corr *)take(sizeof(Corr) * (size_t)nch_max);
    Corr *cdend = (Corr *)take(sizeof(Corr) * (size_t)nch_max);
    i64 *misc = (i64 *)take(64);  // [0] unique count, [1] re-runs
    void *tmp = (void *)q;
    size_t tb = ws_bytes - (size_t)(q - (char *)ws);

    k_fit_flags<<<grid_for(n, 256, 8), 256, 0, st>>>(keys, n, flag);
    LJ_CK_LAUNCH();
    LJ_CK(cub::DeviceSelect::Flagged(tmp, tb, cub::CountingInputIterator<i64>(0), flag, uidx, misc, (int64_t)n, st));
    i64 s = 0;
    LJ_CK(cudaMemcpyAsync(&s, misc, sizeof(i64), cudaMemcpyDeviceToHost, st));
    LJ_CK(cudaMemsetAsync(misc + 1, 0, sizeof(i64), st));
    LJ_CK(cudaStreamSynchronize(st));
    const FitPts P{keys, uidx, (double)max_error};
    i64 k = 0;
    if (s <= 2) {
        // models.py:196-198: every unique point is a knot
        k_fit_all<<<1, 32, 0, st>>>(keys, uidx, s, knot_keys, knot_ranks);
        LJ_CK_LAUNCH();
        k = s;
    } else {
        const i64 nch = (s + FIT_CHUNK - 1) / FIT_CHUNK;
        k_fit_spec<<<grid_for(nch, 64, 8), 64, 0, st>>>(P, s, nch, spk, spn, spend);
        LJ_CK_LAUNCH();
        if (nch > 1) {
            k_fit_conv<<<grid_for(nch, 64, 8), 64, 0, st>>>(P, s, nch, spk, spn, spend, cdk, cdn, cvg, cdend);
            LJ_CK_LAUNCH();
        }
        k_fit_chain<<<1, 32, 0, st>>>(P, s, nch, spk, spn, spend, cdk, cdn, cvg, cdend, cnt,
                                      (unsigned long long *)(misc + 1));
        LJ_CK_LAUNCH();
        size_t t2 = tb;
        LJ_CK(cub::DeviceScan::ExclusiveSum(tmp, t2, cnt, off, (int64_t)nch, st));
        k_fit_emit<<<(unsigned)(nch < 4096 ? nch : 4096), 256, 0, st>>>(keys, uidx, s, nch, spk, spn, cdk, cdn, cvg,
                                                                          off, knot_keys, knot_ranks);
        LJ_CK_LAUNCH();
        i64 last_off = 0, last_cnt = 0;
        LJ_CK(cudaMemcpyAsync(&last_off, off + nch - 1, sizeof(i64), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaMemcpyAsync(&last_cnt, cnt + nch - 1, sizeof(i64), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaStreamSynchronize(st));
        k = last_off + last_cnt;
        // models.py:215-216: the last point closes the spline
        i64 last_rank = -1, s_last_rank = 0;
        LJ_CK(cudaMemcpyAsync(&last_rank, knot_ranks + k - 1, sizeof(i64), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaMemcpyAsync(&s_last_rank, uidx + s - 1, sizeof(i64), cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaStreamSynchronize(st));
        if (last_rank != s_last_rank) {
            LJ_CK(cudaMemcpyAsync(knot_keys + k, keys + s_last_rank, sizeof(u64), cudaMemcpyDeviceToDevice, st));
            LJ_CK(cudaMemcpyAsync(knot_ranks + k, uidx + s - 1, sizeof(i64), cudaMemcpyDeviceToDevice, st));
            ++k;
        }
    }
    // shift from the bit length of the largest knot key; the radix table
    u64 kmax = 0;
    LJ_CK(cudaMemcpyAsync(&kmax, knot_keys + k - 1, sizeof(u64), cudaMemcpyDeviceToHost, st));
    LJ_CK(cudaStreamSynchronize(st));
    int mb = 0;
    for (u64 v = kmax; v; v >>= 1) ++mb;
    const u64 shift = (u64)(mb - radix_bits > 0 ? mb - radix_bits : 0);
    const i64 np1 = ((i64)1 << radix_bits) + 1;
    k_fit_radix<<<grid_for(np1, 256, 8), 256, 0, st>>>(knot_keys, k, shift, np1, radix_out);
    LJ_CK_LAUNCH();
    *npts_out = k;
    *shift_out = shift;
    return LJ_OK;
}

}  // extern "C"
