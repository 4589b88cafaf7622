/*
 * lj_gen.c -- HOST generator of the BASELINE configurations' seeded inputs
 * (TEST / BASELINE INFRASTRUCTURE ONLY, like the rest of oracle/).
 *
 * The CUDA library draws the same streams on the device
 * (paper_2111_08824_b200/csrc/lj_core.cu: lj_fill_mix64, lj_fill_payloads,
 * lj_gather_uniform, lj_fill_normal, lj_fill_lognormal, lj_fill_cluster).
 * Both sides evaluate include/lj_gen.h (IEEE + - * / sqrt only, each
 * rounded separately), so the host regenerates every configuration bit for
 * bit WITHOUT loading the CUDA library: bench.py's reference arm builds its
 * inputs here and oracle/gen.py mirrors paper_2111_08824_b200/configs.py on
 * top of these primitives.  Compiled with -ffp-contract=off (Makefile).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/lj_gen.h"

#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef int64_t i64;

/* draw offset+i of stream seed: mix64(seed ^ (offset + i)) (lj_fill_mix64) */
void orc_gen_mix(u64 *out, i64 n, i64 offset, u64 seed) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) out[i] = ljg_mix64(seed ^ (u64)(offset + i));
}

/* reference data.py:181-192 positional payloads mix64(i + mix64(seed)) | 1
 * at positions offset .. offset+n-1 (lj_fill_payloads) */
void orc_gen_payloads(u64 *out, i64 n, i64 offset, u64 seed) {
    const u64 base = ljg_mix64(seed);
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) out[i] = ljg_mix64((u64)(offset + i) + base) | 1ULL;
}

/* src[mulhi(mix64(seed ^ (offset+i)), src_n)] (lj_gather_uniform) */
void orc_gen_gather_uniform(u64 *out, i64 n, i64 offset, u64 seed, const u64 *src, i64 src_n) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        const u64 r = ljg_mix64(seed ^ (u64)(offset + i));
        out[i] = src[(u64)(((unsigned __int128)r * (u64)src_n) >> 64)];
    }
}

void orc_gen_normal(double *out, i64 n, i64 offset, u64 seed) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) out[i] = ljg_normal(seed, (u64)(offset + i));
}

void orc_gen_lognormal(i64 *out, i64 n, i64 offset, u64 seed, double sigma, double scale, double maxv) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) out[i] = ljg_lognormal_key(seed, (u64)(offset + i), sigma, scale, maxv);
}

void orc_gen_cluster(i64 *out, i64 n, i64 offset, u64 seed, const double *centres, int ncent, double sigma,
                     double maxv) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) out[i] = ljg_cluster_key(seed, (u64)(offset + i), centres, ncent, sigma, maxv);
}

/* keep[i] = 1 iff no j < i has v[j] == v[i] (values != ~0).  Indices are
 * spread over 256 buckets by a hash of the value (stable, so each bucket
 * lists its indices in increasing order); every bucket then inserts its
 * values in that order into its own open-addressing set. */
void orc_first_occurrence(const u64 *v, i64 n, uint8_t *keep) {
    enum { NB = 256 };
    if (n <= 0) return;
    int T = 1;
#ifdef _OPENMP
    T = omp_get_max_threads();
#endif
    i64 *hist = (i64 *)calloc((size_t)T * NB, sizeof(i64));
    i64 *idx = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 bstart[NB + 1];
#pragma omp parallel num_threads(T)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        const i64 lo = n * t / T, hi = n * (t + 1) / T;
        i64 *h = hist + (size_t)t * NB;
        for (i64 i = lo; i < hi; ++i) ++h[ljg_mix64(v[i]) >> 56];
#pragma omp barrier
#pragma omp single
        {
            i64 run = 0;
            for (int b = 0; b < NB; ++b) {
                bstart[b] = run;
                for (int u = 0; u < T; ++u) {
                    const i64 c = hist[(size_t)u * NB + b];
                    hist[(size_t)u * NB + b] = run;
                    run += c;
                }
            }
            bstart[NB] = run;
        }
        for (i64 i = lo; i < hi; ++i) idx[h[ljg_mix64(v[i]) >> 56]++] = i;
#pragma omp barrier
#pragma omp for schedule(dynamic, 1)
        for (int b = 0; b < NB; ++b) {
            const i64 cnt = bstart[b + 1] - bstart[b];
            i64 cap = 16;
            while (cap < 2 * cnt) cap <<= 1;
            u64 *set = (u64 *)malloc(sizeof(u64) * (size_t)cap);
            memset(set, 0xFF, sizeof(u64) * (size_t)cap);
            for (i64 q = bstart[b]; q < bstart[b + 1]; ++q) {
                const i64 i = idx[q];
                const u64 key = v[i];
                u64 s = ljg_mix64(key ^ 0x5bd1e995ULL) & (u64)(cap - 1);
                int fresh = 1;
                while (set[s] != ~0ULL) {
                    if (set[s] == key) {
                        fresh = 0;
                        break;
                    }
                    s = (s + 1) & (u64)(cap - 1);
                }
                if (fresh) set[s] = key;
                keep[i] = (uint8_t)fresh;
            }
            free(set);
        }
    }
    free(idx);
    free(hist);
}

/* np.searchsorted(cdf, u, side="left") for sorted doubles, in parallel */
void orc_searchsorted_f64(const double *cdf, i64 n, const double *u, i64 m, i64 *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < m; ++i) {
        const double v = u[i];
        i64 lo = 0, hi = n;
        while (lo < hi) {
            const i64 mid = (lo + hi) >> 1;
            if (cdf[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        out[i] = lo;
    }
}

/* np.searchsorted(sorted, v, side="left") for u64, in parallel */
void orc_searchsorted_u64(const u64 *sorted, i64 n, const u64 *v, i64 m, i64 *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < m; ++i) {
        const u64 x = v[i];
        i64 lo = 0, hi = n;
        while (lo < hi) {
            const i64 mid = (lo + hi) >> 1;
            if (sorted[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        out[i] = lo;
    }
}
