/*
 * lj_gen.h -- portable, bit-reproducible generator arithmetic for the
 * seeded synthetic inputs of the BASELINE configurations.
 *
 * The configurations' lognormal and normal-cluster keys need log, exp and
 * cos.  libm and CUDA's math library round those differently in the last
 * place, and one ulp moves floor(1e12 * exp(...)) to another integer, so a
 * host regeneration would not reproduce the device's inputs.  The functions
 * below use only IEEE-754 correctly rounded operations (+ - * / sqrt), each
 * rounded separately (device: explicit __d*_rn intrinsics, never contracted
 * into FMA; host: compiled with -ffp-contract=off), so the SAME bits come
 * out of the CUDA kernels (csrc/lj_core.cu lj_fill_normal / _lognormal) and
 * of the host generator in oracle/ (oracle/lj_gen.c), which the reference
 * arm of bench.py uses without loading the CUDA library.
 *
 * Accuracy is ~1-2 ulp (Cody-Waite reductions + Taylor / atanh series), far
 * below what a key generator needs; determinism is the point.
 *
 * Counter-based draws: draw j of stream `seed` is mix64(seed ^ j)
 * (SplitMix64 finaliser, reference util.py:30-44).
 */
#ifndef LJ_GEN_H
#define LJ_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define LJG_FN __host__ __device__ __forceinline__
#else
#include <string.h>
#define LJG_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define LJG_ADD(a, b) __dadd_rn((a), (b))
#define LJG_SUB(a, b) __dsub_rn((a), (b))
#define LJG_MUL(a, b) __dmul_rn((a), (b))
#define LJG_DIV(a, b) __ddiv_rn((a), (b))
#define LJG_SQRT(a) __dsqrt_rn(a)
#else
#include <math.h>
#define LJG_ADD(a, b) ((a) + (b))
#define LJG_SUB(a, b) ((a) - (b))
#define LJG_MUL(a, b) ((a) * (b))
#define LJG_DIV(a, b) ((a) / (b))
#define LJG_SQRT(a) sqrt(a)
#endif

LJG_FN uint64_t ljg_mix64(uint64_t z) {
    z = z + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

LJG_FN uint64_t ljg_bits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t b;
    memcpy(&b, &x, 8);
    return b;
#endif
}

LJG_FN double ljg_from_bits(uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)b);
#else
    double x;
    memcpy(&x, &b, 8);
    return x;
#endif
}

/* uniform double in (0, 1): top 53 bits of a draw, centred in their cell */
LJG_FN double ljg_unit(uint64_t m) {
    return LJG_MUL(LJG_ADD((double)(int64_t)(m >> 11), 0.5), 1.1102230246251565e-16 /* 2^-53 */);
}

/* round half to even for |y| < 2^51 (the 1.5 * 2^52 shift) */
LJG_FN double ljg_rint(double y) {
    return LJG_SUB(LJG_ADD(y, 6755399441055744.0), 6755399441055744.0);
}

#define LJG_LN2_HI 6.93147180369123816490e-01 /* fdlibm ln2_hi: 21 trailing zero bits */
#define LJG_LN2_LO 1.90821492927058770002e-10
#define LJG_INV_LN2 1.44269504088896338700e+00
#define LJG_SQRT2 1.4142135623730951
#define LJG_TWO_PI 6.283185307179586

/* natural log of a positive normal double */
LJG_FN double ljg_log(double x) {
    const uint64_t b = ljg_bits(x);
    int e = (int)((b >> 52) & 0x7FF) - 1023;
    double m = ljg_from_bits((b & 0x000FFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL); /* [1, 2) */
    if (m > LJG_SQRT2) {
        m = LJG_MUL(m, 0.5); /* exact */
        e += 1;
    }
    /* log m = 2 atanh(s), s = (m-1)/(m+1), |s| < 0.1716: s * sum 2 z^j/(2j+1) */
    const double f = LJG_SUB(m, 1.0);
    const double s = LJG_DIV(f, LJG_ADD(2.0, f));
    const double z = LJG_MUL(s, s);
    double p = LJG_DIV(2.0, 25.0);
    for (int j = 11; j >= 0; --j) p = LJG_ADD(LJG_MUL(p, z), LJG_DIV(2.0, (double)(2 * j + 1)));
    const double ed = (double)e;
    return LJG_ADD(LJG_MUL(ed, LJG_LN2_HI), LJG_ADD(LJG_MUL(ed, LJG_LN2_LO), LJG_MUL(s, p)));
}

/* e^x for |x| < 700 */
LJG_FN double ljg_exp(double x) {
    const double kd = ljg_rint(LJG_MUL(x, LJG_INV_LN2));
    const double r = LJG_SUB(LJG_SUB(x, LJG_MUL(kd, LJG_LN2_HI)), LJG_MUL(kd, LJG_LN2_LO)); /* |r| < 0.35 */
    double p = 1.0;
    for (int j = 18; j >= 1; --j) p = LJG_ADD(1.0, LJG_DIV(LJG_MUL(r, p), (double)j));
    const int k = (int)kd;
    return LJG_MUL(p, ljg_from_bits((uint64_t)(int64_t)(k + 1023) << 52));
}

/* cos(2 pi u) for u in [0, 1]; the quadrant reductions are exact (Sterbenz) */
LJG_FN double ljg_cos2pi(double u) {
    double w = u > 0.5 ? LJG_SUB(1.0, u) : u; /* [0, 0.5] */
    double sign = 1.0;
    if (w > 0.25) {
        w = LJG_SUB(0.5, w); /* cos 2pi(1/2 - w) = -cos 2pi w */
        sign = -1.0;
    }
    int use_sin = 0;
    if (w > 0.125) {
        w = LJG_SUB(0.25, w); /* cos 2pi(1/4 - w) = sin 2pi w */
        use_sin = 1;
    }
    const double t = LJG_MUL(w, LJG_TWO_PI); /* [0, pi/4] */
    const double z = LJG_MUL(t, t);
    double p = 1.0;
    if (use_sin) {
        for (int j = 12; j >= 1; --j) p = LJG_SUB(1.0, LJG_DIV(LJG_MUL(z, p), (double)((2 * j) * (2 * j + 1))));
        p = LJG_MUL(t, p);
    } else {
        for (int j = 12; j >= 1; --j) p = LJG_SUB(1.0, LJG_DIV(LJG_MUL(z, p), (double)((2 * j - 1) * (2 * j))));
    }
    return LJG_MUL(sign, p);
}

/* standard normal draw j of stream `seed` (Box-Muller on two counter draws) */
LJG_FN double ljg_normal(uint64_t seed, uint64_t j) {
    const double u1 = ljg_unit(ljg_mix64((seed ^ 0xA5A5ULL) ^ j));
    const double u2 = ljg_unit(ljg_mix64((seed ^ 0x5A5AULL) ^ j));
    return LJG_MUL(LJG_SQRT(LJG_MUL(-2.0, ljg_log(u1))), ljg_cos2pi(u2));
}

/* floor(scale * exp(sigma * normal)) clamped to [0, maxv], as int64 */
LJG_FN int64_t ljg_lognormal_key(uint64_t seed, uint64_t j, double sigma, double scale, double maxv) {
    double v = LJG_MUL(scale, ljg_exp(LJG_MUL(sigma, ljg_normal(seed, j))));
    v = floor(v);
    v = v < 0.0 ? 0.0 : (v > maxv ? maxv : v);
    return (int64_t)v;
}

/* centre[cluster] + sigma * normal as int64 (truncation), or -1 when the
 * draw falls outside [0, maxv); the cluster of draw j is the top bits of
 * mix64((seed ^ 0x32) ^ j), the normal comes from stream seed ^ 0x33 */
LJG_FN int64_t ljg_cluster_key(uint64_t seed, uint64_t j, const double *centres, int ncent, double sigma,
                               double maxv) {
    int bits = 0;
    while ((1 << bits) < ncent) ++bits;
    const uint64_t cl = bits ? (ljg_mix64((seed ^ 0x32ULL) ^ j) >> (64 - bits)) : 0;
    const double v = LJG_ADD(centres[cl], LJG_MUL(sigma, ljg_normal(seed ^ 0x33ULL, j)));
    return (v >= 0.0 && v < maxv) ? (int64_t)v : -1;
}

#endif /* LJ_GEN_H */
