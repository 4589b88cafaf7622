// lj_probe_count.h -- the reference's search_steps of one GRMI lookup
// (gapped.py:86-160: exponential search from the predicted slot, then a
// lower-bound binary search, then one verification probe), computed from
// where the key sits in the gapped array instead of by touching memory.
//
// The key occupies slots [lb, re) (slots < lb hold smaller keys, slots >= re
// larger; lb == re when it is absent).  Coordinates are relative to any
// origin o with all of start, lb, re within 2^30 of it; lim = L - o and
// zero = -o (both clamped to +-2^30).  Plain C++ so the host test
// (tests/test_probe_count.py) checks it exhaustively against the loop.
#pragma once

#ifdef __CUDACC__
#define LJ_HD __host__ __device__ __forceinline__
#else
#define LJ_HD inline
#endif

namespace lj {

// the reference's loop, restated over positions
LJ_HD int ref_probe_count_loop(int start, int lb, int re, int lim, int zero) {
    if (start >= lb && start < re) return 1;
    int probes = 1, lo, hi;
    if (start < lb) {
        int prev = start, step = 1;
        for (;;) {
            const int idx = start + step;
            if (idx >= lim) { lo = prev + 1; hi = lim; break; }
            ++probes;
            if (idx < lb) { prev = idx; step <<= 1; }
            else if (idx < re) return probes;
            else { lo = prev + 1; hi = idx; break; }
        }
    } else {
        int prev = start, step = 1;
        for (;;) {
            const int idx = start - step;
            if (idx < zero) { lo = zero; hi = prev; break; }
            ++probes;
            if (idx >= re) { prev = idx; step <<= 1; }
            else if (idx >= lb) return probes;
            else { lo = idx + 1; hi = prev; break; }
        }
    }
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        ++probes;
        if (mid < lb) lo = mid + 1; else hi = mid;
    }
    if (lo < lim) ++probes;
    return probes;
}

LJ_HD int ceil_log2_pos(int d) {  // d >= 1
#ifdef __CUDA_ARCH__
    return 32 - __clz(d - 1);
#else
    return d <= 1 ? 0 : 32 - __builtin_clz((unsigned)(d - 1));
#endif
}

// Closed form.  With d the distance from start to the first slot past the
// run boundary on the key's side, the exponential phase takes J =
// ceil(log2 d) steps and its last probe either lands inside the run (J + 2
// probes in all) or brackets an interval of exactly 2^(J-1) - 1 slots,
// which the binary search resolves in J - 1 steps whatever the target, plus
// the verification probe (2J + 2; 3 when J = 0).  Only when the exponential
// phase would leave the array [0, L) does the interval length depend on
// the target; that case (within 2^J of either end) runs the loop.
LJ_HD int ref_probe_count(int start, int lb, int re, int lim, int zero) {
    if (start >= lb && start < re) return 1;
    const bool right = start < lb;
    const int d = right ? lb - start : start - re + 1;
    const int J = ceil_log2_pos(d);
    const int reach = right ? lim - start : start - zero;  // largest in-range step is < / <= this
    const bool bounded = right ? ((1 << J) >= reach) : ((1 << J) > reach);
    if (bounded) return ref_probe_count_loop(start, lb, re, lim, zero);
    const bool hit = right ? ((1 << J) < re - start) : ((1 << J) <= start - lb);
    return hit ? J + 2 : (J ? 2 * J + 2 : 3);
}

}  // namespace lj
