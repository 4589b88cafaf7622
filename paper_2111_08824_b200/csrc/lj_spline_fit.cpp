// lj_spline_fit.cpp -- host-side RadixSpline fit (models.py:171-219).
//
// The greedy corridor is a strictly sequential scan over the unique keys
// (each decision depends on the corridor left by the previous one), so it
// runs on the host, in C++, over the device-sorted keys copied back once.
// The model it produces is evaluated on the GPU only.  Compiled with
// -ffp-contract=off: every rounding matches numpy's scalar float64 ops, so
// the chosen spline points equal the reference's (tests pin this).
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "../../include/lj_b200.h"

namespace {

int bit_length(uint64_t v) {
    int b = 0;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

}  // namespace

extern "C" int lj_spline_fit_host(const uint64_t *keys, int64_t n, int64_t max_error, int64_t radix_bits,
                                  uint64_t *keys_out, int64_t *ranks_out, int64_t *radix_out,
                                  int64_t *npts_out, uint64_t *shift_out) {
    if (n <= 0 || max_error < 1 || radix_bits < 1 || radix_bits > 30) return LJ_E_INVALID;
    for (int64_t i = 1; i < n; ++i)
        if (keys[i - 1] > keys[i]) return LJ_E_INVALID;  // must be sorted ascending
    const double err = (double)max_error;

    // unique keys with first-occurrence ranks (np.unique + searchsorted left)
    std::vector<int64_t> uidx;
    uidx.reserve((size_t)n);
    for (int64_t i = 0; i < n; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) uidx.push_back(i);
    const int64_t s = (int64_t)uidx.size();

    std::vector<int64_t> chosen;
    if (s <= 2) {
        for (int64_t i = 0; i < s; ++i) chosen.push_back(i);
    } else {
        // corridor narrowing: keep the slope window reachable from the base
        // point; when a new point leaves it, the previous point becomes a
        // knot and the window restarts from there
        chosen.push_back(0);
        double bx = (double)keys[uidx[0]], by = (double)uidx[0];
        double hi = std::numeric_limits<double>::infinity(), lo = -hi;
        for (int64_t i = 1; i < s; ++i) {
            const double xi = (double)keys[uidx[i]], yi = (double)uidx[i];
            double dx = xi - bx;
            const double slope = (yi - by) / dx;
            if (slope > hi || slope < lo) {
                chosen.push_back(i - 1);
                bx = (double)keys[uidx[i - 1]];
                by = (double)uidx[i - 1];
                dx = xi - bx;
                hi = (yi + err - by) / dx;
                lo = (yi - err - by) / dx;
            } else {
                const double u = (yi + err - by) / dx, l = (yi - err - by) / dx;
                if (u < hi) hi = u;
                if (l > lo) lo = l;
            }
        }
        if (chosen.back() != s - 1) chosen.push_back(s - 1);
    }
    const int64_t k = (int64_t)chosen.size();
    for (int64_t i = 0; i < k; ++i) {
        keys_out[i] = keys[uidx[chosen[i]]];
        ranks_out[i] = uidx[chosen[i]];
    }
    const int mb = bit_length(keys_out[k - 1]);
    const uint64_t shift = (uint64_t)(mb - radix_bits > 0 ? mb - radix_bits : 0);
    // radix_table[p] = first spline point whose prefix >= p, p in [0, 2^r]
    const int64_t np1 = ((int64_t)1 << radix_bits) + 1;
    int64_t j = 0;
    for (int64_t p = 0; p < np1; ++p) {
        while (j < k && (int64_t)(keys_out[j] >> shift) < p) ++j;
        radix_out[p] = j;
    }
    *npts_out = k;
    *shift_out = shift;
    return LJ_OK;
}

// Exact accelerator for the bounded search of models.py:263-282 (see
// LjSpline.aux in lj_b200.h).  Bucket p covers keys with (k >> shift) == p;
// its sub-table splits that range on the next `bits` key bits.
extern "C" int lj_spline_aux_host(const uint64_t *keys, int64_t npts, const int64_t *radix, int64_t radix_bits,
                                  uint64_t shift, uint64_t *aux, uint32_t *sub, int64_t *sub_len) {
    if (npts < 1 || radix_bits < 1 || radix_bits > 30) return LJ_E_INVALID;
    const int64_t nb = (int64_t)1 << radix_bits;
    int64_t off = 0;
    for (int64_t p = 0; p < nb; ++p) {
        const int64_t lo = radix[p], hi = radix[p + 1], c = hi - lo;
        int bits = 0;
        if (c > 8 && shift > 0) {
            while (((int64_t)1 << bits) < c) ++bits;
            bits += 1;
            if ((uint64_t)bits > shift) bits = (int)shift;
            if (bits > 24) bits = 24;
        }
        if (aux) aux[p] = ((uint64_t)off << 8) | (uint64_t)bits;
        if (bits) {
            const int64_t ns = ((int64_t)1 << bits) + 1;
            if (sub) {
                const uint64_t sub_shift = shift - (uint64_t)bits;
                const uint64_t mask = ((uint64_t)1 << bits) - 1;
                int64_t j = lo;
                for (int64_t q = 0; q < ns; ++q) {
                    // first point in [lo, hi) whose sub-prefix is >= q
                    while (j < hi && (int64_t)((keys[j] >> sub_shift) & mask) < q) ++j;
                    sub[off + q] = (uint32_t)j;
                }
            }
            off += ns;
        }
    }
    *sub_len = off;
    return LJ_OK;
}
