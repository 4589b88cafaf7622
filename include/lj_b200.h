/*
 * lj_b200.h -- C ABI of the B200-native learned-join hot paths.
 *
 * This is the drop-in boundary: the Python mirror of the reference's join
 * entry points (paper_2111_08824_b200/, names as in the reference package
 * `learned_joins`) binds exactly these symbols with ctypes; a reference
 * maintainer would bind the same symbols from their runner registry
 * (INTEGRATION.md).  Reference paths are relative to
 * /root/reference/pkg/src/learned_joins/.
 *
 * Conventions
 *  - Every entry point returns int: LJ_OK (0) or a negative LJ_E_* code;
 *    lj_last_error() returns a thread-local message.  No C++ exception
 *    crosses the ABI.
 *  - All array arguments are CALLER-OWNED DEVICE pointers unless the name
 *    ends in `_host`.  The library never allocates device memory: scratch
 *    comes from a caller workspace sized by the matching *_workspace_bytes.
 *  - Every device call is asynchronous on the caller's `stream`
 *    (cudaStream_t passed as void*).  Calls on distinct streams with
 *    distinct workspaces are re-entrant.
 *  - Keys and payloads are uint64.  A key may not equal LJ_SENTINEL_KEY
 *    (util.py:8,15-22).
 *  - Join results are reduced on device to LjChecksum words
 *    {count, sum, xor, search_steps} of t = R.payload + S.payload mod 2^64
 *    (SURVEY.md 8a); pairs are materialised only through the *_count /
 *    *_collect entry points.
 *  - Model evaluation is bit-identical to the reference's numpy arithmetic:
 *    separate rounded multiply and add (no FMA), round-half-even rint,
 *    x86 float->int64 cast semantics (models.py:112-135,221-248).
 */
#ifndef LJ_B200_H
#define LJ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LJ_OK 0
#define LJ_E_INVALID (-1)   /* bad argument (ValueError in the reference) */
#define LJ_E_CUDA (-2)      /* CUDA runtime error */
#define LJ_E_WORKSPACE (-3) /* workspace too small */
#define LJ_E_NCCL (-4)      /* collective error */
#define LJ_E_UNSUPPORTED (-5)

#define LJ_SENTINEL_KEY 0xFFFFFFFFFFFFFFFFULL

/* One RMI leaf, 32 B = one DRAM sector (models.py:121-124 operands). */
typedef struct LjLeaf {
    double slope;
    double icpt;
    int64_t clamp_lo;
    int64_t clamp_hi;
} LjLeaf;

/* Two-level linear RMI view (models.py:39-143, RecursiveModelIndex). */
typedef struct LjRmi {
    double root_slope;
    double root_icpt;
    int64_t m;              /* fanout: number of leaves */
    int64_t n;              /* trained_len */
    const LjLeaf *leaves;   /* [m] */
    const int64_t *err;     /* [2m] interleaved {err_lo, err_hi}; may be NULL
                               when only positions are needed */
    const double *root_dev; /* optional: the root {slope, intercept} in DEVICE
                               memory (a model fitted on the stream, e.g. by
                               lj_lsj_run); NULL = root_slope / root_icpt.
                               Read by the LSJ kernels (K6-K9). */
} LjRmi;

/* Gapped RMI index view (gapped.py:206-338, GappedRmiIndex). */
typedef struct LjGrmi {
    LjRmi model;
    int64_t n;              /* real entries */
    int64_t L;              /* slot count = round(gap_factor * n) */
    const uint64_t *slots;  /* [2L] interleaved {gkey, gpayload}; gaps hold
                               the nearest real key to the left, payload 0 */
    const uint32_t *bitmap; /* [ceil(L/32)] occupancy bits */
    int32_t payload_nonzero;/* 1 if every real payload != 0: then a slot is
                               real iff its payload != 0 and the bitmap is
                               never read */
    int32_t _pad;
} LjGrmi;

/* RadixSpline view (models.py:150-256, RadixSplineIndex). */
typedef struct LjSpline {
    int64_t npts;           /* spline points K */
    int64_t n;              /* trained_len */
    int64_t max_error;
    int64_t radix_bits;
    uint64_t shift;
    const uint64_t *keys;   /* [K] spline keys */
    const double *ranks;    /* [K] spline ranks as float64 (models.py:228) */
    const uint32_t *radix;  /* [2^radix_bits + 1] radix table */
    /* Optional exact search accelerator (NULL = plain bounded binary
     * search, models.py:263-282): for radix bucket p, aux[p] = (offset << 8)
     * | bits; when bits > 0, sub[offset + q] is the first spline point whose
     * next `bits` key bits (below the radix prefix) are >= q, q in
     * [0, 2^bits].  The first spline key >= k inside [radix[p], radix[p+1])
     * is then searched in [sub[offset+q], sub[offset+q+1]) -- the same
     * index by construction (built by lj_spline_aux_host). */
    const uint64_t *aux;    /* [2^radix_bits] */
    const uint32_t *sub;
    int64_t nsub;           /* length of sub (0 without the accelerator) */
} LjSpline;

/* Spline-keyed chained hash view (learned_hash.py:17-101). */
typedef struct LjSplineHash {
    LjSpline model;
    int64_t n;              /* entries */
    int64_t table_len;      /* P */
    int64_t stride;         /* P / n when n divides P (bucket = pos*stride,
                               only every stride-th bucket can be occupied):
                               starts is then indexed by bucket/stride; else 1 */
    const uint64_t *entries;/* [2n] interleaved {key, payload}, chains in
                               insertion order */
    const uint32_t *starts; /* [P/stride + 1] chain offsets (n < 2^32) */
    /* Optional probe table (NULL: the chains are probed): [2 * nslots]
     * interleaved {key, payload}, the entries in key order at slot
     * max(2 * pos, previous slot + 1), gap slots holding the key to their
     * left with payload 0, a final pair of keys ~0.  Built by
     * lj_spline_slots_plan / _fill when every payload is nonzero; the probe
     * scans forward from slot 2*pos(k) (lj_hash_staged.cu). */
    const uint64_t *slots;
    int64_t nslots;
    int32_t slots_unique;   /* 1 if no two build keys are equal: the probe
                               stops at the first match */
    int32_t _pad;
    const double *segs;     /* [4 * model.npts] per spline point li >= 1:
                               {x0 = f64(key[li-1]), RN(1/max(f64(key[li]) - x0, 1)),
                                rank[li-1], RN(rank[li] - rank[li-1])}
                               (lj_spline_segments); required with slots */
} LjSplineHash;

/* ------------------------------------------------------------ library */
const char *lj_last_error(void);
int lj_version(void);
/* 1 if a CUDA device of compute capability 10.x is visible, else 0. */
int lj_device_ok(void);

/* ---------------------------------------------------------- data prep */
/* data.py:181-192 positional payloads: mix64(i + mix64(seed)) | 1, i in
 * [offset, offset+n). */
int lj_fill_payloads(uint64_t *out, int64_t n, int64_t offset, uint64_t seed, void *stream);
/* out[i] = mix64(seed ^ (offset+i)) (util.py:30-44 finaliser as a counter PRF). */
int lj_fill_mix64(uint64_t *out, int64_t n, int64_t offset, uint64_t seed, void *stream);
/* out[i] = src[mulhi64(mix64(seed ^ (offset+i)), src_n)]: uniform draw with
 * replacement from src (SURVEY 8d C3/C5 counter sampler). */
/* Portable generator draws (include/lj_gen.h; bit-identical to the host
 * generator oracle/lj_gen.c): out[i] = draw offset+i of stream `seed`.
 * lj_fill_normal: standard normal (Box-Muller); lj_fill_lognormal:
 * floor(scale * exp(sigma * normal)) clamped to [0, maxv]; lj_fill_cluster:
 * centres[cluster] + sigma * normal truncated, -1 outside [0, maxv)
 * (ncent a power of two, centres a device array). */
int lj_fill_normal(double *out, int64_t n, int64_t offset, uint64_t seed, void *stream);
int lj_fill_lognormal(int64_t *out, int64_t n, int64_t offset, uint64_t seed, double sigma, double scale,
                      double maxv, void *stream);
int lj_fill_cluster(int64_t *out, int64_t n, int64_t offset, uint64_t seed, const double *centres, int ncent,
                    double sigma, double maxv, void *stream);
int lj_gather_uniform(uint64_t *out, int64_t n, int64_t offset, uint64_t seed, const uint64_t *src,
                      int64_t src_n, void *stream);
/* Stable device sort of (key, payload) pairs by key; used by index builds
 * (data.py:84-86) and the LSJ sample.  */
size_t lj_sort_pairs_workspace_bytes(int64_t n);
int lj_sort_pairs(const uint64_t *keys_in, const uint64_t *pay_in, uint64_t *keys_out,
                  uint64_t *pay_out, int64_t n, int begin_bit, int end_bit, void *ws,
                  size_t ws_bytes, void *stream);

/* ----------------------------------------------------------- RMI (K10) */
/* models.py:57-110 on device over sorted keys.  Outputs: root[2]
 * {slope, icpt}, leaves[m], err[2m].  Deterministic (fixed reduction
 * order).  */
size_t lj_rmi_fit_workspace_bytes(int64_t n, int64_t m);
int lj_rmi_fit(const uint64_t *sorted_keys, int64_t n, int64_t m, double *root, LjLeaf *leaves,
               int64_t *err, void *ws, size_t ws_bytes, void *stream);
/* models.py:126-135 predict_many; any output may be NULL. */
int lj_rmi_predict(const LjRmi *model, const uint64_t *keys, int64_t nk, int64_t *pos,
                   int64_t *lo, int64_t *hi, int64_t *leaf, void *stream);
/* rmi-inlj (baselines.py:96-157): INLJ of S against the
 * SORTED R (r_keys/r_pay, nr) indexed by `model` fitted on it: predict
 * [lo, hi] (models.py:126-135), bounded lower bound counting the reference's
 * bisection steps + one verification compare, whole equal run on a hit.
 * out[4] = {count, sum, xor, search_steps}. */
int lj_rmi_probe(const LjRmi *model, const uint64_t *r_keys, const uint64_t *r_pay, int64_t nr,
                 const uint64_t *s_keys, const uint64_t *s_pay, int64_t ns, uint64_t *out, int accumulate,
                 void *stream);
/* models.py:285-299 partition_index for an RMI. */
int lj_rmi_partition_index(const LjRmi *model, const uint64_t *keys, int64_t nk, int64_t P,
                           int64_t *out, void *stream);

/* ---------------------------------------------------------- GRMI (K11, K1) */
/* gapped.py:221-256: model-based insertion of sorted (key, payload) into
 * L slots + bitmap; *payload_nonzero_dev (1 word) gets the flag. */
size_t lj_grmi_build_workspace_bytes(int64_t n, int64_t L);
int lj_grmi_build(const LjRmi *model, const uint64_t *sorted_keys, const uint64_t *sorted_pay,
                  int64_t n, int64_t L, uint64_t *slots, uint32_t *bitmap,
                  int32_t *payload_nonzero_dev, void *ws, size_t ws_bytes, void *stream);
/* gapped.py:258-261 predicted slot per probe. */
int lj_grmi_predict_slots(const LjGrmi *idx, const uint64_t *keys, int64_t nk, int64_t *out,
                          void *stream);
/* gapped.py:86-160 exponential search from given start slots: out_slot
 * (-1 = absent), out_probes. */
int lj_grmi_search(const LjGrmi *idx, const int64_t *slots0, const uint64_t *keys, int64_t nk,
                   int64_t *out_slot, int64_t *out_probes, void *stream);
/* K1: fused predict + search + run scan + checksum of S against the index.
 * out[4] = {count, sum, xor, search_steps}; zeroed first unless accumulate. */
int lj_grmi_probe(const LjGrmi *idx, const uint64_t *s_keys, const uint64_t *s_pay, int64_t nk,
                  uint64_t *out, int accumulate, void *stream);
/* Materialisation, gapped.py:163-203: per-probe leftmost slot + match
 * count, then (after an exclusive scan of counts into offsets) the R
 * payloads and source indices of every match.  slots0 = start slots of the
 * searches (gapped.py:294 search_from), or NULL to predict them. */
int lj_grmi_count(const LjGrmi *idx, const int64_t *slots0, const uint64_t *keys, int64_t nk,
                  int64_t *lefts, int64_t *counts, int64_t *probes, void *stream);
int lj_grmi_collect(const LjGrmi *idx, const uint64_t *keys, int64_t nk, const int64_t *lefts,
                    const int64_t *offsets, uint64_t *out_pay, int64_t *out_src, void *stream);

/* ------------------------------------------------- Request Buffers (K4) */
/* Request-Buffer analogue (buffers.py:73-150: the paper buffers requests per
 * leaf so that lookups walk the index in order).  Groups S by KEY-RANGE
 * window of 2^shift gapped slots: window w takes the keys k with
 * W[w] < k <= W[w+1], W[w] the gapped key at slot w * 2^shift, so every
 * key's lower bound lies inside its window's slot range.  The window is
 * found from the model's predicted slot (gapped.py:258-261) and corrected by
 * the neighbouring window keys.  bins = lj_leaf_bucket_bins(L) <= 2048.
 * Output: pairs_out (capacity lj_leaf_bucket_capacity(nk, L) records) of
 * interleaved {key, payload}; reg_out[lj_leaf_bucket_regions(L)] =
 * {rstart[0..bins], rend[0..bins), overflow}: window w's records are
 * [rstart[w], rend[w]), then `overflow` records of any window follow at
 * rstart[bins].  When the staged probe applies, one pass fills regions sized
 * from a 1/16 sample (gaps after each window, rare overflow); otherwise two
 * passes produce the exact, gap-free layout (overflow 0).  Order inside a
 * window is unspecified. */
int lj_leaf_bucket_bins(int64_t L);
int lj_leaf_bucket_regions(int64_t L);
int64_t lj_leaf_bucket_capacity(int64_t nk, int64_t L);
size_t lj_leaf_bucket_workspace_bytes(int64_t nk, int64_t L);
int lj_leaf_bucket(const LjGrmi *idx, const uint64_t *keys, const uint64_t *pay, int64_t nk,
                   uint64_t *pairs_out, int64_t *reg_out, void *ws, size_t ws_bytes, void *stream);
/* K1 over the output of lj_leaf_bucket: each CTA stages a window's real
 * entries in shared memory and searches there, the overflow records take the
 * plain K1; results and search_steps equal lj_grmi_probe's (the reference's
 * probe count follows from the predicted slot and the key's position).  ws:
 * 8 bytes of device scratch (work counter).  accumulate: bit 0 = add to out
 * instead of overwriting it; bit 1 = leave the reference's probe counter
 * (out[3]) and with it the model evaluation out (the staged search finds
 * the lower bound through the window's radix table; an ablation). */
int lj_grmi_probe_bucketed(const LjGrmi *idx, const uint64_t *s_pairs, const int64_t *reg, void *ws, uint64_t *out,
                           int accumulate, void *stream);
/* The window staging of the probe above, precomputed once per index: for
 * every window the compacted real keys, slot offsets, radix table and RMI
 * leaves in the probe's shared-memory layout (+ a 32-B header), so a CTA
 * stages a window with four bulk copies instead of rebuilding it.  0 bytes:
 * the index is not probed through staged windows.  The image is derived
 * from the index alone (rebuild it if the index changes). */
size_t lj_grmi_stage_image_bytes(const LjGrmi *idx);
int lj_grmi_stage_image_build(const LjGrmi *idx, void *img, size_t bytes, void *stream);
int lj_grmi_probe_bucketed_img(const LjGrmi *idx, const uint64_t *s_pairs, const int64_t *reg, void *ws,
                               const void *img, uint64_t *out, int accumulate, void *stream);
/* K1 over interleaved {key, payload} probe records (e.g. bucketed S). */
int lj_grmi_probe_pairs(const LjGrmi *idx, const uint64_t *s_pairs, int64_t nk, uint64_t *out, int accumulate,
                        void *stream);

/* ------------------------------------------------- RadixSpline (K5) */
/* models.py:171-219 greedy-corridor fit on HOST sorted keys (sequential by
 * nature).  keys_out/ranks_out hold up to n entries, radix_out 2^r+1.  */
int lj_spline_fit_host(const uint64_t *sorted_keys_host, int64_t n, int64_t max_error,
                       int64_t radix_bits, uint64_t *keys_out_host, int64_t *ranks_out_host,
                       int64_t *radix_out_host, int64_t *npts_out, uint64_t *shift_out);
/* The same fit on the DEVICE over device-sorted keys (speculative chunks
 * spliced where they converge, repaired in order on the device when they do
 * not): knot_keys/knot_ranks hold up to n entries, radix_out 2^r+1 (all
 * device); *npts_out / *shift_out on the host.  Identical knots. */
size_t lj_spline_fit_workspace_bytes(int64_t n);
int lj_spline_fit(const uint64_t *sorted_keys, int64_t n, int64_t max_error, int64_t radix_bits,
                  uint64_t *knot_keys, int64_t *knot_ranks, int64_t *radix_out, int64_t *npts_out,
                  uint64_t *shift_out, void *ws, size_t ws_bytes, void *stream);
/* Build the LjSpline.aux/sub accelerator on the host: every radix bucket
 * holding more than 8 spline points gets ceil(log2(count)) + 1 extra key
 * bits.  Call with sub_host = NULL to get the required sub length. */
int lj_spline_aux_host(const uint64_t *keys_host, int64_t npts, const int64_t *radix_host, int64_t radix_bits,
                       uint64_t shift, uint64_t *aux_host, uint32_t *sub_host, int64_t *sub_len);
int lj_spline_predict(const LjSpline *model, const uint64_t *keys, int64_t nk, int64_t *pos,
                      int64_t *lo, int64_t *hi, void *stream);
int lj_spline_partition_index(const LjSpline *model, const uint64_t *keys, int64_t nk, int64_t P,
                              int64_t *out, void *stream);
/* learned_hash.py:55-66: chains by partition_index(model, key, P), stable. */
size_t lj_spline_hash_build_workspace_bytes(int64_t n, int64_t P);
int lj_spline_hash_build(const LjSpline *model, const uint64_t *keys, const uint64_t *pay,
                         int64_t n, int64_t P, uint64_t *entries, uint32_t *starts, void *ws,
                         size_t ws_bytes, void *stream);
/* K5: learned_hash.py:81-96 fused with the checksum. */
int lj_spline_hash_probe(const LjSplineHash *idx, const uint64_t *s_keys, const uint64_t *s_pay,
                         int64_t nk, uint64_t *out, int accumulate, void *stream);
/* Request-Buffer analogue for K5: group S by a window of predicted
 * positions (<= 2048 windows, shared-memory-privatised partition) so that
 * the probe walks chain offsets and entries window by window (cached). */
size_t lj_spline_hash_bucket_workspace_bytes(int64_t nk, int64_t n);
int lj_spline_hash_bucket(const LjSplineHash *idx, const uint64_t *keys, const uint64_t *pay, int64_t nk,
                          uint64_t *pairs_out, int64_t *starts_out, void *ws, size_t ws_bytes, void *stream);
int lj_spline_hash_probe_grouped(const LjSplineHash *idx, const uint64_t *s_pairs, int64_t nk, uint64_t *out,
                                 int accumulate, void *stream);
/* One-pass variant (the default of the buffered runner): S grouped by
 * approximate-position window into est-capacity regions (lj_leaf_bucket's
 * layout: reg[2*bins+2] = region starts, region ends, overflow count; gap
 * records carry the reserved key 2^64-1); pairs_out holds
 * lj_spline_hash_bucket_capacity(nk, n) records; columns 16-B aligned. */
/* Probe table of a spline-hash index (LjSplineHash.slots), from the build
 * keys sorted ascending with their payloads: plan writes plan[0] = the slot
 * count to allocate and plan[1] = the number of zero payloads (a table is
 * only valid when it is 0) to DEVICE memory; fill (same workspace, after
 * plan) writes the 2*nslots words.  Index build, untimed like the
 * reference's (learned_hash.py:35-66). */
size_t lj_spline_slots_workspace_bytes(int64_t n);
int lj_spline_segments(const LjSpline *model, double *segs, void *stream);
int lj_spline_slots_plan(const LjSpline *model, const uint64_t *sorted_keys, const uint64_t *sorted_pay, int64_t n,
                         int64_t *plan, void *ws, size_t ws_bytes, void *stream);
int lj_spline_slots_fill(const uint64_t *sorted_keys, const uint64_t *sorted_pay, int64_t n, uint64_t *slots,
                         int64_t nslots, void *ws, size_t ws_bytes, void *stream);
int64_t lj_spline_hash_bucket_bins(int64_t n);
int64_t lj_spline_hash_bucket_capacity(int64_t nk, int64_t n);
size_t lj_spline_hash_bucket_est_workspace_bytes(const LjSplineHash *idx, int64_t nk);
int lj_spline_hash_bucket_est(const LjSplineHash *idx, const uint64_t *keys, const uint64_t *pay, int64_t nk,
                              uint64_t *pairs_out, int64_t *reg_out, void *ws, size_t ws_bytes, void *stream);
/* K5 over those regions, handed out to the CTAs in record order by a chunk
 * counter (ws >= 8 bytes), so every SM works on the same few windows and
 * their chain offsets and entries stay in L2. */
int lj_spline_hash_probe_regions(const LjSplineHash *idx, const uint64_t *s_pairs, const int64_t *reg,
                                 int64_t nbins, void *ws, size_t ws_bytes, uint64_t *out, int accumulate,
                                 void *stream);
int lj_spline_hash_count(const LjSplineHash *idx, const uint64_t *keys, int64_t nk,
                         int64_t *counts, void *stream);
int lj_spline_hash_collect(const LjSplineHash *idx, const uint64_t *keys, int64_t nk,
                           const int64_t *offsets, uint64_t *out_pay, int64_t *out_src,
                           void *stream);

/* ------------------------------------------------------- LSJ (K6-K9) */
/* lsj.py:95-130 sample: one key per stratum [j*n/total, (j+1)*n/total) at a
 * counter-drawn offset, sorted (results-neutral stand-in for numpy's
 * Generator.choice; the model only steers bucket sizes). */
size_t lj_lsj_sample_workspace_bytes(int64_t total);
int lj_lsj_sample(const uint64_t *keys, int64_t n, int64_t total, uint64_t seed, uint64_t *sample_sorted,
                  void *ws, size_t ws_bytes, void *stream);
/* ... over keys[i * stride] (stride 2: interleaved {key, payload} records). */
int lj_lsj_sample_strided(const uint64_t *keys, int64_t stride, int64_t n, int64_t total, uint64_t seed,
                          uint64_t *sample_sorted, void *ws, size_t ws_bytes, void *stream);
/* An LSJ relation model: the sample-fitted RMI plus equi-depth bins over its
 * predicted positions: bin(key) = table[pos(key)], pb[j] = first predicted
 * position of bin j (pb[nbins] = trained_len).  Monotone in the key. */
typedef struct LjLsjModel {
    LjRmi rmi;
    int64_t nbins;            /* <= 32768 */
    const int64_t *pb;        /* [nbins+1] */
    const uint32_t *table;    /* [rmi.n] */
    const uint64_t *sample;   /* sorted sample the model was fitted on, or NULL;
                                 when present it also places the split points
                                 of the sort's second level (equi-depth) */
    int64_t nsample;
} LjLsjModel;
/* Bin boundaries at equally spaced ranks of the sorted sample. */
size_t lj_lsj_bins_workspace_bytes(int64_t total);
int lj_lsj_bins(const LjRmi *model, const uint64_t *sample_sorted, int64_t total, int64_t nbins, int64_t *pb,
                uint32_t *table, void *ws, size_t ws_bytes, void *stream);
/* Table from explicit bounds (pb[j] = ceil(j*n/nbins) gives exactly the
 * reference's partition_index buckets at scale nbins, models.py:297). */
int lj_lsj_bins_from_bounds(const int64_t *pb, int64_t nbins, int64_t trained_len, uint32_t *table, void *stream);
/* lsj.py:133-209 / 258-263: K6 histogram + K7 scatter of (key, payload)
 * into the model's bins, shared-memory privatised (no per-tuple global
 * atomics).  pairs[2n] interleaved out; starts[nbins+1] bucket bounds. */
size_t lj_lsj_partition_workspace_bytes(int64_t n, int64_t nbins);
int lj_lsj_partition(const LjLsjModel *model, const uint64_t *keys, const uint64_t *pay, int64_t n,
                     uint64_t *pairs, int64_t *starts, void *ws, size_t ws_bytes, void *stream);
/* The same partition in ONE pass (no exact counting pass): a 1/16 strided
 * sample of the keys sizes a region per bin (estimate * 17/16 + 4096), the
 * scatter claims run by run.  pairs: lj_lsj_partition_regions_capacity(n,
 * nbins) records; reg[2 nbins + 2]: bin b = records [reg[b], reg[nbins + 1 +
 * b]) of pairs (gaps between the bins), reg[2 nbins + 1] = 0.  Should a
 * region overflow (the slack is many standard deviations of the estimate),
 * the exact two-pass partition runs over the same buffer instead -- its
 * kernels are always enqueued and return at once otherwise, so the decision
 * stays on the device.  Needs 16-B aligned columns, nbins <= 2048, n < 2^32.
 * lj_lsj_sort_regions sorts such regions into the dense pairs_out and
 * returns the bins' dense starts[nbins+1] (what lj_lsj_partition's starts
 * are for lj_lsj_sort; lj_lsj_join takes them as r_starts). */
int64_t lj_lsj_partition_regions_capacity(int64_t n, int64_t nbins);
size_t lj_lsj_partition_regions_workspace_bytes(int64_t n, int64_t nbins);
int lj_lsj_partition_regions(const LjLsjModel *model, const uint64_t *keys, const uint64_t *pay, int64_t n,
                             uint64_t *pairs, int64_t *reg, void *ws, size_t ws_bytes, void *stream);
/* ... reading the relation as n interleaved 16-B records {key, payload}
 * (16-B aligned) in place -- the form the range shuffle of the distributed
 * LSJ delivers (lsj.py:161-173: the per-worker ranges are contiguous record
 * runs); same output, capacity and workspace. */
int lj_lsj_partition_regions_rec(const LjLsjModel *model, const uint64_t *records, int64_t n, uint64_t *pairs,
                                 int64_t *reg, void *ws, size_t ws_bytes, void *stream);
/* The exact key-range bin function the partition passes evaluate in
 * shared memory (lj_keybin.cuh): bins[i] = #{ j in [1, nbins) :
 * bounds[j] <= keys[i] } for non-decreasing bounds (bounds[0] ignored).
 * lj_lsj_key_bounds: the model's bins as key boundaries (bounds[j] = first
 * key whose predicted position reaches pb[j]).  ws >= lj_keybin_workspace_bytes. */
size_t lj_keybin_workspace_bytes(int64_t nbins);
int lj_keybin_eval(const uint64_t *bounds, int64_t nbins, const uint64_t *keys, int64_t nk, uint32_t *bins,
                   void *ws, size_t ws_bytes, void *stream);
int lj_lsj_key_bounds(const LjLsjModel *model, uint64_t *bounds, void *ws, size_t ws_bytes, void *stream);
/* Range shuffle of the distributed LSJ fused with its partition (the
 * shared model's nbins = destination ranks): _count -> exact counts[nbins+1]
 * (device) and every tuple's destination kept in ws; _scatter (same ws) ->
 * every tuple written to bases[dest] + its claimed position, bases[] =
 * ABSOLUTE record indices (address / 16) of this rank's region in each
 * destination's receive buffer (symmetric memory: NVLink P2P stores). */
size_t lj_lsj_shuffle_workspace_bytes(int64_t n, int64_t nbins);
int lj_lsj_shuffle_count(const LjLsjModel *model, const uint64_t *keys, const uint64_t *pay, int64_t n,
                         int64_t *counts, void *ws, size_t ws_bytes, void *stream);
int lj_lsj_shuffle_scatter(const LjLsjModel *model, const uint64_t *keys, const uint64_t *pay, int64_t n,
                           const int64_t *bases, void *ws, size_t ws_bytes, void *stream);
/* lsj.py:242-286 per-bucket sort (K8, model-placed, shared memory) from the
 * partitioned pairs_in into pairs_out (fully sorted, bucket ranges kept).
 * Asynchronous on the stream (no host readback): sub-buckets above the
 * per-CTA capacity go to a one-CTA-per-SM instance, the rare ones above
 * that to a global-memory chunk sort + merge, through device-side lists.
 * stats (device int64[4], or NULL) = {sub-buckets above the main capacity,
 * bitonic fallbacks, sorted by the big instance, sorted in global memory}. */
size_t lj_lsj_sort_workspace_bytes(int64_t n, int64_t nbins);
int lj_lsj_sort(const LjLsjModel *model, const uint64_t *pairs_in, uint64_t *pairs_out, int64_t n,
                const int64_t *starts, void *ws, size_t ws_bytes, int64_t *stats, void *stream);
int lj_lsj_sort_regions(const LjLsjModel *model, const uint64_t *pairs_in, uint64_t *pairs_out, int64_t n,
                        const int64_t *reg, int64_t *starts_out, void *ws, size_t ws_bytes, int64_t *stats,
                        void *stream);
/* Reference bucket bounds at scale P of a sorted relation (the
 * partition_index buckets of lsj.py:302-305, for its counters). */
int lj_lsj_ref_bounds(const LjRmi *model, const uint64_t *sorted_pairs, int64_t n, int64_t P, int64_t *bounds,
                      void *stream);
/* lsj.py:316-370 chunked join (K9) of sorted S against sorted R through R's
 * model and bucket bounds: every S tile's exact R slice is found first (one
 * thread per tile, into ws), then tile and slice are merged in shared
 * memory.  mode 0: out[4] checksum; mode 1: counts[ns]; mode 2: pairs at
 * offsets[ns] into out_pr/out_ps. */
/* lsj.py:373-405 lsj_join in ONE call, asynchronous on the stream, from one
 * caller workspace (lj_lsj_run_workspace_bytes): per relation the sample
 * (seed for R, seed ^ 0x5DEECE66D for S, lsj.py:388-391), the RMI fit with
 * fanout min(1000, samples // 8), equi-depth bins, partition (K6/K7), the
 * split + model-placed sort (K8); then the chunked merge-join (K9) of S
 * against R through R's model.  out[4] (device) = {count, sum, xor, 0} of
 * R.payload + S.payload over the equal-key pairs.  The same words as the
 * Python orchestration (lsj.lsj_join) and the reference's lsj_join. */
size_t lj_lsj_run_workspace_bytes(int64_t nr, int64_t ns, double sample_rate);
int lj_lsj_run(const uint64_t *r_keys, const uint64_t *r_pay, int64_t nr, const uint64_t *s_keys,
               const uint64_t *s_pay, int64_t ns, double sample_rate, uint64_t seed, uint64_t *out, void *ws,
               size_t ws_bytes, void *stream);
/* ... with both relations held as interleaved 16-B records {key, payload}
 * (16-B aligned, < 2^32 - 1 each): what a range shuffle delivers; same
 * workspace, same result words. */
int lj_lsj_run_rec(const uint64_t *r_records, int64_t nr, const uint64_t *s_records, int64_t ns, double sample_rate,
                   uint64_t seed, uint64_t *out, void *ws, size_t ws_bytes, void *stream);
size_t lj_lsj_join_workspace_bytes(int64_t ns);
int lj_lsj_join(const LjLsjModel *model_r, const uint64_t *r_pairs, int64_t nr, const int64_t *r_starts,
                const uint64_t *s_pairs, int64_t ns, int mode, int64_t *counts, const int64_t *offsets,
                uint64_t *out_pr, uint64_t *out_ps, uint64_t *out, int accumulate, void *ws, size_t ws_bytes,
                void *stream);

/* ---------------------------------------------- multi-GPU (one process)
 * Single-process calls over ndev devices with one NCCL communicator and one
 * stream per device (ncclComm_t / cudaStream_t passed as void*); NCCL is
 * bound at run time (dlopen libnccl.so.2, the copy already loaded in the
 * process if any).  lj_nccl_available() = 1 if it was found. */
int lj_nccl_available(void);
/* ncclCommInitAll over devs (comms[ndev] out) / ncclCommDestroy. */
int lj_nccl_comm_init_all(int ndev, const int *devs, void **comms);
int lj_nccl_comm_destroy(void *comm);
/* The checksum reduction: words[d] = device int64[4]
 * {count, sum, xor, ...} of device d; afterwards every words[d] holds the
 * global {count, sum mod 2^64, xor}.  ws[d] >= lj_reduce_sums_workspace_bytes(nranks). */
size_t lj_reduce_sums_workspace_bytes(int nranks);
int lj_reduce_sums(int ndev, const int *devs, void *const *comms, void *const *streams, uint64_t *const *words,
                   void *const *ws);
/* The distributed learned sort-join (lsj.py:373-405, workers = devices):
 * R / S shards per device, a shared model on the union of the R samples,
 * range partition, ncclSend/ncclRecv exchange, lj_lsj_run per device,
 * lj_reduce_sums.  cap_r / cap_s bound the tuples a device receives (the
 * workspace is sized by them); recv_counts (host int64[2*ndev] or NULL)
 * reports what each device received -- LJ_E_WORKSPACE when above the caps.
 * Reads the partition counts back once (NCCL's exchange sizes are host
 * values).  out[d] = device int64[4]: the global checksum on every device. */
size_t lj_lsj_run_multi_workspace_bytes(int ndev, int64_t nr_local, int64_t ns_local, int64_t nr_total,
                                        int64_t cap_r, int64_t cap_s, double sample_rate);
int lj_lsj_run_multi(int ndev, const int *devs, void *const *comms, void *const *streams,
                     const uint64_t *const *r_keys, const uint64_t *const *r_pay, const int64_t *nr,
                     const uint64_t *const *s_keys, const uint64_t *const *s_pay, const int64_t *ns,
                     int64_t cap_r, int64_t cap_s, double sample_rate, uint64_t seed, uint64_t *const *out,
                     void *const *ws, const size_t *ws_bytes, int64_t *recv_counts);

#ifdef __cplusplus
}
#endif
#endif /* LJ_B200_H */
