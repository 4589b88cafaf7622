// lj_multi.cu -- single-process multi-GPU entry points over NCCL (SURVEY
// 8(b): `(ndev, devs, comms, streams)` calls from one host thread).
//
//  * lj_reduce_sums: the INLJ / LSJ checksum reduction -- count and sum by
//    one ncclAllReduce(sum, uint64) (the sum wraps mod 2^64 exactly like the
//    checksum's), xor by one ncclAllGather of the word and a fold on the
//    device (NCCL has no xor reduction).
//  * lj_lsj_run_multi: the distributed learned sort-join (lsj.py:373-405 with
//    workers = GPUs): every device samples its R shard, the samples are
//    broadcast to every device and sorted there, one RMI + ndev equi-depth
//    range bins are fitted on that global sample (deterministic kernels: the
//    same model everywhere), both relations are range-partitioned by it
//    (K6/K7), the ndev x ndev runs are exchanged with grouped ncclSend /
//    ncclRecv (the path's one exchange step), each device joins its key
//    range with lj_lsj_run, and lj_reduce_sums combines the words.
//
// NCCL is bound at run time (dlopen of libnccl.so.2, reusing the copy the
// process already loaded -- e.g. torch's): the library does not link it,
// and lj_nccl_available() reports whether it was found.  The exchange
// sizes are host values in NCCL, so lj_lsj_run_multi reads the partition
// counts back once (the only synchronisation); everything else is enqueued
// on the per-device streams.
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "lj_common.cuh"

namespace lj {

struct NcclApi {
    bool ok = false;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGetErrorString) err_str = nullptr;
};

static NcclApi &nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
#define LJ_SYM(f, s) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, s))
        LJ_SYM(all_reduce, "ncclAllReduce");
        LJ_SYM(all_gather, "ncclAllGather");
        LJ_SYM(broadcast, "ncclBroadcast");
        LJ_SYM(send, "ncclSend");
        LJ_SYM(recv, "ncclRecv");
        LJ_SYM(group_start, "ncclGroupStart");
        LJ_SYM(group_end, "ncclGroupEnd");
        LJ_SYM(comm_count, "ncclCommCount");
        LJ_SYM(init_all, "ncclCommInitAll");
        LJ_SYM(destroy, "ncclCommDestroy");
        LJ_SYM(err_str, "ncclGetErrorString");
#undef LJ_SYM
        a.ok = a.all_reduce && a.all_gather && a.broadcast && a.send && a.recv && a.group_start && a.group_end &&
               a.comm_count && a.init_all && a.destroy && a.err_str;
        return a;
    }();
    return api;
}

static int nccl_fail(ncclResult_t r, const char *what) {
    set_error(std::string("NCCL error in ") + what + ": " + (nccl().err_str ? nccl().err_str(r) : "?"));
    return LJ_E_NCCL;
}

#define LJ_NC(call)                                          \
    do {                                                     \
        ncclResult_t _r = (call);                            \
        if (_r != ncclSuccess) return nccl_fail(_r, #call);  \
    } while (0)

static size_t alm(size_t v) { return (v + 255) & ~(size_t)255; }

__global__ void k_fold_xor(const u64 *xs, int nranks, u64 *words) {
    u64 x = 0;
    for (int r = 0; r < nranks; ++r) x ^= xs[r];
    words[2] = x;
}

struct DevGuard {
    int prev = 0;
    DevGuard() { cudaGetDevice(&prev); }
    ~DevGuard() { cudaSetDevice(prev); }
};

}  // namespace lj

using namespace lj;

extern "C" {

int lj_nccl_available(void) { return nccl().ok ? 1 : 0; }

int lj_nccl_comm_init_all(int ndev, const int *devs, void **comms) {
    LJ_REQUIRE(ndev >= 1 && devs && comms, "need ndev >= 1, devs and comms");
    if (!nccl().ok) {
        set_error("NCCL (libnccl.so.2) is not available");
        return LJ_E_UNSUPPORTED;
    }
    std::vector<ncclComm_t> c((size_t)ndev);
    LJ_NC(nccl().init_all(c.data(), ndev, devs));
    for (int d = 0; d < ndev; ++d) comms[d] = c[(size_t)d];
    return LJ_OK;
}

int lj_nccl_comm_destroy(void *comm) {
    if (!comm) return LJ_OK;
    if (!nccl().ok) return LJ_E_UNSUPPORTED;
    LJ_NC(nccl().destroy(reinterpret_cast<ncclComm_t>(comm)));
    return LJ_OK;
}

size_t lj_reduce_sums_workspace_bytes(int nranks) { return alm(sizeof(u64) * (size_t)(nranks > 0 ? nranks : 1)); }

int lj_reduce_sums(int ndev, const int *devs, void *const *comms, void *const *streams, uint64_t *const *words,
                   void *const *ws) {
    LJ_REQUIRE(ndev >= 1 && devs && comms && streams && words && ws, "null argument");
    if (!nccl().ok) {
        set_error("NCCL (libnccl.so.2) is not available");
        return LJ_E_UNSUPPORTED;
    }
    DevGuard g;
    int nranks = 0;
    LJ_NC(nccl().comm_count(reinterpret_cast<ncclComm_t>(comms[0]), &nranks));
    LJ_NC(nccl().group_start());
    for (int d = 0; d < ndev; ++d) {
        LJ_CK(cudaSetDevice(devs[d]));
        ncclComm_t c = reinterpret_cast<ncclComm_t>(comms[d]);
        cudaStream_t st = as_stream(streams[d]);
        LJ_NC(nccl().all_reduce(words[d], words[d], 2, ncclUint64, ncclSum, c, st));
        LJ_NC(nccl().all_gather(words[d] + 2, ws[d], 1, ncclUint64, c, st));
    }
    LJ_NC(nccl().group_end());
    for (int d = 0; d < ndev; ++d) {
        LJ_CK(cudaSetDevice(devs[d]));
        k_fold_xor<<<1, 1, 0, as_stream(streams[d])>>>((const u64 *)ws[d], nranks, words[d]);
        LJ_CK_LAUNCH();
    }
    return LJ_OK;
}

static int64_t rate_total(int64_t n, double rate) {
    return n > 0 ? std::max<int64_t>(1, (int64_t)nearbyint(rate * (double)n)) : 0;
}

// a bound of the gathered sample size sum_d max(1, rint(rate * nr_d))
static int64_t ts_bound(int64_t nr_total, int ndev, double rate) {
    return (int64_t)nearbyint(rate * (double)nr_total) + 2 * (int64_t)ndev + 2;
}

size_t lj_lsj_run_multi_workspace_bytes(int ndev, int64_t nr_local, int64_t ns_local, int64_t nr_total,
                                        int64_t cap_r, int64_t cap_s, double sample_rate) {
    const int64_t ts = ts_bound(nr_total, ndev, sample_rate);
    const int64_t fan = std::min<int64_t>(1000, std::max<int64_t>(1, ts / 8));
    size_t sort_t = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, sort_t, (const u64 *)nullptr, (u64 *)nullptr, (int64_t)ts);
    size_t scr = std::max({lj_lsj_sample_workspace_bytes(std::max<int64_t>(1, ts)), lj_rmi_fit_workspace_bytes(ts, fan),
                           lj_lsj_bins_workspace_bytes(ts), lj_lsj_partition_workspace_bytes(nr_local, ndev),
                           lj_lsj_partition_workspace_bytes(ns_local, ndev), alm(sort_t)});
    return 2 * alm(sizeof(u64) * (size_t)ts) +                                           // gathered + sorted sample
           alm(sizeof(double) * 2) + alm(sizeof(LjLeaf) * (size_t)fan) + alm(sizeof(i64) * 2 * (size_t)fan) +
           alm(sizeof(i64) * (size_t)(ndev + 1)) + alm(sizeof(u32) * (size_t)ts) +        // model + bins
           alm(16 * (size_t)std::max<int64_t>(nr_local, 1)) + alm(16 * (size_t)std::max<int64_t>(ns_local, 1)) +
           2 * alm(sizeof(i64) * (size_t)(ndev + 1)) +                                   // partitioned + starts
           alm(16 * (size_t)cap_r) + alm(16 * (size_t)cap_s) +                            // received runs
           alm(scr) + alm(lj_lsj_run_workspace_bytes(cap_r, cap_s, sample_rate)) +
           lj_reduce_sums_workspace_bytes(ndev) + 1024;
}

int lj_lsj_run_multi(int ndev, const int *devs, void *const *comms, void *const *streams,
                     const uint64_t *const *r_keys, const uint64_t *const *r_pay, const int64_t *nr,
                     const uint64_t *const *s_keys, const uint64_t *const *s_pay, const int64_t *ns,
                     int64_t cap_r, int64_t cap_s, double sample_rate, uint64_t seed, uint64_t *const *out,
                     void *const *ws, const size_t *ws_bytes, int64_t *recv_counts) {
    LJ_REQUIRE(ndev >= 1 && devs && comms && streams && out && ws && ws_bytes, "null argument");
    LJ_REQUIRE(sample_rate > 0.0 && sample_rate <= 1.0, "sample_rate must be in (0, 1]");
    if (!nccl().ok) {
        set_error("NCCL (libnccl.so.2) is not available");
        return LJ_E_UNSUPPORTED;
    }
    NcclApi &N = nccl();
    DevGuard g;
    int64_t nr_total = 0;
    std::vector<int64_t> tot((size_t)ndev), soff((size_t)ndev + 1, 0);
    for (int d = 0; d < ndev; ++d) {
        nr_total += nr[d];
        tot[(size_t)d] = rate_total(nr[d], sample_rate);
        soff[(size_t)d + 1] = soff[(size_t)d] + tot[(size_t)d];
    }
    const int64_t ts = soff[(size_t)ndev];
    LJ_REQUIRE(ts >= 1, "R is empty on every device");
    const int64_t fan = std::min<int64_t>(1000, std::max<int64_t>(1, ts / 8));
    struct Lay {
        u64 *gath, *samp;
        double *root;
        LjLeaf *leaves;
        i64 *err, *pb;
        u32 *table;
        u64 *pr, *ps;
        i64 *str, *sts;
        ulonglong2 *rr, *rs;
        char *scr, *run, *red;
        size_t scr_b, run_b;
    };
    std::vector<Lay> L((size_t)ndev);
    std::vector<LjRmi> rmi((size_t)ndev);
    std::vector<LjLsjModel> md((size_t)ndev);
    for (int d = 0; d < ndev; ++d) {
        if (ws_bytes[d] < lj_lsj_run_multi_workspace_bytes(ndev, nr[d], ns[d], nr_total, cap_r, cap_s, sample_rate)) {
            set_error("lj_lsj_run_multi: workspace too small");
            return LJ_E_WORKSPACE;
        }
        char *p = (char *)(((uintptr_t)ws[d] + 255) & ~(uintptr_t)255);
        auto take = [&](size_t b) {
            char *r = p;
            p += alm(b);
            return r;
        };
        Lay &l = L[(size_t)d];
        const int64_t tb = ts_bound(nr_total, ndev, sample_rate);
        const int64_t fb = std::min<int64_t>(1000, std::max<int64_t>(1, tb / 8));
        l.gath = (u64 *)take(sizeof(u64) * (size_t)tb);
        l.samp = (u64 *)take(sizeof(u64) * (size_t)tb);
        l.root = (double *)take(sizeof(double) * 2);
        l.leaves = (LjLeaf *)take(sizeof(LjLeaf) * (size_t)fb);
        l.err = (i64 *)take(sizeof(i64) * 2 * (size_t)fb);
        l.pb = (i64 *)take(sizeof(i64) * (size_t)(ndev + 1));
        l.table = (u32 *)take(sizeof(u32) * (size_t)tb);
        l.pr = (u64 *)take(16 * (size_t)std::max<int64_t>(nr[d], 1));
        l.ps = (u64 *)take(16 * (size_t)std::max<int64_t>(ns[d], 1));
        l.str = (i64 *)take(sizeof(i64) * (size_t)(ndev + 1));
        l.sts = (i64 *)take(sizeof(i64) * (size_t)(ndev + 1));
        l.rr = (ulonglong2 *)take(16 * (size_t)cap_r);
        l.rs = (ulonglong2 *)take(16 * (size_t)cap_s);
        l.red = take(lj_reduce_sums_workspace_bytes(ndev));
        l.run_b = lj_lsj_run_workspace_bytes(cap_r, cap_s, sample_rate);
        l.run = take(l.run_b);
        l.scr = p;
        l.scr_b = ws_bytes[d] - (size_t)(p - (char *)ws[d]);
        rmi[(size_t)d] = LjRmi{0.0, 0.0, fan, ts, l.leaves, l.err, l.root};
        md[(size_t)d] = LjLsjModel{rmi[(size_t)d], ndev, l.pb, l.table, l.samp, ts};
    }
    // (1) every device samples its R shard (the per-rank seed keeps the
    // shards' strata independent), the samples meet on every device
    for (int d = 0; d < ndev; ++d) {
        LJ_CK(cudaSetDevice(devs[d]));
        if (tot[(size_t)d] > 0) {
            const int rc = lj_lsj_sample(r_keys[d], nr[d], tot[(size_t)d], seed ^ ((uint64_t)d << 48),
                                         L[(size_t)d].gath + soff[(size_t)d], L[(size_t)d].scr, L[(size_t)d].scr_b,
                                         streams[d]);
            if (rc) return rc;
        }
    }
    LJ_NC(N.group_start());
    for (int src = 0; src < ndev; ++src) {
        if (!tot[(size_t)src]) continue;
        for (int d = 0; d < ndev; ++d) {
            LJ_CK(cudaSetDevice(devs[d]));
            // the send buffer is read on the root only
            LJ_NC(N.broadcast(d == src ? L[(size_t)src].gath + soff[(size_t)src] : L[(size_t)d].gath + soff[(size_t)src],
                              L[(size_t)d].gath + soff[(size_t)src],
                              (size_t)tot[(size_t)src], ncclUint64, src, reinterpret_cast<ncclComm_t>(comms[d]),
                              as_stream(streams[d])));
        }
    }
    LJ_NC(N.group_end());
    // (2) the same sorted global sample, RMI and ndev range bins everywhere
    for (int d = 0; d < ndev; ++d) {
        LJ_CK(cudaSetDevice(devs[d]));
        Lay &l = L[(size_t)d];
        cudaStream_t st = as_stream(streams[d]);
        size_t t = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, t, (const u64 *)l.gath, l.samp, (int64_t)ts);
        LJ_CK(cub::DeviceRadixSort::SortKeys(l.scr, t, (const u64 *)l.gath, l.samp, (int64_t)ts, 0, 64, st));
        int rc = lj_rmi_fit(l.samp, ts, fan, l.root, l.leaves, l.err, l.scr, l.scr_b, streams[d]);
        if (rc) return rc;
        rc = lj_lsj_bins(&rmi[(size_t)d], l.samp, ts, ndev, l.pb, l.table, l.scr, l.scr_b, streams[d]);
        if (rc) return rc;
        // (3) both relations range-partitioned by the shared model
        rc = lj_lsj_partition(&md[(size_t)d], r_keys[d], r_pay[d], nr[d], l.pr, l.str, l.scr, l.scr_b, streams[d]);
        if (rc) return rc;
        rc = lj_lsj_partition(&md[(size_t)d], s_keys[d], s_pay[d], ns[d], l.ps, l.sts, l.scr, l.scr_b, streams[d]);
        if (rc) return rc;
    }
    // the exchange sizes (NCCL takes host counts): the one readback
    std::vector<int64_t> hr((size_t)ndev * (ndev + 1)), hs((size_t)ndev * (ndev + 1));
    for (int d = 0; d < ndev; ++d) {
        LJ_CK(cudaSetDevice(devs[d]));
        cudaStream_t st = as_stream(streams[d]);
        LJ_CK(cudaMemcpyAsync(&hr[(size_t)d * (ndev + 1)], L[(size_t)d].str, sizeof(i64) * (ndev + 1),
                              cudaMemcpyDeviceToHost, st));
        LJ_CK(cudaMemcpyAsync(&hs[(size_t)d * (ndev + 1)], L[(size_t)d].sts, sizeof(i64) * (ndev + 1),
                              cudaMemcpyDeviceToHost, st));
    }
    for (int d = 0; d < ndev; ++d) {
        LJ_CK(cudaSetDevice(devs[d]));
        LJ_CK(cudaStreamSynchronize(as_stream(streams[d])));
    }
    std::vector<int64_t> rin((size_t)ndev, 0), sin((size_t)ndev, 0);
    for (int src = 0; src < ndev; ++src)
        for (int dst = 0; dst < ndev; ++dst) {
            rin[(size_t)dst] += hr[(size_t)src * (ndev + 1) + dst + 1] - hr[(size_t)src * (ndev + 1) + dst];
            sin[(size_t)dst] += hs[(size_t)src * (ndev + 1) + dst + 1] - hs[(size_t)src * (ndev + 1) + dst];
        }
    for (int d = 0; d < ndev; ++d) {
        if (recv_counts) {
            recv_counts[2 * d] = rin[(size_t)d];
            recv_counts[2 * d + 1] = sin[(size_t)d];
        }
        if (rin[(size_t)d] > cap_r || sin[(size_t)d] > cap_s) {
            set_error("lj_lsj_run_multi: a device receives more than cap_r / cap_s (recv_counts has the sizes)");
            return LJ_E_WORKSPACE;
        }
    }
    // (4) the exchange: every (src, dst) run with one send / recv pair
    LJ_NC(N.group_start());
    for (int rel = 0; rel < 2; ++rel) {
        const std::vector<int64_t> &h = rel ? hs : hr;
        std::vector<int64_t> at((size_t)ndev, 0);
        for (int src = 0; src < ndev; ++src)
            for (int dst = 0; dst < ndev; ++dst) {
                const int64_t a = h[(size_t)src * (ndev + 1) + dst], c = h[(size_t)src * (ndev + 1) + dst + 1] - a;
                if (c <= 0) continue;
                const u64 *sb = (rel ? L[(size_t)src].ps : L[(size_t)src].pr) + 2 * a;
                ulonglong2 *rb = (rel ? L[(size_t)dst].rs : L[(size_t)dst].rr) + at[(size_t)dst];
                at[(size_t)dst] += c;
                LJ_CK(cudaSetDevice(devs[src]));
                LJ_NC(N.send(sb, (size_t)(2 * c), ncclUint64, dst, reinterpret_cast<ncclComm_t>(comms[src]),
                             as_stream(streams[src])));
                LJ_CK(cudaSetDevice(devs[dst]));
                LJ_NC(N.recv(rb, (size_t)(2 * c), ncclUint64, src, reinterpret_cast<ncclComm_t>(comms[dst]),
                             as_stream(streams[dst])));
            }
    }
    LJ_NC(N.group_end());
    // (5) every device joins its key range; (6) the words are combined
    std::vector<uint64_t *> words((size_t)ndev);
    std::vector<void *> red((size_t)ndev);
    for (int d = 0; d < ndev; ++d) {
        LJ_CK(cudaSetDevice(devs[d]));
        Lay &l = L[(size_t)d];
        cudaStream_t st = as_stream(streams[d]);
        // the received records are sampled and partitioned in place (no copy back to columns)
        (void)st;
        const int rc = lj_lsj_run_rec(reinterpret_cast<const u64 *>(l.rr), rin[(size_t)d],
                                      reinterpret_cast<const u64 *>(l.rs), sin[(size_t)d], sample_rate, seed, out[d],
                                      l.run, l.run_b, streams[d]);
        if (rc) return rc;
        words[(size_t)d] = out[d];
        red[(size_t)d] = l.red;
    }
    return lj_reduce_sums(ndev, devs, comms, streams, words.data(), red.data());
}

}  // extern "C"
