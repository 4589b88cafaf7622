#!/usr/bin/env python
"""Benchmark of the learned-join hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl b200|reference]

Default workload = BASELINE.json's metric config, configs[2] (C3, "at
1/2/4/8 B200"): RadixSpline learned-hash INLJ, R = 2*10^8 unique keys from
64 normal clusters, S = 2*10^9 probes drawn uniformly from R, sharded
across the GPUs with R replicated.  One step = one pass of the hot path
over this rank's S (grouping by index window + probe) against the prebuilt
index, reduced to (count, sum, xor) on device.  Metric: join tuples/s =
(|R| + |S|) / step time (reference bench.py:307-314).

``--gpus N`` (N > 1) without a torchrun environment re-launches itself
under ``torch.distributed.run`` with N ranks on 127.0.0.1.  Every rank
builds the same index (untimed, as the reference) and probes its
contiguous 1/N of S; the three checksum words are combined inside the
timed step (sum/count all-reduce, xor all-gather).  The whole-job value
counts the replicated R once and every rank's S shard.

``--impl reference`` times the reference algorithm's CPU implementation
(the C restatement in oracle/, OpenMP over every host thread; the
reference itself is Python+numba and does not exist on the GPU box) on
bounded samples of the same workload, on inputs produced by the HOST
generator oracle/gen.py -- bit-identical to the device inputs, without
loading the CUDA library -- and prints the full-size checksum of the
oracle beside the timing (the GPU line prints its own).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGO_BYTES = {"grmi-inlj": 32, "buffered-grmi-inlj": 32, "spline-hash-inlj": 32, "lsj": 80}
METRIC = "join tuples/s ((|R|+|S|)/time)"
MASK = (1 << 64) - 1

# workload descriptions (identical in both arms; BASELINE.json configs)
WORKLOADS = {
    "c1": ("grmi-inlj", "GRMI INLJ: R=2^20 uniform63 unique, S=2^22 (90% hits), density 0.5, 1024 leaves"),
    "c2": ("grmi-inlj", "GRMI INLJ skewed: R=2^24 lognormal(0,2)x1e12 unique, S=2^28 (95% Zipf(0.8) hits), "
                        "density 0.5, 65536 leaves"),
    "c3": ("spline-hash-inlj", "RadixSpline learned-hash INLJ: R=2e8 clustered-normal unique (64 clusters, "
                               "sigma 2^40), S=2e9 uniform from R sharded over the GPUs, 18 radix bits, max error "
                               "32, P=4|R|"),
    "c4": ("lsj", "LSJ: R=2^28 lognormal(0,1.5)x2^40 unique, S=2^28 Zipf(1.0) over R ranks, 4096 partitions, "
                  "1% sample models"),
    "c5": ("lsj", "LSJ across GPUs: R=S=2e9 (all GPUs) uniform unique (bijective mix) / uniform from R, shared "
                  "model range shuffle"),
}
DEFAULT_VARIANT = {"c1": "direct", "c2": "buffered", "c3": "buffered"}
# configs whose relations are split across the ranks (BASELINE: C3's S is
# sharded with R replicated; C5 range-shuffles both); the others run one
# full-size workload per GPU (weak scaling)
SHARDED = {"c3": ("s",), "c5": ("r", "s")}


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _config_block(args, n_r, n_s):
    algo, desc = WORKLOADS[args.config]
    return {"workload": f"{args.config}: {desc}", "algorithm": algo,
            "variant": (args.variant or DEFAULT_VARIANT.get(args.config, "direct")) if algo != "lsj" else None,
            "scale": args.scale, "n_r": n_r, "n_s": n_s,
            "l2": "inputs larger than L2 and L2 flushed (512 MB write) between steps",
            "parallelism": _parallelism(args.config, algo, args.gpus)}


def _parallelism(cfg, algorithm, n):
    if cfg == "c5":
        return f"lsj range shuffle over {n} GPU(s): shared model, P2P all-to-all, local LSJ"
    if algorithm == "lsj":
        return f"lsj replicas x{n} (one full join per GPU)"
    if cfg in SHARDED:
        return f"inlj replicated R, S sharded 1/{n} per GPU"
    return f"inlj replicated R, full S per GPU x{n}"


# ---------------------------------------------------------------- CPU legs
# (the oracle: the checker and the CPU baseline, never the measured product)


class CpuJoin:
    """The reference algorithm's CPU implementation (oracle/, C + OpenMP)
    over host arrays: rk/rp whole, S through s_slice(lo, hi).  The index
    build is untimed, as in the reference (bench.py:138-144,202-209)."""

    def __init__(self, algorithm, opts, rk, rp, s_slice, n_s):
        import oracle

        self.oracle, self.algorithm, self.opts = oracle, algorithm, opts
        self.rk, self.rp, self.s_slice, self.n_s = rk, rp, s_slice, n_s
        self.idx = None
        if algorithm in ("grmi-inlj", "buffered-grmi-inlj"):
            self.idx = oracle.grmi_build(rk, rp, opts["gap_factor"], opts["rmi_fanout"])
        elif algorithm == "spline-hash-inlj":
            self.idx = oracle.spline_hash_build(rk, rp, opts.get("spline_error", 32), opts.get("radix_bits", 18),
                                                opts.get("table_factor", 4.0))

    def probe(self, sk, sp, threads):
        o = self.oracle
        if self.algorithm == "spline-hash-inlj":
            return o.spline_hash_join(self.idx, sk, sp, threads)[:3]
        return o.grmi_join(self.idx, sk, sp, threads)[:3]

    def lsj(self, m, threads):
        sk, sp = self.s_slice(0, m)
        return self.oracle.lsj_join(self.rk[:m], self.rp[:m], sk, sp, workers=threads,
                                    fanout=self.opts.get("fanout", 4096),
                                    sample_rate=self.opts.get("sample_rate", 0.01))[0]

    def sample_size(self, threads, target_s):
        """Smallest power-of-4 sample whose run takes >= target_s / 4."""
        m = min(self.n_s, 1 << 18)
        while True:
            dt = self.time_sample(m, threads)
            if dt >= target_s / 4 or m >= self.n_s:
                return m, dt
            m = min(self.n_s, m * 4)

    def time_sample(self, m, threads):
        if self.algorithm == "lsj":
            t0 = time.perf_counter()
            self.lsj(m, threads)
            return time.perf_counter() - t0
        sk, sp = self.s_slice(0, m)
        t0 = time.perf_counter()
        self.probe(sk, sp, threads)
        return time.perf_counter() - t0

    def value(self, m, dt, n_r):
        """Whole-workload tuples/s from a sample run (time extrapolated
        linearly in |S| for INLJ, in |R|+|S| for LSJ -- optimistic for the
        CPU's n log n sort)."""
        if self.algorithm == "lsj":
            return (n_r + self.n_s) / (dt * (n_r + self.n_s) / (2 * m))
        return (n_r + self.n_s) / (dt * self.n_s / m)

    def describe(self, m, dt, threads):
        if self.algorithm == "lsj":
            return (f"LSJ with {threads} workers over the first {m} tuples of R and of S ({dt:.2f} s), time "
                    f"scaled linearly to |R|+|S|")
        return (f"first {m} of {self.n_s} S probes against the full R index on {threads} thread(s) ({dt:.2f} s), "
                f"time extrapolated x{self.n_s / m:.1f}; index build untimed as in the reference")

    def full_checksum(self, threads, slice_n=1 << 25):
        """The oracle's (count, sum, xor) over the whole workload: S in
        slices against the index (sums add, xors xor); LSJ through the
        ground-truth sort-merge join (baselines.py:337-348)."""
        if self.algorithm == "lsj":
            sk, sp = self.s_slice(0, self.n_s)
            return tuple(self.oracle.smj_checksum(self.rk, self.rp, sk, sp))
        c = s = x = 0
        for lo in range(0, self.n_s, slice_n):
            sk, sp = self.s_slice(lo, min(self.n_s, lo + slice_n))
            w = self.probe(sk, sp, threads)
            c, s, x = c + w[0], (s + w[1]) & MASK, x ^ w[2]
        return (c, s, x)


def cpu_baseline(cj: CpuJoin, n_r, target_s=8.0):
    """All host threads, plus W = 1 beside it."""
    cores = cj.oracle.num_threads()
    m, dt = cj.sample_size(cores, target_s)
    info = {"value": cj.value(m, dt, n_r), "unit": "tuples/s", "cores": cores, "kind": "port",
            "sample": cj.describe(m, dt, cores)}
    m1, dt1 = cj.sample_size(1, target_s / 2)
    info["w1"] = {"value": cj.value(m1, dt1, n_r), "cores": 1, "sample": cj.describe(m1, dt1, 1)}
    return info, m


def run_reference_arm(args):
    """The reference's CPU path on host-generated inputs: no CUDA library
    is loaded in this process (oracle/ only)."""
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    import oracle
    from oracle import gen

    t0 = time.perf_counter()
    kw = {} if args.scale is None else {"scale": args.scale}
    h = gen.CONFIGS[args.config](**kw)
    gen_s = time.perf_counter() - t0
    algo = WORKLOADS[args.config][0]
    n_r, n_s = h.rk.size, h.n_s
    if args.config in SHARDED and args.gpus > 1:
        pass  # the reference joins the whole workload (its W threads share the host)
    t0 = time.perf_counter()
    cj = CpuJoin(algo, dict(h.opts, seed=42), h.rk, h.rp, h.s_slice, n_s)
    build_s = time.perf_counter() - t0
    cores = oracle.num_threads()
    m, dt = cj.sample_size(cores, 4.0)
    steps = []
    for i in range(args.warmup + args.steps):
        dt = cj.time_sample(m, cores)
        if i >= args.warmup:
            steps.append(dt)
    dt = statistics.median(steps)
    value = cj.value(m, dt, n_r)
    t_full = n_r + n_s
    ms = t_full / value * 1e3
    info = {"value": value, "unit": "tuples/s", "cores": cores, "kind": "port", "sample": cj.describe(m, dt, cores)}
    try:
        m1, dt1 = cj.sample_size(1, 2.0)
        info["w1"] = {"value": cj.value(m1, dt1, n_r), "cores": 1, "sample": cj.describe(m1, dt1, 1)}
    except Exception as exc:  # reported, never required
        info["w1"] = {"error": repr(exc)}
    checksum = None
    if not args.no_full_checksum:
        t0 = time.perf_counter()
        c, sm, x = cj.full_checksum(cores)
        checksum = {"count": c, "sum": sm, "xor": x, "full_pass_s": time.perf_counter() - t0,
                    "how": ("oracle spline-hash / GRMI probe over all of S in 2^25-probe slices" if algo != "lsj"
                            else "oracle sort-merge join (baselines.py:337-348) over all of R and S")}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if args.config in SHARDED else "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (host generator oracle/gen.py, bit-identical to the device inputs)",
            "config": _config_block(args, n_r, n_s), "cpu_baseline": info,
            "e2e": {"value": value, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "checksum": checksum, "prep": {"gen_s": gen_s, "index_build_s": build_s}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm


def make_inputs(cfg: str, shard: int = 0, shards: int = 1, scale=None):
    import inspect

    from paper_2111_08824_b200 import configs

    fn = configs.CONFIGS[cfg]
    kw = {"shard": shard}
    if "shards" in inspect.signature(fn).parameters:
        kw["shards"] = shards
    if scale is not None:
        kw["scale"] = scale
    return fn(**kw)


def build_index(inp):
    import paper_2111_08824_b200 as lj

    o = dict(lj.DEFAULT_OPTS, **inp.opts)
    if inp.algorithm in ("grmi-inlj", "buffered-grmi-inlj"):
        return lj.GappedRmiIndex(o["gap_factor"], o["rmi_fanout"]).fit(inp.r)
    if inp.algorithm == "spline-hash-inlj":
        return lj.SplineHashIndex(o["spline_error"], o["radix_bits"], o["table_factor"]).fit(inp.r)
    return None  # lsj builds nothing ahead of time: it is timed end to end


class Step:
    """One step of the hot path: `parts` run in order on the current stream;
    `dominant` names the part the roofline is reported for and `dom_bytes`
    its algorithmic bytes per launch."""

    def __init__(self, parts, dominant, dom_bytes, kernel, bytes_note):
        self.parts, self.dominant, self.dom_bytes = parts, dominant, dom_bytes
        self.kernel, self.bytes_note = kernel, bytes_note
        self.holder = {}

    def __call__(self, out):
        for _, fn in self.parts:
            fn(out)
        return out


def make_step(inp, index, variant="buffered", world: int = 1, distributed: bool = False):
    """A step is one pass of the hot path over the whole (local) S (INLJ,
    index prebuilt as in the reference, bench.py:138-144 of the reference)
    or the whole LSJ (sample, fit, partition, sort, join)."""
    import torch

    import paper_2111_08824_b200 as lj

    n_r, n_s = len(inp.r), len(inp.s)
    if index is not None:
        keys, pays = inp.s.keys, inp.s.payloads
        grmi = "grmi" in inp.algorithm
        if variant == "buffered":
            scratch = index.bucket_scratch(n_s)
            parts = [("bucket", lambda out: index.bucket_records(keys, pays, scratch)),
                     ("probe", lambda out: index.probe_records(n_s, scratch, out))]
            kern = "k_grmi_probe_staged" if grmi else "k_hash_probe_staged"
            st = Step(parts, "probe", 32 * n_s, kern,
                      f"32 B/probe x {n_s} probes (16 B S record + 16 B R entry); the one-pass grouping by "
                      "index window runs before it in the step")
            st.scratch = scratch
            return st
        fn = (lambda out: index.join_checksum(keys, pays, out=out))
        return Step([("probe", fn)], "probe", 32 * n_s, "k_grmi_probe" if grmi else "k_hash_probe",
                    f"32 B/probe x {n_s} probes (16 B S record + 16 B R entry)")
    o = dict(lj.DEFAULT_OPTS, **inp.opts)
    cfg = lj.LsjConfig(workers=1, fanout=o["fanout"], sample_rate=o["sample_rate"], seed=o["seed"])
    if distributed:
        # C5 across GPUs: shared model, range shuffle, local LSJ, 3-word
        # reduction (dist.lsj_join); the words come back reduced on every rank
        from paper_2111_08824_b200 import dist as ljdist

        def dist_step(out):
            (c, sm, x), ph = ljdist.lsj_join(inp.r.keys, inp.r.payloads, inp.s.keys, inp.s.payloads, cfg)
            st.holder["phases"] = ph
            sg = [v - (1 << 64) if v >= (1 << 63) else v for v in (c, sm, x, 0)]
            out.copy_(torch.tensor(sg, dtype=torch.int64))
            return out

        st = Step([("lsj", dist_step)], "lsj", 80 * (n_r + n_s), "distributed LSJ step (partition, all-to-all, "
                  "local LSJ)", f"80 B/tuple x {n_r + n_s} local tuples (partition 32, sort 32, merge 16)")
        st.reduced = True
        return st

    def lsj_phases(out):
        # the same LSJ through the Python orchestration (one C call per
        # phase), which records the phase events
        res, br = lj.lsj_join(inp.r, inp.s, cfg, counters=False)
        st.holder["br"] = br
        out.copy_(res._words)
        return out

    # The step: the whole LSJ as ONE asynchronous C call (lj_lsj_run: sample,
    # fit, bins, partition, sort, join of both relations from one workspace;
    # no host readback, the partition's overflow fallback decided on the
    # device), captured into a CUDA graph on first use and replayed.
    from paper_2111_08824_b200 import _lib

    lib = _lib.lib()
    dev = inp.r.keys.device
    ws = _lib.workspace(lib.lj_lsj_run_workspace_bytes(n_r, n_s, float(o["sample_rate"])), dev)
    cap = {}

    def one_call(out):
        _lib.check(lib.lj_lsj_run(_lib.ptr(inp.r.keys), _lib.ptr(inp.r.payloads), n_r, _lib.ptr(inp.s.keys),
                                  _lib.ptr(inp.s.payloads), n_s, float(o["sample_rate"]), int(o["seed"]) & MASK,
                                  _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "lsj_run")

    def lsj_step(out):
        if cap.get("ptr") != out.data_ptr():
            one_call(out)  # kernel attributes are set outside the capture
            torch.cuda.synchronize()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(graph, stream=side):
                    one_call(out)
            torch.cuda.current_stream().wait_stream(side)
            cap.update(ptr=out.data_ptr(), graph=graph)
        cap["graph"].replay()
        return out

    st = Step([("lsj", lsj_step)], "sort", 32 * (n_r + n_s), "lsj sort phase (k_split_*, k_lsj_sort)",
              f"sort phase: 32 B/tuple (read 16 + write 16) x {n_r + n_s} tuples; whole pipeline 80 B/tuple")
    st.phases = lsj_phases
    st.path = "lj_lsj_run (one C call) replayed as a CUDA graph"
    return st


def count_launches(step, out):
    """Kernels launched by one step, counted with the CUDA profiler (CUPTI):
    every kernel except torch's own elementwise fills."""
    import torch

    try:
        import warnings

        from torch.profiler import ProfilerActivity, profile

        warnings.filterwarnings("ignore", module="torch.profiler")
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(out)
            torch.cuda.synchronize()
        n = 0
        for e in prof.events():
            if getattr(e, "device_type", None) is not None and str(e.device_type).endswith("CUDA"):
                name = e.name
                if "Memset" in name or "Memcpy" in name or name.startswith("void at::") or "native::" in name:
                    continue
                n += 1
        return n
    except Exception:
        return None


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    use_pg = world > 1 or args.config == "c5"  # C5 always runs the distributed LSJ
    if use_pg:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
    inp = make_inputs(args.config, shard=rank, shards=world, scale=args.scale)
    index = build_index(inp)
    dev = torch.device("cuda", local)
    variant = args.variant or DEFAULT_VARIANT.get(args.config, "direct")
    args.variant = variant
    run_step = make_step(inp, index, variant, world, distributed=args.config == "c5")
    reduced = getattr(run_step, "reduced", False)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = torch.zeros(4, dtype=torch.int64, device=dev)
    xors = torch.zeros(world, dtype=torch.int64, device=dev)
    # whole-job tuples: sharded relations summed over the ranks, replicated
    # ones counted once (R of C3), per-GPU workloads N times (weak scaling)
    sizes = torch.tensor([len(inp.r), len(inp.s)], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(sizes)
    sh = SHARDED.get(args.config, ())
    job_r = int(sizes[0]) if "r" in sh else (len(inp.r) if index is not None else world * len(inp.r))
    job_s = int(sizes[1]) if "s" in sh else world * len(inp.s)
    args.scaling = "strong" if sh else "weak"
    args.job_tuples = job_r + job_s

    def step():
        run_step(out)
        if world > 1 and not reduced:
            dist.all_gather_into_tensor(xors, out[2:3].contiguous())
            dist.all_reduce(out, op=dist.ReduceOp.SUM)  # count, sum, steps (wrap mod 2^64)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # evict the index and S from L2 between steps
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = float(total.item()) / args.steps
    n_r, n_s = len(inp.r), len(inp.s)
    value = (job_r + job_s) / (ms_per_step / 1e3)
    w = out.cpu().tolist()
    xor_all = 0
    if world > 1 and not reduced:
        for v in xors.cpu().tolist():
            xor_all ^= v & MASK
    else:
        xor_all = w[2] & MASK

    # the dominant kernel timed alone, live, with CUDA events on its stream
    dom = []
    phase_ms = []
    for i in range(args.steps):
        flush.zero_()
        if run_step.dominant == "sort":  # LSJ: phase events recorded by lsj_join itself
            getattr(run_step, "phases", run_step)(out)
            torch.cuda.synchronize()
            br = run_step.holder["br"]
            dom.append(br.sort * 1e3)
            phase_ms.append((br.part * 1e3, br.sort * 1e3, br.join * 1e3))
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for name, fn in run_step.parts:
            if name == run_step.dominant:
                e0.record()
                fn(out)
                e1.record()
            else:
                fn(out)
        torch.cuda.synchronize()
        dom.append(e0.elapsed_time(e1))
    k_ms = statistics.mean(dom)
    peak, peak_kind = _peaks()
    achieved = run_step.dom_bytes / (k_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": _ncu_traffic(args.config), "kernel": run_step.kernel, "kernel_ms": k_ms,
                "peak_kind": peak_kind, "algorithmic_bytes": run_step.bytes_note,
                "step_frac": (ALGO_BYTES[inp.algorithm] * (n_s if index is not None else n_r + n_s))
                / (ms_per_step / 1e3) / 1e9 / peak}
    if run_step.kernel == "k_grmi_probe_staged" and hasattr(index, "probe_records"):
        # ablation: the staged probe without the reference's probe counter
        # (search_steps): the staged search never uses the model's prediction,
        # so its evaluation goes with the counter; the checksum is unchanged
        nc = []
        o2 = torch.zeros(4, dtype=torch.int64, device=dev)
        for i in range(args.steps):
            flush.zero_()
            run_step.parts[0][1](o2)  # regroup S (the probe consumes the grouped records)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            index.probe_records(n_s, run_step.scratch, o2, count_steps=False)
            e1.record()
            torch.cuda.synchronize()
            nc.append(e0.elapsed_time(e1))
        nc_ms = statistics.mean(nc)
        w2 = o2.cpu().tolist()
        roofline["no_probe_counter"] = {
            "kernel_ms": nc_ms, "achieved": run_step.dom_bytes / (nc_ms / 1e3) / 1e9,
            "frac": run_step.dom_bytes / (nc_ms / 1e3) / 1e9 / peak,
            "same_checksum": [v & MASK for v in w2[:3]] == [w[0] & MASK, w[1] & MASK, xor_all],
            "note": "probe_records(count_steps=False): no search_steps, no model evaluation"}
    if phase_ms:
        # LSJ per phase (partition 32 B, sort 32 B, merge 16 B per tuple of |R| + |S|)
        roofline["lsj_phases"] = {}
        for i, (name, bpt) in enumerate((("partition", 32), ("sort", 32), ("merge", 16))):
            ms = statistics.mean(p[i] for p in phase_ms)
            gbs = bpt * (n_r + n_s) / (ms / 1e3) / 1e9
            roofline["lsj_phases"][name] = {"ms": ms, "achieved": gbs, "frac": gbs / peak,
                                            "algorithmic_bytes": f"{bpt} B/tuple x {n_r + n_s}"}
    if phase_ms and hasattr(run_step, "phases"):
        # the step is lj_lsj_run replayed as one CUDA graph; the phase times
        # above come from the same LSJ run phase by phase from Python
        pm = []
        o3 = torch.zeros(4, dtype=torch.int64, device=dev)
        for i in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run_step.phases(o3)
            e1.record()
            torch.cuda.synchronize()
            pm.append(e0.elapsed_time(e1))
        w3 = o3.cpu().tolist()
        roofline["step_path"] = run_step.path
        roofline["python_orchestration"] = {
            "ms_per_step": statistics.mean(pm),
            "same_checksum": [v & MASK for v in w3[:3]] == [w[0] & MASK, w[1] & MASK, xor_all],
            "note": "lsj_join: one C call per phase with CUDA events between them (the source of lsj_phases)"}
    ph = run_step.holder.get("phases")
    if ph is not None and "shuffle" in ph:
        # the range shuffle against NVLink (16 B x (|R|+|S|)/G x
        # (G-1)/G per GPU leave the GPU)
        moved = 16 * (n_r + n_s) * (world - 1) / world
        sh_ms = (ph["part"] + ph["xchg"]) * 1e3
        roofline["nvlink"] = {"bytes_per_gpu": moved, "shuffle_ms": sh_ms, "peak": 900.0, "unit": "GB/s",
                              "achieved": moved / (sh_ms / 1e3) / 1e9 if sh_ms > 0 else 0.0,
                              "frac": (moved / (sh_ms / 1e3) / 1e9 / 900.0) if sh_ms > 0 else 0.0,
                              "shuffle": ph["shuffle"]}
    launches = count_launches(run_step, out)

    e2e = None
    if not args.no_e2e:
        e2e = _e2e(args, inp, world)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                from paper_2111_08824_b200.util import to_numpy_u64

                s_keys, s_pays = inp.s.keys, inp.s.payloads
                cj = CpuJoin(inp.algorithm, dict(inp.opts, seed=42), to_numpy_u64(inp.r.keys),
                             to_numpy_u64(inp.r.payloads),
                             lambda lo, hi: (to_numpy_u64(s_keys[lo:hi]), to_numpy_u64(s_pays[lo:hi])), n_s)
                cpu, _ = cpu_baseline(cj, n_r)
            except Exception as exc:  # the baseline is reported, never required
                cpu = {"error": repr(exc)}
        line = {"metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (device generator, seeded; == host generator oracle/gen.py)",
                "config": _config_block(args, job_r if "r" in sh else n_r, job_s if "s" in sh else n_s),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": (launches * args.steps) if launches is not None else None,
                "clocks": clk.summary(),
                "checksum": {"count": w[0], "sum": w[1] & MASK, "xor": xor_all, "search_steps": w[3]}}
        print(json.dumps(line), flush=True)
    if use_pg:
        dist.destroy_process_group()


def _e2e(args, inp, world):
    """The same metric through the reference-facing registry entry point
    ``ALGORITHMS[name](r, s, 1, opts)`` with HOST-resident relations
    (pinned): the runner copies S host->device inside its timed region
    (chunked, overlapped with the join; LSJ: R and S, overlapped with R's
    side) and reads the 3 result words back.  The INLJ index over R is
    built untimed inside the runner, as the reference's runners do."""
    import torch

    import paper_2111_08824_b200 as lj

    r_host = lj.Relation.on_host(inp.r.keys.cpu(), inp.r.payloads.cpu())
    s_host = lj.Relation.on_host(inp.s.keys.cpu(), inp.s.payloads.cpu())
    opts = dict(lj.DEFAULT_OPTS, **inp.opts)
    algo = inp.algorithm if inp.algorithm != "grmi-inlj" or args.variant == "direct" else "buffered-grmi-inlj"
    h2d = 16 * len(inp.s) + (16 * len(inp.r) if inp.algorithm == "lsj" else 0)
    steps = max(1, min(args.steps, 3))
    times = []
    for i in range(steps + 1):
        torch.cuda.synchronize()
        if args.config == "c5":
            from paper_2111_08824_b200 import dist as ljdist

            t0 = time.perf_counter()
            r, s = r_host.to_device(), s_host.to_device()
            cfg = lj.LsjConfig(workers=1, fanout=opts["fanout"], sample_rate=opts["sample_rate"], seed=opts["seed"])
            ljdist.lsj_join(r.keys, r.payloads, s.keys, s.payloads, cfg)
            rt = time.perf_counter() - t0
            del r, s
        else:
            _, _, rt = lj.ALGORITHMS[algo](r_host, s_host, 1, opts)
        if i:
            times.append(rt)
    t = statistics.median(times)
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    path = (f"lj.ALGORITHMS[{algo!r}](Relation.on_host(R), Relation.on_host(S), 1, opts): runner-timed probe "
            "(S in 2^25-tuple chunks, H2D on a copy stream overlapped with the grouping + probe)"
            if inp.algorithm != "lsj" else
            f"lj.ALGORITHMS['lsj'](host R, host S, 1, opts): lsj_join_host, R's side overlaps S's H2D")
    if args.config == "c5":
        path = "dist.lsj_join over R and S copied from pinned host memory"
    return {"value": getattr(args, "job_tuples", len(inp.r) + world * len(inp.s)) / t, "unit": "tuples/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 3 * 8, "ms_per_step": t * 1e3, "steps": steps,
            "path": path}


def _ncu_traffic(cfg):
    p = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args_list, n):
    """``--gpus N`` outside torchrun: one process per GPU via
    torch.distributed.run on this node; rank 0's JSON line passes through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + args_list
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default=None, choices=["buffered", "direct"],
                    help="INLJ: group S by index window on device first (Request-Buffer analogue) or probe "
                         "directly; default per config (c2/c3 buffered, c1 direct)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-checksum", action="store_true", help="reference arm: skip the full-size oracle pass")
    ap.add_argument("--scale", type=int, default=None, help="config size divisor / shift (tests only; not a bench "
                                                            "number)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(sys.argv[1:], args.gpus))
    run_b200(args)


if __name__ == "__main__":
    main()
