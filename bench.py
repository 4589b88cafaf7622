#!/usr/bin/env python
"""Benchmark of the learned-join hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

Default workload = BASELINE.json configs[1] (C2): Gapped-RMI INLJ, R = 2^24
unique floor(1e12*lognormal(0,2)) keys, S = 2^28 probes (95% Zipf(0.8)
hits), RMI with 2^16 leaves at density 0.5.  One step = one fused probe
(K1) of the whole S relation against the prebuilt index, with the result
reduced to (count, sum, xor) on device.  Metric: join tuples/s =
(|R| + |S|) / step time (bench.py:307-314 of the reference).

Multi-GPU (torchrun, one process per GPU): the R index is replicated and
every rank probes its own full-size S shard (weak scaling); the per-rank
checksums are combined with NCCL (sum/count all-reduce, xor all-gather) inside
the timed step.  value = (|R| + N*|S|) / max-over-ranks step time.

``--impl reference`` times the reference algorithm's CPU implementation --
the C restatement in oracle/ (the reference itself is Python+numba and is
not installed on the GPU box) -- with every host thread, on a bounded
sample of the same workload, extrapolated to the full S.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGO_BYTES = {"grmi-inlj": 32, "buffered-grmi-inlj": 32, "spline-hash-inlj": 32, "lsj": 80}


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
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


# configs whose relations are split across the ranks (BASELINE: C3's S is
# sharded with R replicated; C5 range-shuffles both); the others run one
# full-size workload per GPU (weak scaling)
SHARDED = {"c3": ("s",), "c5": ("r", "s")}


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


DEFAULT_VARIANT = {"c1": "direct", "c2": "buffered", "c3": "buffered"}


class Step:
    """One step of the hot path: `parts` run in order on the current stream;
    `dominant` names the part the roofline is reported for and `dom_bytes`
    its algorithmic bytes per launch."""

    def __init__(self, parts, dominant, dom_bytes, kernel, bytes_note):
        self.parts, self.dominant, self.dom_bytes = parts, dominant, dom_bytes
        self.kernel, self.bytes_note = kernel, bytes_note
        self.last_breakdown = None

    def __call__(self, out):
        for _, fn in self.parts:
            fn(out)
        return out


def make_step(inp, index, variant="buffered", world: int = 1, distributed: bool = False):
    """A step is one pass of the hot path over the whole S (INLJ, index
    prebuilt as in the reference, bench.py:138-144 of the reference) or the
    whole LSJ (sample, fit, partition, sort, join)."""
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
            kern = "k_grmi_probe_staged" if grmi else "k_hash_probe_chunks"
            st = Step(parts, "probe", 32 * n_s, kern,
                      f"32 B/probe x {n_s} probes (16 B S record + 16 B R entry); the one-pass bucketing "
                      "(k_est_sample + k_bin_scatter_est) runs before it in the step")
            st.scratch = scratch  # reused by the e2e leg (C3's is ~66 GB)
            return st
        fn = (lambda out: index.join_checksum(keys, pays, out=out))
        return Step([("probe", fn)], "probe", 32 * n_s, "k_grmi_probe" if grmi else "k_hash_probe",
                    f"32 B/probe x {n_s} probes (16 B S record + 16 B R entry)")
    o = dict(lj.DEFAULT_OPTS, **inp.opts)
    cfg = lj.LsjConfig(workers=1, fanout=o["fanout"], sample_rate=o["sample_rate"], seed=o["seed"])
    holder = {}
    if distributed:
        # C5 across GPUs: shared model, range shuffle (NCCL all-to-all-v),
        # local LSJ, 3-word reduction (dist.lsj_join); the words come back
        # reduced on every rank
        from paper_2111_08824_b200 import dist as ljdist

        def dist_step(out):
            (c, sm, x), ph = ljdist.lsj_join(inp.r.keys, inp.r.payloads, inp.s.keys, inp.s.payloads, cfg)
            holder["phases"] = ph
            sg = [v - (1 << 64) if v >= (1 << 63) else v for v in (c, sm, x, 0)]
            out.copy_(torch.tensor(sg, dtype=torch.int64))
            return out

        st = Step([("lsj", dist_step)], "lsj", 80 * (n_r + n_s), "distributed LSJ step (partition, all-to-all, "
                  "local LSJ)", f"80 B/tuple x {n_r + n_s} local tuples (partition 32, sort 32, merge 16)")
        st.holder = holder
        st.reduced = True
        return st

    def lsj_step(out):
        res, br = lj.lsj_join(inp.r, inp.s, cfg)
        holder["br"] = br
        out.copy_(res._words)
        return out

    st = Step([("lsj", lsj_step)], "sort", 32 * (n_r + n_s), "lsj sort phase (k_split_*, k_lsj_sort)",
              f"sort phase: 32 B/tuple (read 16 + write 16) x {n_r + n_s} tuples; whole pipeline 80 B/tuple")
    st.holder = holder
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


# ---------------------------------------------------------------- CPU arms


def cpu_inlj(inp, target_s: float = 8.0, threads: int = 0):
    """Oracle (C restatement of the reference path, OpenMP) on a bounded
    sample, extrapolated to the whole workload.  Returns (value, info, rerun)."""
    import numpy as np

    import oracle

    o = inp.opts
    rk, rp = inp.r.numpy()
    n_r, n_s = len(inp.r), len(inp.s)
    cores = threads or oracle.num_threads()
    if inp.algorithm == "lsj":
        # LSJ is timed end to end on prefixes of R and S (all phases), then
        # scaled linearly in |R|+|S| (optimistic for the CPU: the sort is
        # n log n)
        sample = min(n_r, 1 << 20)
        while True:
            sk = inp.s.keys[:sample].cpu().numpy().view(np.uint64)
            sp = inp.s.payloads[:sample].cpu().numpy().view(np.uint64)
            rks, rps = rk[:sample], rp[:sample]
            run = lambda a, b, rks=rks, rps=rps: oracle.lsj_join(rks, rps, a, b, workers=cores,
                                                                  fanout=o.get("fanout", 4096),
                                                                  sample_rate=o.get("sample_rate", 0.01))
            t0 = time.perf_counter()
            run(sk, sp)
            dt = time.perf_counter() - t0
            if dt >= target_s / 4 or sample >= min(n_r, n_s):
                break
            sample = min(n_r, n_s, sample * 4)
        scale = (n_r + n_s) / (2 * sample)
        value = (n_r + n_s) / (dt * scale)
        info = {"value": value, "unit": "tuples/s", "cores": cores, "kind": "port",
                "sample": f"LSJ with {cores} workers (one thread each, as the reference's share-nothing "
                          f"workers) over the first {sample} tuples of R and of S ({dt:.2f} s), "
                          f"time scaled x{scale:.1f} linearly to |R|+|S|"}
        return value, info, (sk, sp, run)
    if inp.algorithm in ("grmi-inlj", "buffered-grmi-inlj"):
        idx = oracle.grmi_build(rk, rp, o["gap_factor"], o["rmi_fanout"])
        run = lambda k, p: oracle.grmi_join(idx, k, p, threads)
    else:
        idx = oracle.spline_hash_build(rk, rp, o.get("spline_error", 32), o.get("radix_bits", 18),
                                       o.get("table_factor", 4.0))
        run = lambda k, p: oracle.spline_hash_join(idx, k, p, threads)
    sample = min(n_s, 1 << 20)
    while True:
        sk = inp.s.keys[:sample].cpu().numpy().view(np.uint64)
        sp = inp.s.payloads[:sample].cpu().numpy().view(np.uint64)
        t0 = time.perf_counter()
        run(sk, sp)
        dt = time.perf_counter() - t0
        if dt >= target_s / 4 or sample >= n_s:
            break
        sample = min(n_s, sample * 4)
    t_full = dt * n_s / sample
    value = (n_r + n_s) / t_full
    info = {"value": value, "unit": "tuples/s", "cores": cores, "kind": "port",
            "sample": f"first {sample} of {n_s} S probes against the full R index ({dt:.2f} s), "
                      f"time extrapolated x{n_s / sample:.1f}; index build untimed as in the reference"}
    return value, info, (sk, sp, run)


def run_reference_arm(args):
    import torch

    rank, world, local = _env_rank()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    inp = make_inputs(args.config)
    value, info, (sk, sp, run) = cpu_inlj(inp)
    steps = []
    n_s = len(inp.s)
    scale = (n_s / sk.size) if inp.algorithm != "lsj" else (len(inp.r) + n_s) / (2 * sk.size)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        run(sk, sp)
        dt = (time.perf_counter() - t0) * scale
        if i >= args.warmup:
            steps.append(dt)
    t = statistics.median(steps)
    value = (len(inp.r) + n_s) / t
    info["value"] = value
    line = {"impl": "reference", "metric": "join tuples/s ((|R|+|S|)/time)", "value": value, "unit": "tuples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": _config_block(args, inp), "cpu_baseline": info,
            "e2e": {"value": value, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config_block(args, inp):
    return {"workload": f"{args.config}: {inp.description}", "algorithm": inp.algorithm,
            "variant": getattr(args, "variant", None) if inp.algorithm != "lsj" else None,
            "n_r": len(inp.r), "n_s": len(inp.s), "l2": "inputs larger than L2 and L2 flushed between steps",
            "parallelism": _parallelism(args.config, inp.algorithm, args.gpus)}


def _parallelism(cfg, algorithm, n):
    if cfg == "c5":
        return f"lsj range shuffle over {n} GPU(s): shared model, NCCL all-to-all-v, local LSJ"
    if algorithm == "lsj":
        return f"lsj replicas x{n} (one full join per GPU)"
    if cfg in SHARDED:
        return f"inlj replicated R, S sharded 1/{n} per GPU"
    return f"inlj replicated R, full S per GPU x{n}"


# ---------------------------------------------------------------- GPU arm


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _env_rank()
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
            xor_all ^= v & (2**64 - 1)
    else:
        xor_all = w[2] & (2**64 - 1)

    # the dominant kernel timed alone, live, with CUDA events on its stream
    dom = []
    phase_ms = []
    for i in range(args.steps):
        flush.zero_()
        if run_step.dominant == "sort":  # LSJ: phase events recorded by lsj_join itself
            run_step(out)
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
    if phase_ms:
        # LSJ per phase (partition 32 B, sort 32 B, merge 16 B per tuple of |R| + |S|)
        roofline["lsj_phases"] = {}
        for i, (name, bpt) in enumerate((("partition", 32), ("sort", 32), ("merge", 16))):
            ms = statistics.mean(p[i] for p in phase_ms)
            gbs = bpt * (n_r + n_s) / (ms / 1e3) / 1e9
            roofline["lsj_phases"][name] = {"ms": ms, "achieved": gbs, "frac": gbs / peak,
                                            "algorithmic_bytes": f"{bpt} B/tuple x {n_r + n_s}"}
    ph = getattr(run_step, "holder", {}).get("phases") if hasattr(run_step, "holder") else None
    if ph is not None and "shuffle" in ph:
        # the range shuffle against NVLink (16 B x (|R|+|S|)/G x
        # (G-1)/G per GPU leave the GPU); partition and exchange are one fused
        # step, timed on the host around its stream syncs
        moved = 16 * (n_r + n_s) * (world - 1) / world
        sh_ms = (ph["part"] + ph["xchg"]) * 1e3
        roofline["nvlink"] = {"bytes_per_gpu": moved, "shuffle_ms": sh_ms, "peak": 900.0, "unit": "GB/s",
                              "achieved": moved / (sh_ms / 1e3) / 1e9 if sh_ms > 0 else 0.0,
                              "frac": (moved / (sh_ms / 1e3) / 1e9 / 900.0) if sh_ms > 0 else 0.0,
                              "shuffle": ph["shuffle"]}
    launches = count_launches(run_step, out)

    e2e = None
    if not args.no_e2e:
        e2e = _e2e(args, inp, index, world, run_step)
    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                _, cpu, _ = cpu_inlj(inp)
            except Exception as exc:  # the baseline is reported, never required
                cpu = {"error": repr(exc)}
        line = {"metric": "join tuples/s ((|R|+|S|)/time)", "value": value, "unit": "tuples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": _config_block(args, inp), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": (launches * args.steps) if launches is not None else None,
                "clocks": clk.summary(),
                "checksum": {"count": w[0], "sum": w[1] & (2**64 - 1), "xor": xor_all, "search_steps": w[3]}}
        print(json.dumps(line), flush=True)
    if use_pg:
        dist.destroy_process_group()


def _e2e(args, inp, index, world, run_step=None):
    """Same metric through the public API from pinned HOST buffers: every
    step copies S (INLJ) or R and S (LSJ) host->device into a validated
    Relation, runs the join and reads the 3-word result back."""
    import torch

    import paper_2111_08824_b200 as lj

    hk = inp.s.keys.cpu().pin_memory()
    hp = inp.s.payloads.cpu().pin_memory()
    h2d = 16 * len(inp.s)
    if index is None:
        rk = inp.r.keys.cpu().pin_memory()
        rp = inp.r.payloads.cpu().pin_memory()
        h2d += 16 * len(inp.r)
        o = dict(lj.DEFAULT_OPTS, **inp.opts)
        cfg = lj.LsjConfig(workers=1, fanout=o["fanout"], sample_rate=o["sample_rate"], seed=o["seed"])
    scratch = getattr(run_step, "scratch", None) if (index is not None and args.variant == "buffered") else None
    steps = max(1, min(args.steps, 3))
    times = []
    for i in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if index is None:
            s = r = None
            if args.config == "c5":
                s = lj.Relation(hk.to("cuda", non_blocking=True), hp.to("cuda", non_blocking=True), validate=True)
                r = lj.Relation(rk.to("cuda", non_blocking=True), rp.to("cuda", non_blocking=True), validate=True)
                from paper_2111_08824_b200 import dist as ljdist

                (c, sm, x), _ = ljdist.lsj_join(r.keys, r.payloads, s.keys, s.payloads, cfg)
                res = lj.JoinResult(checksum=(c, sm, x))
            else:
                res = lj.lsj_join_host(rk, rp, hk, hp, cfg)
            del s, r
        else:
            # S streamed from pinned host memory: chunk copies on a copy
            # stream overlapped with the bucketing + probe of the previous one
            words = lj.join_checksum_host(index, hk, hp, buffered=scratch is not None, scratch=scratch)
            res = lj.JoinResult(words=words)
        _ = res.checksum
        dt = time.perf_counter() - t0
        if i:
            times.append(dt)
    t = statistics.median(times)
    n_s = len(inp.s)
    how = ("lj.lsj_join_host: R's sample/fit/partition/sort overlap S's H2D" if index is None else
           "lj.join_checksum_host: S in 2^25-tuple chunks, H2D on a copy stream overlapped with the join")
    return {"value": getattr(args, "job_tuples", len(inp.r) + world * n_s) / t, "unit": "tuples/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 4 * 8, "ms_per_step": t * 1e3, "steps": steps, "path": how}


def _ncu_traffic(cfg):
    p = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variant", default=None, choices=["buffered", "direct"],
                    help="INLJ: group S by index window on device first (Request-Buffer analogue) or probe "
                         "directly; default per config (c2 buffered, c1/c3 direct)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scale", type=int, default=None, help="config size shift (tests only; not a bench number)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
