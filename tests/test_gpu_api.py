"""The reference-facing APIs around the hot paths, mirroring the
reference's own tests (-m gpu): request buffers (tests/test_buffers.py:
70-160 -> buffers.py:73-150) and the LSJ range partition
(tests/test_lsj.py:70-110 -> lsj.py:133-209)."""

import math
from collections import Counter

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lj():
    import paper_2111_08824_b200 as lj

    return lj


@pytest.fixture(scope="module")
def index(lj):
    # seq_h-like keys (the reference fixture: gen_dataset("seq_h", 4000, 3)):
    # sorted, gappy, unique
    rng = np.random.default_rng(3)
    keys = np.cumsum(rng.integers(1, 4, 4000)).astype(np.uint64)
    return lj.GappedRmiIndex(4.0, 32).fit(lj.make_relation(keys, 7))


def _collect_first(lj, index, keys, plan):
    got = {}

    def sink(tags, payloads, found):
        for t, p, f in zip(tags.tolist(), payloads.tolist(), found.tolist()):
            assert t not in got  # exactly one result per input key
            got[t] = (f, p if f else None)

    stats = lj.buffered_probe(index, keys, plan, sink)
    return got, stats


def _lookup(index, k):
    v = index.lookup(np.uint64(k))
    return None if v is None else int(v)


def test_buffered_single_key(lj, index):
    key = index.gkeys[index.bitmap][100]
    got, _ = _collect_first(lj, index, np.asarray([key], dtype=np.uint64), lj.plan_buffers(33, 32, cap=5))
    assert got[0] == (True, _lookup(index, key))


def test_buffered_multiset_equals_unbuffered(lj, index):
    probes = np.random.default_rng(0).integers(0, 12000, 3000).astype(np.uint64)
    got, stats = _collect_first(lj, index, probes, lj.plan_buffers(33, 32, cap=37))
    assert len(got) == probes.size
    for i, k in enumerate(probes):
        e = _lookup(index, k)
        assert got[i] == ((e is not None), e)
    assert stats.predictions == probes.size


def test_buffered_any_cap_and_order(lj, index):
    base = np.random.default_rng(1).integers(0, 12000, 600).astype(np.uint64)
    ref = Counter((_lookup(index, k) is not None, _lookup(index, k)) for k in base)
    for cap in (1, 2, 19, 600, 10_000):
        for seed in (0, 1):
            probes = np.random.default_rng(seed).permutation(base)
            got, _ = _collect_first(lj, index, probes, lj.plan_buffers(33, 32, cap=cap))
            assert Counter(got.values()) == ref


def test_buffered_flush_counts_presorted(lj, index):
    cap = 200
    rng = np.random.default_rng(2)
    probes = rng.choice(index.gkeys[index.bitmap], 3000, replace=True)
    leaf = index.leaf_of(probes).cpu().numpy()
    probes = probes[np.argsort(leaf, kind="stable")]
    flushes = []
    lj.buffered_probe(index, probes, lj.plan_buffers(33, 32, cap=cap), lambda t, p, f: flushes.append(len(t)))
    counts = np.bincount(index.leaf_of(probes).cpu().numpy())
    assert len(flushes) == int(sum(math.ceil(c / cap) for c in counts if c))


def test_buffered_collect_all_duplicates(lj):
    keys = np.array([4, 4, 9, 9, 9, 12], dtype=np.uint64)
    rel = lj.make_relation(keys, 3)
    idx = lj.GappedRmiIndex(2.0, 4).fit(rel)
    pairs = []
    lj.buffered_probe(idx, np.array([9, 4, 1], dtype=np.uint64), lj.plan_buffers(5, 4, cap=2),
                      lambda t, p: pairs.extend(zip(t.tolist(), p.tolist())), collect="all")
    by_tag = Counter(t for t, _ in pairs)
    assert by_tag[0] == 3 and by_tag[1] == 2 and 2 not in by_tag


def test_buffered_invalid_collect(lj, index):
    with pytest.raises(ValueError):
        lj.buffered_probe(index, np.array([1], dtype=np.uint64), lj.plan_buffers(33, 32), lambda *a: None,
                          collect="x")


def test_buffered_leaf_switches_match_the_schedule(lj, index):
    """The stats' leaf switches are those of the flush schedule, which the
    buffered runner counts without a per-flush loop (bench.py:174-179)."""
    from paper_2111_08824_b200.buffers import schedule_leaf_switches

    probes = np.random.default_rng(5).integers(0, 12000, 5000).astype(np.uint64)
    stats = lj.buffered_probe(index, probes, lj.plan_buffers(33, 32, cap=7), lambda *a: None)
    assert stats.leaf_switches == schedule_leaf_switches(index.leaf_of(probes), 7)
    assert stats.leaf_switches < probes.size  # buffering groups leaves


def test_range_partition_perfect_quartiles(lj):
    from paper_2111_08824_b200.lsj import range_partition

    rel = lj.make_relation(np.arange(100, dtype=np.uint64), 1)
    model = lj.RecursiveModelIndex(1).fit(np.arange(100, dtype=np.uint64))
    part = range_partition(rel, model, 4, lj.LsjConfig(workers=4, fanout=100))
    assert part.ranges == [(0, 25), (25, 50), (50, 75), (75, 100)]
    k = part.keys.cpu().numpy().view(np.uint64)
    for i, (a, b) in enumerate(part.ranges):
        assert set(k[a:b].tolist()) == set(range(25 * i, 25 * i + 25))


def test_range_partition_skewed_multiset_boundaries_histogram(lj):
    from paper_2111_08824_b200.lsj import range_partition

    rng = np.random.default_rng(6)
    keys = np.floor(1e9 * rng.lognormal(0, 2, 100_000)).astype(np.uint64)
    rel = lj.make_relation(keys, 6)
    model = lj.RecursiveModelIndex(1000).fit(np.sort(keys[::100]))
    cfg = lj.LsjConfig(workers=8, fanout=10000)
    part = range_partition(rel, model, 8, cfg)
    pk = part.keys.cpu().numpy().view(np.uint64)
    assert np.array_equal(np.sort(pk), np.sort(keys))
    # every key of range i maps to worker i at the reference's scale
    fine = lj.partition_index(model, part.keys, cfg.effective_fanout()).cpu().numpy()
    per_worker = fine // (cfg.effective_fanout() // 8)
    for i, (a, b) in enumerate(part.ranges):
        assert np.all(per_worker[a:b] == i)
    assert part.histogram.shape == (8, 8) and part.histogram.sum() == len(rel)
    assert np.array_equal(part.histogram.sum(axis=0), [b - a for a, b in part.ranges])
    # prefix sums: worker w's slice of target t starts where the reference writes it
    assert np.array_equal(part.prefix_sums[0], [a for a, _ in part.ranges])
