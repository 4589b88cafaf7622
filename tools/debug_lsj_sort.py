import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2111_08824_b200 as lj
from paper_2111_08824_b200.lsj import sort_relation, sort_diag, LsjModel
def _np(t): return t.detach().cpu().numpy().view(np.uint64)
rng = np.random.default_rng(5)
base = np.unique(np.floor(2.0**40 * rng.lognormal(0, 1.5, 60000)).astype(np.uint64))
w = 1.0 / np.arange(1, base.size + 1)
keys = base[rng.choice(base.size, 200000, p=w / w.sum())]
pays = np.arange(1, keys.size + 1, dtype=np.uint64)
r = lj.Relation(keys, pays)
m = lj.RecursiveModelIndex(100).fit(np.sort(keys[::10]))
srt = sort_relation(r.keys, r.payloads, m, 64)
k = _np(srt.keys.contiguous())
bad = np.nonzero(k[:-1] > k[1:])[0]
print("diag", sort_diag(srt.diag), "nbad", bad.size, "first bad", bad[:10])
vals, cnts = np.unique(keys, return_counts=True)
print("top counts", np.sort(cnts)[-5:])
if bad.size:
    i = bad[0]
    print("around", k[max(0,i-3):i+4])
    # find which run of equal keys
    top = vals[np.argmax(cnts)]
    pos = np.nonzero(k == top)[0]
    print("top key", top, "count", cnts.max(), "positions", pos.min(), pos.max(), "expected start", np.searchsorted(np.sort(keys), top))
for n in (2000, 9000, 50000):
    rng = np.random.default_rng(n)
    kk = rng.integers(0, 2**63, n, dtype=np.uint64); kk[: n // 10] = kk[n // 10]
    pp = rng.integers(1, 2**63, n, dtype=np.uint64)
    rr = lj.Relation(kk, pp)
    rmi = lj.RecursiveModelIndex(1).fit(np.array([12345], np.uint64))
    s2 = sort_relation(rr.keys, rr.payloads, LsjModel.uniform(rmi, 1), 1)
    k2 = _np(s2.keys.contiguous())
    print(n, "sorted", bool(np.all(k2[:-1] <= k2[1:])), "perm", sorted(zip(k2.tolist(), _np(s2.payloads.contiguous()).tolist())) == sorted(zip(kk.tolist(), pp.tolist())), sort_diag(s2.diag))
