"""Per-call timing of score_fetch with fresh page-locked result arrays vs preallocated ones (development probe)."""
import os, sys, time, gc
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N
from bench import pinned
rng = np.random.default_rng(1)
n, L = 4_000_000, 150
(q, kq), (s, ks) = pinned(rng.integers(0, 4, (n, L), dtype=np.uint8)), pinned(rng.integers(0, 4, (n, L), dtype=np.uint8))
hq, hs = W.SequencePool.from_uniform(q).to_packed(), W.SequencePool.from_uniform(s).to_packed()
k1 = pinned(hq.packed); k2 = pinned(hs.packed); hq.packed, hs.packed = k1[0], k2[0]
ctx = W.get_context(0)
sch = W.ScoringScheme()
def one(dest):
    t0 = time.perf_counter()
    b = N.Batch.uniform(ctx, hq.packed, 150, hs.packed, 150, n, packed=True)
    ms, nl, r = b.score_fetch(sch, "local", "auto", dest=dest)
    b.close()
    return (time.perf_counter() - t0) * 1e3, r
for mode in ("fresh", "prealloc", "fresh-keep-prev", "fresh-gc-off"):
    if mode == "fresh-gc-off": gc.disable()
    ts = []; prev = None
    dest = tuple(N.pinned_empty(n) for _ in range(3)) if mode == "prealloc" else None
    for k in range(8):
        t, r = one(dest)
        ts.append(round(t, 1))
        if mode == "fresh-keep-prev": prev = r
        del r
    print(mode, ts)
