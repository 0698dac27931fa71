import os, sys
sys.path.insert(0, "/root/repo/tools"); sys.path.insert(0, "/root/repo")
import numpy as np, bench
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme
pairs = 100_000
(qc, qo, ql), (sc, so, sl) = bench.make_pareto(pairs, 220507615)
idx = np.arange(pairs, dtype=np.int32)
ctx = N.Context(0); sch = ScoringScheme(2, -1, 2, 1, "affine")
total = float((ql.astype(np.int64) * sl).sum())
for world in (8, 1):
    shard_of, cells = N.plan_shards(ql, sl, idx, idx, world)
    times = []
    for r in range(world):
        sub = idx[shard_of == r]
        b = N.Batch(ctx, qc, qo, ql, sc, so, sl, sub, sub)
        ms = min(b.score(sch, "local", "auto")[0] for _ in range(2)); times.append(ms); b.close()
    print(f"N={world}: shard ms {[round(t,1) for t in times]} max {max(times):.1f}", flush=True)
