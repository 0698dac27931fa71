"""Projected multi-GPU behaviour of cfg5 on ONE GPU: shard the 100 000-pair batch with wsb_plan_shards for N = 1, 2, 4, 8,
run every shard alone (kernel-only time, CUDA events) and report the slowest shard -- what an N-GPU run would be bound by,
since shards share no state.  A projection for DESIGN.md, not a bench value."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
(qc, qo, ql), (sc, so, sl) = bench.make_pareto(pairs, 220507615)
idx = np.arange(pairs, dtype=np.int32)
ctx = N.Context(0)
sch = ScoringScheme(2, -1, 2, 1, "affine")
total = float((ql.astype(np.int64) * sl).sum())
base = None
for world in (1, 2, 4, 8):
    shard_of, cells = N.plan_shards(ql, sl, idx, idx, world)
    times = []
    for r in range(world):
        sub = idx[shard_of == r]
        b = N.Batch(ctx, qc, qo, ql, sc, so, sl, sub, sub)
        ms = min(b.score(sch, "local", "auto")[0] for _ in range(2))
        times.append(ms)
        b.close()
    worst = max(times)
    base = base or worst
    print(f"N={world}: shard ms min {min(times):8.1f} max {worst:8.1f}  cells/shard {cells.min():.3e}..{cells.max():.3e}  "
          f"projected {total / worst / 1e6:8.0f} GCUPS  speed-up {base / worst:4.2f}x  efficiency {base / worst / world:4.2f}", flush=True)
