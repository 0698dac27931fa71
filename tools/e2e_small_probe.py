"""Host-side timeline of one small end-to-end step (cfg1's shape: 10 000 x 150 bp, global linear): general create path
against the metadata-free uniform one, and run_batch as a whole."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N
from bench import pinned

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
L = 150
rng = np.random.default_rng(1)
(q, kq), (s, ks) = pinned(rng.integers(0, 4, (n, L), dtype=np.uint8)), pinned(rng.integers(0, 4, (n, L), dtype=np.uint8))
scheme = W.ScoringScheme(2, -1, 1, 1, "linear")
ctx = W.get_context(0)
off = np.arange(n, dtype=np.int64) * L; ln = np.full(n, L, np.int32); idx = np.arange(n, dtype=np.int32)
for name in ("general", "uniform"):
    best = None
    for rep_ in range(20):
        t0 = time.perf_counter()
        if name == "general":
            b = N.Batch(ctx, q.reshape(-1), off, ln, s.reshape(-1), off, ln, idx, idx)
        else:
            b = N.Batch.uniform(ctx, q, L, s, L, n, packed=False)
        t1 = time.perf_counter()
        ms, nl, r = b.score_fetch(scheme, "global", "auto")
        t2 = time.perf_counter()
        b.close()
        t3 = time.perf_counter()
        cur = ((t3 - t0) * 1e6, (t1 - t0) * 1e6, (t2 - t1) * 1e6, (t3 - t2) * 1e6, ms * 1e3, nl)
        if rep_ >= 5 and (best is None or cur[0] < best[0]):
            best = cur
    print("%-8s n=%d total %.0f us: create %.0f score_fetch %.0f close %.0f (kernel %.0f us, %d launches)" % ((name, n) + best))
qp, sp = W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s)
job = W.BatchJob(qp, sp, np.stack([idx, idx], 1), W.AlignConfig("global", "linear"), scheme)
ts = []
for rep_ in range(20):
    t0 = time.perf_counter(); rep = W.run_batch(job); ts.append((time.perf_counter() - t0) * 1e6)
print("run_batch n=%d: min %.0f us median %.0f us (wall_time field %.0f us)" % (n, min(ts[5:]), sorted(ts[5:])[7], rep.wall_time * 1e6))
