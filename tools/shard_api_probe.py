"""Where the time of run_batch(devices=[0, 0, ...]) goes on ONE GPU (shards of one device serialise on the context lock):
per-shard timings of create / score / fetch from pinned host pools.  Development probe."""
import os, sys, time, threading
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N
from bench import pinned

rng = np.random.default_rng(1)
n, L = 4_000_000, 150
(q, kq), (s, ks) = pinned(rng.integers(0, 4, (n, L), dtype=np.uint8)), pinned(rng.integers(0, 4, (n, L), dtype=np.uint8))
pairs = np.stack([np.arange(n, dtype=np.int32)] * 2, 1)
scheme = W.ScoringScheme()
for devs in ([0], [0, 0], [0, 0, 0, 0]):
    job = W.BatchJob(W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s), pairs, W.AlignConfig("local", "affine"), scheme, devices=devs)
    W.run_batch(job); W.run_batch(job)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); rep = W.run_batch(job); ts.append(time.perf_counter() - t0)
    print(len(devs), "shards: run_batch %.1f ms (wall_time %.1f), kernel_ms(max) %.2f" % (min(ts) * 1e3, rep.wall_time * 1e3, rep.kernel_ms))
# one quarter by hand
ctx = W.get_context(0)
k = n // 4
for rep_ in range(3):
    t0 = time.perf_counter()
    b = N.Batch.uniform(ctx, q[:k], L, s[:k], L, k, packed=False)
    t1 = time.perf_counter()
    b.score(scheme, "local", "auto")
    t2 = time.perf_counter()
    r = b.fetch_scores()
    t3 = time.perf_counter()
    b.close()
    t4 = time.perf_counter()
    print("quarter by hand: create %.2f score %.2f fetch %.2f close %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3))
