"""Host-side timeline of one end-to-end step (create -> score -> fetch) for byte pools and 2-bit pools from pinned memory."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N
from bench import pinned

rng = np.random.default_rng(1)
n, L = 4_000_000, 150
(q, kq), (s, ks) = pinned(rng.integers(0, 4, (n, L), dtype=np.uint8)), pinned(rng.integers(0, 4, (n, L), dtype=np.uint8))
scheme = W.ScoringScheme()
ctx = W.get_context(0)
pq, ps = W.SequencePool.from_uniform(q).to_packed(), W.SequencePool.from_uniform(s).to_packed()
(pqp, k1), (psp, k2) = pinned(pq.packed), pinned(ps.packed)
for name, a, b_, packed in (("bytes", q, s, False), ("packed2", pqp, psp, True)):
    for rep_ in range(4):
        t0 = time.perf_counter()
        b = N.Batch.uniform(ctx, a, L, b_, L, n, packed=packed)
        t1 = time.perf_counter()
        ms, nl = b.score(scheme, "local", "auto")
        t2 = time.perf_counter()
        r = b.fetch_scores()
        t3 = time.perf_counter()
        b.close()
        t4 = time.perf_counter()
    for rep_ in range(4):
        t0 = time.perf_counter()
        b = N.Batch.uniform(ctx, a, L, b_, L, n, packed=packed)
        ms2, nl2, r2 = b.score_fetch(scheme, "local", "auto")
        b.close()
        t5 = time.perf_counter()
    print("%-8s create + score_fetch + close %.2f ms (kernel_ms %.2f, %d launches)" % (name, (t5 - t0) * 1e3, ms2, nl2))
    print("%-8s create %.2f score %.2f (kernel_ms %.2f, %d launches) fetch %.2f close %.2f  total %.2f ms" % (
        name, (t1 - t0) * 1e3, (t2 - t1) * 1e3, ms, nl, (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t4 - t0) * 1e3))
