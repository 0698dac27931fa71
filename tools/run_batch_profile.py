import os, sys, time, cProfile, pstats
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2205_07610_b200 as W
from bench import pinned
rng = np.random.default_rng(1)
n, L = 4_000_000, 150
(q, kq), (s, ks) = pinned(rng.integers(0, 4, (n, L), dtype=np.uint8)), pinned(rng.integers(0, 4, (n, L), dtype=np.uint8))
pairs = np.stack([np.arange(n, dtype=np.int32)] * 2, 1)
hq, hs = W.SequencePool.from_uniform(q).to_packed(), W.SequencePool.from_uniform(s).to_packed()
k1 = pinned(hq.packed); k2 = pinned(hs.packed); hq.packed, hs.packed = k1[0], k2[0]
job = W.BatchJob(hq, hs, pairs, W.AlignConfig("local", "affine"), W.ScoringScheme(), tuning=W.EngineTuning(packed=True), devices=[0])
W.run_batch(job); W.run_batch(job)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); rep = W.run_batch(job); ts.append(time.perf_counter() - t0)
print("run_batch ms:", [round(t * 1e3, 2) for t in ts], "wall_time", rep.wall_time * 1e3, "kernel_ms", rep.kernel_ms, "launches", rep.gpu_launches, "h2d", rep.h2d_bytes)
pr = cProfile.Profile(); pr.enable(); rep = W.run_batch(job); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
from paper_2205_07610_b200 import batch as B, _native as N
ident = np.arange(n, dtype=np.int32)
cfg = W.validate_config(W.AlignConfig("local", "affine"), W.ScoringScheme())
for _ in range(4):
    out = {}
    t0 = time.perf_counter(); B._run_shard(0, hq, hs, ident, ident, cfg, W.ScoringScheme(), "auto", out, True); t1 = time.perf_counter()
print("_run_shard %.2f ms, kernel %.2f, launches %d" % ((t1 - t0) * 1e3, out["ms"], out["launches"]))
ctx = W.get_context(0)
for _ in range(4):
    t0 = time.perf_counter()
    b = N.Batch.uniform(ctx, hq.packed, 150, hs.packed, 150, n, packed=True)
    t1 = time.perf_counter()
    ms2, nl2, r2 = b.score_fetch(W.ScoringScheme(), "local", "auto")
    t2 = time.perf_counter()
    b.close()
    t3 = time.perf_counter()
print("by hand: create %.2f score_fetch %.2f close %.2f (kernel %.2f)" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, ms2))
for _ in range(4):
    t0 = time.perf_counter()
    b = N.Batch.uniform(ctx, hq.packed, 150, hs.packed, 150, n, packed=True)
    ms3, nl3 = b.score(W.ScoringScheme(), "local", "auto")
    t1 = time.perf_counter()
    r3 = b.fetch_scores()
    t2 = time.perf_counter()
    b.close()
print("by hand separate: create+score %.2f fetch %.2f (kernel %.2f)" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, ms3))
print("packed dtype/shape/flags", hq.packed.dtype, hq.packed.shape, hq.packed.flags.c_contiguous, hq.packed.ctypes.data % 4096)
dest = tuple(N.pinned_empty(n) for _ in range(3))
for _ in range(4):
    t0 = time.perf_counter()
    b = N.Batch.uniform(ctx, hq.packed, 150, hs.packed, 150, n, packed=True)
    t1 = time.perf_counter()
    ms2, nl2, r2 = b.score_fetch(W.ScoringScheme(), "local", "auto", dest=dest)
    t2 = time.perf_counter()
    b.close()
print("by hand, preallocated dest: create %.2f score_fetch %.2f (kernel %.2f)" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, ms2))
keep = []
for _ in range(4):
    b = N.Batch.uniform(ctx, hq.packed, 150, hs.packed, 150, n, packed=True)
    t0 = time.perf_counter()
    d3 = tuple(N.pinned_empty(n) for _ in range(3))
    t1 = time.perf_counter()
    st_ = np.empty(n, np.int32); z_ = np.zeros(n, np.int32)
    t2 = time.perf_counter()
    ms2, nl2, r2 = b.score_fetch(W.ScoringScheme(), "local", "auto", dest=d3)
    t3 = time.perf_counter()
    b.close()
    keep = [d3]
print("pinned_empty x3 during upload %.2f ms, np.empty+zeros %.2f ms, score_fetch %.2f" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))
