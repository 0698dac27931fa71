"""Where does the end-to-end time of a 4M-pair batch go? (host buffers -> results), byte pools vs 2-bit pools."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N
n, L = int(os.environ.get("PAIRS", 4_000_000)), 150
rng = np.random.default_rng(1)
def pin(a):
    t = torch.empty(a.shape, dtype=torch.uint8, pin_memory=True); v = t.numpy(); v[...] = a; return v, t
q, qk = pin(rng.integers(0, 4, (n, L), dtype=np.uint8)); s, sk = pin(rng.integers(0, 4, (n, L), dtype=np.uint8))
off = np.arange(n, dtype=np.int64) * L; ln = np.full(n, L, np.int32); idx = np.arange(n, dtype=np.int32)
ctx = W.get_context(0); sch = W.ScoringScheme()
pq, ps = W.SequencePool(q.reshape(-1), off, ln), W.SequencePool(s.reshape(-1), off, ln)
t0 = time.perf_counter(); kq, ks = pq.to_packed(), ps.to_packed(); print(f"host packing of both pools {time.perf_counter() - t0:.2f} s")
kq.packed, kqk = pin(kq.packed); ks.packed, ksk = pin(ks.packed)
for name, packed in (("bytes", None), ("packed2", ((kq.packed, None), (ks.packed, None)))):
    for rep in range(4):
        t0 = time.perf_counter()
        b = N.Batch(ctx, q.reshape(-1), off, ln, s.reshape(-1), off, ln, idx, idx, packed=packed)
        t1 = time.perf_counter(); ms, nl = b.score(sch, "local", "f16x2")
        t2 = time.perf_counter(); res = b.fetch_scores()
        t3 = time.perf_counter(); b.close(); t4 = time.perf_counter()
        print(f"{name:8s} create {t1-t0:.3f}  score {t2-t1:.3f} (kernel {ms:.1f} ms, {nl} launches)  fetch {t3-t2:.3f}  close {t4-t3:.3f}  total {t4-t0:.3f}")
for name, a, b_ in (("bytes", pq, ps), ("packed2", kq, ks)):
    job = W.BatchJob(a, b_, np.stack([idx, idx], 1), W.AlignConfig("local", "affine"), sch)
    for rep in range(4):
        t0 = time.perf_counter(); r = W.run_batch(job); t1 = time.perf_counter()
        print(f"{name:8s} run_batch {t1-t0:.3f} s  -> {r.total_cells/(t1-t0)/1e9:.0f} GCUPS  (wall_time field {r.wall_time:.3f})")
