"""Where does the end-to-end time of the cfg3 traceback batch go?  (host buffers -> spans + CIGAR runs on the host)"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N
n, L = int(os.environ.get("PAIRS", 1_000_000)), 250
rng = np.random.default_rng(1)
def pin(a):
    t = torch.empty(a.shape, dtype=torch.uint8, pin_memory=True); v = t.numpy(); v[...] = a; return v, t
q, qk = pin(rng.integers(0, 4, (n, L), dtype=np.uint8)); s, sk = pin(rng.integers(0, 4, (n, L), dtype=np.uint8))
s[::2] = q[::2]   # half the pairs related (few runs), half unrelated (~77 runs)
off = np.arange(n, dtype=np.int64) * L; ln = np.full(n, L, np.int32); idx = np.arange(n, dtype=np.int32)
ctx = W.get_context(0); sch = W.ScoringScheme()
for rep in range(4):
    t0 = time.perf_counter()
    b = N.Batch(ctx, q.reshape(-1), off, ln, s.reshape(-1), off, ln, idx, idx)
    t1 = time.perf_counter(); ms, nl = b.traceback(sch, "semiglobal")
    t2 = time.perf_counter(); res = b.fetch_traceback()
    t3 = time.perf_counter(); b.close(); t4 = time.perf_counter()
    print(f"create {t1-t0:.4f}  traceback {t2-t1:.4f} (kernels {ms:.1f} ms, {nl} launches)  fetch {t3-t2:.4f} ({res['cigar'].nbytes/1e6:.0f} MB runs)"
          f"  close {t4-t3:.4f}  total {t4-t0:.4f}", flush=True)
pq, ps = W.SequencePool(q.reshape(-1), off, ln), W.SequencePool(s.reshape(-1), off, ln)
job = W.BatchJob(pq, ps, np.stack([idx, idx], 1), W.AlignConfig("semiglobal", "affine", "traceback"), sch)
for rep in range(4):
    t0 = time.perf_counter(); r = W.run_batch(job); t1 = time.perf_counter()
    print(f"run_batch {t1-t0:.4f} s -> {r.total_cells/(t1-t0)/1e9:.0f} GCUPS", flush=True)
