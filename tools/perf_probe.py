"""Quick kernel-only throughput probe (not the bench contract): uniform random-ACGT batches through the C ABI."""
import argparse, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", type=int, default=1_000_000)
ap.add_argument("--len", type=int, default=150)
ap.add_argument("--type", default="local")
ap.add_argument("--gap", default="affine")
ap.add_argument("--variants", default="f16x2,i32")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
rng = np.random.default_rng(1)
n, L = a.pairs, a.len
q = rng.integers(0, 4, n * L, dtype=np.uint8); s = rng.integers(0, 4, n * L, dtype=np.uint8)
off = np.arange(n, dtype=np.int64) * L; ln = np.full(n, L, np.int32); idx = np.arange(n, dtype=np.int32)
ctx = N.Context(0)
t0 = time.time(); b = N.Batch(ctx, q, off, ln, s, off, ln, idx, idx); t1 = time.time()
print(f"upload {t1 - t0:.3f}s  cells {b.total_cells:.3e}  SMs {ctx.sm_count}")
sch = ScoringScheme(2, -1, 2, 1, "affine") if a.gap == "affine" else ScoringScheme(2, -1, 1, 1, "linear")
for var in a.variants.split(","):
    for r in range(a.reps):
        ms, nl = b.score(sch, a.type, var)
        print(f"{var:6s} {a.type}/{a.gap} L={L} pairs={n}: {ms:8.3f} ms  {b.total_cells / ms / 1e6:9.1f} GCUPS  launches={nl}")
    sc = b.fetch_scores()
    print("  checksum", int(sc[0].astype(np.int64).sum()), int(sc[1].astype(np.int64).sum()), int(sc[2].astype(np.int64).sum()))
