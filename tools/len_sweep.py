"""int32 kernel-only GCUPS over read length (uniform batches), long-read kernel vs general kernel."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme
ctx = N.Context(0)
sch = ScoringScheme(2, -1, 2, 1, "affine")
atype = sys.argv[1] if len(sys.argv) > 1 else "local"
for L in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "300,400,512,600,800,1024,1500,2048,4096,10000").split(",")]:
    n = max(256, int(6e10 / (L * L)))
    rng = np.random.default_rng(L)
    q = rng.integers(0, 4, n * L, dtype=np.uint8); s = rng.integers(0, 4, n * L, dtype=np.uint8)
    off = np.arange(n, dtype=np.int64) * L; ln = np.full(n, L, np.int32); idx = np.arange(n, dtype=np.int32)
    b = N.Batch(ctx, q, off, ln, s, off, ln, idx, idx)
    best = min(b.score(sch, atype, os.environ.get("SWEEP_VARIANT", "i32"))[0] for _ in range(3))
    r = b.fetch_scores()
    print(f"{atype} L={L:6d} pairs={n:7d} {best:9.3f} ms {b.total_cells / best / 1e6:8.1f} GCUPS  checksum {int(r[0].astype(np.int64).sum())} {int(r[1].astype(np.int64).sum())} {int(r[2].astype(np.int64).sum())}", flush=True)
    b.close()
