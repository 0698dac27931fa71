"""Kernel-only traceback throughput outside the BASELINE configs: local alignments and ragged short-read batches.
Run twice (default and WSB_TB_NO16=1) to compare the packed int16 fill with the int32 fill.  Development probe.

    python tools/tb_probe.py [--pairs 400000]
"""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", type=int, default=400_000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = N.Context(0)
AFF = ScoringScheme(2, -1, 2, 1, "affine")
rng = np.random.default_rng(5)


def pools(lens_q, lens_s):
    def pool(lens):
        off = np.zeros(len(lens), np.int64); off[1:] = np.cumsum(lens[:-1])
        return rng.integers(0, 4, int(lens.sum()), dtype=np.uint8), off, lens.astype(np.int32)
    return pool(lens_q), pool(lens_s), np.arange(len(lens_q), dtype=np.int32)


def run(name, qp, sp, idx, atype):
    b = N.Batch(ctx, qp[0], qp[1], qp[2], sp[0], sp[1], sp[2], idx, idx)
    best = min(b.traceback(AFF, atype)[0] for _ in range(a.reps))
    print(f"{name:44s} pairs={len(idx):8d} cells={b.total_cells:.3e} best {best:9.3f} ms {b.total_cells / best / 1e6:8.1f} GCUPS"
          f" ({'int32 fill' if os.environ.get('WSB_TB_NO16') else 'packed int16 fill'})", flush=True)
    b.close()


n = a.pairs
L = np.full(n, 150, np.int64)
run("local affine 150 bp uniform + CIGAR", *pools(L, L), "local")
run("global affine 150 bp uniform + CIGAR", *pools(L, L), "global")
lq = rng.integers(100, 251, n); ls = np.clip(np.rint(lq * rng.uniform(0.85, 1.15, n)), 50, 256).astype(np.int64)
for at in ("semiglobal", "local"):
    run(f"{at} affine 100-250 bp ragged + CIGAR", *pools(lq, ls), at)
