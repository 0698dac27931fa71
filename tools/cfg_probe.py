"""Kernel-only throughput of every BASELINE.json config at a reduced pair count, with an oracle spot check.

    python tools/cfg_probe.py [--cfgs 1,2,3,4,5] [--scale 1.0] [--check 64]

Not the bench contract (that is bench.py); this is the development probe behind the per-config table in DESIGN.md.
"""
import argparse, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

ap = argparse.ArgumentParser()
ap.add_argument("--cfgs", default="1,2,3,4,5")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--check", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = N.Context(0)
AFF = ScoringScheme(2, -1, 2, 1, "affine")
LIN = ScoringScheme(2, -1, 1, 1, "linear")


def uniform(n, L, seed):
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 4, n * L, dtype=np.uint8); s = rng.integers(0, 4, n * L, dtype=np.uint8)
    off = np.arange(n, dtype=np.int64) * L; ln = np.full(n, L, np.int32); idx = np.arange(n, dtype=np.int32)
    return (q, off, ln), (s, off, ln), idx


def pareto(n, seed, cap=100_000):
    """cfg5 lengths: L = min(cap, floor(100/(1-u))), n = clip(round(L*v), 100, cap), v ~ U[0.8, 1.25]."""
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    L = np.minimum(cap, np.floor(100.0 / (1.0 - u))).astype(np.int64)
    v = rng.uniform(0.8, 1.25, n)
    M = np.clip(np.rint(L * v), 100, cap).astype(np.int64)
    def pool(lens):
        off = np.zeros(n, np.int64); off[1:] = np.cumsum(lens[:-1])
        return rng.integers(0, 4, int(lens.sum()), dtype=np.uint8), off, lens.astype(np.int32)
    return pool(L), pool(M), np.arange(n, dtype=np.int32)


def check(qp, sp, idx, got, atype, sch, limit):
    if limit <= 0:
        return "unchecked"
    cells = qp[2][idx].astype(np.int64) * sp[2][idx]
    cand = np.nonzero(cells <= 4e8)[0]
    sel = cand[np.linspace(0, len(cand) - 1, min(limit, len(cand))).astype(np.int64)] if len(cand) else cand
    big = np.argsort(cells)[-2:] if cells.max() <= 1.2e10 else np.array([], np.int64)
    sel = np.unique(np.concatenate([sel, big]))
    t0 = time.time()
    w = oracle.score_batch(qp[0], qp[1], qp[2], sp[0], sp[1], sp[2], idx[sel], idx[sel], atype, sch.gap_model == "affine",
                           sch.match_score, sch.mismatch_score, sch.gap_open, sch.gap_extend)
    ok = all((g[sel] == x).all() for g, x in zip(got[:3], w))
    return f"oracle {'OK' if ok else 'MISMATCH'} on {len(sel)} pairs ({time.time() - t0:.1f}s)"


def run(name, qp, sp, idx, atype, sch, variant="auto", traceback=False, chk=a.check):
    b = N.Batch(ctx, qp[0], qp[1], qp[2], sp[0], sp[1], sp[2], idx, idx)
    best = 1e30
    for r in range(a.reps):
        ms, nl = b.traceback(sch, atype) if traceback else b.score(sch, atype, variant)
        best = min(best, ms)
    got = b.fetch_scores()
    msg = check(qp, sp, idx, got, atype, sch, chk)
    print(f"{name:34s} pairs={len(idx):8d} cells={b.total_cells:.3e} best {best:9.3f} ms {b.total_cells / best / 1e6:8.1f} GCUPS "
          f"launches={nl} {msg}", flush=True)
    b.close()


for c in a.cfgs.split(","):
    if c == "1":
        qp, sp, idx = uniform(10_000, 150, 1)
        run("cfg1 global/linear 150bp f16", qp, sp, idx, "global", LIN, "auto")
        run("cfg1 global/linear 150bp i32", qp, sp, idx, "global", LIN, "i32")
        qp, sp, idx = uniform(1_000_000, 150, 1)
        run("cfg1x100 global/linear 150bp f16", qp, sp, idx, "global", LIN, "auto")
    if c == "2":
        qp, sp, idx = uniform(int(1_000_000 * a.scale), 150, 2)
        run("cfg2 local/affine 150bp f16", qp, sp, idx, "local", AFF, "f16x2")
        run("cfg2 local/affine 150bp i32", qp, sp, idx, "local", AFF, "i32")
    if c == "3":
        qp, sp, idx = uniform(int(200_000 * a.scale), 250, 3)
        run("cfg3 semiglobal/affine 250bp score", qp, sp, idx, "semiglobal", AFF, "auto")
        run("cfg3 semiglobal/affine 250bp tb", qp, sp, idx, "semiglobal", AFF, traceback=True)
    if c == "4":
        qp, sp, idx = uniform(int(2_500 * a.scale), 10_000, 4)
        run("cfg4 global/affine 10kbp i32", qp, sp, idx, "global", AFF, "auto", chk=min(a.check, 8))
    if c == "5":
        qp, sp, idx = pareto(int(20_000 * a.scale), 5, cap=int(os.environ.get("CFG5_CAP", 100_000)))
        print("cfg5 max lens", int(qp[2].max()), int(sp[2].max()), "pairs > 10k:", int((qp[2] > 10_000).sum()))
        run("cfg5 local/affine pareto", qp, sp, idx, "local", AFF, "auto", chk=min(a.check, 32))
