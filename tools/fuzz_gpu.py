"""Randomised cross-check on the GPU: AUTO == forced int32 == oracle on mixed batches (all alignment types, random
schemes, lengths 1..4000 with repeated shapes so that packed units form, flagged symbols).  Development aid."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

ctx = N.Context(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 12
bad = 0
for rd in range(rounds):
    n = int(rng.integers(20, 400))
    shapes = [(int(rng.integers(1, 4000)), int(rng.integers(1, 4000))) for _ in range(6)] + [(150, 150), (250, 250), (600, 2100)]
    qs, ss = [], []
    for k in range(n):
        if rng.random() < 0.6:
            m, nn = shapes[int(rng.integers(0, len(shapes)))]
        else:
            m, nn = int(rng.integers(1, 600)), int(rng.integers(1, 600))
        q = rng.integers(0, 4, m).astype(np.uint8); s = rng.integers(0, 4, nn).astype(np.uint8)
        if rng.random() < 0.5 and nn >= m:
            at = int(rng.integers(0, nn - m + 1)); s[at:at + m] = q
            flip = rng.random(m) < 0.06; s[at:at + m][flip] = (s[at:at + m][flip] + 1) % 4
        if rng.random() < 0.15: q[int(rng.integers(0, m))] = 4
        if rng.random() < 0.15: s[int(rng.integers(0, nn))] = 4
        qs.append(q); ss.append(s)
    ql = np.array([len(x) for x in qs], np.int32); sl = np.array([len(x) for x in ss], np.int32)
    qo = np.zeros(n, np.int64); qo[1:] = np.cumsum(ql[:-1]); so = np.zeros(n, np.int64); so[1:] = np.cumsum(sl[:-1])
    qc, sc = np.concatenate(qs), np.concatenate(ss)
    idx = np.arange(n, dtype=np.int32)
    affine = rng.random() < 0.7
    match = int(rng.integers(1, 6)); mism = -int(rng.integers(0, 5)); a = int(rng.integers(1, 8)); bb = int(rng.integers(1, a + 1)) if affine else a
    sch = ScoringScheme(match, mism, a, bb if affine else a, "affine" if affine else "linear")
    for at in ("global", "local", "semiglobal"):
        want = oracle.score_batch(qc, qo, ql, sc, so, sl, idx, idx, at, affine, match, mism, a, bb if affine else a)
        for var in ("auto", "i32", "s16x2"):
            b = N.Batch(ctx, qc, qo, ql, sc, so, sl, idx, idx)
            b.score(sch, at, var); got = b.fetch_scores(); b.close()
            ok = all((g == w).all() for g, w in zip(got[:3], want))
            if not ok:
                bad += 1
                k = int(np.nonzero((got[0] != want[0]) | (got[1] != want[1]) | (got[2] != want[2]))[0][0])
                print(f"MISMATCH round {rd} {at} {var} scheme {(match, mism, a, bb)} {sch.gap_model} pair {k} shape {(ql[k], sl[k])} "
                      f"got {(got[0][k], got[1][k], got[2][k])} want {(want[0][k], want[1][k], want[2][k])}", flush=True)
    print(f"round {rd}: n={n} scheme {(match, mism, a, bb)} {sch.gap_model} ok so far, mismatches {bad}", flush=True)
print("TOTAL MISMATCHES", bad)
