"""Randomised cross-check of the packed int16 short-read kernels on the GPU (both lane-group shapes; run once with
WSB_S16_LAT=0 and once with WSB_S16_LAT=2): AUTO == oracle for local and global alignment over ragged batches of reads up
to 154 x 152 symbols, uniform batches, random schemes inside the kernels' limits, flagged symbols, mutated copies.
Development aid: python tools/fuzz_short16.py <seed> <rounds>."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

ctx = N.Context(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bad = 0
for rd in range(rounds):
    n = int(rng.choice([3, 17, 200, 1500, 6000, 12000]))
    uniform = rng.random() < 0.4
    um, un = int(rng.integers(1, 155)), int(rng.integers(1, 153))
    qs, ss = [], []
    for k in range(n):
        m, nn = (um, un) if uniform else (int(rng.integers(1, 155)), int(rng.integers(1, 153)))
        q = rng.integers(0, 4, m).astype(np.uint8); s = rng.integers(0, 4, nn).astype(np.uint8)
        if rng.random() < 0.5:
            w = min(m, nn); at = int(rng.integers(0, nn - w + 1)); s[at:at + w] = q[:w]
            flip = rng.random(w) < 0.06; s[at:at + w][flip] = (s[at:at + w][flip] + 1) % 4
        if rng.random() < 0.05: q[int(rng.integers(0, m))] = 4
        if rng.random() < 0.03: s[int(rng.integers(0, nn))] = 4
        qs.append(q); ss.append(s)
    ql = np.array([len(x) for x in qs], np.int32); sl = np.array([len(x) for x in ss], np.int32)
    qo = np.zeros(n, np.int64); qo[1:] = np.cumsum(ql[:-1]); so = np.zeros(n, np.int64); so[1:] = np.cumsum(sl[:-1])
    qc, sc = np.concatenate(qs), np.concatenate(ss)
    idx = np.arange(n, dtype=np.int32)
    affine = rng.random() < 0.6
    if rng.random() < 0.5:
        match, mism, a, bb = 2, -1, (2 if affine else 1), 1
    else:
        match = int(rng.integers(1, 6)); mism = -int(rng.integers(0, 5)); a = int(rng.integers(1, 8)); bb = int(rng.integers(1, a + 1))
    sch = ScoringScheme(match, mism, a, bb if affine else a, "affine" if affine else "linear")
    for at in ("global", "local"):
        want = oracle.score_batch(qc, qo, ql, sc, so, sl, idx, idx, at, affine, match, mism, a, bb if affine else a)
        b = N.Batch(ctx, qc, qo, ql, sc, so, sl, idx, idx)
        b.score(sch, at, "auto"); got = b.fetch_scores(); b.close()
        if not all((g == w).all() for g, w in zip(got[:3], want)):
            bad += 1
            k = int(np.nonzero((got[0] != want[0]) | (got[1] != want[1]) | (got[2] != want[2]))[0][0])
            print(f"MISMATCH round {rd} {at} scheme {(match, mism, a, bb)} {sch.gap_model} uniform={uniform} n={n} pair {k} "
                  f"shape {(ql[k], sl[k])} got {(got[0][k], got[1][k], got[2][k])} want {(want[0][k], want[1][k], want[2][k])}", flush=True)
    print(f"round {rd}: n={n} uniform={uniform} scheme {(match, mism, a, bb)} {sch.gap_model}: mismatches so far {bad}", flush=True)
print("TOTAL MISMATCHES", bad)
