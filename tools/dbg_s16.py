"""Debug aid: packed int16 short kernel against the oracle on small batches; prints the first mismatches."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
from helpers import gpu_scores, oracle_scores, scheme_of
from paper_2205_07610_b200 import _native as N

ctx = N.Context(0)
rng = np.random.default_rng(5)
for name, lens, npairs in (("uniform150", (150, 150), 64), ("uniform40", (40, 40), 64), ("ragged", None, 400)):
    for gap in ("affine", "linear"):
        scheme = scheme_of((2, -1, 2, 1) if gap == "affine" else (2, -1, 1, 1), gap)
        qs, ss = [], []
        for i in range(npairs):
            m = lens[0] if lens else int(rng.integers(20, 154)); n = lens[1] if lens else int(rng.integers(20, 152))
            q = rng.integers(0, 4, m, dtype=np.uint8); s = rng.integers(0, 4, n, dtype=np.uint8)
            if i % 2: s[: min(m, n)] = q[: min(m, n)]; s[n // 2] = (s[n // 2] + 1) % 4
            qs.append(q); ss.append(s)
        pairs = [(i, i) for i in range(npairs)]
        want = oracle_scores(qs, ss, pairs, scheme, "local")
        got = gpu_scores(ctx, qs, ss, pairs, scheme, "local", "s16x2")
        bad_s = np.nonzero(got[0] != want[0])[0]
        bad_p = np.nonzero((got[0] == want[0]) & ((got[1] != want[1]) | (got[2] != want[2])))[0]
        print(f"{name} {gap}: score mismatches {len(bad_s)}, position-only mismatches {len(bad_p)} of {npairs}")
        for k in list(bad_s[:6]) + list(bad_p[:6]):
            print(f"   pair {k} m={len(qs[k])} n={len(ss[k])}: got {(got[0][k], got[1][k], got[2][k])} want {(want[0][k], want[1][k], want[2][k])}")
