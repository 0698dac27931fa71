"""Randomised traceback cross-check on the GPU: spans and CIGAR runs == oracle (refdp.ref_traceback restatement) on
mixed batches, all alignment types, random schemes, flagged symbols, several code-scratch chunk sizes.  Development aid."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

ctx = N.Context(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 10
bad = 0
for rd in range(rounds):
    os.environ["WSB_TB_SCRATCH_MB"] = str(int(rng.choice([1, 4, 64, 4096])))
    n = int(rng.integers(10, 300))
    short = rng.random() < 0.5   # every subject within one stage: affine global / semiglobal take the packed int16 fill
    qs, ss = [], []
    for k in range(n):
        m = int(rng.integers(1, 1200)) if (rng.random() < 0.3 and not short) else int(rng.integers(1, 300))
        q = rng.integers(0, 4, m).astype(np.uint8)
        if rng.random() < 0.6:
            keep = rng.random(m) > 0.04
            s = q[keep].copy()
            ins = np.nonzero(rng.random(len(s)) < 0.04)[0]
            s = np.insert(s, ins, rng.integers(0, 4, len(ins)).astype(np.uint8)) if len(s) else rng.integers(0, 4, 3).astype(np.uint8)
            flip = rng.random(len(s)) < 0.05; s[flip] = (s[flip] + 1) % 4
        else:
            s = rng.integers(0, 4, int(rng.integers(1, 400))).astype(np.uint8)
        if len(s) == 0: s = np.array([1], np.uint8)
        if short: s = s[:int(rng.choice([128, 256]))].copy()
        if rng.random() < 0.15: q[int(rng.integers(0, len(q)))] = 4
        if rng.random() < 0.15: s[int(rng.integers(0, len(s)))] = 4
        qs.append(q); ss.append(s)
    ql = np.array([len(x) for x in qs], np.int32); sl = np.array([len(x) for x in ss], np.int32)
    qo = np.zeros(n, np.int64); qo[1:] = np.cumsum(ql[:-1]); so = np.zeros(n, np.int64); so[1:] = np.cumsum(sl[:-1])
    qc, sc = np.concatenate(qs), np.concatenate(ss)
    idx = np.arange(n, dtype=np.int32)
    affine = rng.random() < 0.7
    match = int(rng.integers(1, 6)); mism = -int(rng.integers(0, 5)); a = int(rng.integers(1, 8)); bb = int(rng.integers(0, a + 2)) if affine else a
    sch = ScoringScheme(match, mism, a, bb if affine else a, "affine" if affine else "linear")
    for at in ("global", "local", "semiglobal"):
        ref = oracle.traceback_batch(qc, qo, ql, sc, so, sl, idx, idx, at, affine, match, mism, a, bb if affine else a)
        b = N.Batch(ctx, qc, qo, ql, sc, so, sl, idx, idx)
        b.traceback(sch, at); tb = b.fetch_traceback(); b.close()
        ok = all((tb[k] == ref[k]).all() for k in ("score", "q_start", "q_end", "s_start", "s_end"))
        off = tb["cigar_off"]
        for k in range(n):
            got = tb["cigar"][off[k]:off[k + 1]]
            if len(got) != ref["n_ops"][k] or not (got == ref["ops_packed"][k, :len(got)]).all():
                ok = False
                print(f"CIGAR MISMATCH round {rd} {at} pair {k} shape {(ql[k], sl[k])} scheme {(match, mism, a, bb)} {sch.gap_model}", flush=True)
                break
        if not ok:
            bad += 1
            print(f"MISMATCH round {rd} {at} scheme {(match, mism, a, bb)} {sch.gap_model}", flush=True)
    print(f"round {rd}: n={n} scheme {(match, mism, a, bb)} {sch.gap_model} scratch {os.environ['WSB_TB_SCRATCH_MB']} MB, mismatches {bad}", flush=True)
print("TOTAL MISMATCHES", bad)
