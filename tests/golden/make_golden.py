"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (the reference tree does not travel to the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Outputs (committed):
    tests/golden/kat.json          frozen known-answer cases from the reference's own tests / SPEC
    tests/golden/random_small.json seeded random pairs, all 6 (type x gap) combos, several schemes, with
                                   ref_score, ref_traceback, engine_score and (where legal) engine_score_packed results
    tests/golden/adversarial.json  flagged symbols, homopolymers, 1xL, lengths straddling lane-group widths, ...

Every record carries the inputs as text so the tests need nothing but this file.
"""
import json
import os
import sys
import warnings

import numpy as np

import waveseq as W
from waveseq.io import cigar_string

HERE = os.path.dirname(os.path.abspath(__file__))
BASES = np.array(list("ACGT"))
COMBOS = [(a, g) for a in ("global", "local", "semiglobal") for g in ("linear", "affine")]
AFFINE = [(2, -1, 2, 1), (3, -2, 4, 1), (1, -3, 2, 2), (5, -4, 10, 1), (2, -9, 2, 1), (2, -1, 1, 3), (1, -1, 0, 0)]
LINEAR = [(2, -1, 1, 1), (2, -1, 2, 2), (1, -1, 1, 1), (3, -2, 5, 5), (4, -3, 0, 0)]


def text(rng, n, alphabet=BASES):
    return "".join(alphabet[rng.integers(0, len(alphabet), n)])


def mutate(rng, t, sub=0.05, ins=0.02, dele=0.02):
    out = []
    for ch in t:
        r = rng.random()
        if r < dele:
            continue
        if r < dele + ins:
            out.append(BASES[rng.integers(0, 4)])
        if rng.random() < sub:
            out.append(BASES[rng.integers(0, 4)])
        else:
            out.append(ch)
    return "".join(out) or "A"


def record(q, s, at, gm, sch, with_tb=True, with_engine=True):
    scheme = W.ScoringScheme(sch[0], sch[1], sch[2], sch[3], gm)
    cfg = W.AlignConfig(at, gm, "score_only")
    Q, S = W.encode_sequence("q", q), W.encode_sequence("s", s)
    score, end = W.ref_score(Q, S, cfg, scheme)
    rec = dict(q=q, s=s, align_type=at, gap_model=gm, scheme=list(sch), score=int(score), end=[int(end[0]), int(end[1])])
    if with_engine:
        es, ee, ec = W.engine_score(Q, S, cfg, scheme)
        assert (es, tuple(ee)) == (score, tuple(end)), (q, s, at, gm, sch)
        rec["engine"] = [int(es), int(ee[0]), int(ee[1]), int(ec)]
    if with_tb:
        tb = W.ref_traceback(Q, S, W.AlignConfig(at, gm, "traceback"), scheme)
        assert tb.score == score
        rs = W.rescore_alignment(tb, Q, S, scheme)
        if rs != score:
            assert gm == "affine" and sch[3] > sch[2], (q, s, at, gm, sch, rs, score)  # beta > alpha: adjacent opens beat a run
        rec_rescore = int(rs)
        rec["tb"] = dict(q_start=tb.q_start, q_end=tb.q_end, s_start=tb.s_start, s_end=tb.s_end,
                         cigar=cigar_string(tb), cells=tb.cells_computed, rescore=rec_rescore)
    return rec


def main():
    warnings.simplefilter("ignore")
    # ---- frozen KATs (pkg/tests/test_refdp.py:18-72) ----
    kat = [
        record("ACGT", "AGT", "global", "linear", (2, -1, 1, 1)),
        record("AAAA", "AA", "global", "affine", (2, -1, 2, 1)),
        record("ACG", "TTACGTT", "semiglobal", "affine", (2, -1, 2, 1)),
        record("TTACGTT", "ACG", "local", "affine", (2, -1, 2, 1)),
        record("TTTT", "CCCC", "local", "affine", (2, -1, 2, 1)),
        record("AA", "A", "global", "linear", (2, -1, 1, 1)),
        record("ACGT", "ACGT", "global", "linear", (2, -1, 1, 1)),
        record("A" * 40, "A" * 20, "global", "affine", (2, -1, 2, 1)),
        record("A" * 20, "A" * 40, "global", "affine", (2, -1, 2, 1)),
    ]
    expect = [(5, [4, 3], "1M1I2M"), (1, [4, 2], None), (6, None, "3M"), (6, None, "3M"), (0, [0, 0], ""),
              (1, None, "1I1M"), (8, [4, 4], "4M")]
    for rec, (sc, end, cig) in zip(kat, expect):
        assert rec["score"] == sc
        assert end is None or rec["end"] == end
        assert cig is None or rec["tb"]["cigar"] == cig, (rec, cig)
    json.dump(kat, open(os.path.join(HERE, "kat.json"), "w"), indent=0)

    # ---- seeded random, short (traceback + engine), every combo x several schemes ----
    rng = np.random.default_rng(220507610)
    rnd = []
    for at, gm in COMBOS:
        pool = AFFINE if gm == "affine" else LINEAR
        for k in range(70):
            sch = pool[k % len(pool)]
            m, n = int(rng.integers(1, 90)), int(rng.integers(1, 90))
            q = text(rng, m)
            s = mutate(rng, q) if k % 3 == 0 else text(rng, n)
            rnd.append(record(q, s, at, gm, sch))
    # longer pairs, score + end only (engine + ref), lengths up to 300 like test_acceptance C1
    for at, gm in COMBOS:
        pool = AFFINE if gm == "affine" else LINEAR
        for k in range(16):
            sch = pool[k % len(pool)]
            m, n = int(rng.integers(100, 301)), int(rng.integers(100, 301))
            q = text(rng, m)
            s = mutate(rng, q, 0.08, 0.03, 0.03) if k % 2 == 0 else text(rng, n)
            rnd.append(record(q, s, at, gm, sch, with_tb=(k % 4 == 0)))
    # packed-16 engine results: both halves must equal the unpacked results (test_engine.py:150-184)
    packed = []
    for at, gm in COMBOS:
        sch = (2, -1, 2, 1) if gm == "affine" else (2, -1, 1, 1)
        scheme = W.ScoringScheme(*sch, gm)
        cfg = W.AlignConfig(at, gm, "score_only")
        for k in range(6):
            qa, sa = text(rng, int(rng.integers(20, 200))), text(rng, int(rng.integers(20, 200)))
            qb, sb = text(rng, int(rng.integers(20, 200))), text(rng, int(rng.integers(20, 200)))
            ra, rb, cells = W.engine_score_packed((W.encode_sequence("a", qa), W.encode_sequence("a", sa)),
                                                  (W.encode_sequence("b", qb), W.encode_sequence("b", sb)), cfg, scheme)
            packed.append(dict(align_type=at, gap_model=gm, scheme=list(sch), qa=qa, sa=sa, qb=qb, sb=sb,
                               a=[int(ra[0]), int(ra[1][0]), int(ra[1][1])], b=[int(rb[0]), int(rb[1][0]), int(rb[1][1])],
                               cells=int(cells)))
    json.dump(dict(pairs=rnd, packed=packed), open(os.path.join(HERE, "random_small.json"), "w"), indent=0)

    # ---- adversarial ----
    adv = []
    acgtn = np.array(list("ACGTN"))
    for at, gm in COMBOS:
        pool = AFFINE if gm == "affine" else LINEAR
        sch0 = pool[0]
        for k in range(10):  # flagged symbols on both sides, N never matches N
            adv.append(record(text(rng, int(rng.integers(5, 70)), acgtn), text(rng, int(rng.integers(5, 70)), acgtn),
                              at, gm, pool[k % len(pool)]))
        adv.append(record("N" * 12, "N" * 9, at, gm, sch0))
        adv.append(record("A" * 33, "A" * 31, at, gm, sch0))          # homopolymers: maximal tie density
        adv.append(record("AC" * 20, "CA" * 21, at, gm, sch0))
        adv.append(record("G", text(rng, 200), at, gm, sch0))           # 1 x L and L x 1
        adv.append(record(text(rng, 200), "T", at, gm, sch0))
        adv.append(record("C", "C", at, gm, sch0))
        adv.append(record("C", "G", at, gm, sch0))
        for L in (31, 32, 33, 63, 64, 65, 127, 128, 129, 151, 152, 153, 255, 256, 257):  # lane-group / stage straddles
            q = text(rng, L)
            adv.append(record(q, mutate(rng, q) if L % 2 else text(rng, L), at, gm, sch0, with_tb=(L < 140)))
        adv.append(record(text(rng, 40), text(rng, 600), at, gm, sch0, with_tb=False))   # several stages wide
        adv.append(record(text(rng, 600), text(rng, 40), at, gm, sch0, with_tb=False))
    json.dump(adv, open(os.path.join(HERE, "adversarial.json"), "w"), indent=0)
    print("kat", len(kat), "random", len(rnd), "packed", len(packed), "adversarial", len(adv))


if __name__ == "__main__":
    sys.exit(main())
