"""Test helpers: pools, oracle comparisons.  Imports oracle/ (allowed: tests are the checker's home)."""
import numpy as np

import oracle
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme


def make_pool(seqs):
    lens = np.array([len(s) for s in seqs], np.int32)
    off = np.zeros(len(seqs), np.int64)
    if len(seqs) > 1:
        off[1:] = np.cumsum(lens[:-1])
    codes = np.concatenate([np.asarray(s, np.uint8) for s in seqs]) if lens.sum() else np.zeros(1, np.uint8)
    return codes, off, lens


def scheme_of(t, gap_model):
    return ScoringScheme(t[0], t[1], t[2], t[3], gap_model)


def gpu_scores(ctx, queries, subjects, pairs, scheme, align_type, variant="auto"):
    qc, qo, ql = make_pool(queries)
    sc, so, sl = make_pool(subjects)
    pq = np.array([p[0] for p in pairs], np.int32)
    ps = np.array([p[1] for p in pairs], np.int32)
    b = N.Batch(ctx, qc, qo, ql, sc, so, sl, pq, ps)
    try:
        b.score(scheme, align_type, variant)
        return b.fetch_scores()
    finally:
        b.close()


def oracle_scores(queries, subjects, pairs, scheme, align_type):
    qc, qo, ql = make_pool(queries)
    sc, so, sl = make_pool(subjects)
    pq = np.array([p[0] for p in pairs], np.int32)
    ps = np.array([p[1] for p in pairs], np.int32)
    return oracle.score_batch(qc, qo, ql, sc, so, sl, pq, ps, align_type, scheme.gap_model == "affine",
                              scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend)


def assert_scores_equal(got, want, ctx_msg=""):
    gs, gi, gj = got[0], got[1], got[2]
    ws, wi, wj = want
    bad = np.nonzero((gs != ws) | (gi != wi) | (gj != wj))[0]
    assert len(bad) == 0, (f"{ctx_msg}: {len(bad)} mismatches, first pair {bad[0]}: "
                           f"got {(gs[bad[0]], gi[bad[0]], gj[bad[0]])} want {(ws[bad[0]], wi[bad[0]], wj[bad[0]])}")
