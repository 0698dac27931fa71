"""GPU parity at the BASELINE.json sizes (cfg1..cfg5): oracle comparison on seeded samples plus size-independent
properties over every pair (variant agreement, swap symmetry, CIGAR span consumption)."""
import numpy as np
import pytest

import bench
import oracle
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.core import ScoringScheme

pytestmark = pytest.mark.gpu

AFF = ScoringScheme(2, -1, 2, 1, "affine")
LIN = ScoringScheme(2, -1, 1, 1, "linear")


@pytest.fixture(scope="module")
def ctx():
    c = N.Context(0)
    yield c
    c.close()


def _uniform(n, L, seed, related=0.0):
    q, s = bench.make_batch(dict(pairs=n, length=L, related=related), seed)
    off = np.arange(n, dtype=np.int64) * L
    ln = np.full(n, L, np.int32)
    return (q.reshape(-1), off, ln), (s.reshape(-1), off, ln), np.arange(n, dtype=np.int32)


def _oracle(qp, sp, sel, atype, sch):
    return oracle.score_batch(qp[0], qp[1], qp[2], sp[0], sp[1], sp[2], sel, sel, atype, sch.gap_model == "affine",
                              sch.match_score, sch.mismatch_score, sch.gap_open, sch.gap_extend)


def _score(ctx, qp, sp, idx, atype, sch, variant="auto"):
    b = N.Batch(ctx, *qp, *sp, idx, idx)
    try:
        b.score(sch, atype, variant)
        return b.fetch_scores()
    finally:
        b.close()


def test_cfg1_global_linear_10k_pairs_all_against_oracle(ctx):
    qp, sp, idx = _uniform(10_000, 150, 220507611)
    want = _oracle(qp, sp, idx, "global", LIN)
    for variant in ("auto", "i32"):
        got = _score(ctx, qp, sp, idx, "global", LIN, variant)
        for g, w in zip(got[:3], want):
            assert (g == w).all(), variant


def test_cfg2_local_affine_4m_pairs_half2_equals_int32_and_oracle_sample(ctx):
    qp, sp, idx = _uniform(4_000_000, 150, 220507612)
    f16 = _score(ctx, qp, sp, idx, "local", AFF, "f16x2")
    i32 = _score(ctx, qp, sp, idx, "local", AFF, "i32")
    for a, b_ in zip(f16[:3], i32[:3]):
        assert (a == b_).all()
    assert not f16[3].any() and not i32[3].any()
    sel = np.random.default_rng(1).choice(4_000_000, 50_000, replace=False).astype(np.int32)
    want = _oracle(qp, sp, sel, "local", AFF)
    for g, w in zip(f16[:3], want):
        assert (g[sel] == w).all()


def test_cfg3_semiglobal_traceback_1m_pairs_spans_and_oracle_sample(ctx):
    n = 1_000_000
    qp, sp, idx = _uniform(n, 250, 220507613, related=0.5)
    b = N.Batch(ctx, *qp, *sp, idx, idx)
    try:
        b.traceback(AFF, "semiglobal")
        tb = b.fetch_traceback()
    finally:
        b.close()
    # every pair: the runs consume exactly the reported spans (M both, I query, D subject)
    runs, off = tb["cigar"], tb["cigar_off"]
    ln = (runs >> 2).astype(np.int64)
    op = runs & 3
    owner = np.repeat(np.arange(n), np.diff(off))
    q_used = np.bincount(owner, weights=ln * (op != 2), minlength=n)
    s_used = np.bincount(owner, weights=ln * (op != 1), minlength=n)
    assert (q_used == tb["q_end"] - tb["q_start"]).all()
    assert (s_used == tb["s_end"] - tb["s_start"]).all()
    assert (op < 3).all() and (ln > 0).all()
    # semiglobal: the alignment ends on the last row or last column and starts on the first row or column
    assert ((tb["q_end"] == 250) | (tb["s_end"] == 250)).all()
    assert ((tb["q_start"] == 0) | (tb["s_start"] == 0)).all()
    # seeded sample (both halves of the workload: related and unrelated pairs) against the oracle walk
    sel = np.random.default_rng(3).choice(n, 4000, replace=False).astype(np.int32)
    ref = oracle.traceback_batch(qp[0], qp[1], qp[2], sp[0], sp[1], sp[2], sel, sel, "semiglobal", True, 2, -1, 2, 1)
    for key in ("score", "q_start", "q_end", "s_start", "s_end"):
        assert (tb[key][sel] == ref[key]).all(), key
    for k, p in enumerate(sel):
        got = runs[off[p]:off[p + 1]]
        assert len(got) == ref["n_ops"][k] and (got == ref["ops_packed"][k, :len(got)]).all(), int(p)


def test_cfg4_global_affine_10kbp_swap_symmetry_and_oracle_sample(ctx):
    n, L = 10_000, 10_000
    qp, sp, idx = _uniform(n, L, 220507614)
    a = _score(ctx, qp, sp, idx, "global", AFF)
    b_ = _score(ctx, sp, qp, idx, "global", AFF)        # swapped roles: a symmetric scheme gives the same score
    assert (a[0] == b_[0]).all()
    assert (a[1] == L).all() and (a[2] == L).all()
    sel = np.arange(0, n, n // 16, dtype=np.int32)[:16]
    want = _oracle(qp, sp, sel, "global", AFF)
    assert (a[0][sel] == want[0]).all()


def test_cfg5_pareto_lengths_swap_symmetry_and_oracle_sample(ctx):
    n = 100_000
    qp, sp = bench.make_pareto(n, 220507615)
    idx = np.arange(n, dtype=np.int32)
    a = _score(ctx, qp, sp, idx, "local", AFF)
    b_ = _score(ctx, sp, qp, idx, "local", AFF)         # local score is symmetric under swapping the roles
    assert (a[0] == b_[0]).all()
    assert not a[3].any()
    cells = qp[2].astype(np.int64) * sp[2]
    small = np.nonzero(cells <= 2e7)[0]
    mid = np.nonzero((cells > 2e7) & (cells <= 1.5e9))[0]
    rng = np.random.default_rng(5)
    sel = np.concatenate([rng.choice(small, 3000, replace=False), rng.choice(mid, 24, replace=False)]).astype(np.int32)
    want = _oracle(qp, sp, sel, "local", AFF)
    for g, w in zip(a[:3], want):
        assert (g[sel] == w).all()
    # end cells stay inside the matrix, and a positive score ends on a matching pair of symbols
    assert (a[1] <= qp[2]).all() and (a[2] <= sp[2]).all()
    pos = np.nonzero(a[0] > 0)[0]
    qe = qp[0][qp[1][pos] + a[1][pos] - 1]
    se = sp[0][sp[1][pos] + a[2][pos] - 1]
    assert (qe == se).all()
