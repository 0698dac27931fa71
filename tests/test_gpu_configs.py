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


def test_cfg2_local_affine_4m_pairs_every_variant_equals_the_oracle_on_every_pair(ctx):
    """forced half2 and forced int32 must agree, and ALL 4 M pairs are checked against the C restatement
    (11 s of oracle time on 16 cores); AUTO is the packed int16 kernel, the headline path."""
    n = 4_000_000
    qp, sp, idx = _uniform(n, 150, 220507612)
    want = _oracle(qp, sp, idx, "local", AFF)
    for variant in ("auto", "f16x2", "i32"):
        got = _score(ctx, qp, sp, idx, "local", AFF, variant)
        for name, g, w in zip(("score", "end_i", "end_j"), got[:3], want):
            bad = np.nonzero(g != w)[0]
            assert len(bad) == 0, f"{variant}: {len(bad)} {name} mismatches, first at pair {bad[0]}: {g[bad[0]]} != {w[bad[0]]}"
        assert not got[3].any()


def _runs_match_oracle(tb, lo, ref):
    """Array-wise CIGAR comparison of pairs [lo, lo + n) of a GPU traceback against an oracle chunk."""
    n = len(ref["n_ops"])
    off = tb["cigar_off"][lo:lo + n + 1]
    if not (np.diff(off) == ref["n_ops"]).all():
        return int(lo + np.nonzero(np.diff(off) != ref["n_ops"])[0][0])
    packed = ref["ops_packed"]
    mask = np.arange(packed.shape[1])[None, :] < ref["n_ops"][:, None]
    got = tb["cigar"][off[0]:off[-1]]
    want = packed[mask]                      # row-major: the pairs' runs back to back, as the device stores them
    if (got == want).all():
        return -1
    at = int(np.nonzero(got != want)[0][0])
    return int(lo + np.searchsorted(off - off[0], at, side="right") - 1)


def test_cfg3_semiglobal_traceback_1m_pairs_spans_and_every_cigar_against_the_oracle(ctx):
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
    # EVERY pair (both halves of the workload: related and unrelated) against the oracle walk, in chunks that keep the
    # oracle's run buffer small; comparison is array-wise (about 30 s of oracle time on 16 cores)
    step = 50_000
    for lo in range(0, n, step):
        sel = np.arange(lo, min(n, lo + step), dtype=np.int32)
        ref = oracle.traceback_batch(qp[0], qp[1], qp[2], sp[0], sp[1], sp[2], sel, sel, "semiglobal", True, 2, -1, 2, 1,
                                     unpack=False)
        for key in ("score", "q_start", "q_end", "s_start", "s_end"):
            bad = np.nonzero(tb[key][sel] != ref[key])[0]
            assert len(bad) == 0, f"{key}: first mismatch at pair {lo + bad[0]}"
        bad_pair = _runs_match_oracle(tb, lo, ref)
        assert bad_pair < 0, f"CIGAR differs from the oracle at pair {bad_pair}"


def test_cfg4_global_affine_10kbp_swap_symmetry_and_1024_pairs_against_the_oracle(ctx):
    n, L = 10_000, 10_000
    qp, sp, idx = _uniform(n, L, 220507614)
    a = _score(ctx, qp, sp, idx, "global", AFF)
    b_ = _score(ctx, sp, qp, idx, "global", AFF)        # swapped roles: a symmetric scheme gives the same score
    assert (a[0] == b_[0]).all()
    assert (a[1] == L).all() and (a[2] == L).all()
    # 1024 pairs against the oracle (~40 s on 16 cores): 512 consecutive (both halves of the packed int16 twins the
    # planner forms from neighbours) plus 512 spread over the batch
    sel = np.unique(np.concatenate([np.arange(512), np.arange(512, n, (n - 512) // 512)[:512]])).astype(np.int32)
    want = _oracle(qp, sp, sel, "global", AFF)
    bad = np.nonzero(a[0][sel] != want[0])[0]
    assert len(bad) == 0, f"{len(bad)} score mismatches, first at pair {sel[bad[0]]}"
    # the int32 long-read kernel on the same pairs, and a flagged subject symbol (the packed kernel hands that pair back)
    sub = sel[:64]
    i32 = _score(ctx, qp, sp, sub, "global", AFF, "i32")
    assert (i32[0] == want[0][:64]).all()
    s_flag = sp[0].copy()
    s_flag[int(sp[1][3]) + 4321] = 4
    spf = (s_flag, sp[1], sp[2])
    first = np.arange(8, dtype=np.int32)
    got = _score(ctx, qp, spf, first, "global", AFF)
    wantf = _oracle(qp, spf, first, "global", AFF)
    assert (got[0] == wantf[0]).all() and got[0][3] != a[0][3] - 10_000_000


def test_cfg5_pareto_lengths_swap_symmetry_and_every_giant_against_the_oracle(ctx):
    n = 100_000
    qp, sp = bench.make_pareto(n, 220507615)
    idx = np.arange(n, dtype=np.int32)
    a = _score(ctx, qp, sp, idx, "local", AFF)
    b_ = _score(ctx, sp, qp, idx, "local", AFF)         # local score is symmetric under swapping the roles
    assert (a[0] == b_[0]).all()
    assert not a[3].any()
    cells = qp[2].astype(np.int64) * sp[2]
    small = np.nonzero(cells <= 2e7)[0]
    mid = np.nonzero((cells > 2e7) & (cells < 1e9))[0]
    giant = np.nonzero(cells >= 1e9)[0]          # the pairs the planner gives a thread-block cluster
    capped = giant[(qp[2][giant] == 100_000) | (sp[2][giant] == 100_000)]   # EVERY pair with a capped 100 kbp side
    others = np.setdiff1d(giant, capped)
    rng = np.random.default_rng(5)
    assert len(capped) >= 50 and int(cells[capped].max()) == 10_000_000_000
    # giants first: the oracle hands small lists out pair by pair, largest work at the front keeps its threads level
    sel = np.concatenate([capped, rng.choice(others, 40, replace=False), rng.choice(mid, 48, replace=False),
                          rng.choice(small, 10_000, replace=False)]).astype(np.int32)
    want = _oracle(qp, sp, sel, "local", AFF)    # rolling-row oracle: ~1.2e12 cells, two to three minutes on 16 cores
    for name, g, w in zip(("score", "end_i", "end_j"), a[:3], want):
        bad = np.nonzero(g[sel] != w)[0]
        assert len(bad) == 0, f"{name}: {len(bad)} mismatches, first at pair {sel[bad[0]]} ({qp[2][sel[bad[0]]]} x {sp[2][sel[bad[0]]]})"
    # end cells stay inside the matrix, and a positive score ends on a matching pair of symbols
    assert (a[1] <= qp[2]).all() and (a[2] <= sp[2]).all()
    pos = np.nonzero(a[0] > 0)[0]
    qe = qp[0][qp[1][pos] + a[1][pos] - 1]
    se = sp[0][sp[1][pos] + a[2][pos] - 1]
    assert (qe == se).all()
