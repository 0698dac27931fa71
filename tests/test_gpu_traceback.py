"""GPU parity: spans + CIGARs of the direction-code traceback (through the C ABI) == oracle ref_traceback, bit-exact."""
import numpy as np
import pytest

import oracle
from conftest import AFFINE_SCHEMES, COMBOS, LINEAR_SCHEMES, cigar_of, codes, load_golden, mutate_codes, random_codes
from helpers import make_pool, scheme_of
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.io import unpack_runs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = N.Context(0)
    yield c
    c.close()


def gpu_traceback(ctx, qs, ss, pairs, scheme, align_type):
    qc, qo, ql = make_pool(qs); sc, so, sl = make_pool(ss)
    pq = np.array([p[0] for p in pairs], np.int32); ps = np.array([p[1] for p in pairs], np.int32)
    b = N.Batch(ctx, qc, qo, ql, sc, so, sl, pq, ps)
    try:
        b.traceback(scheme, align_type)
        return b.fetch_traceback()
    finally:
        b.close()


def oracle_traceback(qs, ss, pairs, scheme, align_type):
    qc, qo, ql = make_pool(qs); sc, so, sl = make_pool(ss)
    pq = np.array([p[0] for p in pairs], np.int32); ps = np.array([p[1] for p in pairs], np.int32)
    return oracle.traceback_batch(qc, qo, ql, sc, so, sl, pq, ps, align_type, scheme.gap_model == "affine",
                                  scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend)


def assert_tb_equal(got, want, msg=""):
    n = len(want["score"])
    for key in ("score", "q_start", "q_end", "s_start", "s_end"):
        bad = np.nonzero(got[key] != want[key])[0]
        assert len(bad) == 0, f"{msg}: {key} differs at pair {bad[0]}: got {got[key][bad[0]]} want {want[key][bad[0]]}"
    for k in range(n):
        runs = unpack_runs(got["cigar"][int(got["cigar_off"][k]):int(got["cigar_off"][k + 1])])
        assert runs == want["ops"][k], f"{msg}: CIGAR differs at pair {k}: got {cigar_of(runs)} want {cigar_of(want['ops'][k])}"


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_golden_cigars(ctx, align_type, gap_model):
    recs = [r for name in ("kat.json", "adversarial.json") for r in load_golden(name)]
    recs += load_golden("random_small.json")["pairs"]
    recs = [r for r in recs if r["align_type"] == align_type and r["gap_model"] == gap_model and "tb" in r]
    assert recs
    by_scheme = {}
    for r in recs:
        by_scheme.setdefault(tuple(r["scheme"]), []).append(r)
    for sch, rs in by_scheme.items():
        scheme = scheme_of(sch, gap_model)
        got = gpu_traceback(ctx, [codes(r["q"]) for r in rs], [codes(r["s"]) for r in rs], [(i, i) for i in range(len(rs))],
                            scheme, align_type)
        for k, r in enumerate(rs):
            runs = unpack_runs(got["cigar"][int(got["cigar_off"][k]):int(got["cigar_off"][k + 1])])
            t = r["tb"]
            assert int(got["score"][k]) == r["score"], (sch, k)
            assert (int(got["q_start"][k]), int(got["q_end"][k]), int(got["s_start"][k]), int(got["s_end"][k])) == (
                t["q_start"], t["q_end"], t["s_start"], t["s_end"]), (sch, k, r["q"], r["s"])
            assert cigar_of(runs) == t["cigar"], (sch, k, r["q"], r["s"])


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_random_vs_oracle(ctx, align_type, gap_model):
    rng = np.random.default_rng(2026)
    pool = AFFINE_SCHEMES + [(2, -9, 2, 1), (2, -1, 1, 3)] if gap_model == "affine" else LINEAR_SCHEMES
    for sch in pool:
        scheme = scheme_of(sch, gap_model)
        qs, ss = [], []
        for k in range(200):
            q = random_codes(rng, int(rng.integers(1, 280)))
            s = mutate_codes(rng, q, 0.06, 0.03, 0.03) if k % 2 else random_codes(rng, int(rng.integers(1, 280)))
            if k % 7 == 0:
                q = q.copy(); q[rng.integers(0, len(q))] = 4
            qs.append(q); ss.append(s)
        pairs = [(i, i) for i in range(len(qs))]
        assert_tb_equal(gpu_traceback(ctx, qs, ss, pairs, scheme, align_type), oracle_traceback(qs, ss, pairs, scheme, align_type),
                        f"{align_type}/{gap_model}/{sch}")


def test_uniform_250bp_semiglobal_affine_cfg3_shape(ctx):
    rng = np.random.default_rng(220507613)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    n = 3000
    qs = [random_codes(rng, 250) for _ in range(n)]
    ss = []
    for i, q in enumerate(qs):
        if i % 2:
            s = mutate_codes(rng, q, 0.03, 0.01, 0.01)[:250]
            s = np.concatenate([s, random_codes(rng, 250 - len(s))])
        else:
            s = random_codes(rng, 250)
        ss.append(s)
    pairs = [(i, i) for i in range(n)]
    assert_tb_equal(gpu_traceback(ctx, qs, ss, pairs, scheme, "semiglobal"), oracle_traceback(qs, ss, pairs, scheme, "semiglobal"), "cfg3")


def test_multi_stage_and_chunked(ctx, monkeypatch):
    monkeypatch.setenv("WSB_TB_SCRATCH_MB", "1")  # force several chunks
    rng = np.random.default_rng(77)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    qs, ss = [], []
    for L in (600, 900, 1300, 513, 40, 700):
        q = random_codes(rng, L)
        qs.append(q); ss.append(mutate_codes(rng, q, 0.08, 0.04, 0.04))
    qs.append(random_codes(rng, 30)); ss.append(random_codes(rng, 1500))
    pairs = [(i, i) for i in range(len(qs))]
    for at in ("global", "local", "semiglobal"):
        assert_tb_equal(gpu_traceback(ctx, qs, ss, pairs, scheme, at), oracle_traceback(qs, ss, pairs, scheme, at), at)


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_empty_and_single_symbol_sides(ctx, align_type, gap_model):
    """The Python API refuses empty sequences like the reference (core.py:103-104); the C ABI accepts them and resolves
    them like refdp's zero-row / zero-column matrices.  One-symbol sides run through the kernels."""
    rng = np.random.default_rng(3)
    seqs = [np.zeros(0, np.uint8), codes("A"), codes("N"), codes("C"), random_codes(rng, 7), random_codes(rng, 130),
            random_codes(rng, 600)]
    pairs = [(a, b) for a in range(len(seqs)) for b in range(len(seqs))]
    scheme = scheme_of((2, -1, 2, 1) if gap_model == "affine" else (2, -1, 1, 1), gap_model)
    want = oracle_traceback(seqs, seqs, pairs, scheme, align_type)
    got = gpu_traceback(ctx, seqs, seqs, pairs, scheme, align_type)
    assert_tb_equal(got, want, f"{align_type}/{gap_model}")
    from helpers import assert_scores_equal, gpu_scores, oracle_scores
    assert_scores_equal(gpu_scores(ctx, seqs, seqs, pairs, scheme, align_type), oracle_scores(seqs, seqs, pairs, scheme, align_type),
                        f"{align_type}/{gap_model}")


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_long_pairs_rescore_to_their_score(ctx, align_type):
    """Lengths the oracle's full matrices cannot hold: the CIGAR must re-score (from first principles) to the score the
    score-only long-read kernel reports, and consume exactly the recorded spans (the reference's own contract for
    align_traceback, tests/test_traceback.py:85-100)."""
    import paper_2205_07610_b200 as W
    from helpers import gpu_scores
    rng = np.random.default_rng(2205)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    qs, ss = [], []
    for L in (21_000, 9_000):
        q = random_codes(rng, L)
        qs.append(q); ss.append(mutate_codes(rng, q, 0.06, 0.03, 0.03))
    if align_type != "global":   # a short read against a long window
        qs.append(ss[0][5000:5400].copy()); ss.append(ss[0])
    pairs = [(i, i) for i in range(len(qs))]
    got = gpu_traceback(ctx, qs, ss, pairs, scheme, align_type)
    score = gpu_scores(ctx, qs, ss, pairs, scheme, align_type)
    assert (got["score"] == score[0]).all()
    for k in range(len(qs)):
        ops = unpack_runs(got["cigar"][int(got["cigar_off"][k]):int(got["cigar_off"][k + 1])])
        res = W.AlignmentResult(int(got["score"][k]), int(got["q_start"][k]), int(got["q_end"][k]), int(got["s_start"][k]),
                                int(got["s_end"][k]), ops, len(qs[k]) * len(ss[k]))
        q = W.Sequence(f"q{k}", qs[k], np.zeros(len(qs[k]), bool))
        s = W.Sequence(f"s{k}", ss[k], np.zeros(len(ss[k]), bool))
        assert W.rescore_alignment(res, q, s, scheme) == res.score
        if align_type == "global":
            assert (res.q_start, res.q_end, res.s_start, res.s_end) == (0, len(qs[k]), 0, len(ss[k]))
        elif align_type == "semiglobal":
            assert res.q_end == len(qs[k]) or res.s_end == len(ss[k])
        assert all(a[0] != b[0] for a, b in zip(ops, ops[1:]))      # runs arrive merged
    if align_type != "global":
        assert got["score"][2] == 800 and (got["s_start"][2], got["s_end"][2]) == (5000, 5400)


@pytest.mark.parametrize("align_type", ["global", "semiglobal", "local"])
def test_packed_int16_fill_uniform_batches(ctx, align_type):
    """Uniform affine batches of one stage take the packed int16 fill (traceback_fill16.cuh): two
    alignments per thread.  Odd counts, flagged symbols on both sides, rectangular shapes, several schemes."""
    rng = np.random.default_rng(1607)
    for (m, n, count), sch in zip([(250, 250, 301), (100, 128, 64), (37, 256, 33), (250, 90, 17), (1, 1, 5), (200, 256, 1),
                                   (129, 131, 40), (256, 255, 9), (150, 150, 101), (180, 192, 21)],
                                  [(2, -1, 2, 1), (2, -1, 2, 1), (1, -3, 5, 2), (2, -1, 2, 1), (2, -1, 2, 1), (5, -4, 10, 1),
                                   (3, -2, 0, 1), (2, -1, 2, 1), (2, -1, 2, 1), (4, -3, 3, 2)]):
        linear = (m + n) % 3 == 0   # a third of the shapes run the linear-gap form
        scheme = scheme_of((sch[0], sch[1], max(1, sch[2]), max(1, sch[2])), "linear") if linear else scheme_of(sch, "affine")
        qs, ss = [], []
        for k in range(count):
            q = random_codes(rng, m)
            if k % 2 == 0 and m == n:
                s = mutate_codes(rng, q, 0.05, 0.0, 0.0)
                cut = int(rng.integers(1, max(2, n - 1)))
                s = np.concatenate([s[:cut], s[cut + 1:], random_codes(rng, 1)]) if k % 4 == 0 and n >= 3 else s   # one deletion
            else:
                s = random_codes(rng, n)
            if k % 5 == 0:
                q = q.copy(); q[rng.integers(0, m)] = 4
            if k % 7 == 0:
                s = s.copy(); s[rng.integers(0, n)] = 4
            assert len(q) == m and len(s) == n
            qs.append(q); ss.append(s)
        pairs = [(i, i) for i in range(count)]
        assert_tb_equal(gpu_traceback(ctx, qs, ss, pairs, scheme, align_type), oracle_traceback(qs, ss, pairs, scheme, align_type),
                        f"{align_type} {m}x{n} {sch}")


@pytest.mark.parametrize("align_type", ["global", "semiglobal", "local"])
def test_packed_int16_fill_ragged_batches(ctx, align_type):
    """Pairs of different sizes share a thread's halves (masked form of the packed fill): every half must store and track
    only inside its own rectangle.  Includes empty sides, one-symbol sides, flagged symbols and an odd pair count."""
    rng = np.random.default_rng(4242)
    for sch, hi, count in (((2, -1, 2, 1), 256, 401), ((1, -3, 5, 2), 128, 77), ((5, -4, 10, 1), 200, 150), ((2, -1, 2, 1), 190, 99),
                           ((2, -1, 1, 1), 256, 203), ((3, -2, 4, 4), 150, 64)):
        scheme = scheme_of(sch, "linear" if sch[2] == sch[3] and sch[2] in (1, 4) else "affine")
        qs, ss = [], []
        for k in range(count):
            m = int(rng.integers(1, hi + 1)); n = int(rng.integers(1, hi + 1))
            if k % 9 == 0:
                m = int(rng.integers(1, 4))
            if k % 11 == 0:
                n = hi
            q = random_codes(rng, m)
            s = mutate_codes(rng, q, 0.06, 0.03, 0.03)[:hi] if k % 2 else random_codes(rng, n)
            if k % 5 == 0:
                q = q.copy(); q[rng.integers(0, len(q))] = 4
            if k % 7 == 0 and len(s):
                s = s.copy(); s[rng.integers(0, len(s))] = 4
            if k in (13, 14, 200):
                s = np.zeros(0, np.uint8)
            if k in (14, 15):
                q = np.zeros(0, np.uint8)
            qs.append(q); ss.append(s)
        pairs = [(i, i) for i in range(count)]
        assert_tb_equal(gpu_traceback(ctx, qs, ss, pairs, scheme, align_type), oracle_traceback(qs, ss, pairs, scheme, align_type),
                        f"{align_type} ragged {sch}")


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_schemes_beyond_the_byte_profile(ctx, align_type, gap_model):
    """|match + gap_open| or |mismatch + gap_open| > 127: the fill takes its compare / select form instead of the signed-byte
    profile (the reference has no such limit); spans and CIGARs still equal ref_traceback."""
    rng = np.random.default_rng(127)
    for sch in ((200, -150, 100, 3), (90, -60, 70, 70), (3, -250, 5, 2)):
        scheme = scheme_of(sch, gap_model)
        qs, ss = [], []
        for k in range(120):
            q = random_codes(rng, int(rng.integers(1, 700 if k < 6 else 200)))
            s = mutate_codes(rng, q, 0.06, 0.03, 0.03) if k % 2 else random_codes(rng, int(rng.integers(1, 700 if k < 6 else 200)))
            if k % 9 == 0:
                q = q.copy(); q[rng.integers(0, len(q))] = 4
            if k % 11 == 0:
                s = s.copy(); s[rng.integers(0, len(s))] = 4
            qs.append(q); ss.append(s)
        pairs = [(i, i) for i in range(len(qs))]
        assert_tb_equal(gpu_traceback(ctx, qs, ss, pairs, scheme, align_type), oracle_traceback(qs, ss, pairs, scheme, align_type),
                        f"{align_type}/{gap_model}/{sch}")
