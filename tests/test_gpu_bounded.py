"""GPU parity: bounded-memory traceback of pairs whose direction codes exceed the scratch budget (
csrc/traceback_band.cuh).  The path must be the full-matrix walk's, bit for bit (oracle = refdp.ref_traceback restated in
oracle/wsoracle.c); beyond the oracle's reach the bounded path is compared with the plain direction-code path and with
the reference's own contract for hirschberg / locate_endpoints (tests/test_traceback.py:22-59,111-132,
tests/test_acceptance.py:115-135)."""
import numpy as np
import pytest

import oracle
from conftest import AFFINE_SCHEMES, COMBOS, LINEAR_SCHEMES, mutate_codes, random_codes
from helpers import make_pool, scheme_of
from paper_2205_07610_b200 import _native as N
from paper_2205_07610_b200.io import unpack_runs
from test_gpu_traceback import assert_tb_equal, oracle_traceback

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = N.Context(0)
    yield c
    c.close()


def bounded_traceback(ctx, qs, ss, pairs, scheme, align_type, scratch_bytes):
    qc, qo, ql = make_pool(qs); sc, so, sl = make_pool(ss)
    pq = np.array([p[0] for p in pairs], np.int32); ps = np.array([p[1] for p in pairs], np.int32)
    b = N.Batch(ctx, qc, qo, ql, sc, so, sl, pq, ps)
    try:
        if scratch_bytes is not None:
            b.set_tb_scratch(scratch_bytes)
        b.traceback(scheme, align_type)
        return b.fetch_traceback(), b.tb_info()
    finally:
        b.close()


def _mixed_pairs(rng, n, lo, hi, flagged=True):
    qs, ss = [], []
    for k in range(n):
        q = random_codes(rng, int(rng.integers(lo, hi)))
        s = mutate_codes(rng, q, 0.06, 0.03, 0.03) if k % 2 else random_codes(rng, int(rng.integers(lo, hi)))
        if flagged and k % 5 == 0:
            q = q.copy(); q[rng.integers(0, len(q))] = 4
        if flagged and k % 7 == 0:
            s = s.copy(); s[rng.integers(0, len(s))] = 4
        qs.append(q); ss.append(s)
    return qs, ss


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_every_pair_through_the_bounded_path_equals_the_oracle(ctx, align_type, gap_model):
    """A one-byte budget sends every pair through checkpoint sweep + tile walk: several bands (R = 128), several tile
    columns (512), flagged symbols, unrelated and related pairs, 1 x L shapes."""
    rng = np.random.default_rng(8001)
    pool = (AFFINE_SCHEMES[:2] + [(2, -9, 2, 1), (2, -1, 1, 3)]) if gap_model == "affine" else LINEAR_SCHEMES[:2]
    for sch in pool:
        scheme = scheme_of(sch, gap_model)
        qs, ss = _mixed_pairs(rng, 24, 1, 1400)
        qs += [random_codes(rng, 1), random_codes(rng, 900), random_codes(rng, 513), random_codes(rng, 129)]
        ss += [random_codes(rng, 1100), random_codes(rng, 1), random_codes(rng, 512), random_codes(rng, 128)]
        pairs = [(i, i) for i in range(len(qs))]
        got, info = bounded_traceback(ctx, qs, ss, pairs, scheme, align_type, 1)
        assert info["pairs"] == len(pairs)
        assert_tb_equal(got, oracle_traceback(qs, ss, pairs, scheme, align_type), f"bounded {align_type}/{gap_model}/{sch}")


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_batch_mixing_plain_and_bounded_pairs(ctx, align_type):
    """Under a 64 KiB code budget the larger pairs of a batch take the bounded path, the others the plain one, in pair
    order, with empty sides and rejected sizes riding along."""
    rng = np.random.default_rng(8002)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    qs, ss = _mixed_pairs(rng, 40, 20, 900)
    qs.append(np.zeros(0, np.uint8)); ss.append(random_codes(rng, 50))
    pairs = [(i, i) for i in range(len(qs))] + [(3, 7), (7, 3)]
    got, info = bounded_traceback(ctx, qs, ss, pairs, scheme, align_type, 64 << 10)
    assert 0 < info["pairs"] < len(pairs)
    assert_tb_equal(got, oracle_traceback(qs, ss, pairs, scheme, align_type), f"mixed {align_type}")


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_bounded_equals_plain_at_30kbp(ctx, align_type):
    """Beyond the oracle's matrices: same CIGAR through both GPU paths (the plain path is pinned to the oracle at small
    sizes and re-scores at 21 kbp, test_gpu_traceback.py); the bounded one keeps 1/10 of the plain path's scratch."""
    rng = np.random.default_rng(8003)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    q = random_codes(rng, 30_000)
    s = mutate_codes(rng, q, 0.08, 0.04, 0.04)
    qs, ss = [q, random_codes(rng, 12_000)], [s, random_codes(rng, 17_000)]
    pairs = [(0, 0), (1, 1)]
    plain, info0 = bounded_traceback(ctx, qs, ss, pairs, scheme, align_type, None)
    small, info1 = bounded_traceback(ctx, qs, ss, pairs, scheme, align_type, 32 << 20)
    assert info0["pairs"] == 0 and info1["pairs"] == 2
    for key in ("score", "q_start", "q_end", "s_start", "s_end", "cigar_off", "cigar"):
        assert np.array_equal(plain[key], small[key]), key
    assert info1["peak_bytes"] < 0.1 * (0.5 * 30_000 * len(s))


def test_100kbp_global_cigar_in_bounded_memory(ctx):
    """a 100 kbp x 100 kbp global CIGAR that rescoring accepts, with a scratch budget (256 MiB)
    twenty times below the 5 GB its direction codes would take."""
    import paper_2205_07610_b200 as W
    from helpers import gpu_scores
    rng = np.random.default_rng(8004)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    q = random_codes(rng, 100_000)
    s = mutate_codes(rng, q, 0.10, 0.05, 0.05)
    got, info = bounded_traceback(ctx, [q], [s], [(0, 0)], scheme, "global", 256 << 20)
    assert info["pairs"] == 1 and info["peak_bytes"] <= 300 << 20
    assert info["cells"] <= 1.1 * len(q) * len(s)          # checkpoint sweep + the tiles under the path
    score = gpu_scores(ctx, [q], [s], [(0, 0)], scheme, "global")
    assert int(got["score"][0]) == int(score[0][0])
    ops = unpack_runs(got["cigar"])
    res = W.AlignmentResult(int(got["score"][0]), 0, len(q), 0, len(s), ops, len(q) * len(s))
    qq = W.Sequence("q", q, np.zeros(len(q), bool)); sq = W.Sequence("s", s, np.zeros(len(s), bool))
    assert W.rescore_alignment(res, qq, sq, scheme) == res.score
    assert (int(got["q_start"][0]), int(got["q_end"][0]), int(got["s_start"][0]), int(got["s_end"][0])) == (0, len(q), 0, len(s))


def _seq(name, c):
    import paper_2205_07610_b200 as W
    return W.Sequence(name, np.asarray(c, np.uint8) & 3, np.asarray(c) >= 4)


def test_hirschberg_contract_of_the_reference(ctx):
    """tests/test_traceback.py:22-59 + test_acceptance.py:115-135 restated: score == reference DP, operations re-score to
    it, whole sequences consumed, deterministic, cells <= 2.1 m n, no quadratic growth of the working memory."""
    import paper_2205_07610_b200 as W

    class Meter:
        current = peak = 0
        def add(self, n): self.current += n; self.peak = max(self.peak, self.current)
        def sub(self, n): self.current -= n

    rng = np.random.default_rng(8005)
    for gap_model, sch in (("affine", (2, -1, 2, 1)), ("affine", (2, -9, 2, 1)), ("linear", (2, -1, 2, 2))):
        scheme = scheme_of(sch, gap_model)
        cfg = W.AlignConfig("global", gap_model, "traceback")
        peaks = {}
        for size in (90, 256, 512, 1024):
            q = random_codes(rng, size); s = mutate_codes(rng, q, 0.1, 0.05, 0.05) if size != 90 else random_codes(rng, 110)
            Q, S = _seq("q", q), _seq("s", s)
            meter = Meter()
            res = W.hirschberg(Q, S, cfg, scheme, meter=meter)
            want = oracle_traceback([q], [s], [(0, 0)], scheme, "global")
            assert res.score == int(want["score"][0]) and res.ops == want["ops"][0]
            assert W.rescore_alignment(res, Q, S, scheme) == res.score
            assert (res.q_start, res.q_end, res.s_start, res.s_end) == (0, len(q), 0, len(s))
            assert W.hirschberg(Q, S, cfg, scheme) == res
            if size >= 512:
                assert res.cells_computed <= 2.1 * len(q) * len(s), size
            assert meter.current == 0 and meter.peak > 0
            peaks[size] = meter.peak
        assert peaks[1024] / peaks[512] < 3 and peaks[512] / peaks[256] < 3
    # midline-gap family and extreme shapes of the reference's tests
    scheme = scheme_of((2, -1, 2, 1), "affine")
    cfg = W.AlignConfig("global", "affine", "traceback")
    for a, b in ((40, 20), (20, 40), (1, 200), (200, 1), (64, 64)):
        Q, S = W.encode_sequence("q", "A" * a), W.encode_sequence("s", "A" * b)
        res = W.hirschberg(Q, S, cfg, scheme)
        assert res.score == W.engine_score(Q, S, W.AlignConfig("global", "affine"), scheme)[0]
        assert W.rescore_alignment(res, Q, S, scheme) == res.score
    with pytest.raises(ValueError):
        W.hirschberg(Q, S, W.AlignConfig("local", "affine", "traceback"), scheme)


def test_locate_endpoints_contract_of_the_reference(ctx):
    """tests/test_traceback.py:111-132 restated."""
    import paper_2205_07610_b200 as W
    rng = np.random.default_rng(3)
    for trial in range(30):
        q = random_codes(rng, int(rng.integers(1, 121))); s = random_codes(rng, int(rng.integers(1, 121)))
        Q, S = _seq("q", q), _seq("s", s)
        for at in ("local", "semiglobal"):
            sch = AFFINE_SCHEMES[trial % len(AFFINE_SCHEMES)]
            scheme = scheme_of(sch, "affine")
            cfg = W.AlignConfig(at, "affine")
            score, (q0, s0), (q1, s1), cells = W.locate_endpoints(Q, S, cfg, scheme)
            qc, qo, ql = make_pool([q]); sc, so, sl = make_pool([s])
            z = np.zeros(1, np.int32)
            want = oracle.score_batch(qc, qo, ql, sc, so, sl, z, z, at, True, *sch)
            assert score == int(want[0][0])
            assert 0 <= q0 <= q1 <= len(q) and 0 <= s0 <= s1 <= len(s)
            if at == "local" and score > 0:
                assert (q1, s1) == (int(want[1][0]), int(want[2][0]))
            assert cells >= len(q) * len(s)
    with pytest.raises(ValueError):
        W.locate_endpoints(Q, Q, W.AlignConfig("global", "affine"), scheme_of((2, -1, 2, 1), "affine"))
