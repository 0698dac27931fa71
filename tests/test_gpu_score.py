"""GPU parity: score + end cell of the CUDA kernels (through the C ABI) == the oracle, bit-exact."""
import numpy as np
import pytest

from conftest import AFFINE_SCHEMES, COMBOS, LINEAR_SCHEMES, codes, load_golden, mutate_codes, random_codes
from helpers import assert_scores_equal, gpu_scores, oracle_scores, scheme_of
from paper_2205_07610_b200 import _native as N

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = N.Context(0)
    yield c
    c.close()


def _random_batch(rng, count, lo, hi, related=0.5, flagged=0.0):
    qs, ss = [], []
    for _ in range(count):
        q = random_codes(rng, int(rng.integers(lo, hi + 1)))
        s = mutate_codes(rng, q) if rng.random() < related else random_codes(rng, int(rng.integers(lo, hi + 1)))
        if flagged and rng.random() < flagged:
            q = q.copy(); q[rng.integers(0, len(q))] = 4
            s = s.copy(); s[rng.integers(0, len(s))] = 4
        qs.append(q); ss.append(s)
    return qs, ss, [(i, i) for i in range(count)]


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
@pytest.mark.parametrize("variant", ["auto", "i32", "f16x2"])
def test_golden_vectors(ctx, align_type, gap_model, variant):
    recs = [r for name in ("kat.json", "adversarial.json") for r in load_golden(name)]
    recs += load_golden("random_small.json")["pairs"]
    recs = [r for r in recs if r["align_type"] == align_type and r["gap_model"] == gap_model]
    by_scheme = {}
    for r in recs:
        by_scheme.setdefault(tuple(r["scheme"]), []).append(r)
    for sch, rs in by_scheme.items():
        scheme = scheme_of(sch, gap_model)
        if variant == "f16x2":
            if gap_model == "affine" and not N.merged_state_exact(scheme):
                continue
            rs = [r for r in rs if N.f16_range_ok(scheme, len(r["q"]), len(r["s"])) and scheme.mismatch_score <= 0 <= scheme.match_score]
            if not rs:
                continue
        qs = [codes(r["q"]) for r in rs]; ss = [codes(r["s"]) for r in rs]
        got = gpu_scores(ctx, qs, ss, [(i, i) for i in range(len(rs))], scheme, align_type, variant)
        want = (np.array([r["score"] for r in rs]), np.array([r["end"][0] for r in rs]), np.array([r["end"][1] for r in rs]))
        assert (got[3] == 0).all()
        assert_scores_equal(got, want, f"{align_type}/{gap_model}/{variant}/{sch}")


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_random_vs_oracle_all_variants(ctx, align_type, gap_model):
    rng = np.random.default_rng(101)
    pool = AFFINE_SCHEMES if gap_model == "affine" else LINEAR_SCHEMES
    for k, sch in enumerate(pool):
        scheme = scheme_of(sch, gap_model)
        qs, ss, pairs = _random_batch(rng, 300, 1, 300, flagged=0.2)
        want = oracle_scores(qs, ss, pairs, scheme, align_type)
        for variant in ("auto", "i32"):
            got = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, variant)
            assert_scores_equal(got, want, f"{align_type}/{gap_model}/{variant}/{sch}")


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_uniform_150bp_f16_equals_i32_equals_oracle(ctx, align_type, gap_model):
    rng = np.random.default_rng(7)
    scheme = scheme_of((2, -1, 2, 1) if gap_model == "affine" else (2, -1, 1, 1), gap_model)
    n = 4001  # odd: the last packed unit has an empty half
    qs = [random_codes(rng, 150) for _ in range(n)]
    ss = [mutate_codes(rng, q)[:150] if i % 2 else random_codes(rng, 150) for i, q in enumerate(qs)]
    ss = [np.concatenate([s, random_codes(rng, 150 - len(s))]) for s in ss]
    pairs = [(i, i) for i in range(n)]
    want = oracle_scores(qs, ss, pairs, scheme, align_type)
    f16 = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, "f16x2")
    i32 = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, "i32")
    assert_scores_equal(f16, want, "f16x2")
    assert_scores_equal(i32, want, "i32")


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_multi_stage_long_reads(ctx, align_type):
    rng = np.random.default_rng(11)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    qs, ss = [], []
    for L in (700, 1500, 2500, 513, 512, 1025):
        q = random_codes(rng, L)
        qs.append(q); ss.append(mutate_codes(rng, q, 0.1, 0.05, 0.05))
    qs.append(random_codes(rng, 40)); ss.append(random_codes(rng, 3000))
    qs.append(random_codes(rng, 3000)); ss.append(random_codes(rng, 40))
    pairs = [(i, i) for i in range(len(qs))]
    want = oracle_scores(qs, ss, pairs, scheme, align_type)
    got = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, "auto")
    assert_scores_equal(got, want, align_type)
    lin = scheme_of((2, -1, 1, 1), "linear")
    assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, lin, align_type), oracle_scores(qs, ss, pairs, lin, align_type), "linear")


def test_all_pairs_index_pools(ctx):
    rng = np.random.default_rng(3)
    qs = [random_codes(rng, int(rng.integers(20, 200))) for _ in range(9)]
    ss = [random_codes(rng, int(rng.integers(20, 200))) for _ in range(7)]
    pairs = [(a, b) for a in range(9) for b in range(7)]
    scheme = scheme_of((2, -1, 2, 1), "affine")
    for at in ("global", "local", "semiglobal"):
        assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, scheme, at), oracle_scores(qs, ss, pairs, scheme, at), at)


def test_forced_f16_reports_range_status(ctx):
    rng = np.random.default_rng(4)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    qs = [random_codes(rng, 100), random_codes(rng, 900)]
    ss = [random_codes(rng, 100), random_codes(rng, 900)]
    got = gpu_scores(ctx, qs, ss, [(0, 0), (1, 1)], scheme, "local", "f16x2")
    assert got[3][0] == 0 and got[3][1] == N.WSB_E_RANGE
    with pytest.raises(ValueError):
        gpu_scores(ctx, qs, ss, [(0, 0)], scheme_of((2, -9, 2, 1), "affine"), "local", "f16x2")


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_long_read_kernel_mixed_lengths(ctx, align_type, gap_model):
    """Pipelined long-read kernel (score_long.cuh): skewed lengths so that several warps-per-pair classes launch side
    by side, flagged symbols, related and unrelated pairs, lengths straddling the 512-column stage width."""
    rng = np.random.default_rng(2205)
    pool = AFFINE_SCHEMES[:2] if gap_model == "affine" else LINEAR_SCHEMES[:2]
    lens = [257, 300, 511, 512, 513, 1023, 1024, 1025, 1536, 2049, 3000, 4100, 64, 65, 9000, 12000]
    qs, ss = [], []
    for L in lens:
        q = random_codes(rng, L)
        s = mutate_codes(rng, q, 0.08, 0.03, 0.03) if rng.random() < 0.6 else random_codes(rng, int(L * rng.uniform(0.8, 1.25)))
        if rng.random() < 0.3:
            q = q.copy(); q[rng.integers(0, len(q), 3)] = 4
            s = s.copy(); s[rng.integers(0, len(s), 3)] = 4
        qs.append(q); ss.append(s)
    for _ in range(40):
        L = int(rng.integers(260, 2000))
        qs.append(random_codes(rng, L)); ss.append(mutate_codes(rng, qs[-1], 0.1, 0.05, 0.05))
    qs.append(random_codes(rng, 70)); ss.append(random_codes(rng, 5000))    # wide and flat
    qs.append(random_codes(rng, 5000)); ss.append(random_codes(rng, 300))   # tall and narrow
    pairs = [(i, i) for i in range(len(qs))]
    for sch in pool:
        scheme = scheme_of(sch, gap_model)
        want = oracle_scores(qs, ss, pairs, scheme, align_type)
        got = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, "auto")
        assert_scores_equal(got, want, f"long {align_type}/{gap_model}/{sch}")


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_long_read_kernel_uniform_batch(ctx, align_type):
    rng = np.random.default_rng(77)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    qs = [random_codes(rng, 2600) for _ in range(48)]
    ss = [np.resize(mutate_codes(rng, q, 0.05, 0.02, 0.02), 2600) if i % 2 else random_codes(rng, 2600) for i, q in enumerate(qs)]
    pairs = [(i, i) for i in range(len(qs))]
    assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, scheme, align_type), oracle_scores(qs, ss, pairs, scheme, align_type),
                        f"uniform long {align_type}")


def test_long_reads_with_non_merged_scheme_use_exact_model(ctx):
    rng = np.random.default_rng(78)
    scheme = scheme_of((2, -9, 2, 1), "affine")   # merged state not exact -> three-state kernel
    qs = [random_codes(rng, 1400) for _ in range(6)]
    ss = [mutate_codes(rng, q, 0.1, 0.05, 0.05) for q in qs]
    pairs = [(i, i) for i in range(len(qs))]
    for at in ("global", "local", "semiglobal"):
        assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, scheme, at), oracle_scores(qs, ss, pairs, scheme, at), at)


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_wide_substitution_scores_use_compare_select_kernel(ctx, align_type):
    """|match - mismatch| > 127 does not fit the byte profile of the dp4a kernels: the planner falls back to ArI32W."""
    rng = np.random.default_rng(79)
    scheme = scheme_of((100, -90, 120, 10), "affine")
    qs, ss, pairs = _random_batch(rng, 60, 1, 700, flagged=0.2)
    assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, scheme, align_type), oracle_scores(qs, ss, pairs, scheme, align_type),
                        f"wide {align_type}")
    lin = scheme_of((90, -80, 100, 100), "linear")
    assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, lin, align_type), oracle_scores(qs, ss, pairs, lin, align_type),
                        f"wide linear {align_type}")


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_long_read_kernel_cluster_classes(ctx, align_type):
    """A batch whose largest pairs dwarf the rest: the planner gives them whole thread-block clusters (2, 4, 8 blocks of
    16 warps), with progress counters in global memory."""
    rng = np.random.default_rng(4242)
    scheme = scheme_of((2, -1, 2, 1), "affine")
    shapes = [(1500, 70000), (2500, 40000), (3000, 20000), (1200, 9000), (900, 5000), (700, 2500)]
    shapes += [(300, 600)] * 6
    qs, ss = [], []
    for m, n in shapes:
        q = random_codes(rng, m)
        s = random_codes(rng, n)
        at = int(rng.integers(0, n - m))
        s[at:at + m] = mutate_codes(rng, q, 0.05, 0.0, 0.0)[:m]   # a diagonal band worth finding
        qs.append(q); ss.append(s)
    pairs = [(i, i) for i in range(len(qs))]
    want = oracle_scores(qs, ss, pairs, scheme, align_type)
    got = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, "auto")
    assert_scores_equal(got, want, f"cluster {align_type}")


@pytest.mark.parametrize("gap_model", ["linear", "affine"])
def test_packed_int16_variant_equals_oracle_including_flagged_subjects(ctx, gap_model):
    """Opt-in S16X2 variant (score_short16.cuh): short local pairs run in packed int16; a pair whose subject holds a
    flagged symbol cannot be encoded there and is re-scored by the half2 kernel inside the same call."""
    rng = np.random.default_rng(16)
    scheme = scheme_of((2, -1, 2, 1) if gap_model == "affine" else (2, -1, 1, 1), gap_model)
    n = 3001
    qs = [random_codes(rng, int(rng.integers(30, 161))) for _ in range(n)]
    ss = [mutate_codes(rng, q)[:150] if i % 2 else random_codes(rng, int(rng.integers(30, 151))) for i, q in enumerate(qs)]
    for i in range(0, n, 7):      # flagged symbols on either side, sometimes both
        if i % 3 != 1:
            s = ss[i].copy(); s[rng.integers(0, len(s))] = 4; ss[i] = s
        if i % 3 != 0:
            q = qs[i].copy(); q[rng.integers(0, len(q))] = 4; qs[i] = q
    qs.append(random_codes(rng, 600)); ss.append(random_codes(rng, 700))    # too long for the kernel: routed as in AUTO
    pairs = [(i, i) for i in range(len(qs))]
    want = oracle_scores(qs, ss, pairs, scheme, "local")
    got = gpu_scores(ctx, qs, ss, pairs, scheme, "local", "s16x2")
    assert_scores_equal(got, want, f"s16x2 {gap_model}")
    # other alignment types: S16X2 is simply AUTO
    assert_scores_equal(gpu_scores(ctx, qs[:200], ss[:200], pairs[:200], scheme, "global", "s16x2"),
                        oracle_scores(qs[:200], ss[:200], pairs[:200], scheme, "global"), "s16x2 global")


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_packed_int16_long_read_kernel_twins_and_hand_backs(ctx, align_type, gap_model):
    """Long pairs of identical shape run two per block in packed int16 (score_long16.cuh); pairs whose subject holds a
    flagged symbol are handed back to the int32 kernel inside the same call; odd counts leave a single."""
    rng = np.random.default_rng(1616)
    scheme = scheme_of((2, -1, 2, 1) if gap_model == "affine" else (2, -1, 2, 2), gap_model)
    qs, ss = [], []
    for (m, n, count) in ((1100, 1300, 5), (2600, 2600, 4), (700, 3100, 3), (4000, 1024, 2)):
        for k in range(count):
            q = random_codes(rng, m)
            s = random_codes(rng, n)
            if k % 2 == 0:
                at = int(rng.integers(0, max(1, n - m))) if n > m else 0
                piece = mutate_codes(rng, q, 0.05, 0.0, 0.0)[:min(m, n - at)]
                s[at:at + len(piece)] = piece
            qs.append(q); ss.append(s)
    ss[1] = ss[1].copy(); ss[1][700] = 4          # flagged subject symbol: hand-back
    qs[6] = qs[6].copy(); qs[6][1234] = 4         # flagged query symbol: exact in the packed kernel
    ss[10] = ss[10].copy(); ss[10][3000] = 4; qs[10] = qs[10].copy(); qs[10][5] = 4
    pairs = [(i, i) for i in range(len(qs))]
    want = oracle_scores(qs, ss, pairs, scheme, align_type)
    got = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, "auto")
    assert_scores_equal(got, want, f"long16 {align_type}/{gap_model}")
    i32 = gpu_scores(ctx, qs, ss, pairs, scheme, align_type, "i32")
    assert_scores_equal(i32, want, f"long int32 {align_type}/{gap_model}")


@pytest.mark.parametrize("gap_model", ["linear", "affine"])
def test_packed_int16_global_short_kernel(ctx, gap_model):
    """AUTO sends short global pairs to score_short16g.cuh: uniform batches (row m captured in the last P trips), ragged
    ones (captured in every trip), reads shorter than the lane group, flagged symbols on both sides (a flagged subject
    symbol hands the pair to the int32 kernel inside the same call), schemes with positive mismatch / beta > alpha."""
    rng = np.random.default_rng(1601)
    schemes = [(2, -1, 2, 1), (3, -2, 4, 1), (1, -3, 2, 2), (5, -4, 10, 1), (2, 1, 3, 1), (2, -1, 1, 3), (1, -1, 0, 0)] \
        if gap_model == "affine" else [(2, -1, 1, 1), (2, -1, 2, 2), (3, -2, 5, 5), (1, 1, 1, 1), (2, -1, 0, 0)]
    for sch in schemes:
        scheme = scheme_of(sch, gap_model)
        if gap_model == "affine" and not N.merged_state_exact(scheme):
            continue
        # uniform 150 x 150 (and 150 x 140), odd pair count
        for L, Ls in ((150, 150), (150, 140), (17, 152), (154, 9)):
            n = 1001
            qs = [random_codes(rng, L) for _ in range(n)]
            ss = [mutate_codes(rng, q, 0.1, 0.05, 0.05)[:Ls] if i % 2 else random_codes(rng, Ls) for i, q in enumerate(qs)]
            ss = [np.concatenate([s, random_codes(rng, Ls - len(s))]) for s in ss]
            for i in range(0, n, 11):
                if i % 3 != 1:
                    s = ss[i].copy(); s[rng.integers(0, len(s))] = 4; ss[i] = s
                if i % 3 != 0:
                    q = qs[i].copy(); q[rng.integers(0, len(q))] = 4; qs[i] = q
            pairs = [(i, i) for i in range(n)]
            assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, scheme, "global", "auto"),
                                oracle_scores(qs, ss, pairs, scheme, "global"), f"uniform {L}x{Ls} {gap_model} {sch}")
        # ragged: 1 .. 154 x 1 .. 152, plus pairs too long for the kernel
        qs, ss, pairs = _random_batch(rng, 1500, 1, 152, flagged=0.1)
        qs.append(random_codes(rng, 154)); ss.append(random_codes(rng, 1))
        qs.append(random_codes(rng, 400)); ss.append(random_codes(rng, 90))
        qs.append(random_codes(rng, 3)); ss.append(random_codes(rng, 3))
        pairs = [(i, i) for i in range(len(qs))]
        assert_scores_equal(gpu_scores(ctx, qs, ss, pairs, scheme, "global", "auto"),
                            oracle_scores(qs, ss, pairs, scheme, "global"), f"ragged {gap_model} {sch}")


@pytest.mark.gpu
@pytest.mark.parametrize("lat", ["0", "2"])
def test_packed_int16_short_kernels_agree_with_the_oracle_in_both_lane_group_shapes(lat):
    """The planner picks the lane-group shape of the packed int16 short-read kernels by launch size (8 x K groups, or the
    16 x 10 latency shape for small launch groups); WSB_S16_LAT pins one of them for a whole process, so the randomized
    cross-check (ragged and uniform batches of 3 .. 12 000 pairs up to 154 x 152, random schemes, flagged symbols, local and
    global) runs once per shape in a subprocess."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WSB_S16_LAT=lat)
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_short16.py"), "31", "10"], env=env, cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "TOTAL MISMATCHES 0" in out.stdout, out.stdout[-2000:]
