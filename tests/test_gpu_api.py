"""GPU: the reference-facing Python API (run_batch, engine_score, align, ...) behaves like the reference's."""
import os

import numpy as np
import pytest

import oracle
import paper_2205_07610_b200 as W
from conftest import COMBOS, load_golden
from paper_2205_07610_b200 import _native as N

pytestmark = pytest.mark.gpu


def _seqs(texts):
    return [W.encode_sequence(f"s{i}", t) for i, t in enumerate(texts)]


def test_frozen_kats_through_public_api():
    # pkg/tests/test_refdp.py:18-72 restated against the GPU path
    lin = W.ScoringScheme(2, -1, 1, 1, "linear")
    aff = W.ScoringScheme(2, -1, 2, 1, "affine")
    q, s = _seqs(["ACGT", "AGT"])
    assert W.engine_score(q, s, W.AlignConfig("global", "linear"), lin) == (5, (4, 3), 12)
    r = W.align_traceback(q, s, W.AlignConfig("global", "linear", "traceback"), lin)
    assert r.ops == [("M", 1), ("I", 1), ("M", 2)] and r.score == 5 and W.rescore_alignment(r, q, s, lin) == 5
    q, s = _seqs(["AAAA", "AA"])
    assert W.engine_score(q, s, W.AlignConfig("global", "affine"), aff)[:2] == (1, (4, 2))
    r = W.align("ACG", "TTACGTT", "semiglobal", aff)
    assert (r.score, r.ops, r.q_start, r.q_end, r.s_start, r.s_end) == (6, [("M", 3)], 0, 3, 2, 5)
    r = W.align("TTACGTT", "ACG", "local", aff)
    assert (r.score, r.ops, r.q_start) == (6, [("M", 3)], 2)
    r = W.align("TTTT", "CCCC", "local", aff)
    assert (r.score, r.ops) == (0, []) and r.q_start == r.q_end
    r = W.align("AA", "A", "global", lin)
    assert (r.score, r.ops) == (1, [("I", 1), ("M", 1)])
    assert W.cigar_string(r) == "1I1M"
    r = W.align("ACGT", "ACGT", "global", lin, traceback=False)
    assert (r.score, r.q_end, r.s_end, r.ops) == (8, 4, 4, None)


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_run_batch_matches_oracle_and_single_pair_api(align_type, gap_model):
    rng = np.random.default_rng(9)
    bases = np.array(list("ACGT"))
    qs = _seqs(["".join(bases[rng.integers(0, 4, int(rng.integers(5, 200)))]) for _ in range(6)])
    ss = _seqs(["".join(bases[rng.integers(0, 4, int(rng.integers(5, 200)))]) for _ in range(5)])
    scheme = W.ScoringScheme(2, -1, 2, 1, "affine") if gap_model == "affine" else W.ScoringScheme(2, -1, 1, 1, "linear")
    pairs = W.all_pairs(qs, ss)
    assert pairs[:6] == [(0, 0), (0, 1), (0, 2), (0, 3), (0, 4), (1, 0)]
    rep = W.run_batch(W.BatchJob(qs, ss, pairs, W.AlignConfig(align_type, gap_model), scheme))
    assert rep.total_cells == sum(len(qs[a]) * len(ss[b]) for a, b in pairs)
    for (a, b), res in zip(pairs, rep.results):
        score, end = oracle.ref_score(qs[a].device_codes(), ss[b].device_codes(), align_type, gap_model == "affine",
                                      scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend)
        assert res.score == score and res.ops is None and res.cells_computed == len(qs[a]) * len(ss[b])
        if align_type == "global":
            assert (res.q_start, res.q_end, res.s_start, res.s_end) == (0, len(qs[a]), 0, len(ss[b]))
        else:
            assert (res.q_start, res.q_end, res.s_start, res.s_end) == (end[0], end[0], end[1], end[1])
        single = W.engine_score(qs[a], ss[b], W.AlignConfig(align_type, gap_model), scheme)
        assert single == (score, end, len(qs[a]) * len(ss[b]))
    # packed tuning gives the same results (tests/test_batch.py:102-113)
    rep2 = W.run_batch(W.BatchJob(qs, ss, pairs, W.AlignConfig(align_type, gap_model), scheme, tuning=W.EngineTuning(packed=True)))
    assert rep2.results == rep.results
    # traceback mode follows ref_traceback
    rep3 = W.run_batch(W.BatchJob(qs, ss, pairs[:8], W.AlignConfig(align_type, gap_model, "traceback"), scheme))
    for (a, b), res in zip(pairs[:8], rep3.results):
        want = oracle.ref_traceback(qs[a].device_codes(), ss[b].device_codes(), align_type, gap_model == "affine",
                                    scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend)
        assert (res.score, res.q_start, res.q_end, res.s_start, res.s_end, res.ops) == (
            want["score"], want["q_start"], want["q_end"], want["s_start"], want["s_end"], want["ops"])
        assert W.rescore_alignment(res, qs[a], ss[b], scheme) == res.score


def test_packed_engine_and_errors():
    aff = W.ScoringScheme(2, -1, 2, 1, "affine")
    cfg = W.AlignConfig("local", "affine")
    for rec in load_golden("random_small.json")["packed"][:12]:
        scheme = W.ScoringScheme(*rec["scheme"], rec["gap_model"])
        c = W.AlignConfig(rec["align_type"], rec["gap_model"])
        qa, sa, qb, sb = _seqs([rec["qa"], rec["sa"], rec["qb"], rec["sb"]])
        ra, rb, cells = W.engine_score_packed((qa, sa), (qb, sb), c, scheme)
        assert [ra[0], ra[1][0], ra[1][1]] == rec["a"] and [rb[0], rb[1][0], rb[1][1]] == rec["b"] and cells == rec["cells"]
    big = _seqs(["A" * 5000, "A" * 5000])
    with pytest.raises(W.PackedRangeOverflow):
        W.engine_score_packed((big[0], big[1]), (big[0], big[1]), cfg, aff)
    with pytest.raises(ValueError):
        q, s = _seqs(["ACGT", "ACGT"])
        W.engine_score_packed((q, s), (q, s), cfg, W.ScoringScheme(2, -9, 2, 1, "affine"))
    with pytest.raises(W.ConfigMismatch):
        W.engine_score(*_seqs(["AC", "AC"]), W.AlignConfig("local", "linear"), aff)
    with pytest.raises(ValueError):
        W.BatchJob(_seqs(["AC"]), _seqs(["AC"]), [(0, 1)], cfg, aff)
    with pytest.raises(ValueError):
        W.BatchJob(_seqs(["AC"]), _seqs(["AC"]), [], cfg, aff)


def _recipe_pair(seed, m, n, related):
    """tests/golden/make_golden_packed_long.py:make_pair, restated (the fixture stores recipes + CRCs, not the text)."""
    rng = np.random.default_rng(seed)
    bases = np.array(list("ACGT"))
    q = rng.integers(0, 4, m)
    if related:
        s = np.resize(q, n).copy()
        mut = rng.random(n) < 0.08
        s[mut] = (s[mut] + rng.integers(1, 4, int(mut.sum()))) % 4
    else:
        s = rng.integers(0, 4, n)
    return "".join(bases[q]), "".join(bases[s])


def test_packed_entry_accepts_the_reference_range_up_to_2_pow_14():
    """engine_score_packed over the reference's whole packed range (max_step * (m + n) < 2^14, engine.py:504-536): 27
    results of the REFERENCE's engine_score_packed on pairs of 600..4000 symbols; tuning.packed stays a hint."""
    import zlib
    for rec in load_golden("packed_long.json")["packed_long"]:
        scheme = W.ScoringScheme(*rec["scheme"], rec["gap_model"])
        c = W.AlignConfig(rec["align_type"], rec["gap_model"])
        (qa, sa), (qb, sb) = _recipe_pair(*rec["a_recipe"]), _recipe_pair(*rec["b_recipe"])
        assert [zlib.crc32((qa + "|" + sa).encode()), zlib.crc32((qb + "|" + sb).encode())] == rec["crc"]
        qa, sa, qb, sb = _seqs([qa, sa, qb, sb])
        assert W.packed_range_ok(scheme, len(qa), len(sa)) and W.packed_range_ok(scheme, len(qb), len(sb))
        ra, rb, cells = W.engine_score_packed((qa, sa), (qb, sb), c, scheme)
        assert [ra[0], ra[1][0], ra[1][1]] == rec["a"] and [rb[0], rb[1][0], rb[1][1]] == rec["b"] and cells == rec["cells"], rec
        one = W.engine_score(qa, sa, c, scheme, tuning=W.EngineTuning(packed=True))     # never raises on range
        assert [one[0], one[1][0], one[1][1]] == rec["a"]
    aff = W.ScoringScheme(2, -1, 2, 1, "affine")
    edge = _seqs(["A" * 4096, "C" * 4095, "A" * 4096, "C" * 4096])        # 2 * 8191 < 2^14 <= 2 * 8192
    W.engine_score_packed((edge[0], edge[1]), (edge[0], edge[1]), W.AlignConfig("local", "affine"), aff)
    with pytest.raises(W.PackedRangeOverflow):
        W.engine_score_packed((edge[2], edge[3]), (edge[0], edge[1]), W.AlignConfig("local", "affine"), aff)


def test_flagged_symbols_never_match():
    aff = W.ScoringScheme(2, -1, 2, 1, "affine")
    q, s = _seqs(["NNNN", "NNNN"])
    assert W.engine_score(q, s, W.AlignConfig("local", "affine"), aff)[0] == 0
    q, s = _seqs(["ACNGT", "ACNGT"])
    assert W.engine_score(q, s, W.AlignConfig("global", "affine"), aff)[0] == 2 * 4 - 1


def test_pool_inputs_and_lazy_results():
    rng = np.random.default_rng(1)
    n = 120_001
    q = rng.integers(0, 4, (n, 40), dtype=np.uint8); s = rng.integers(0, 4, (n, 40), dtype=np.uint8)
    job = W.BatchJob(W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s), np.stack([np.arange(n), np.arange(n)], 1),
                     W.AlignConfig("local", "affine"), W.ScoringScheme())
    rep = W.run_batch(job)
    assert isinstance(rep.results, W.ResultArray) and len(rep.results) == n
    for k in (0, 1, n // 2, n - 1):
        score, end = oracle.ref_score(q[k], s[k], "local", True, 2, -1, 2, 1)
        assert (rep.results[k].score, rep.results[k].q_end, rep.results[k].s_end) == (score, end[0], end[1])
    assert rep.gpu_launches >= 1 and rep.h2d_bytes >= 2 * n * 40 and rep.kernel_ms > 0   # regular metadata is generated on the device


def test_packed_pools_give_identical_results():
    """Pools in the reference's 2-bit layout are expanded on the device (wsb_batch_create_packed_async)."""
    rng = np.random.default_rng(21)
    n = 70_000   # large enough for the piecewise upload path when unflagged
    L = 150
    q = rng.integers(0, 4, (n, L), dtype=np.uint8)
    s = rng.integers(0, 4, (n, L), dtype=np.uint8)
    idx = np.arange(n, dtype=np.int32)
    pairs = np.stack([idx, idx], 1)
    for flagged in (False, True):
        if flagged:
            q[5, 7] = 4; s[11, 3] = 4; s[n - 1, L - 1] = 4
        pq, ps = W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s)
        for cfg in (W.AlignConfig("local", "affine"), W.AlignConfig("global", "affine"),
                    W.AlignConfig("semiglobal", "affine", "traceback")):
            count = n if cfg.result_mode == "score_only" else 3000
            a = W.run_batch(W.BatchJob(pq, ps, pairs[:count], cfg, W.ScoringScheme()))
            b = W.run_batch(W.BatchJob(pq.to_packed(), ps.to_packed(), pairs[:count], cfg, W.ScoringScheme()))
            assert b.h2d_bytes < a.h2d_bytes
            ra, rb = a.results, b.results
            if isinstance(ra, list):
                assert ra == rb
            else:
                for f in ("score", "q_start", "q_end", "s_start", "s_end"):
                    assert (getattr(ra, f) == getattr(rb, f)).all(), (flagged, cfg.align_type, f)
                if ra.runs is not None:
                    assert (ra.runs == rb.runs).all() and (ra.run_off == rb.run_off).all()


@pytest.mark.parametrize("result_mode", ["score_only", "traceback"])
def test_multi_shard_assembly_on_one_gpu(monkeypatch, result_mode):
    """run_batch(devices=[...]) with three shards: every shard gets its own context (here all on GPU 0, one context per
    shard thread) and the results are scattered back into pair order, identical to the single-shard run."""
    from paper_2205_07610_b200 import _native as N, batch as B
    rng = np.random.default_rng(33)
    n = 900
    lens = rng.integers(30, 400, n)
    qs = [rng.integers(0, 4, int(L)).astype(np.uint8) for L in lens]
    ss = [rng.integers(0, 4, int(L * rng.uniform(0.7, 1.3)) + 1).astype(np.uint8) for L in lens]

    def pool(seqs):
        ln = np.array([len(s) for s in seqs], np.int32)
        off = np.zeros(len(seqs), np.int64); off[1:] = np.cumsum(ln[:-1])
        return W.SequencePool(np.concatenate(seqs), off, ln)

    pairs = np.stack([rng.permutation(n), rng.permutation(n)], 1).astype(np.int32)
    cfg = W.AlignConfig("local" if result_mode == "score_only" else "semiglobal", "affine", result_mode)
    job1 = W.BatchJob(pool(qs), pool(ss), pairs, cfg, W.ScoringScheme(), devices=[0])
    one = W.run_batch(job1)
    made = []
    monkeypatch.setattr(B, "get_context", lambda device: made.append(N.Context(0)) or made[-1])
    job3 = W.BatchJob(pool(qs), pool(ss), pairs, cfg, W.ScoringScheme(), devices=[0, 0, 0])
    three = W.run_batch(job3)
    assert len(made) == 3 and len(three.shard_cells) == 3 and sum(three.shard_cells) == one.total_cells == three.total_cells
    assert max(three.shard_cells) - min(three.shard_cells) <= 400 * 520     # balanced to within one large pair
    assert list(one.results) == list(three.results)
    for c in made:
        c.close()


def _contexts_per_shard(monkeypatch):
    from paper_2205_07610_b200 import _native as N, batch as B
    made = []
    monkeypatch.setattr(B, "get_context", lambda device: made.append(N.Context(0)) or made[-1])
    return made


@pytest.mark.parametrize("result_mode", ["score_only", "traceback"])
def test_sharded_run_uploads_every_pool_byte_once(monkeypatch, result_mode):
    """a shard uploads only what its pairs reference.  Arbitrary pair lists over pools four times larger than
    any shard needs: the four shards together move about as many bytes as one shard would, results identical."""
    rng = np.random.default_rng(44)
    n_seq, n = 4000, 1000
    lens = rng.integers(60, 300, n_seq)
    qs = [rng.integers(0, 4, int(L)).astype(np.uint8) for L in lens]
    ss = [rng.integers(0, 4, int(L)).astype(np.uint8) for L in lens]

    def pool(seqs):
        ln = np.array([len(s) for s in seqs], np.int32)
        off = np.zeros(len(seqs), np.int64); off[1:] = np.cumsum(ln[:-1])
        return W.SequencePool(np.concatenate(seqs), off, ln)

    used = rng.choice(n_seq, n, replace=False)
    pairs = np.stack([used, rng.permutation(used)], 1).astype(np.int32)      # a quarter of either pool is referenced
    cfg = W.AlignConfig("local" if result_mode == "score_only" else "global", "affine", result_mode)
    one = W.run_batch(W.BatchJob(pool(qs), pool(ss), pairs, cfg, W.ScoringScheme(), devices=[0]))
    made = _contexts_per_shard(monkeypatch)
    four = W.run_batch(W.BatchJob(pool(qs), pool(ss), pairs, cfg, W.ScoringScheme(), devices=[0, 0, 0, 0]))
    assert len(made) == 4 and list(one.results) == list(four.results)
    referenced = int(lens[pairs[:, 0]].sum() + lens[pairs[:, 1]].sum())
    metadata = 4 * (8 + 4) * n // 2 + 2 * 4 * n          # offsets + lengths of the compact pools, pair columns
    assert four.h2d_bytes <= referenced + 2 * metadata + 4096, (four.h2d_bytes, referenced)
    assert four.h2d_bytes * 3 < one.h2d_bytes            # the single shard sends the whole pools
    for c in made:
        c.close()


def test_sharded_reads_matrix_takes_the_metadata_free_path_per_shard(monkeypatch):
    """Uniform pools with the identity pair list: contiguous blocks, zero-copy slices, every shard on the regular upload
    (no offset / length / pair arrays), bytes and 2-bit pools alike."""
    rng = np.random.default_rng(45)
    n, L = 140_000, 64
    q = rng.integers(0, 4, (n, L), dtype=np.uint8); s = rng.integers(0, 4, (n, L), dtype=np.uint8)
    s[::3] = q[::3]
    pairs = np.stack([np.arange(n), np.arange(n)], 1).astype(np.int32)
    cfg = W.AlignConfig("local", "affine", "score_only")
    one = W.run_batch(W.BatchJob(W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s), pairs, cfg,
                                 W.ScoringScheme(), devices=[0]))
    made = _contexts_per_shard(monkeypatch)
    for packed in (False, True):
        pq, ps = W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s)
        if packed:
            pq, ps = pq.to_packed(), ps.to_packed()
        two = W.run_batch(W.BatchJob(pq, ps, pairs, cfg, W.ScoringScheme(), devices=[0, 0]))
        assert (two.results.score == one.results.score).all() and (two.results.q_end == one.results.q_end).all()
        assert (two.results.s_end == one.results.s_end).all()
        assert two.h2d_bytes == (2 * n * L // 4 if packed else 2 * n * L)      # pool bytes only, each once
        assert len(two.shard_cells) == 2 and sum(two.shard_cells) == n * L * L
    for c in made:
        c.close()


@pytest.mark.parametrize("align_type,gap_model", COMBOS)
def test_small_reads_matrix_takes_the_metadata_free_path(align_type, gap_model):
    """cfg1-sized regular jobs (uniform pools, identity pairs, score only) skip the offset / length / pair arrays like the
    big ones: same results as the general upload of the same reads and as the oracle, and only pool bytes on the bus."""
    rng = np.random.default_rng(77)
    n, L = 3000, 150
    q = rng.integers(0, 4, (n, L), dtype=np.uint8); s = rng.integers(0, 4, (n, L), dtype=np.uint8)
    s[::2] = q[::2]; s[::2, 40:43] = 3 - s[::2, 40:43]
    scheme = W.ScoringScheme(2, -1, 2, 1, "affine") if gap_model == "affine" else W.ScoringScheme(2, -1, 1, 1, "linear")
    cfg = W.AlignConfig(align_type, gap_model)
    ident = np.stack([np.arange(n), np.arange(n)], 1).astype(np.int32)
    fast = W.run_batch(W.BatchJob(W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s), ident, cfg, scheme))
    assert fast.h2d_bytes == 2 * n * L
    # the same pairs in reverse order: not an identity list, so the general upload carries them
    rev = ident[::-1].copy()
    slow = W.run_batch(W.BatchJob(W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s), rev, cfg, scheme))
    assert slow.h2d_bytes > 2 * n * L
    off = np.arange(n, dtype=np.int64) * L; ln = np.full(n, L, np.int32); idx = np.arange(n, dtype=np.int32)
    sc, ei, ej = oracle.score_batch(q.reshape(-1), off, ln, s.reshape(-1), off, ln, idx, idx, align_type, gap_model == "affine",
                                    scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend)[:3]
    for k in range(n):
        a, b = fast.results[k], slow.results[n - 1 - k]
        assert (a.score, a.q_end, a.s_end) == (b.score, b.q_end, b.s_end) == (int(sc[k]), int(ei[k]), int(ej[k]))


def test_selftest_draws_the_reference_cases_and_agrees_with_the_oracle():
    """selftest() mirrors cli.cmd_selftest (cli.py:264-301): same random cases per seed, AUTO kernels vs the int32 kernel on
    the GPU, here with the CPU oracle as a third voice; a planted wrong answer must come back as a JSON-able repro blob."""
    import json
    import oracle
    from helpers import make_pool
    import paper_2205_07610_b200 as W

    def checker(queries, subjects, scheme, align_type):
        qc, qo, ql = make_pool([np.where(q.flags, 4, q.codes).astype(np.uint8) for q in queries])
        sc, so, sl = make_pool([np.where(s.flags, 4, s.codes).astype(np.uint8) for s in subjects])
        idx = np.arange(len(queries), dtype=np.int32)
        return oracle.score_batch(qc, qo, ql, sc, so, sl, idx, idx, align_type, scheme.gap_model == "affine",
                                  scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend)

    rep = W.selftest(cases=600, seed=11, checker=checker)
    assert rep == {"ok": True, "cases": 600, "failure": None}

    def liar(queries, subjects, scheme, align_type):
        sc, ei, ej = (np.array(a) for a in checker(queries, subjects, scheme, align_type))
        sc[-1] += 1
        return sc, ei, ej

    rep = W.selftest(cases=40, seed=3, checker=liar)
    assert not rep["ok"]
    blob = json.loads(json.dumps(rep["failure"]))
    assert set(blob) >= {"case", "seed", "query", "subject", "align_type", "gap_model", "scheme", "engine", "reference"}
    assert blob["reference"][0] == blob["engine"][0] + 1 and set(blob["query"]) <= set("ACGT")


def test_engine_stats_from_the_planner():
    """EngineStats in the spirit of tests/test_engine.py:187-245: stages, wavefront iterations and ops per executed cell
    update come back from the native planner (padding included, the reference's definition)."""
    rng = np.random.default_rng(4)
    q = W.Sequence("q", rng.integers(0, 4, 150).astype(np.uint8), np.zeros(150, bool))
    s = W.Sequence("s", rng.integers(0, 4, 150).astype(np.uint8), np.zeros(150, bool))
    scheme = W.ScoringScheme(2, -1, 2, 1, "affine")
    st = W.EngineStats()
    W.engine_score(q, s, W.AlignConfig("local", "affine"), scheme, stats=st, instrument=True)
    # packed int16 short kernel, two alignments per register (the second half rides empty); a batch this small runs on the
    # latency shape: lane groups of 16 x 10 columns
    assert (st.stages, st.iterations, st.cells) == (1, 150 + 16 - 1, 150 * 150)
    assert st.updates == 1 * 150 * 160 * 2
    assert st.ops_max * 4 == st.updates * 5 and st.ops_addsub * 4 == st.updates * 6 and st.ops_lookup * 2 == st.updates
    st2 = W.EngineStats()
    lin = W.ScoringScheme(2, -1, 1, 1, "linear")
    W.engine_score(q, s, W.AlignConfig("global", "linear"), lin, stats=st2, instrument=True)
    assert st2.ops_max * 2 == st2.updates and st2.ops_addsub == st2.updates      # VIMNMX3 + VIADD, PRMT + VIADD per two cells
    # a long pair: 512-column stages of the long-read kernel, int32 (5 instructions per cell: 2 max, 2 add, 1 lookup)
    ql = W.Sequence("q", rng.integers(0, 4, 3000).astype(np.uint8), np.zeros(3000, bool))
    sl = W.Sequence("s", rng.integers(0, 4, 5000).astype(np.uint8), np.zeros(5000, bool))
    st3 = W.EngineStats()
    W.engine_score(ql, sl, W.AlignConfig("global", "affine"), scheme, stats=st3)
    assert st3.stages == 10 and st3.iterations == 10 * (3000 + 31) and st3.updates == 10 * 3000 * 512
    assert st3.ops_total == 4 * st3.updates and st3.ops_lookup == st3.updates
    st3.cells == 3000 * 5000
    # counters accumulate over calls like the reference's absorb()
    W.engine_score(q, s, W.AlignConfig("local", "affine"), scheme, stats=st)
    assert st.stages == 2 and st.cells == 2 * 150 * 150


def _gpu_rank_main(rank, world, port, out_dir):
    """One rank of a two-rank job over gloo, both ranks on GPU 0: plan the shards natively, run MY shard through the product's
    run_batch, gather the shard results by pair index; rank 0 compares the gathered job with the oracle."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(77)                      # every rank builds the same job
    n = 3000
    seqs_q = [rng.integers(0, 4, int(rng.integers(20, 400))).astype(np.uint8) for _ in range(n)]
    seqs_s = [rng.integers(0, 4, int(rng.integers(20, 400))).astype(np.uint8) for _ in range(n)]
    seqs_q[7] = rng.integers(0, 4, 5000).astype(np.uint8); seqs_s[7] = rng.integers(0, 4, 6000).astype(np.uint8)   # one heavy pair
    pool = lambda xs: W.SequencePool.from_sequences([W.Sequence(f"x{i}", x, np.zeros(len(x), bool)) for i, x in enumerate(xs)])
    pq, ps = pool(seqs_q), pool(seqs_s)
    idx = np.arange(n, dtype=np.int32)
    shard_of, cells = N.plan_shards(pq.len, ps.len, idx, idx, world)
    mine = np.nonzero(shard_of == rank)[0]
    cfg = W.AlignConfig("local", "affine", "traceback")
    rep = W.run_batch(W.BatchJob(pq, ps, np.stack([mine, mine], 1), cfg, W.ScoringScheme(), devices=[0]))
    assert rep.total_cells == int(cells[rank])
    local = torch.zeros(n, 3, dtype=torch.int64)
    res = rep.results
    local[torch.from_numpy(mine)] = torch.tensor([[r.score, r.q_end, r.s_end] for r in res], dtype=torch.int64)
    dist.all_reduce(local, op=dist.ReduceOp.SUM)         # disjoint shards: the sum is the gather
    cig = [None] * world
    dist.all_gather_object(cig, {int(p): W.cigar_string(r) for p, r in zip(mine, res)})
    if rank == 0:
        import oracle
        from helpers import make_pool
        qc, qo, ql = make_pool(seqs_q); sc, so, sl = make_pool(seqs_s)
        want = oracle.traceback_batch(qc, qo, ql, sc, so, sl, idx, idx, "local", True, 2, -1, 2, 1)
        got = local.numpy()
        assert (got[:, 0] == want["score"]).all() and (got[:, 1] == want["q_end"]).all() and (got[:, 2] == want["s_end"]).all()
        merged = {k: v for d in cig for k, v in d.items()}
        from conftest import cigar_of
        assert all(merged[k] == cigar_of(want["ops"][k]) for k in range(n))
        with open(os.path.join(out_dir, "ok"), "w") as fh:
            fh.write("ok")
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_over_gloo_run_their_shards_on_the_gpu(tmp_path):
    """The multi-rank protocol of bench.py / a multi-process deployment with real GPU work: world size 2 over gloo, both ranks on
    GPU 0."""
    import torch.multiprocessing as mp
    port = 29600 + (os.getpid() % 2000)
    mp.spawn(_gpu_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    assert open(tmp_path / "ok").read() == "ok"


def test_host_packed_upload_matches_the_plain_upload(monkeypatch):
    """Large byte pools are packed into the 2-bit layout by host threads, piece by piece, and expanded on the device
    (hostpack.cpp, HostPacker in wsb200.cu): a quarter of the bytes on the bus, identical results.  Covered: a reads
    matrix (metadata-free path), ragged pools whose piece boundaries fall inside a packed byte, flagged symbols (their
    slice travels as plain bytes, also next to a shared byte), score-only and traceback, and the oracle on a sample."""
    from paper_2205_07610_b200 import batch as B
    from paper_2205_07610_b200.engine import get_context
    monkeypatch.delenv("WSB_HOST_PACK_THREADS", raising=False)
    monkeypatch.delenv("LOCAL_WORLD_SIZE", raising=False)
    assert N.load().wsb_host_pack_isa().decode() in ("avx512bw", "bmi2", "plain")
    rng = np.random.default_rng(77)
    scheme = W.ScoringScheme()

    def run(pq, ps, pairs, cfg, threads):
        monkeypatch.setattr(B, "_host_pack_policy", lambda: threads)
        return W.run_batch(W.BatchJob(pq, ps, pairs, cfg, scheme))

    def same(a, b, what):
        for f in ("score", "q_start", "q_end", "s_start", "s_end"):
            assert (getattr(a.results, f) == getattr(b.results, f)).all(), (what, f)
        if a.results.runs is not None:
            assert (a.results.runs == b.results.runs).all() and (a.results.run_off == b.results.run_off).all(), what

    # 1. reads matrix, 300 k x 150 bp (90 MB): the bench's path
    n, L = 300_000, 150
    q = rng.integers(0, 4, (n, L), dtype=np.uint8)
    s = q.copy()
    mut = rng.random((n, L)) < 0.1
    s[mut] = rng.integers(0, 4, int(mut.sum()), dtype=np.uint8)
    idx = np.arange(n, dtype=np.int32)
    pairs = np.stack([idx, idx], 1)
    for flagged in (False, True):
        if flagged:   # first piece, a middle piece, the very last symbol
            q[5, 7] = 4; s[n // 2 + 3, 1] = 4; s[n - 1, L - 1] = 4
        pq, ps = W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s)
        for cfg in (W.AlignConfig("local", "affine"), W.AlignConfig("semiglobal", "affine", "traceback")):
            plain = run(pq, ps, pairs, cfg, 0)
            packed = run(pq, ps, pairs, cfg, 5)   # an odd thread count: slices of unequal size
            same(plain, packed, (flagged, cfg.align_type))
            assert plain.h2d_bytes >= 2 * n * L
            if not flagged:
                assert 2 * n * L // 4 <= packed.h2d_bytes <= plain.h2d_bytes // 4 + 4096
            else:
                assert packed.h2d_bytes < plain.h2d_bytes
        if not flagged:
            sample = np.sort(rng.choice(n, 2000, replace=False)).astype(np.int32)
            off = np.arange(n, dtype=np.int64) * L
            ln = np.full(n, L, np.int32)
            want, wi, wj = oracle.score_batch(q.reshape(-1), off, ln, s.reshape(-1), off, ln, sample, sample, "local", True,
                                              scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend)
            got = run(pq, ps, pairs, W.AlignConfig("local", "affine"), -1).results
            assert (got.score[sample] == want).all() and (got.q_end[sample] == wi).all() and (got.s_end[sample] == wj).all()

    # 2. ragged pools with explicit offsets: 270 k pairs of 101..163 symbols, piece boundaries inside packed bytes
    n = 270_000
    ql = rng.integers(101, 164, n).astype(np.int32)
    sl = rng.integers(101, 164, n).astype(np.int32)
    qo = np.zeros(n, np.int64); qo[1:] = np.cumsum(ql[:-1])
    so = np.zeros(n, np.int64); so[1:] = np.cumsum(sl[:-1])
    qc = rng.integers(0, 4, int(ql.sum()), dtype=np.uint8)
    sc = rng.integers(0, 4, int(sl.sum()), dtype=np.uint8)
    idx = np.arange(n, dtype=np.int32)
    pairs = np.stack([idx, idx], 1)
    for flagged in (False, True):
        if flagged:
            sc[int(so[n // 8 * 3]) - 1] = 4    # the last symbol before a boundary region
            qc[int(qo[n // 2]) + 2] = 4
        pq, ps = W.SequencePool(qc, qo, ql), W.SequencePool(sc, so, sl)
        for cfg in (W.AlignConfig("global", "affine"), W.AlignConfig("local", "affine")):
            plain = run(pq, ps, pairs, cfg, 0)
            packed = run(pq, ps, pairs, cfg, 16)
            same(plain, packed, ("ragged", flagged, cfg.align_type))
            assert packed.h2d_bytes < plain.h2d_bytes
    get_context(0).set_host_pack_threads(-1)
