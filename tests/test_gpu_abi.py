"""The one-shot C ABI exactly as INTEGRATION.md section 1 binds it (wsb_score_batch / wsb_traceback_batch through raw
ctypes, no helper classes), the TSV writer that reads the device's run buffer, and the reference-style bench report."""
import ctypes
import json

import numpy as np
import pytest

import oracle
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N
from conftest import random_codes, mutate_codes

pytestmark = pytest.mark.gpu


class _Scheme(ctypes.Structure):   # struct wsb_scheme, as in INTEGRATION.md
    _fields_ = [(n, ctypes.c_int32) for n in ("match", "mismatch", "gap_open", "gap_extend", "gap_model")]


_ATYPE = {"global": 0, "local": 1, "semiglobal": 2}
_p = lambda a: a.ctypes.data_as(ctypes.c_void_p)


@pytest.fixture(scope="module")
def raw():
    lib = ctypes.CDLL(N._LIB_PATH)
    lib.wsb_strerror.restype = ctypes.c_char_p
    ctx = ctypes.c_void_p()
    assert lib.wsb_ctx_create(0, ctypes.byref(ctx)) == 0
    yield lib, ctx
    lib.wsb_ctx_destroy(ctx)


def _pools(rng, n, lo=20, hi=400):
    qs = [random_codes(rng, int(rng.integers(lo, hi))) for _ in range(n)]
    ss = [mutate_codes(rng, q) if i % 2 else random_codes(rng, int(rng.integers(lo, hi))) for i, q in enumerate(qs)]
    qs[3] = qs[3].copy(); qs[3][5] = 4          # flagged symbols ride along
    ss[4] = ss[4].copy(); ss[4][7] = 4
    def pool(seqs):
        lens = np.array([len(s) for s in seqs], np.int32)
        off = np.concatenate([[0], np.cumsum(lens[:-1])]).astype(np.int64)
        return np.concatenate(seqs).astype(np.uint8), off, lens
    return pool(qs), pool(ss)


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_wsb_score_batch_one_shot(raw, align_type):
    lib, ctx = raw
    rng = np.random.default_rng(91)
    (qc, qo, ql), (sc, so, sl) = _pools(rng, 300)
    pq = rng.integers(0, 300, 1000).astype(np.int32); ps = rng.integers(0, 300, 1000).astype(np.int32)   # not the identity
    n = len(pq)
    score, ei, ej, st = (np.empty(n, np.int32) for _ in range(4))
    sch = _Scheme(2, -1, 2, 1, 1)
    rc = lib.wsb_score_batch(ctx, ctypes.byref(sch), _ATYPE[align_type], 0, _p(qc), _p(qo), _p(ql),
                             ctypes.c_int64(len(ql)), _p(sc), _p(so), _p(sl), ctypes.c_int64(len(sl)), _p(pq), _p(ps),
                             ctypes.c_int64(n), _p(score), _p(ei), _p(ej), _p(st))
    assert rc == 0, lib.wsb_strerror(rc)
    want = oracle.score_batch(qc, qo, ql, sc, so, sl, pq, ps, align_type, True, 2, -1, 2, 1)
    assert not st.any()
    assert (score == want[0]).all() and (ei == want[1]).all() and (ej == want[2]).all()


@pytest.mark.parametrize("align_type", ["global", "local", "semiglobal"])
def test_wsb_traceback_batch_one_shot_with_capacity_retry(raw, align_type):
    lib, ctx = raw
    rng = np.random.default_rng(92)
    (qc, qo, ql), (sc, so, sl) = _pools(rng, 120, hi=300)
    pq = np.arange(120, dtype=np.int32); ps = np.roll(pq, 1) if align_type == "local" else pq.copy()
    n = len(pq)
    outs = {k: np.empty(n, np.int32) for k in ("score", "q_start", "q_end", "s_start", "s_end", "status")}
    off = np.empty(n + 1, np.int64)
    sch = _Scheme(2, -1, 2, 1, 1)

    def call(cap):
        cigar = np.empty(max(cap, 1), np.uint32)
        rc = lib.wsb_traceback_batch(ctx, ctypes.byref(sch), _ATYPE[align_type], _p(qc), _p(qo), _p(ql),
                                     ctypes.c_int64(len(ql)), _p(sc), _p(so), _p(sl), ctypes.c_int64(len(sl)), _p(pq), _p(ps),
                                     ctypes.c_int64(n), _p(outs["score"]), _p(outs["q_start"]), _p(outs["q_end"]),
                                     _p(outs["s_start"]), _p(outs["s_end"]), _p(cigar), ctypes.c_int64(cap), _p(off),
                                     _p(outs["status"]))
        return rc, cigar

    rc, _ = call(8)                      # far too small: the call reports it and cigar_off[n] says what is needed
    assert rc == N.WSB_E_CAPACITY, lib.wsb_strerror(rc)
    need = int(off[n])
    assert need > 8
    rc, cigar = call(need)
    assert rc == 0, lib.wsb_strerror(rc)
    ref = oracle.traceback_batch(qc, qo, ql, sc, so, sl, pq, ps, align_type, True, 2, -1, 2, 1)
    for key in ("score", "q_start", "q_end", "s_start", "s_end"):
        assert (outs[key] == ref[key]).all(), key
    for k in range(n):
        assert W.io.unpack_runs(cigar[off[k]:off[k + 1]]) == ref["ops"][k], k


def _job(rng, n, mode):
    text = lambda codes: "".join("ACGT"[int(c)] for c in codes)
    qc = [random_codes(rng, int(rng.integers(40, 200))) for _ in range(n)]
    qs = [W.encode_sequence(f"q{i}", text(c)) for i, c in enumerate(qc)]
    ss = [W.encode_sequence(f"s{i}", text(mutate_codes(rng, c))) for i, c in enumerate(qc)]
    pairs = [(i, i) for i in range(n)]
    return W.BatchJob(qs, ss, pairs, W.AlignConfig("semiglobal", "affine", mode), W.ScoringScheme(2, -1, 2, 1, "affine"))


def test_write_batch_tsv_equals_write_results_tsv(tmp_path):
    rng = np.random.default_rng(93)
    job = _job(rng, 64, "traceback")
    rep = W.run_batch(job)
    qid = [f"q{i}" for i in range(64)]; sid = [f"s{i}" for i in range(64)]
    a, b = tmp_path / "a.tsv", tmp_path / "b.tsv"
    W.io.write_batch_tsv(rep.results, job.pairs, qid, sid, a)
    results = list(rep.results)             # AlignmentResult objects, the reference's shape
    W.io.write_results_tsv(((qid[q], sid[s], r) for (q, s), r in zip(job.pairs, results)), b)
    ta, tb = a.read_text(), b.read_text()
    assert ta == tb
    lines = ta.splitlines()
    assert lines[0].split("\t") == list(W.io.TSV_HEADER) and len(lines) == 65
    assert all(ln.split("\t")[7] for ln in lines[1:])      # traceback mode: every row carries a CIGAR


def test_measure_gcups_and_report_json():
    rng = np.random.default_rng(94)
    job = _job(rng, 200, "score_only")
    rep = W.bench.measure_gcups(job, 4, W.bench.HardwareModel.b200())
    assert rep.repetitions == 4 and rep.cells == sum(len(job.queries[q]) * len(job.subjects[s]) for q, s in job.pairs)
    assert rep.achieved_gcups > 0 and 0 < rep.efficiency < 1 and rep.extra_cells == 0
    keys = list(json.loads(rep.to_json()).keys())       # the reference's key order (tests/test_bench.py:87-93)
    assert keys == ["achieved_gcups", "tpp_gcups", "efficiency", "cells", "extra_cells", "wall_s", "repetitions", "workload",
                    "median_rule"]
    with pytest.raises(ValueError):
        W.bench.measure_gcups(job, 0)
