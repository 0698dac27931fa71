"""CPU oracle for the batched pairwise-alignment hot path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may import this
package.  The product package (paper_2205_07610_b200) never does: it fails loudly when the CUDA library is missing.

The arithmetic lives in wsoracle.c, a plain-C restatement of the reference's full-matrix DP
(pkg/src/waveseq/refdp.py:44-235, engine.py:281-288 for empty sides).  Parity is pinned against the reference's
own frozen known-answer tests and against golden vectors produced by running the reference in the build container
(tests/golden/make_golden.py -> tests/golden/*.json, checked by tests/test_oracle.py).

Sequences are uint8 arrays, one byte per symbol: 0..3 = ACGT, 4 = flagged.  CIGAR runs come back as
[(op, length)] with op in "MID" (I consumes the query, D the subject).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libwsoracle.so")
_SRC_PATH = os.path.join(_HERE, "wsoracle.c")
_lib = None

ALIGN_TYPE_ID = {"global": 0, "local": 1, "semiglobal": 2}
OPS = "MID"


def build(force: bool = False) -> str:
    """Compile wsoracle.c into libwsoracle.so (gcc, OpenMP).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC_PATH):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, _SRC_PATH])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i32, i64, p = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        lib.ws_oracle_score.argtypes = [p, i32, p, i32, ctypes.c_int, ctypes.c_int, i32, i32, i32, i32, p, p, p]
        lib.ws_oracle_traceback.argtypes = [p, i32, p, i32, ctypes.c_int, ctypes.c_int, i32, i32, i32, i32,
                                            p, p, p, p, p, p, i64, p]
        lib.ws_oracle_score_batch.argtypes = [p, p, p, p, p, p, p, p, i64, ctypes.c_int, ctypes.c_int,
                                              i32, i32, i32, i32, p, p, p, ctypes.c_int]
        lib.ws_oracle_traceback_batch.argtypes = [p, p, p, p, p, p, p, p, i64, ctypes.c_int, ctypes.c_int,
                                                  i32, i32, i32, i32, p, p, p, p, p, p, i64, p, ctypes.c_int]
        lib.ws_oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(_load().ws_oracle_max_threads())


def ref_score(q, s, align_type: str, affine: bool, match: int, mismatch: int, alpha: int, beta: int):
    """(score, (i, j)) exactly as refdp.ref_score (refdp.py:151-155)."""
    lib = _load()
    q, s = _u8(q), _u8(s)
    out = np.zeros(3, np.int32)
    rc = lib.ws_oracle_score(_ptr(q), len(q), _ptr(s), len(s), ALIGN_TYPE_ID[align_type], int(affine),
                             match, mismatch, alpha, beta, _ptr(out[0:]), _ptr(out[1:]), _ptr(out[2:]))
    if rc:
        raise MemoryError("oracle allocation failed")
    return int(out[0]), (int(out[1]), int(out[2]))


def unpack_ops(packed: np.ndarray) -> list[tuple[str, int]]:
    return [(OPS[int(v) & 3], int(v) >> 2) for v in packed]


def ref_traceback(q, s, align_type: str, affine: bool, match: int, mismatch: int, alpha: int, beta: int):
    """dict(score, q_start, q_end, s_start, s_end, ops) exactly as refdp.ref_traceback (refdp.py:158-235)."""
    lib = _load()
    q, s = _u8(q), _u8(s)
    cap = len(q) + len(s) + 2
    ops = np.zeros(cap, np.uint32)
    out = np.zeros(5, np.int32)
    n_ops = np.zeros(1, np.int64)
    rc = lib.ws_oracle_traceback(_ptr(q), len(q), _ptr(s), len(s), ALIGN_TYPE_ID[align_type], int(affine),
                                 match, mismatch, alpha, beta, _ptr(out[0:]), _ptr(out[1:]), _ptr(out[2:]),
                                 _ptr(out[3:]), _ptr(out[4:]), _ptr(ops), cap, _ptr(n_ops))
    if rc:
        raise RuntimeError(f"oracle traceback failed rc={rc}")
    return dict(score=int(out[0]), q_start=int(out[1]), q_end=int(out[2]), s_start=int(out[3]),
                s_end=int(out[4]), ops=unpack_ops(ops[:int(n_ops[0])]))


def score_batch(q_codes, q_off, q_len, s_codes, s_off, s_len, pair_q, pair_s, align_type: str, affine: bool,
                match: int, mismatch: int, alpha: int, beta: int, threads: int = 0):
    """Batched ref_score over sequence pools; returns (score, end_i, end_j) int32 arrays."""
    lib = _load()
    q_codes, s_codes = _u8(q_codes), _u8(s_codes)
    q_off = np.ascontiguousarray(q_off, np.int64); s_off = np.ascontiguousarray(s_off, np.int64)
    q_len = np.ascontiguousarray(q_len, np.int32); s_len = np.ascontiguousarray(s_len, np.int32)
    pair_q = np.ascontiguousarray(pair_q, np.int32); pair_s = np.ascontiguousarray(pair_s, np.int32)
    n = len(pair_q)
    score = np.zeros(n, np.int32); ei = np.zeros(n, np.int32); ej = np.zeros(n, np.int32)
    threads = threads or max_threads()
    rc = lib.ws_oracle_score_batch(_ptr(q_codes), _ptr(q_off), _ptr(q_len), _ptr(s_codes), _ptr(s_off), _ptr(s_len),
                                   _ptr(pair_q), _ptr(pair_s), n, ALIGN_TYPE_ID[align_type], int(affine),
                                   match, mismatch, alpha, beta, _ptr(score), _ptr(ei), _ptr(ej), threads)
    if rc:
        raise MemoryError("oracle allocation failed")
    return score, ei, ej


def traceback_batch(q_codes, q_off, q_len, s_codes, s_off, s_len, pair_q, pair_s, align_type: str, affine: bool,
                    match: int, mismatch: int, alpha: int, beta: int, threads: int = 0, unpack: bool = True):
    """Batched ref_traceback; returns dict of int32 arrays plus a list of per-pair op lists (unpack=False: only the
    packed run words `ops_packed[n, stride]` with `n_ops[n]`, for array-wise comparison of large batches)."""
    lib = _load()
    q_codes, s_codes = _u8(q_codes), _u8(s_codes)
    q_off = np.ascontiguousarray(q_off, np.int64); s_off = np.ascontiguousarray(s_off, np.int64)
    q_len = np.ascontiguousarray(q_len, np.int32); s_len = np.ascontiguousarray(s_len, np.int32)
    pair_q = np.ascontiguousarray(pair_q, np.int32); pair_s = np.ascontiguousarray(pair_s, np.int32)
    n = len(pair_q)
    stride = int((q_len[pair_q].astype(np.int64) + s_len[pair_s]).max()) + 2 if n else 2
    ops = np.zeros((n, stride), np.uint32)
    n_ops = np.zeros(n, np.int32)
    outs = {k: np.zeros(n, np.int32) for k in ("score", "q_start", "q_end", "s_start", "s_end")}
    threads = threads or max_threads()
    rc = lib.ws_oracle_traceback_batch(_ptr(q_codes), _ptr(q_off), _ptr(q_len), _ptr(s_codes), _ptr(s_off),
                                       _ptr(s_len), _ptr(pair_q), _ptr(pair_s), n, ALIGN_TYPE_ID[align_type],
                                       int(affine), match, mismatch, alpha, beta, _ptr(outs["score"]),
                                       _ptr(outs["q_start"]), _ptr(outs["q_end"]), _ptr(outs["s_start"]),
                                       _ptr(outs["s_end"]), _ptr(ops), stride, _ptr(n_ops), threads)
    if rc:
        raise RuntimeError(f"oracle traceback batch failed rc={rc}")
    if unpack:
        outs["ops"] = [unpack_ops(ops[i, :n_ops[i]]) for i in range(n)]
    outs["ops_packed"] = ops
    outs["n_ops"] = n_ops
    return outs
