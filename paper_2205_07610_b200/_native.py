"""ctypes binding of libwsb200.so (include/wsb200.h).  There is no CPU fallback: if the library is missing or no
CUDA device is present, every compute entry point raises DeviceError."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .core import DeviceError, LengthOverflow, PackedRangeOverflow, WaveseqError

_LIB_PATH = os.environ.get("WSB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwsb200.so")  # WSB_LIB: tuning aid
_lib = None

ALIGN_TYPE_ID = {"global": 0, "local": 1, "semiglobal": 2}
GAP_MODEL_ID = {"linear": 0, "affine": 1}
VARIANT_ID = {"auto": 0, "f16x2": 1, "i32": 2, "s16x2": 3}

WSB_OK, WSB_E_CUDA, WSB_E_ARG, WSB_E_NOMEM, WSB_E_LENGTH, WSB_E_RANGE, WSB_E_SCHEME, WSB_E_CAPACITY, WSB_E_NODEVICE = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)

EXPORTED_SYMBOLS = (
    "wsb_strerror", "wsb_version", "wsb_device_count", "wsb_ctx_create", "wsb_ctx_destroy", "wsb_last_error",
    "wsb_ctx_sm_count", "wsb_batch_create", "wsb_batch_create_async", "wsb_batch_create_packed_async", "wsb_batch_create_uniform_async", "wsb_batch_destroy", "wsb_batch_score", "wsb_batch_fetch_scores",
    "wsb_batch_traceback", "wsb_batch_fetch_traceback", "wsb_batch_total_cells", "wsb_score_batch",
    "wsb_traceback_batch", "wsb_merged_state_exact", "wsb_f16_range_ok", "wsb_plan_shards", "wsb_batch_has_faults", "wsb_pinned_alloc",
    "wsb_pinned_free", "wsb_batch_total_runs", "wsb_batch_h2d_bytes", "wsb_compact_pool", "wsb_batch_kernel_cycles",
    "wsb_batch_set_tb_scratch", "wsb_batch_tb_info", "wsb_batch_plan_stats", "wsb_batch_score_fetch",
    "wsb_ctx_set_host_pack_threads", "wsb_host_pack_isa",
)


class SchemeStruct(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32), ("gap_open", ctypes.c_int32),
                ("gap_extend", ctypes.c_int32), ("gap_model", ctypes.c_int32)]


def lib_path() -> str:
    return _LIB_PATH


def load():
    """Load the shared library (no GPU needed for loading or for the host-only helpers)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise DeviceError(f"{_LIB_PATH} is missing: build it with `python -m paper_2205_07610_b200.build` "
                          "(there is no CPU fallback)")
    # upload, download, compute and the launch-group streams of a context should not share hardware connections (default 8
    # per process); takes effect when CUDA has not been initialised yet in this process
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    lib = ctypes.CDLL(_LIB_PATH)
    p, i32, i64, ci = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
    lib.wsb_strerror.restype = ctypes.c_char_p
    lib.wsb_strerror.argtypes = [ci]
    lib.wsb_version.restype = ctypes.c_char_p
    lib.wsb_last_error.restype = ctypes.c_char_p
    lib.wsb_last_error.argtypes = [p]
    lib.wsb_device_count.argtypes = [p]
    lib.wsb_ctx_create.argtypes = [ci, p]
    lib.wsb_ctx_destroy.argtypes = [p]
    lib.wsb_ctx_destroy.restype = None
    lib.wsb_ctx_sm_count.argtypes = [p]
    lib.wsb_ctx_set_host_pack_threads.argtypes = [p, ci]
    lib.wsb_host_pack_isa.restype = ctypes.c_char_p
    lib.wsb_batch_create.argtypes = [p, p, p, p, i64, p, p, p, i64, p, p, i64, p]
    lib.wsb_batch_create_async.argtypes = [p, p, p, p, i64, p, p, p, i64, p, p, i64, p]
    lib.wsb_batch_create_packed_async.argtypes = [p, p, p, i64, p, p, i64, p, p, i64, p, p, i64, p, p, i64, p]
    lib.wsb_batch_create_uniform_async.argtypes = [p, p, p, i32, p, p, i32, i64, p]
    lib.wsb_batch_destroy.argtypes = [p]
    lib.wsb_batch_destroy.restype = None
    lib.wsb_batch_score.argtypes = [p, p, ci, ci, p, p]
    lib.wsb_batch_fetch_scores.argtypes = [p, p, p, p, p]
    lib.wsb_batch_score_fetch.argtypes = [p, p, ci, ci, p, p, p, p, p, p]
    lib.wsb_batch_traceback.argtypes = [p, p, ci, p, p]
    lib.wsb_batch_fetch_traceback.argtypes = [p, p, p, p, p, p, p, i64, p, p]
    lib.wsb_batch_total_cells.argtypes = [p]
    lib.wsb_batch_total_cells.restype = i64
    lib.wsb_score_batch.argtypes = [p, p, ci, ci, p, p, p, i64, p, p, p, i64, p, p, i64, p, p, p, p]
    lib.wsb_traceback_batch.argtypes = [p, p, ci, p, p, p, i64, p, p, p, i64, p, p, i64, p, p, p, p, p, p, i64, p, p]
    lib.wsb_batch_has_faults.argtypes = [p]
    lib.wsb_batch_h2d_bytes.argtypes = [p]
    lib.wsb_batch_h2d_bytes.restype = i64
    lib.wsb_batch_total_runs.argtypes = [p]
    lib.wsb_batch_total_runs.restype = i64
    lib.wsb_batch_set_tb_scratch.argtypes = [p, i64]
    lib.wsb_batch_tb_info.argtypes = [p, p]
    lib.wsb_batch_plan_stats.argtypes = [p, p]
    lib.wsb_pinned_alloc.argtypes = [ctypes.c_size_t, p]
    lib.wsb_pinned_free.argtypes = [p]
    lib.wsb_pinned_free.restype = None
    lib.wsb_merged_state_exact.argtypes = [p]
    lib.wsb_f16_range_ok.argtypes = [p, i32, i32]
    lib.wsb_plan_shards.argtypes = [p, p, p, p, i64, i32, p, p]
    _lib = lib
    return lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def zeros_view(n: int) -> np.ndarray:
    """n int32 zeros that cost nothing: a read-only broadcast of one element (numpy zero-fills a real 16 MB array, ~2 ms per
    4 M pairs -- the per-pair status of a batch without faults is only ever read)."""
    return np.broadcast_to(np.zeros(1, np.int32), (int(n),))


def pinned_empty(n: int, dtype=np.int32) -> np.ndarray:
    """Uninitialised array in page-locked host memory from the library's block cache; the block goes back to the
    cache when the array (and every view of it) is garbage collected."""
    import weakref
    lib = load()
    dt = np.dtype(dtype)
    nbytes = max(int(n) * dt.itemsize, 1)
    ptr = ctypes.c_void_p()
    if lib.wsb_pinned_alloc(nbytes, ctypes.byref(ptr)) != WSB_OK or not ptr.value:
        return np.empty(n, dt)  # no pinned memory to be had: a pageable array still works, only slower
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    weakref.finalize(buf, lib.wsb_pinned_free, ptr.value)
    return np.frombuffer(buf, dtype=dt, count=int(n))


def scheme_struct(scheme) -> SchemeStruct:
    return SchemeStruct(int(scheme.match_score), int(scheme.mismatch_score), int(scheme.gap_open),
                        int(scheme.gap_extend), GAP_MODEL_ID[scheme.gap_model])


def status_exception(status: int, detail: str = "") -> Exception:
    msg = load().wsb_strerror(status).decode()
    if detail:
        msg = f"{msg}: {detail}"
    if status == WSB_E_LENGTH:
        return LengthOverflow(msg)
    if status == WSB_E_RANGE:
        return PackedRangeOverflow(msg)
    if status in (WSB_E_ARG, WSB_E_SCHEME):
        return ValueError(msg)
    if status == WSB_E_NOMEM:
        return MemoryError(msg)
    if status in (WSB_E_CUDA, WSB_E_NODEVICE):
        return DeviceError(msg)
    return WaveseqError(msg)


def device_count() -> int:
    n = ctypes.c_int(0)
    load().wsb_device_count(ctypes.byref(n))
    return n.value


def merged_state_exact(scheme) -> bool:
    s = scheme_struct(scheme)
    return bool(load().wsb_merged_state_exact(ctypes.byref(s)))


def f16_range_ok(scheme, m: int, n: int) -> bool:
    s = scheme_struct(scheme)
    return bool(load().wsb_f16_range_ok(ctypes.byref(s), int(m), int(n)))


def plan_shards(q_len, s_len, pair_q, pair_s, n_shards: int):
    q_len = np.ascontiguousarray(q_len, np.int32); s_len = np.ascontiguousarray(s_len, np.int32)
    pair_q = np.ascontiguousarray(pair_q, np.int32); pair_s = np.ascontiguousarray(pair_s, np.int32)
    shard_of = np.zeros(len(pair_q), np.int32)
    cells = np.zeros(n_shards, np.int64)
    rc = load().wsb_plan_shards(_ptr(q_len), _ptr(s_len), _ptr(pair_q), _ptr(pair_s), len(pair_q), n_shards,
                                _ptr(shard_of), _ptr(cells))
    if rc:
        raise status_exception(rc)
    return shard_of, cells


def compact_pool(codes, off, lengths, ids):
    """(codes, off) of the pool made of sequences `ids` only, in that order (wsb_compact_pool; host memory, no GPU)."""
    codes = np.ascontiguousarray(codes, np.uint8); off = np.ascontiguousarray(off, np.int64)
    lengths = np.ascontiguousarray(lengths, np.int32); ids = np.ascontiguousarray(ids, np.int64)
    total = int(lengths[ids].astype(np.int64).sum()) if len(ids) else 0
    out_codes = np.empty(max(total, 1), np.uint8)
    out_off = np.zeros(len(ids), np.int64)
    lib = load()
    lib.wsb_compact_pool.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    rc = lib.wsb_compact_pool(_ptr(codes), _ptr(off), _ptr(lengths), _ptr(ids), len(ids), _ptr(out_codes), _ptr(out_off))
    if rc:
        raise status_exception(rc)
    return out_codes, out_off


class Context:
    """One per GPU (wsb_ctx): owns the stream, events and scratch.  Not re-entrant."""

    def __init__(self, device: int = 0):
        self._lib = load()
        h = ctypes.c_void_p()
        rc = self._lib.wsb_ctx_create(int(device), ctypes.byref(h))
        if rc:
            raise status_exception(rc, f"device {device}")
        self._h = h
        self.device = device

    @property
    def sm_count(self) -> int:
        return int(self._lib.wsb_ctx_sm_count(self._h))

    def last_error(self) -> str:
        return self._lib.wsb_last_error(self._h).decode()

    def set_host_pack_threads(self, threads: int) -> None:
        """Host threads that pack large byte pools into the 2-bit layout before upload (0: off, -1: library default)."""
        rc = self._lib.wsb_ctx_set_host_pack_threads(self._h, int(threads))
        if rc:
            raise status_exception(rc, "host_pack_threads")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wsb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Batch:
    """Device-resident pools + pair list (wsb_batch)."""

    _h2d_final = 0

    @property
    def h2d_bytes(self) -> int:
        """Bytes that crossed the bus for this batch so far (regular metadata is generated on the device; host-packed
        pools count as packed).  Final once the first score / traceback call has returned."""
        return int(self._lib.wsb_batch_h2d_bytes(self._h)) if getattr(self, "_h", None) else self._h2d_final

    def __init__(self, ctx: Context, q_codes, q_off, q_len, s_codes, s_off, s_len, pair_q, pair_s, packed=None):
        """packed = ((q_packed, q_flag_pos), (s_packed, s_flag_pos)): both pools in the 2-bit layout (four symbols per
        byte, low bits first over the concatenated pool) plus the positions of flagged symbols; q_codes / s_codes are
        then ignored (may be None)."""
        self._lib = load()
        self.ctx = ctx
        meta = [np.ascontiguousarray(q_off, np.int64), np.ascontiguousarray(q_len, np.int32),
                np.ascontiguousarray(s_off, np.int64), np.ascontiguousarray(s_len, np.int32),
                np.ascontiguousarray(pair_q, np.int32), np.ascontiguousarray(pair_s, np.int32)]
        self.n_pairs = len(meta[4])
        h = ctypes.c_void_p()
        if packed is None:
            pools = [np.ascontiguousarray(q_codes, np.uint8), np.ascontiguousarray(s_codes, np.uint8)]
            self._keep = pools + meta  # the upload is asynchronous: the arrays must outlive it (released in close())
            rc = self._lib.wsb_batch_create_async(ctx._h, _ptr(pools[0]), _ptr(meta[0]), _ptr(meta[1]), len(meta[1]),
                                                  _ptr(pools[1]), _ptr(meta[2]), _ptr(meta[3]), len(meta[3]),
                                                  _ptr(meta[4]), _ptr(meta[5]), self.n_pairs, ctypes.byref(h))
        else:
            (qp, qf), (sp, sf) = packed
            pools = [np.ascontiguousarray(qp, np.uint8), np.ascontiguousarray(sp, np.uint8),
                     np.ascontiguousarray(qf if qf is not None else [], np.int64),
                     np.ascontiguousarray(sf if sf is not None else [], np.int64)]
            self._keep = pools + meta
            rc = self._lib.wsb_batch_create_packed_async(
                ctx._h, _ptr(pools[0]), _ptr(pools[2]) if len(pools[2]) else None, len(pools[2]), _ptr(meta[0]), _ptr(meta[1]),
                len(meta[1]), _ptr(pools[1]), _ptr(pools[3]) if len(pools[3]) else None, len(pools[3]), _ptr(meta[2]),
                _ptr(meta[3]), len(meta[3]), _ptr(meta[4]), _ptr(meta[5]), self.n_pairs, ctypes.byref(h))
        if rc:
            self._keep = None
            raise status_exception(rc, ctx.last_error())
        self._h = h

    @classmethod
    def uniform(cls, ctx: Context, q_pool, q_len: int, s_pool, s_len: int, n_pairs: int, packed: bool = False) -> "Batch":
        """Regular batch (wsb_batch_create_uniform_async): read i of either pool at i * length, pair i = (i, i); the pools
        are byte arrays or, with packed=True, 2-bit packed arrays without flagged symbols."""
        self = cls.__new__(cls)
        self._lib = load()
        self.ctx = ctx
        self.n_pairs = int(n_pairs)
        pools = [np.ascontiguousarray(q_pool, np.uint8), np.ascontiguousarray(s_pool, np.uint8)]
        self._keep = pools
        h = ctypes.c_void_p()
        qa = (None, _ptr(pools[0])) if packed else (_ptr(pools[0]), None)
        sa = (None, _ptr(pools[1])) if packed else (_ptr(pools[1]), None)
        rc = self._lib.wsb_batch_create_uniform_async(ctx._h, qa[0], qa[1], int(q_len), sa[0], sa[1], int(s_len),
                                                      self.n_pairs, ctypes.byref(h))
        if rc:
            self._keep = None
            raise status_exception(rc, ctx.last_error())
        self._h = h
        return self

    @property
    def kernel_cycles(self) -> int:
        """SM cycles of the last packed int16 short-read launch (0 when another kernel carried the batch)."""
        self._lib.wsb_batch_kernel_cycles.restype = ctypes.c_int64
        self._lib.wsb_batch_kernel_cycles.argtypes = [ctypes.c_void_p]
        return int(self._lib.wsb_batch_kernel_cycles(self._h))

    @property
    def total_cells(self) -> int:
        return int(self._lib.wsb_batch_total_cells(self._h))

    def score(self, scheme, align_type: str, variant: str = "auto", timed: bool = True):
        """Run the score kernels; returns (kernel_ms, launches).  Results stay on the device."""
        s = scheme_struct(scheme)
        ms = ctypes.c_float(0.0)
        nl = ctypes.c_int32(0)
        rc = self._lib.wsb_batch_score(self._h, ctypes.byref(s), ALIGN_TYPE_ID[align_type], VARIANT_ID[variant],
                                       ctypes.byref(ms) if timed else None, ctypes.byref(nl))
        if rc:
            raise status_exception(rc, self.ctx.last_error())
        return float(ms.value), int(nl.value)

    def score_fetch(self, scheme, align_type: str, variant: str = "auto", dest=None, timed: bool = True):
        """score() + fetch_scores() in one native call: the results of pieces that have finished travel back while later
        pieces are still uploading and running.  Returns (kernel_ms, launches, (score, end_i, end_j, status))."""
        n = self.n_pairs
        if dest is not None:
            score, ei, ej = dest
            assert all(a.dtype == np.int32 and a.flags.c_contiguous and len(a) == n for a in dest)
        else:
            # page-locked destinations from 1 024 pairs on: three downloads into pageable memory are staged one by one
            # (~15 us each), which is a third of a cfg1-sized call
            score, ei, ej = (pinned_empty(n) for _ in range(3)) if n >= 1024 else (np.empty(n, np.int32) for _ in range(3))
        s = scheme_struct(scheme)
        ms = ctypes.c_float(0.0)
        nl = ctypes.c_int32(0)
        rc = self._lib.wsb_batch_score_fetch(self._h, ctypes.byref(s), ALIGN_TYPE_ID[align_type], VARIANT_ID[variant],
                                             ctypes.byref(ms) if timed else None, ctypes.byref(nl), _ptr(score), _ptr(ei), _ptr(ej),
                                             None)
        if rc:
            raise status_exception(rc, self.ctx.last_error())
        self.has_faults = bool(self._lib.wsb_batch_has_faults(self._h))
        if self.has_faults:
            status = np.empty(n, np.int32)
            rc = self._lib.wsb_batch_fetch_scores(self._h, _ptr(score), _ptr(ei), _ptr(ej), _ptr(status))
            if rc:
                raise status_exception(rc, self.ctx.last_error())
        else:
            status = zeros_view(n)
        return float(ms.value), int(nl.value), (score, ei, ej, status)

    def fetch_scores(self, dest=None):
        """(score, end_i, end_j, status).  dest: three preallocated int32 arrays of n_pairs elements to download into (the
        multi-GPU runner passes slices of the job-wide result arrays, so shard results land in place)."""
        n = self.n_pairs
        big = n >= 65536
        if dest is not None:
            score, ei, ej = dest
            assert all(a.dtype == np.int32 and a.flags.c_contiguous and len(a) == n for a in dest)
        else:
            score, ei, ej = (pinned_empty(n) for _ in range(3)) if big else (np.empty(n, np.int32) for _ in range(3))
        # the per-pair status array only carries information when the plan recorded a fault
        self.has_faults = bool(self._lib.wsb_batch_has_faults(self._h))
        status = np.empty(n, np.int32) if self.has_faults else None
        rc = self._lib.wsb_batch_fetch_scores(self._h, _ptr(score), _ptr(ei), _ptr(ej), _ptr(status))
        if rc:
            raise status_exception(rc, self.ctx.last_error())
        if status is None:
            status = zeros_view(n)
        return score, ei, ej, status

    def plan_stats(self) -> dict:
        """Geometry counters of the last plan (stages, wavefront iterations, executed cell updates, instruction counts)."""
        out = (ctypes.c_int64 * 8)()
        rc = self._lib.wsb_batch_plan_stats(self._h, out)
        if rc:
            raise status_exception(rc, self.ctx.last_error())
        keys = ("stages", "iterations", "updates", "ops_max", "ops_addsub", "ops_lookup", "groups", "pairs")
        return {k: int(v) for k, v in zip(keys, out)}

    def set_tb_scratch(self, nbytes: int) -> None:
        """Direction-code scratch budget of this batch; pairs whose codes exceed it take the bounded-memory path."""
        rc = self._lib.wsb_batch_set_tb_scratch(self._h, int(nbytes))
        if rc:
            raise status_exception(rc, self.ctx.last_error())

    def tb_info(self) -> dict:
        """Counters of the bounded-memory path in the last traceback call."""
        out = (ctypes.c_int64 * 4)()
        rc = self._lib.wsb_batch_tb_info(self._h, out)
        if rc:
            raise status_exception(rc, self.ctx.last_error())
        return {"pairs": int(out[0]), "cells": int(out[1]), "tiles": int(out[2]), "peak_bytes": int(out[3])}

    def traceback(self, scheme, align_type: str, timed: bool = True):
        s = scheme_struct(scheme)
        ms = ctypes.c_float(0.0)
        nl = ctypes.c_int32(0)
        rc = self._lib.wsb_batch_traceback(self._h, ctypes.byref(s), ALIGN_TYPE_ID[align_type],
                                           ctypes.byref(ms) if timed else None, ctypes.byref(nl))
        if rc:
            raise status_exception(rc, self.ctx.last_error())
        return float(ms.value), int(nl.value)

    def fetch_traceback(self, cigar_cap: int | None = None):
        n = self.n_pairs
        big = n >= 65536
        alloc = pinned_empty if big else (lambda k, dt=np.int32: np.empty(k, dt))
        out = {k: alloc(n) for k in ("score", "q_start", "q_end", "s_start", "s_end")}
        self.has_faults = bool(self._lib.wsb_batch_has_faults(self._h))
        status = np.empty(n, np.int32) if self.has_faults else None
        off = alloc(n + 1, np.int64)
        total = int(self._lib.wsb_batch_total_runs(self._h))
        cap = int(cigar_cap) if cigar_cap is not None else max(total, 1)   # exact: one download, no retry
        cig = alloc(cap, np.uint32)
        rc = self._lib.wsb_batch_fetch_traceback(self._h, _ptr(out["score"]), _ptr(out["q_start"]), _ptr(out["q_end"]),
                                                 _ptr(out["s_start"]), _ptr(out["s_end"]), _ptr(cig), cap, _ptr(off),
                                                 _ptr(status))
        if rc:
            raise status_exception(rc, self.ctx.last_error())
        out["status"] = status if status is not None else zeros_view(n)
        out["cigar"] = cig[:int(off[n])]
        out["cigar_off"] = off
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._h2d_final = int(self._lib.wsb_batch_h2d_bytes(self._h))
            self._lib.wsb_batch_destroy(self._h)
            self._h = None
        self._keep = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
