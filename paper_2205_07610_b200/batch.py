"""Batch runner: BatchJob -> GPU shards -> BatchReport.

Drop-in for the reference's thread-pool runner (pkg/src/waveseq/batch.py): same BatchJob / BatchReport / run_batch /
all_pairs / resolve_workers names, the same validation and error contract (BatchError carries the smallest failing
pair index, batch.py:179-180, 241-242) and results in per-pair slots, independent of scheduling (batch.py:206).

What replaces the worker pool: the pairs are sharded over the visible GPUs by cell count (native wsb_plan_shards,
longest-processing-time first), every shard runs on its own context / stream from its own host thread, and the shard
results are scattered back into the pair slots.  The shards share no state, so there is no collective.

Score-only results follow batch._score_result (batch.py:105-115).  Traceback results follow refdp.ref_traceback (the
full-matrix walk): see DESIGN.md "CIGAR oracle".
"""
from __future__ import annotations

import os
import threading
import time
from collections.abc import Sequence as _SequenceABC
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .core import (AlignConfig, AlignmentResult, BatchError, ScoringScheme, Sequence, validate_config)
from .engine import EngineTuning, get_context, packed_range_ok
from .io import unpack_runs
from .pool import SequencePool

CHUNK_PAIRS = 64  # kept for API compatibility; the GPU planner does its own bucketing


def resolve_workers(requested: int = 0) -> int:
    """WAVESEQ_WORKERS wins, then the request, then the CPU count (reference semantics; the GPU path only validates it)."""
    env = os.environ.get("WAVESEQ_WORKERS")
    if env is not None:
        try:
            w = int(env)
        except ValueError:
            raise ValueError(f"WAVESEQ_WORKERS must be an integer, got {env!r}") from None
    elif requested:
        w = requested
    else:
        w = os.cpu_count() or 1
    if w < 1:
        raise ValueError(f"worker count must be positive, got {w}")
    return w


def resolve_devices(requested=None) -> list[int]:
    """GPUs a batch is sharded over: explicit list / count, else WAVESEQ_DEVICES (count or comma list), else GPU 0."""
    if requested is None:
        env = os.environ.get("WAVESEQ_DEVICES")
        if env:
            requested = [int(x) for x in env.split(",")] if "," in env else int(env)
        else:
            requested = 1
    if isinstance(requested, int):
        if requested < 1:
            raise ValueError("device count must be positive")
        return list(range(requested))
    return [int(d) for d in requested]


def all_pairs(queries, subjects) -> list[tuple[int, int]]:
    """Cartesian product of index pairs, row-major."""
    if not len(queries) or not len(subjects):
        raise ValueError("both sequence lists must be non-empty")
    ns = len(subjects)
    return [(qi, si) for qi in range(len(queries)) for si in range(ns)]


@dataclass
class BatchJob:
    """Sequence pools (lists of Sequence or SequencePool), index pairs (list of tuples or (n, 2) array), config, scheme.

    tuning.packed=True forces the packed half2 kernel (pairs outside its range fail like the reference's packed mode
    would not: the reference silently runs them unpacked, batch.py:136-138, and so does this runner).  workers is
    accepted for compatibility.  devices (extension) picks the GPUs to shard over.
    """

    queries: object
    subjects: object
    pairs: object
    cfg: AlignConfig
    scheme: ScoringScheme
    tuning: EngineTuning | None = None
    workers: int = 0
    devices: object = None

    def __post_init__(self):
        if len(self.pairs) == 0:
            raise ValueError("pairs must be non-empty")
        arr = np.asarray(self.pairs)
        if arr.ndim != 2 or arr.shape[1] != 2:
            raise ValueError("pairs must be (query index, subject index) tuples")
        nq, ns = len(self.queries), len(self.subjects)
        bad = np.nonzero((arr[:, 0] < 0) | (arr[:, 0] >= nq) | (arr[:, 1] < 0) | (arr[:, 1] >= ns))[0]
        if len(bad):
            qi, si = arr[bad[0]]
            raise ValueError(f"pair ({int(qi)}, {int(si)}) is out of range")
        self._pair_array = np.ascontiguousarray(arr, np.int32)
        # the device wants the two index columns as separate contiguous arrays: split once, here
        self._pair_q = np.ascontiguousarray(self._pair_array[:, 0])
        self._pair_s = np.ascontiguousarray(self._pair_array[:, 1])
        # pair i = (i, i)?  (checked once here; lets run_batch take the metadata-free upload for uniform pools)
        n = len(self._pair_q)
        self._identity = bool(n and self._pair_q[0] == 0 and self._pair_q[-1] == n - 1 and
                              np.array_equal(self._pair_q, self._pair_s) and
                              np.array_equal(self._pair_q, np.arange(n, dtype=np.int32)))


class ResultArray(_SequenceABC):
    """results[i] belongs to pairs[i].  Backed by arrays; AlignmentResult objects are built on access so that batches of
    millions of pairs do not pay for millions of Python objects up front."""

    def __init__(self, score, q_start, q_end, s_start, s_end, cells, runs=None, run_off=None):
        self.score, self.q_start, self.q_end, self.s_start, self.s_end, self._cells = (
            score, q_start, q_end, s_start, s_end, cells)
        self.runs, self.run_off = runs, run_off

    @property
    def cells(self):
        """m * n per pair; computed on first use (a callable is stored until then)."""
        if callable(self._cells):
            self._cells = self._cells()
        return self._cells

    def __len__(self) -> int:
        return int(self.score.shape[0])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        ops = None
        if self.runs is not None:
            ops = unpack_runs(self.runs[int(self.run_off[i]):int(self.run_off[i + 1])])
        return AlignmentResult(score=int(self.score[i]), q_start=int(self.q_start[i]), q_end=int(self.q_end[i]),
                               s_start=int(self.s_start[i]), s_end=int(self.s_end[i]), ops=ops,
                               cells_computed=int(self.cells[i]))

    def __eq__(self, other):
        if isinstance(other, (list, ResultArray)):
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        return NotImplemented


@dataclass
class BatchReport:
    """results[i] belongs to pairs[i]; total_cells = sum of m*n over pairs; wall_time covers upload, kernels, download."""

    results: object
    wall_time: float
    total_cells: int
    kernel_ms: float = 0.0          # device time of the alignment kernels (max over shards)
    gpu_launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    shard_cells: list = field(default_factory=list)

    @property
    def gcups(self) -> float:
        return self.total_cells / max(self.wall_time, 1e-12) / 1e9


def plan_shards(queries: SequencePool, subjects: SequencePool, pair_array: np.ndarray, n_shards: int):
    """Cell-count balanced shard of every pair (native longest-processing-time planner)."""
    return N.plan_shards(queries.len, subjects.len, pair_array[:, 0], pair_array[:, 1], n_shards)


def _variant_for(job: BatchJob, cfg: AlignConfig) -> str:
    if job.tuning is not None and job.tuning.packed and cfg.result_mode == "score_only":
        return "auto"  # packed where exact, int32 elsewhere: the reference's _plan_units falls back the same way
    env = os.environ.get("WSB_VARIANT")
    return env if env in ("auto", "f16x2", "i32") else "auto"


def _host_pack_policy() -> int:
    """Host threads for the packed upload of a single-shard job: the library default (-1: min(16, cores)) when this process
    has the host to itself, 0 (plain uploads) when torchrun runs one rank per GPU on it -- every rank has its own PCIe link
    but they all share the cores.  Jobs sharded over several devices never pack (same reason).  WSB_HOST_PACK_THREADS overrides."""
    if os.environ.get("WSB_HOST_PACK_THREADS") is not None:
        return -1
    try:
        ranks = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    except ValueError:
        ranks = 1
    return -1 if ranks <= 1 else 0


def host_pack_info() -> dict:
    """What the packed upload of a single-shard job would use in this process: {"threads": default (-1), forced count or 0
    (off), "isa": packing body of the running CPU}."""
    env = os.environ.get("WSB_HOST_PACK_THREADS")
    return {"threads": int(env) if env is not None else _host_pack_policy(), "isa": N.load().wsb_host_pack_isa().decode(),
            "cores": os.cpu_count()}


def _run_shard(device: int, queries: SequencePool, subjects: SequencePool, pair_q: np.ndarray, pair_s: np.ndarray,
               cfg: AlignConfig, scheme: ScoringScheme, variant: str, out: dict, regular: bool = False, dest=None,
               host_pack: int = -1):
    try:
        ctx = get_context(device)
        ctx.set_host_pack_threads(host_pack)
        both_packed = queries.packed is not None and subjects.packed is not None
        no_flags = both_packed and not (queries.flag_pos is not None and len(queries.flag_pos)) and \
            not (subjects.flag_pos is not None and len(subjects.flag_pos))
        # (score-only jobs take it from 1 024 pairs on: the six metadata arrays of the general upload cost ~120 us per call,
        # more than the kernel of a cfg1-sized batch; tools/e2e_small_probe.py)
        small_ok = cfg.result_mode != "traceback" and len(pair_q) >= 1024 and min(queries.uniform_len or 0, subjects.uniform_len or 0) > 0
        if regular and (len(pair_q) >= 65536 or small_ok) and (no_flags or (queries.packed is None and subjects.packed is None)):
            # uniform pools, identity pairs: no offset / length / pair arrays at all
            batch = N.Batch.uniform(ctx, queries.packed if both_packed else queries.codes, queries.uniform_len,
                                    subjects.packed if both_packed else subjects.codes, subjects.uniform_len,
                                    len(pair_q), packed=both_packed)
        elif queries.packed is not None and subjects.packed is not None:   # 2-bit pools: a quarter of the bytes to upload
            batch = N.Batch(ctx, None, queries.off, queries.len, None, subjects.off, subjects.len, pair_q, pair_s,
                            packed=((queries.packed, queries.flag_pos), (subjects.packed, subjects.flag_pos)))
        else:
            batch = N.Batch(ctx, queries.codes, queries.off, queries.len, subjects.codes, subjects.off, subjects.len,
                            pair_q, pair_s)
        try:
            out["cells"] = batch.total_cells
            if cfg.result_mode == "traceback":
                out["ms"], out["launches"] = batch.traceback(scheme, cfg.align_type)
                out["tb"] = batch.fetch_traceback()
                out["faults"] = batch.has_faults
            else:
                out["ms"], out["launches"], out["scores"] = batch.score_fetch(scheme, cfg.align_type, variant, dest)
                out["faults"] = batch.has_faults
            out["h2d"] = batch.h2d_bytes   # read after the run: a host-packed upload counts its bytes as the pieces are queued
        finally:
            batch.close()
    except BaseException as exc:  # re-raised by the caller in the submitting thread
        out["error"] = exc


def _run_sliced_shard(device: int, queries: SequencePool, subjects: SequencePool, pair_q: np.ndarray, pair_s: np.ndarray,
                      idx: np.ndarray, regular: bool, cfg: AlignConfig, scheme: ScoringScheme, variant: str, out: dict,
                      dest=None):
    """One GPU's share of a multi-GPU job: the pools are cut down to what the shard's pairs reference before anything is
    uploaded (a contiguous block of a reads matrix is a zero-copy slice; an arbitrary pair list is gathered into compact
    pools with remapped indices; a shard that references most of a pool anyway takes it whole)."""
    try:
        if regular:
            lo, hi = int(idx[0]), int(idx[-1]) + 1
            q_sub, s_sub = queries.slice_uniform(lo, hi), subjects.slice_uniform(lo, hi)
            ident = np.arange(hi - lo, dtype=np.int32)
            return _run_shard(device, q_sub, s_sub, ident, ident, cfg, scheme, variant, out, True, dest, host_pack=0)
        pq, ps = pair_q[idx], pair_s[idx]

        def cut(pool, col):
            used, inv = np.unique(col, return_inverse=True)
            if len(used) * 4 > len(pool) * 3:
                return pool, col
            return pool.subset(used), inv.astype(np.int32)
        q_sub, pq = cut(queries, pq)
        s_sub, ps = cut(subjects, ps)
        _run_shard(device, q_sub, s_sub, np.ascontiguousarray(pq, np.int32), np.ascontiguousarray(ps, np.int32), cfg, scheme,
                   variant, out, False, host_pack=0)
    except BaseException as exc:
        out["error"] = exc


def run_batch(job: BatchJob) -> BatchReport:
    """Align every pair of the job on the GPU(s); results keep the pairs' order.

    A failing pair aborts the batch with BatchError carrying its index (the smallest one if several fail).
    """
    cfg = validate_config(job.cfg, job.scheme)
    resolve_workers(job.workers)
    devices = resolve_devices(job.devices)
    queries = SequencePool.from_sequences(job.queries)
    subjects = SequencePool.from_sequences(job.subjects)
    pairs = job._pair_array
    pair_q, pair_s = job._pair_q, job._pair_s
    n = len(pairs)
    variant = _variant_for(job, cfg)
    lens = {}

    def pair_lengths():  # per-pair (m, n) as int64, only materialised when something needs them
        if not lens:
            lens["m"] = queries.len.take(pair_q).astype(np.int64)
            lens["n"] = subjects.len.take(pair_s).astype(np.int64)
        return lens["m"], lens["n"]

    t0 = time.perf_counter()
    regular = (job._identity and queries.uniform_len is not None and subjects.uniform_len is not None and
               n <= len(queries) and n <= len(subjects))
    if len(devices) == 1:
        shard_index = [np.arange(n) if cfg.result_mode == "traceback" else range(n)]
        shard_cells = []
    elif regular:   # a reads matrix: contiguous blocks (whole packed units, whole 2-bit bytes), no planner pass
        cuts = [min(n, (n * k // len(devices) + 2047) // 2048 * 2048) for k in range(len(devices))] + [n]
        shard_index = [np.arange(cuts[k], cuts[k + 1]) for k in range(len(devices))]
        shard_cells = [int(len(ix)) * queries.uniform_len * subjects.uniform_len for ix in shard_index]
    else:
        shard_of, sc = N.plan_shards(queries.len, subjects.len, pair_q, pair_s, len(devices))
        shard_index = [np.nonzero(shard_of == k)[0] for k in range(len(devices))]
        shard_cells = [int(x) for x in sc]
    outs = [dict() for _ in devices]
    threads = []
    # contiguous shards of a score-only job download straight into their block of the job-wide (page-locked) result arrays
    in_place = len(devices) > 1 and regular and cfg.result_mode != "traceback" and n >= 65536
    whole = tuple(N.pinned_empty(n) for _ in range(3)) if in_place else None
    for dev, idx, out in zip(devices, shard_index, outs):
        if len(idx) == 0:
            continue
        if len(devices) == 1:  # no thread hop for the common single-GPU case
            _run_shard(dev, queries, subjects, pair_q, pair_s, cfg, job.scheme, variant, out, regular, host_pack=_host_pack_policy())
            continue
        dest = tuple(a[int(idx[0]):int(idx[-1]) + 1] for a in whole) if in_place else None
        th = threading.Thread(target=_run_sliced_shard, name=f"waveseq-gpu-{dev}",
                              args=(dev, queries, subjects, pair_q, pair_s, idx, regular, cfg, job.scheme, variant, out, dest))
        threads.append(th)
        th.start()
    for th in threads:
        th.join()
    wall = time.perf_counter() - t0
    for out in outs:
        if "error" in out:
            raise out["error"]

    single = len(devices) == 1
    runs = run_off = None
    if single and cfg.result_mode != "traceback":  # one shard: the fetched arrays are the result arrays
        score, qe, se, status = outs[0]["scores"]
        if cfg.align_type == "global":   # the kernels report (m, n) as the end cell
            qs = N.zeros_view(n); ss = qs
        else:
            qs, ss = qe, se
    elif in_place:
        score, qe, se = whole
        qs = ss = None
        status = None
    else:
        score = np.empty(n, np.int32); qs = np.zeros(n, np.int32); qe = np.empty(n, np.int32)
        ss = np.zeros(n, np.int32); se = np.empty(n, np.int32); status = np.zeros(n, np.int32)
    if single and cfg.result_mode != "traceback":
        pass
    elif cfg.result_mode == "traceback" and single:   # one shard: the fetched arrays are the result arrays
        tb = outs[0]["tb"]
        score, qs, qe, ss, se, status = tb["score"], tb["q_start"], tb["q_end"], tb["s_start"], tb["s_end"], tb["status"]
        runs, run_off = tb["cigar"], tb["cigar_off"]
    elif cfg.result_mode == "traceback":
        counts = np.zeros(n, np.int64)
        for idx, out in zip(shard_index, outs):
            if len(idx) == 0:
                continue
            tb = out["tb"]
            score[idx], qs[idx], qe[idx], ss[idx], se[idx], status[idx] = (
                tb["score"], tb["q_start"], tb["q_end"], tb["s_start"], tb["s_end"], tb["status"])
            counts[idx] = np.diff(tb["cigar_off"])
        run_off = np.zeros(n + 1, np.int64)
        np.cumsum(counts, out=run_off[1:])
        runs = np.empty(int(run_off[-1]), np.uint32)
        for idx, out in zip(shard_index, outs):
            if len(idx) == 0:
                continue
            tb = out["tb"]
            # shard run k of pair idx[j] goes to run_off[idx[j]] + (k - shard offset of that pair): one fancy-index store
            src_off = tb["cigar_off"]
            shift = np.repeat(run_off[idx] - src_off[:-1], np.diff(src_off))
            runs[shift + np.arange(len(shift), dtype=np.int64)] = tb["cigar"][:len(shift)]
    elif in_place:   # the shards wrote their blocks themselves; the status array exists only if a shard reported faults
        if any(o.get("faults", False) for o in outs if o):
            status = np.zeros(n, np.int32)
            for idx, out in zip(shard_index, outs):
                if len(idx):
                    status[int(idx[0]):int(idx[-1]) + 1] = out["scores"][3]
        else:
            status = N.zeros_view(n)
        if cfg.align_type == "global":
            qs = N.zeros_view(n); ss = qs
        else:
            qs, ss = qe, se
    else:
        for idx, out in zip(shard_index, outs):
            if len(idx) == 0:
                continue
            sc_, ei, ej, st = out["scores"]
            # contiguous shards (reads matrices) land with four block copies; index arrays only for planner-made shards
            at = slice(int(idx[0]), int(idx[-1]) + 1) if int(idx[-1]) - int(idx[0]) + 1 == len(idx) else idx
            score[at], qe[at], se[at], status[at] = sc_, ei, ej, st
        if cfg.align_type != "global":  # start is unknown without a traceback pass: both span ends carry the argmax cell (batch.py:111-115)
            qs, ss = qe, se
    any_fault = any(o.get("faults", True) for o in outs if o)
    bad = np.nonzero(status)[0] if any_fault else ()
    if len(bad):
        i = int(bad[0])
        m_arr, n_arr = pair_lengths()
        raise BatchError(i, N.status_exception(int(status[i]), f"problem of size {int(m_arr[i])}x{int(n_arr[i])}"))

    def cell_counts():
        m_arr, n_arr = pair_lengths()
        return m_arr * n_arr

    results = ResultArray(score, qs, qe, ss, se, cell_counts, runs, run_off)
    if n <= 4096:  # small batches: a plain list like the reference's; larger ones stay array-backed (same Sequence API)
        results = list(results)
    # bytes actually downloaded: score + end cell (+ starts and run offsets in traceback mode, + status only on faults)
    words = (5 if cfg.result_mode == "traceback" else 3) + (1 if any_fault else 0)
    d2h = sum(4 * words * len(idx) for idx in shard_index)
    if runs is not None:
        d2h += runs.nbytes + 8 * (n + 1)
    if not shard_cells:
        shard_cells = [int(outs[0].get("cells", 0))]
    return BatchReport(results=results, wall_time=wall, total_cells=int(sum(o.get("cells", 0) for o in outs)),
                       kernel_ms=max((o.get("ms", 0.0) for o in outs), default=0.0),
                       gpu_launches=sum(o.get("launches", 0) for o in outs),
                       h2d_bytes=sum(o.get("h2d", 0) for o in outs), d2h_bytes=d2h, shard_cells=shard_cells)
