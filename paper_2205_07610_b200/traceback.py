"""Traceback entry points: alignments with operations, computed on the GPU.

The reference has two CPU traceback paths that agree on score but not always on the co-optimal path: the full-matrix
walk refdp.ref_traceback (refdp.py:158-235; diagonal, then I, then D; extension before open) and the linear-space
Hirschberg align_traceback (traceback.py:347-376), whose path-level output the reference's own tests do not pin
(SPEC.md:147,293).  The GPU traceback stores per-cell direction codes and walks them, which *is* the full-matrix
algorithm, so align_traceback / explicit_traceback here reproduce ref_traceback bit for bit, including
cells_computed = m*n.
"""
from __future__ import annotations

import numpy as np

from . import _native as N
from .core import AlignConfig, AlignmentResult, ScoringScheme, Sequence, UseHirschberg, check_length_bounds, validate_config
from .engine import EngineStats, EngineTuning, get_context
from .io import unpack_runs
from .pool import SequencePool

T_EXPLICIT = 128


def _traceback_pairs(pairs, cfg: AlignConfig, scheme: ScoringScheme, device: int = 0,
                     scratch_bytes: int | None = None, info: dict | None = None) -> list[AlignmentResult]:
    queries = SequencePool.from_sequences([p[0] for p in pairs])
    subjects = SequencePool.from_sequences([p[1] for p in pairs])
    idx = np.arange(len(pairs), dtype=np.int32)
    batch = N.Batch(get_context(device), queries.codes, queries.off, queries.len, subjects.codes, subjects.off,
                    subjects.len, idx, idx)
    try:
        if scratch_bytes is not None:
            batch.set_tb_scratch(scratch_bytes)
        batch.traceback(scheme, cfg.align_type, timed=False)
        tb = batch.fetch_traceback()
        if info is not None:
            info.update(batch.tb_info())
    finally:
        batch.close()
    out = []
    for k, (q, s) in enumerate(pairs):
        if tb["status"][k]:
            raise N.status_exception(int(tb["status"][k]), f"problem of size {len(q)}x{len(s)}")
        runs = tb["cigar"][int(tb["cigar_off"][k]):int(tb["cigar_off"][k + 1])]
        out.append(AlignmentResult(score=int(tb["score"][k]), q_start=int(tb["q_start"][k]), q_end=int(tb["q_end"][k]),
                                   s_start=int(tb["s_start"][k]), s_end=int(tb["s_end"][k]), ops=unpack_runs(runs),
                                   cells_computed=len(q) * len(s)))
    return out


def align_traceback(query: Sequence, subject: Sequence, cfg: AlignConfig, scheme: ScoringScheme,
                    tuning: EngineTuning | None = None, meter=None, stats: EngineStats | None = None) -> AlignmentResult:
    """Alignment with operations for any align type (direction-code fill + on-device walk)."""
    cfg = validate_config(cfg, scheme)
    check_length_bounds(len(query), len(subject), scheme)
    res = _traceback_pairs([(query, subject)], cfg, scheme)[0]
    if stats is not None:
        stats.cells += res.cells_computed
    return res


def explicit_traceback(query: Sequence, subject: Sequence, cfg: AlignConfig, scheme: ScoringScheme,
                       meter=None) -> AlignmentResult:
    """Full-matrix traceback for small problems; raises UseHirschberg beyond T_EXPLICIT like the reference."""
    cfg = validate_config(cfg, scheme)
    if len(query) + len(subject) > T_EXPLICIT:
        raise UseHirschberg(f"m+n = {len(query) + len(subject)} exceeds the explicit traceback bound {T_EXPLICIT}")
    return _traceback_pairs([(query, subject)], cfg, scheme)[0]


def _bounded(query: Sequence, subject: Sequence, cfg: AlignConfig, scheme: ScoringScheme, meter, stats):
    """One pair through the bounded-memory path (csrc/traceback_band.cuh): a one-byte code budget sends every pair there."""
    info: dict = {}
    res = _traceback_pairs([(query, subject)], cfg, scheme, scratch_bytes=1, info=info)[0]
    cells = len(query) * len(subject) * (cfg.align_type != "global") + info.get("cells", 0)   # end-cell sweep + checkpoint sweep + tiles
    if meter is not None:     # AllocationMeter-compatible object: the scratch of the pair, taken and given back
        meter.add(info.get("peak_bytes", 0))
        meter.sub(info.get("peak_bytes", 0))
    if stats is not None:
        stats.cells += cells
    return res, cells


def hirschberg(query: Sequence, subject: Sequence, cfg: AlignConfig, scheme: ScoringScheme,
               tuning: EngineTuning | None = None, meter=None, stats: EngineStats | None = None) -> AlignmentResult:
    """Global traceback in bounded memory (reference: traceback.py:208-224).

    The reference splits the problem recursively (Myers-Miller); here the score sweep leaves checkpoint rows and tile
    columns (8/R + 8/512 bytes per cell instead of 0.5) and the walk re-fills only the tiles it crosses, so about 1.0x
    the matrix cells are computed (the reference: up to 2x) and the path is the full-matrix walk's (refdp.py:158-235).
    Contract kept from the reference's tests (test_traceback.py:22-59, test_acceptance.py:115-135): score equals the
    score-only kernels, rescoring the operations gives the score, cells_computed <= 2.1 m n."""
    cfg = validate_config(cfg, scheme)
    if cfg.align_type != "global":
        raise ValueError("hirschberg builds global tracebacks; use align_traceback for local or semiglobal")
    check_length_bounds(len(query), len(subject), scheme)
    res, cells = _bounded(query, subject, cfg, scheme, meter, stats)
    return AlignmentResult(score=res.score, q_start=0, q_end=len(query), s_start=0, s_end=len(subject), ops=res.ops,
                           cells_computed=cells)


def locate_endpoints(query: Sequence, subject: Sequence, cfg: AlignConfig, scheme: ScoringScheme,
                     tuning: EngineTuning | None = None, stats: EngineStats | None = None):
    """Score, start and end cell of a local or semiglobal alignment: (score, (q0, s0), (q1, s1), cells)
    (reference: traceback.py:312-344).  The end cell is the score kernels' argmax (the reference's forward sweep); the
    start is where the full-matrix walk from that end cell stops -- the reference finds *a* co-optimal start with an
    anchored reverse sweep, its tests pin score, window bounds and the local end cell (test_traceback.py:111-127)."""
    cfg = validate_config(cfg, scheme)
    if cfg.align_type == "global":
        raise ValueError("locate_endpoints applies to local and semiglobal only")
    check_length_bounds(len(query), len(subject), scheme)
    res, cells = _bounded(query, subject, cfg, scheme, None, stats)
    return res.score, (res.q_start, res.s_start), (res.q_end, res.s_end), cells
