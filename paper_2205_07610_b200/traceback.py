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


def _traceback_pairs(pairs, cfg: AlignConfig, scheme: ScoringScheme, device: int = 0) -> list[AlignmentResult]:
    queries = SequencePool.from_sequences([p[0] for p in pairs])
    subjects = SequencePool.from_sequences([p[1] for p in pairs])
    idx = np.arange(len(pairs), dtype=np.int32)
    batch = N.Batch(get_context(device), queries.codes, queries.off, queries.len, subjects.codes, subjects.off,
                    subjects.len, idx, idx)
    try:
        batch.traceback(scheme, cfg.align_type, timed=False)
        tb = batch.fetch_traceback()
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
