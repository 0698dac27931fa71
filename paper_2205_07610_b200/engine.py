"""Engine entry points: single-pair scoring through the CUDA kernels.

Mirrors the reference's engine API (pkg/src/waveseq/engine.py): engine_score (:383-400), engine_score_packed
(:512-597), EngineTuning (:39-55), auto_tuning (:58-68), merged_state_exact (:71-94), packed_range_ok (:504-509),
EngineStats (:109-146).  Every call runs on the GPU through the C ABI; there is no CPU path.

Mapping of the reference's tuning knobs: lanes / cols_per_lane are accepted for compatibility but the lane-group shape
is chosen by the native planner per length bucket; packed=True asks for the packed half2 kernel, which raises
PackedRangeOverflow when a problem leaves the reference's packed range (max_step*(m+n) < 2^14, checked first, as the
reference does) or the kernel's exact fp16 window, and ValueError for affine schemes the merged state cannot represent.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import (AlignConfig, PackedRangeOverflow, ScoringScheme, Sequence, check_length_bounds, validate_config)
from .pool import SequencePool

_ALLOWED_LANES = (4, 8, 16, 32, 64)
_PACK_LIMIT = 1 << 14

_ctx_lock = threading.Lock()
_contexts: dict[int, N.Context] = {}


def get_context(device: int = 0) -> N.Context:
    """Process-wide context per GPU (created on first use)."""
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = _contexts[device] = N.Context(device)
        return ctx


@dataclass(frozen=True)
class EngineTuning:
    """Lane-group shape request: lanes per group, matrix columns per lane, packed two-alignment mode."""

    lanes: int = 32
    cols_per_lane: int = 4
    packed: bool = False

    def __post_init__(self):
        if self.lanes not in _ALLOWED_LANES:
            raise ValueError(f"lanes must be one of {_ALLOWED_LANES}, got {self.lanes}")
        if not 1 <= self.cols_per_lane <= 16:
            raise ValueError(f"cols_per_lane must be in 1..16, got {self.cols_per_lane}")

    @property
    def stage_width(self) -> int:
        return self.lanes * self.cols_per_lane


def auto_tuning(max_len: int, packed: bool = False) -> EngineTuning:
    k = 1
    while k < 16 and 32 * k < max_len:
        k *= 2
    return EngineTuning(lanes=32, cols_per_lane=k, packed=packed)


def merged_state_exact(scheme: ScoringScheme) -> bool:
    """True when the merged gap state G = max(E, F) reproduces exact Gotoh H values for the scheme."""
    return N.merged_state_exact(scheme)


def packed_range_ok(scheme: ScoringScheme, m: int, n: int) -> bool:
    """The reference's packed-range rule: every finite score of an m x n problem fits 16-bit halves."""
    return scheme.max_step * (m + n) < _PACK_LIMIT


def f16_range_ok(scheme: ScoringScheme, m: int, n: int) -> bool:
    """True when the packed half2 kernel is exact for an m x n problem (all DP values are fp16 integers)."""
    return N.f16_range_ok(scheme, m, n)


@dataclass
class EngineStats:
    """Counters of the reference's engine (engine.py:109-146), filled from the native planner (wsb_batch_plan_stats):
    stages, wavefront iterations, and the max / add-sub instructions of the executed cell updates (padding included) as
    thread-instruction counts of the kernel the planner picked -- the packed kernels advance two cells per instruction, so
    ops per update can be fractional; ops_lookup counts the substitution lookups (PRMT / IDP.4A / HSET2), which the
    reference's tally folds into its adds.  The block counters count the CPU emulation's memory touches and stay zero
    (the kernels' traffic is measured with ncu instead)."""

    query_load_blocks: int = 0
    query_load_misaligned: int = 0
    boundary_load_blocks: int = 0
    boundary_load_misaligned: int = 0
    boundary_store_blocks: int = 0
    boundary_store_misaligned: int = 0
    ops_max: int = 0
    ops_addsub: int = 0
    iterations: int = 0
    cells: int = 0
    stages: int = 0
    ops_lookup: int = 0      # extension: substitution lookups
    updates: int = 0         # extension: cell updates executed, padding included (stages * m * stage width per alignment)

    @property
    def ops_total(self) -> int:
        return self.ops_max + self.ops_addsub

    def absorb_plan(self, plan: dict, cells: int) -> None:
        self.cells += cells
        self.stages += plan["stages"]
        self.iterations += plan["iterations"]
        self.updates += plan["updates"]
        self.ops_max += plan["ops_max"]
        self.ops_addsub += plan["ops_addsub"]
        self.ops_lookup += plan["ops_lookup"]


def _score_pairs(pairs, cfg: AlignConfig, scheme: ScoringScheme, variant: str, device: int = 0, stats=None):
    queries = SequencePool.from_sequences([p[0] for p in pairs])
    subjects = SequencePool.from_sequences([p[1] for p in pairs])
    idx = np.arange(len(pairs), dtype=np.int32)
    batch = N.Batch(get_context(device), queries.codes, queries.off, queries.len, subjects.codes, subjects.off,
                    subjects.len, idx, idx)
    try:
        batch.score(scheme, cfg.align_type, variant, timed=False)
        score, ei, ej, status = batch.fetch_scores()
        if stats is not None:
            stats.absorb_plan(batch.plan_stats(), sum(len(q) * len(s) for q, s in pairs))
    finally:
        batch.close()
    for k in range(len(pairs)):
        if status[k]:
            raise N.status_exception(int(status[k]), f"problem of size {len(pairs[k][0])}x{len(pairs[k][1])}")
    return score, ei, ej


def engine_score(query: Sequence, subject: Sequence, cfg: AlignConfig, scheme: ScoringScheme,
                 tuning: EngineTuning | None = None, stats: EngineStats | None = None,
                 instrument: bool = False) -> tuple[int, tuple[int, int], int]:
    """(score, end cell, computed cells).  Global: end = (m, n); local / semiglobal: argmax cell, ties broken toward the
    smallest query then subject coordinate."""
    cfg = validate_config(cfg, scheme)
    m, n = len(query), len(subject)
    check_length_bounds(m, n, scheme)
    # tuning.packed is a hint, as in the reference (engine.py:383-400 never looks at it): the planner packs two
    # alignments per register wherever that is exact (int16 / half2) and runs int32 elsewhere
    score, ei, ej = _score_pairs([(query, subject)], cfg, scheme, "auto", stats=stats)
    return int(score[0]), (int(ei[0]), int(ej[0])), m * n


def engine_score_packed(pair_a: tuple[Sequence, Sequence], pair_b: tuple[Sequence, Sequence], cfg: AlignConfig,
                        scheme: ScoringScheme, tuning: EngineTuning | None = None, stats: EngineStats | None = None,
                        instrument: bool = False):
    """Two problems scored in one call: ((score_a, end_a), (score_b, end_b), cells).  Accepts and rejects exactly what
    the reference does (engine.py:512-536): PackedRangeOverflow beyond max_step * (m + n) < 2^14, ValueError for affine
    schemes outside the merged-state rule.  Inside that range the planner picks the widest exact kernel: packed int16
    (short local pairs, long twins), packed half2 (values within 2^11) or int32 -- every one of them bit-exact."""
    cfg = validate_config(cfg, scheme)
    for q, s in (pair_a, pair_b):
        if not packed_range_ok(scheme, len(q), len(s)):
            raise PackedRangeOverflow(f"problem of size {len(q)}x{len(s)} exceeds the packed 16-bit range "
                                      f"(max |score| step {scheme.max_step})")
    if scheme.gap_model == "affine" and not merged_state_exact(scheme):
        raise ValueError("packed affine mode requires a merged-state-exact scheme")
    score, ei, ej = _score_pairs([pair_a, pair_b], cfg, scheme, "auto", stats=stats)
    cells = len(pair_a[0]) * len(pair_a[1]) + len(pair_b[0]) * len(pair_b[1])
    return (int(score[0]), (int(ei[0]), int(ej[0]))), (int(score[1]), (int(ei[1]), int(ej[1]))), cells
