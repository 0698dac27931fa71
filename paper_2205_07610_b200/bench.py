"""Throughput measurement in the reference's conventions (bench.py:30-115): GCUPS = score cells / wall time, median of
the repetitions with the even-count rule, next to a theoretical peak from a simple hardware model.

For a B200 the model's "cores" are issue lanes: HardwareModel.b200(...) = SMs x 128 thread-instructions per clock, and
cycles_per_cell = the reference's score ops per cell divided by the cells a thread instruction advances (2 in the
packed kernels), which makes theoretical_peak() the ALU-issue roofline of BASELINE.md / DESIGN.md.
"""
from __future__ import annotations

import json
from dataclasses import dataclass

from .batch import BatchJob, run_batch

MEDIAN_RULE = "mean of the two middle values of the sorted run speeds"


@dataclass(frozen=True)
class HardwareModel:
    """cores x clock_ghz / cycles_per_cell = peak GCUPS (reference: bench.HardwareModel, bench.py:12-27)."""

    cores: float
    clock_ghz: float
    cycles_per_cell: float

    def __post_init__(self):
        if min(self.cores, self.clock_ghz, self.cycles_per_cell) <= 0:
            raise ValueError("hardware model fields must all be positive")

    @classmethod
    def b200(cls, ops_per_cell: float = 8.0, cells_per_instruction: int = 2, sm_count: int = 148,
             clock_ghz: float = 1.965) -> "HardwareModel":
        return cls(cores=sm_count * 128, clock_ghz=clock_ghz, cycles_per_cell=ops_per_cell / cells_per_instruction)


def theoretical_peak(hw: HardwareModel) -> float:
    return hw.cores * hw.clock_ghz / hw.cycles_per_cell


def median_rate(values) -> float:
    """Median; with an even count, the mean of the two middle values (the paper's rule)."""
    vals = sorted(values)
    if not vals:
        raise ValueError("median of an empty list")
    mid = len(vals) // 2
    return vals[mid] if len(vals) % 2 else (vals[mid - 1] + vals[mid]) / 2.0


@dataclass
class BenchReport:
    achieved_gcups: float
    tpp_gcups: float | None
    efficiency: float | None
    cells: int
    extra_cells: int
    wall_s: float
    repetitions: int
    workload: str
    median_rule: str = MEDIAN_RULE

    def to_json(self) -> str:
        return json.dumps({k: getattr(self, k) for k in ("achieved_gcups", "tpp_gcups", "efficiency", "cells", "extra_cells",
                                                         "wall_s", "repetitions", "workload", "median_rule")}, indent=2)


def measure_gcups(job: BatchJob, repetitions: int, hw: HardwareModel | None = None) -> BenchReport:
    """Median GCUPS of `repetitions` run_batch calls (upload + kernels + download inside the timing, parsing and
    writing outside, as in the reference).  Traceback mode counts score cells only; this implementation's direction-code
    traceback touches every cell exactly once, so extra_cells is 0."""
    if repetitions < 1:
        raise ValueError("repetitions must be at least 1")
    rates, last = [], None
    for _ in range(repetitions):
        last = run_batch(job)
        rates.append(last.gcups)
    achieved = median_rate(rates)
    peak = theoretical_peak(hw) if hw is not None else None
    return BenchReport(achieved_gcups=achieved, tpp_gcups=peak, efficiency=(achieved / peak if peak else None),
                       cells=last.total_cells, extra_cells=0,
                       wall_s=(last.total_cells / achieved / 1e9 if achieved > 0 else 0.0), repetitions=repetitions,
                       workload=f"{len(job.pairs)} pairs, {job.cfg.align_type}/{job.scheme.gap_model}, {job.cfg.result_mode}")
