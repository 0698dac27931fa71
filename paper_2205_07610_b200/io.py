"""CIGAR text for results (the one piece of the reference's io module on the path: io.py:80-95)."""
from __future__ import annotations

from .core import AlignmentResult, merge_ops

OPS = "MID"


def cigar_string(result: AlignmentResult) -> str:
    """Run-length CIGAR (M/I/D, I consumes the query); empty for score-only or empty alignments."""
    if not result.ops:
        return ""
    return "".join(f"{n}{op}" for op, n in merge_ops(result.ops))


def unpack_runs(packed) -> list[tuple[str, int]]:
    """(length << 2 | op) words from the device -> [("M", 4), ...]."""
    return [(OPS[int(w) & 3], int(w) >> 2) for w in packed]
