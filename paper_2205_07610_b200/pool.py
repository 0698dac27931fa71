"""SequencePool: the device-facing layout of a list of sequences (one byte per symbol, offsets, lengths).

The reference hands kernels one numpy array per sequence (engine._encode_q5, engine.py:203-207).  A GPU batch wants one
contiguous pool per side, indexed by the job's (query, subject) pairs, so sequences shared by many pairs (all_pairs,
batch.py:58-64) are stored once.
"""
from __future__ import annotations

import numpy as np

from .core import FLAGGED_CODE, Sequence


class SequencePool:
    """codes[off[k] : off[k] + len[k]] are the symbols of sequence k: 0..3 = ACGT, 4 = flagged."""

    def __init__(self, codes: np.ndarray, off: np.ndarray, lengths: np.ndarray, ids=None):
        self.codes = np.ascontiguousarray(codes, np.uint8)
        self.off = np.ascontiguousarray(off, np.int64)
        self.len = np.ascontiguousarray(lengths, np.int32)
        self.ids = ids
        if self.off.shape != self.len.shape:
            raise ValueError("offset and length arrays must have the same shape")

    def __len__(self) -> int:
        return int(self.len.shape[0])

    def __getitem__(self, k: int) -> Sequence:
        """Materialise one Sequence (reference type) on demand."""
        o, n = int(self.off[k]), int(self.len[k])
        raw = self.codes[o:o + n]
        flags = raw >= FLAGGED_CODE
        return Sequence(self.ids[k] if self.ids is not None else str(k), np.where(flags, 0, raw).astype(np.uint8), flags)

    @classmethod
    def from_sequences(cls, seqs) -> "SequencePool":
        if isinstance(seqs, SequencePool):
            return seqs
        lengths = np.fromiter((len(s) for s in seqs), np.int32, len(seqs))
        off = np.zeros(len(seqs), np.int64)
        if len(seqs) > 1:
            np.cumsum(lengths[:-1], out=off[1:])
        codes = np.empty(max(int(lengths.sum()), 1), np.uint8)
        for s, o, n in zip(seqs, off, lengths):
            codes[o:o + n] = s.device_codes()
        return cls(codes, off, lengths, [s.id for s in seqs])

    @classmethod
    def from_uniform(cls, codes2d: np.ndarray) -> "SequencePool":
        """Pool over the rows of an (n_sequences, length) uint8 matrix, without copying."""
        n, length = codes2d.shape
        return cls(codes2d.reshape(-1), np.arange(n, dtype=np.int64) * length, np.full(n, length, np.int32))
