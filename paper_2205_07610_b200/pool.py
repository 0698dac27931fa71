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
        self.packed = None       # optional 2-bit form of the pool (from_packed): what run_batch uploads when present
        self.flag_pos = None
        self.uniform_len = None  # set by from_uniform: read k starts at k * uniform_len
        self._codes = np.ascontiguousarray(codes, np.uint8) if codes is not None else None
        self.off = np.ascontiguousarray(off, np.int64)
        self.len = np.ascontiguousarray(lengths, np.int32)
        self.ids = ids
        if self.off.shape != self.len.shape:
            raise ValueError("offset and length arrays must have the same shape")

    def __len__(self) -> int:
        return int(self.len.shape[0])

    @property
    def codes(self) -> np.ndarray:
        """One byte per symbol (expanded on first use when the pool was built from packed data)."""
        if self._codes is None:
            total = int((self.off + self.len).max()) if len(self.len) else 0
            sym = np.arange(total, dtype=np.int64)
            c = (self.packed[sym >> 2] >> ((sym & 3) << 1).astype(np.uint8)) & 3
            if self.flag_pos is not None and len(self.flag_pos):
                c[self.flag_pos] = FLAGGED_CODE
            self._codes = c.astype(np.uint8)
        return self._codes

    @classmethod
    def from_packed(cls, packed: np.ndarray, off: np.ndarray, lengths: np.ndarray, flag_pos=None, ids=None) -> "SequencePool":
        """Pool in the reference's 2-bit layout (Sequence.data, core.py:78-87: four symbols per byte, low bits first)
        over the concatenated pool: symbol k sits in bits 2*(k%4) of byte k//4.  flag_pos lists the pool positions of
        flagged (non-ACGT) symbols, which the packed data stores as 0 like the reference does."""
        pool = cls(None, off, lengths, ids)
        pool.packed = np.ascontiguousarray(packed, np.uint8)
        pool.flag_pos = None if flag_pos is None else np.ascontiguousarray(flag_pos, np.int64)
        return pool

    def to_packed(self) -> "SequencePool":
        """The same pool in 2-bit form (host-side packing; meant for pools that are reused across batches)."""
        c = self.codes
        flags = np.nonzero(c >= FLAGGED_CODE)[0].astype(np.int64)
        v = np.where(c >= FLAGGED_CODE, 0, c).astype(np.uint8)
        pad = (-len(v)) % 4
        if pad:
            v = np.concatenate([v, np.zeros(pad, np.uint8)])
        v = v.reshape(-1, 4)
        packed = (v[:, 0] | (v[:, 1] << 2) | (v[:, 2] << 4) | (v[:, 3] << 6)).astype(np.uint8)
        out = SequencePool.from_packed(packed, self.off, self.len, flags, self.ids)
        out.uniform_len = self.uniform_len
        return out

    def subset(self, ids: np.ndarray) -> "SequencePool":
        """Compact pool of the sequences `ids` (in that order): what one GPU shard uploads when its pairs reference only a
        part of the pool.  Uniform pools keep their shape, so a contiguous id range of one is a zero-copy slice."""
        from . import _native as N
        ids = np.asarray(ids, np.int64)
        if self.uniform_len is not None and len(ids) and int(ids[-1]) - int(ids[0]) + 1 == len(ids) and \
                (len(ids) == 1 or bool((np.diff(ids) == 1).all())):
            return self.slice_uniform(int(ids[0]), int(ids[-1]) + 1)
        codes, off = N.compact_pool(self.codes, self.off, self.len, ids)
        out = SequencePool(codes, off, self.len[ids], None if self.ids is None else [self.ids[int(k)] for k in ids])
        if self.uniform_len is not None:
            out.uniform_len = self.uniform_len
        return out

    def slice_uniform(self, lo: int, hi: int) -> "SequencePool":
        """Reads lo .. hi-1 of a uniform pool without copying (2-bit pools: lo * length must be a multiple of four symbols,
        else the slice falls back to the byte form)."""
        L = self.uniform_len
        if L is None:
            raise ValueError("slice_uniform needs a pool built by from_uniform")
        n = hi - lo
        off = np.arange(n, dtype=np.int64) * L
        lens = np.full(n, L, np.int32)
        ids = None if self.ids is None else self.ids[lo:hi]
        no_flags = self.flag_pos is None or len(self.flag_pos) == 0
        if self.packed is not None and (lo * L) % 4 == 0 and no_flags:
            out = SequencePool.from_packed(self.packed[lo * L // 4:(hi * L + 3) // 4], off, lens, None, ids)
        else:
            out = SequencePool(self.codes[lo * L:hi * L], off, lens, ids)
        out.uniform_len = L
        return out

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
        pool = cls(codes2d.reshape(-1), np.arange(n, dtype=np.int64) * length, np.full(n, length, np.int32))
        pool.uniform_len = int(length)
        return pool
