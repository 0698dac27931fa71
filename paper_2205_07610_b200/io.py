"""Result wire formats: CIGAR text and the results TSV (reference: io.cigar_string io.py:80-95, io.write_results_tsv
io.py:98-110, TSV_HEADER io.py:21-22).  FASTA parsing and the read simulator stay out of scope."""
from __future__ import annotations

import os

import numpy as np

from .core import AlignmentResult, merge_ops

OPS = "MID"
TSV_HEADER = ("query_id", "subject_id", "score", "q_start", "q_end", "s_start", "s_end", "cigar")


def cigar_string(result: AlignmentResult) -> str:
    """Run-length CIGAR (M/I/D, I consumes the query); empty for score-only or empty alignments."""
    if not result.ops:
        return ""
    return "".join(f"{n}{op}" for op, n in merge_ops(result.ops))


def unpack_runs(packed) -> list[tuple[str, int]]:
    """(length << 2 | op) words from the device -> [("M", 4), ...]."""
    return [(OPS[int(w) & 3], int(w) >> 2) for w in packed]


def runs_to_cigar(packed) -> str:
    """CIGAR text straight from the device's run words (already merged and in forward order)."""
    return "".join(f"{int(w) >> 2}{OPS[int(w) & 3]}" for w in packed)


def write_results_tsv(rows, path: str | os.PathLike) -> None:
    """One TSV row per aligned pair under the reference's header; rows yields (query_id, subject_id, AlignmentResult).
    The cigar column is empty for score-only results."""
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\t".join(TSV_HEADER) + "\n")
        for qid, sid, r in rows:
            fh.write(f"{qid}\t{sid}\t{r.score}\t{r.q_start}\t{r.q_end}\t{r.s_start}\t{r.s_end}\t{cigar_string(r)}\n")


def write_batch_tsv(results, pairs, query_ids, subject_ids, path: str | os.PathLike) -> None:
    """Same file as write_results_tsv, written from a run_batch result without building AlignmentResult objects: the
    columns come from the result arrays, the CIGAR text from the device's run-length buffer."""
    from .batch import ResultArray
    if not isinstance(results, ResultArray):
        write_results_tsv(((query_ids[q], subject_ids[s], r) for (q, s), r in zip(pairs, results)), path)
        return
    pairs = np.asarray(pairs)
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\t".join(TSV_HEADER) + "\n")
        for i in range(len(results)):
            cig = "" if results.runs is None else runs_to_cigar(results.runs[int(results.run_off[i]):int(results.run_off[i + 1])])
            fh.write(f"{query_ids[int(pairs[i, 0])]}\t{subject_ids[int(pairs[i, 1])]}\t{int(results.score[i])}\t"
                     f"{int(results.q_start[i])}\t{int(results.q_end[i])}\t{int(results.s_start[i])}\t"
                     f"{int(results.s_end[i])}\t{cig}\n")
