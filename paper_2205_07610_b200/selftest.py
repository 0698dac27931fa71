"""Randomised self-check of the GPU engine (reference: cli.cmd_selftest, cli.py:264-301).

The reference draws random short problems (m, n in 1..120, five schemes, three alignment types, random lane-group shapes),
runs its engine and compares score and end cell with its own full-matrix DP; on the first mismatch it prints a JSON blob
that reproduces the case.  Here both sides run on the GPU: the kernel family AUTO picks (packed int16 / half2 / long-read
kernels) is compared with the general int32 kernel -- independent code with its own cell update, edge handling and
end-cell tracking -- and, when the caller passes `checker` (the tests pass the CPU oracle), with that as well.  The cases
are drawn exactly like the reference's, so a seed means the same problems in both packages.  There is no CPU fallback: the
product never computes an alignment on the host.
"""
from __future__ import annotations

import json

import numpy as np

from . import _native as N
from .core import ScoringScheme, decode_sequence, encode_sequence
from .engine import get_context
from .pool import SequencePool

SELFTEST_SCHEMES = (
    ScoringScheme(2, -1, 2, 1, "affine"),
    ScoringScheme(3, -2, 4, 1, "affine"),
    ScoringScheme(1, -3, 2, 2, "affine"),
    ScoringScheme(2, -1, 1, 1, "linear"),
    ScoringScheme(1, -1, 3, 3, "linear"),
)
SELFTEST_TYPES = ("global", "local", "semiglobal")
_LANES = (4, 8, 16, 32)
_COLS = (1, 2, 4)


def draw_cases(cases: int, seed: int):
    """The reference's case generator (cli.py:265-279), draw for draw -- the lane-group shape draws are consumed too."""
    rng = np.random.default_rng(seed)
    alphabet = np.array(list("ACGT"))
    out = []
    for _ in range(cases):
        m = int(rng.integers(1, 121))
        n = int(rng.integers(1, 121))
        q = encode_sequence("q", "".join(alphabet[rng.integers(0, 4, m)]))
        s = encode_sequence("s", "".join(alphabet[rng.integers(0, 4, n)]))
        scheme = SELFTEST_SCHEMES[int(rng.integers(0, len(SELFTEST_SCHEMES)))]
        atype = SELFTEST_TYPES[int(rng.integers(0, 3))]
        lanes = _LANES[int(rng.integers(0, len(_LANES)))]
        cols = _COLS[int(rng.integers(0, len(_COLS)))]
        out.append((q, s, scheme, atype, lanes, cols))
    return out


def selftest(cases: int = 200, seed: int = 0, device: int = 0, checker=None, variants=("auto", "i32")) -> dict:
    """Run `cases` random problems; returns {"ok": bool, "cases": n, "failure": blob or None}.

    checker(queries, subjects, scheme, align_type) -> (scores, end_i, end_j) may add an external reference (arrays in
    case order of that group)."""
    drawn = draw_cases(cases, seed)
    groups: dict = {}
    for k, (q, s, scheme, atype, lanes, cols) in enumerate(drawn):
        groups.setdefault((scheme, atype), []).append(k)
    ctx = get_context(device)
    for (scheme, atype), idx in groups.items():
        qs = SequencePool.from_sequences([drawn[k][0] for k in idx])
        ss = SequencePool.from_sequences([drawn[k][1] for k in idx])
        ident = np.arange(len(idx), dtype=np.int32)
        results = {}
        batch = N.Batch(ctx, qs.codes, qs.off, qs.len, ss.codes, ss.off, ss.len, ident, ident)
        try:
            for v in variants:
                batch.score(scheme, atype, v, timed=False)
                results[v] = tuple(np.array(a) for a in batch.fetch_scores()[:3])
        finally:
            batch.close()
        if checker is not None:
            results["checker"] = tuple(np.asarray(a) for a in checker([drawn[k][0] for k in idx], [drawn[k][1] for k in idx],
                                                                      scheme, atype))
        names = list(results)
        base = results[names[0]]
        for other in names[1:]:
            got = results[other]
            bad = np.nonzero((base[0] != got[0]) | (base[1] != got[1]) | (base[2] != got[2]))[0]
            if len(bad):
                j = int(bad[0]); k = idx[j]
                q, s, _, _, lanes, cols = drawn[k]
                blob = {"case": k, "seed": seed, "query": decode_sequence(q), "subject": decode_sequence(s),
                        "align_type": atype, "gap_model": scheme.gap_model,
                        "scheme": [scheme.match_score, scheme.mismatch_score, scheme.gap_open, scheme.gap_extend],
                        "lanes": lanes, "cols_per_lane": cols,
                        "engine": [int(base[0][j]), [int(base[1][j]), int(base[2][j])]], "engine_variant": names[0],
                        "reference": [int(got[0][j]), [int(got[1][j]), int(got[2][j])]], "reference_variant": other}
                return {"ok": False, "cases": cases, "failure": blob}
    return {"ok": True, "cases": cases, "failure": None}


def main(argv=None) -> int:
    import argparse, sys
    ap = argparse.ArgumentParser(description="random cross-check of the GPU kernels (AUTO vs int32)")
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args(argv)
    rep = selftest(a.cases, a.seed)
    if not rep["ok"]:
        b = rep["failure"]
        print(f"FAIL at case {b['case']}: engine {b['engine']}, reference {b['reference']}", file=sys.stderr)
        print(json.dumps(b), file=sys.stderr)
        return 1
    print(f"{a.cases}/{a.cases} ok")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
