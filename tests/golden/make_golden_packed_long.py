"""Golden vectors for the reference's full packed range (max_step * (m + n) < 2^14): engine_score_packed of the REFERENCE
on pairs of 600..4000 symbols, all three alignment types, linear and merged affine schemes.

Run in the build container only (the reference tree does not travel to the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_packed_long.py

Output (committed): tests/golden/packed_long.json.  Sequences are stored as (seed, length, mutation) recipes plus a
CRC, not as text, to keep the file small; tests/helpers_golden.py:regen rebuilds them with the same generator.
"""
import json
import os
import zlib

import numpy as np

import waveseq as W

HERE = os.path.dirname(os.path.abspath(__file__))
BASES = np.array(list("ACGT"))


def make_pair(seed, m, n, related):
    """Deterministic sequences from a recipe (also used by the test, so keep it in sync with tests/test_gpu_api.py)."""
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 4, m)
    if related:
        s = np.resize(q, n).copy()
        mut = rng.random(n) < 0.08
        s[mut] = (s[mut] + rng.integers(1, 4, int(mut.sum()))) % 4
    else:
        s = rng.integers(0, 4, n)
    return "".join(BASES[q]), "".join(BASES[s])


def main():
    out = []
    shapes = [(600, 700), (1000, 1000), (1500, 2400), (4000, 4000), (3900, 650), (2048, 2049)]
    k = 0
    for at in ("global", "local", "semiglobal"):
        for gm, sch in (("affine", (2, -1, 2, 1)), ("linear", (2, -1, 1, 1)), ("affine", (1, -1, 2, 2))):
            scheme = W.ScoringScheme(*sch, gm)
            cfg = W.AlignConfig(at, gm)
            for (m, n) in shapes[k % 2::2]:
                k += 1
                ra_recipe = (1000 + k, m, n, k % 2 == 0)
                rb_recipe = (2000 + k, n if k % 3 == 0 else m, m if k % 3 == 0 else n, k % 2 == 1)
                qa, sa = make_pair(*ra_recipe)
                qb, sb = make_pair(*rb_recipe)
                if not (W.packed_range_ok(scheme, len(qa), len(sa)) and W.packed_range_ok(scheme, len(qb), len(sb))):
                    continue
                ra, rb, cells = W.engine_score_packed((W.encode_sequence("a", qa), W.encode_sequence("a", sa)),
                                                      (W.encode_sequence("b", qb), W.encode_sequence("b", sb)), cfg, scheme)
                out.append(dict(align_type=at, gap_model=gm, scheme=list(sch), a_recipe=list(ra_recipe), b_recipe=list(rb_recipe),
                                crc=[zlib.crc32((qa + "|" + sa).encode()), zlib.crc32((qb + "|" + sb).encode())],
                                a=[int(ra[0]), int(ra[1][0]), int(ra[1][1])], b=[int(rb[0]), int(rb[1][0]), int(rb[1][1])],
                                cells=int(cells)))
                print(at, gm, sch, len(qa), len(sa), len(qb), len(sb), ra, rb, flush=True)
    json.dump(dict(packed_long=out), open(os.path.join(HERE, "packed_long.json"), "w"), indent=0)
    print("packed_long", len(out))


if __name__ == "__main__":
    main()
