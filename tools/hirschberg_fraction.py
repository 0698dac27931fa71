"""how often does the reference's linear-space path (waveseq.align_traceback: Hirschberg splits) return the SAME
CIGAR and spans as the full-matrix walk (waveseq.refdp.ref_traceback) that this library reproduces bit for bit on the GPU?
Both paths are optimal (equal score, rescoring accepts both); they pick different co-optimal paths.  Reported, not required.
Build container only: needs /root/reference.
PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tools/hirschberg_fraction.py [pairs]"""
import os, sys, time
import numpy as np
import waveseq as W
from waveseq import refdp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle

B = np.array(list("ACGT"))
n_pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rows = []
for at, gm, L, sch in (("semiglobal", "affine", 250, (2, -1, 2, 1)), ("local", "affine", 250, (2, -1, 2, 1)),
                       ("global", "affine", 250, (2, -1, 2, 1)), ("global", "linear", 150, (2, -1, 1, 1))):
    scheme = W.ScoringScheme(*sch, gm)
    cfg = W.AlignConfig(at, gm, "traceback")
    for kind in ("unrelated", "mutated copy (3 % sub, 1 % ins, 1 % del)"):
        rng = np.random.default_rng(220507613 + len(rows))
        same_ops = same_span = same_score = ours_eq_ref = 0
        t0 = time.perf_counter()
        for k in range(n_pairs):
            q = rng.integers(0, 4, L)
            if kind == "unrelated":
                s = rng.integers(0, 4, L)
            else:
                out = []
                for x in q:
                    u = rng.random()
                    if u < 0.01: continue
                    if u < 0.02: out.append(int(rng.integers(0, 4)))
                    out.append(int((x + 1 + rng.integers(0, 3)) % 4) if rng.random() < 0.03 else int(x))
                s = np.array(out[:L] + list(rng.integers(0, 4, max(0, L - len(out)))))
            qs, ss = W.encode_sequence("q", "".join(B[q])), W.encode_sequence("s", "".join(B[s]))
            full = refdp.ref_traceback(qs, ss, cfg, scheme)
            lin = W.align_traceback(qs, ss, cfg, scheme)
            mine = oracle.ref_traceback(q.astype(np.uint8), s.astype(np.uint8), at, gm == "affine", *sch)
            ours_eq_ref += (mine["score"], mine["q_start"], mine["q_end"], mine["s_start"], mine["s_end"], list(map(tuple, mine["ops"]))) == (
                full.score, full.q_start, full.q_end, full.s_start, full.s_end, [tuple(o) for o in full.ops])
            same_score += lin.score == full.score
            same_span += (lin.q_start, lin.q_end, lin.s_start, lin.s_end) == (full.q_start, full.q_end, full.s_start, full.s_end)
            same_ops += [tuple(o) for o in lin.ops] == [tuple(o) for o in full.ops] and (lin.q_start, lin.s_start) == (full.q_start, full.s_start)
        rows.append((at, gm, L, kind, n_pairs, same_score, same_span, same_ops, ours_eq_ref, time.perf_counter() - t0))
        print(rows[-1], flush=True)
print("\n| alignment | reads | pairs | equal score | equal spans | identical CIGAR + start | this library's oracle == ref_traceback |")
print("|---|---|---|---|---|---|---|")
for at, gm, L, kind, n, sc, sp, op, me, dt in rows:
    print(f"| {at} {gm}, {L} bp | {kind} | {n} | {sc}/{n} | {sp}/{n} | **{op}/{n}** | {me}/{n} |")
