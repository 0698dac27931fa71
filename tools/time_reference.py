"""Time the REAL reference (waveseq.run_batch, numba engine) on bounded samples of the five configs.  Build container
only: needs /root/reference.  PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tools/time_reference.py"""
import json, os, sys, time
import numpy as np
import waveseq as W

B = np.array(list("ACGT"))
def seqs(rng, n, L, pref): return [W.encode_sequence(f"{pref}{i}", "".join(B[rng.integers(0, 4, L)])) for i in range(n)]
workers = os.cpu_count()
out = []
def run(name, n, L, at, gm, sch, mode="score_only", packed=False):
    rng = np.random.default_rng(7)
    q, s = seqs(rng, n, L, "q"), seqs(rng, n, L, "s")
    job = W.BatchJob(q, s, [(i, i) for i in range(n)], W.AlignConfig(at, gm, mode), W.ScoringScheme(*sch, gm),
                     tuning=W.EngineTuning(packed=True) if packed else None, workers=workers)
    W.run_batch(W.BatchJob(q[:8], s[:8], [(i, i) for i in range(8)], job.cfg, job.scheme, tuning=job.tuning, workers=2))  # JIT warm-up
    t0 = time.perf_counter(); rep = W.run_batch(job); dt = time.perf_counter() - t0
    rec = dict(config=name, pairs=n, length=L, workers=workers, packed=packed, seconds=round(dt, 2), gcups=round(rep.total_cells / dt / 1e9, 4))
    print(json.dumps(rec), flush=True); out.append(rec)
run("cfg1 global linear", 4000, 150, "global", "linear", (2, -1, 1, 1))
run("cfg2 local affine", 4000, 150, "local", "affine", (2, -1, 2, 1))
run("cfg2 local affine packed16", 4000, 150, "local", "affine", (2, -1, 2, 1), packed=True)
run("cfg3 semiglobal affine traceback", 300, 250, "semiglobal", "affine", (2, -1, 2, 1), mode="traceback")
run("cfg4 global affine 10 kbp", 8, 10000, "global", "affine", (2, -1, 2, 1))
