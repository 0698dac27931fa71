import os, sys, time, cProfile, pstats
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2205_07610_b200 as W
from bench import pinned
rng = np.random.default_rng(1)
n, L = 4_000_000, 150
(q, kq), (s, ks) = pinned(rng.integers(0, 4, (n, L), dtype=np.uint8)), pinned(rng.integers(0, 4, (n, L), dtype=np.uint8))
idx = np.arange(n, dtype=np.int32)
pair_arr = np.stack([idx, idx], 1)
host_q, host_s = W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s)
job = W.BatchJob(host_q, host_s, pair_arr, W.AlignConfig("local", "affine", "score_only"), W.ScoringScheme(), tuning=W.EngineTuning(packed=True), devices=[0])
for _ in range(4): rep = W.run_batch(job)
pq2, ps2 = host_q.to_packed(), host_s.to_packed()
keep2 = [pinned(hp.packed) for hp in (pq2, ps2)]
pq2.packed, ps2.packed = keep2[0][0], keep2[1][0]
job_p = W.BatchJob(pq2, ps2, pair_arr, job.cfg, W.ScoringScheme(), tuning=job.tuning, devices=[0])
W.run_batch(job_p); W.run_batch(job_p)
ts = []
for _ in range(6):
    t0 = time.perf_counter(); rep_p = W.run_batch(job_p); _ = int(rep_p.results.score[0]); ts.append(round((time.perf_counter() - t0) * 1e3, 1))
print("packed leg per step:", ts, "wall", rep_p.wall_time * 1e3)
pr = cProfile.Profile(); pr.enable(); rep_p = W.run_batch(job_p); _ = int(rep_p.results.score[0]); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
