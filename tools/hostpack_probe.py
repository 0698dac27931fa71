"""Timeline of the host-packed upload: WSB_TRACE lines of one run_batch call at bench size (cfg2: 4 M x 150 bp)."""
import os, sys, time
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ["WSB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N

n, L = 4_000_000, 150
rng = np.random.default_rng(1)
def pinned(shape):
    a = N.pinned_empty(int(np.prod(shape)), np.uint8).reshape(shape)
    a[...] = rng.integers(0, 4, shape, dtype=np.uint8)
    return a
q, s = pinned((n, L)), pinned((n, L))
idx = np.arange(n, dtype=np.int32)
job = W.BatchJob(W.SequencePool.from_uniform(q), W.SequencePool.from_uniform(s), np.stack([idx, idx], 1),
                 W.AlignConfig("local", "affine"), W.ScoringScheme(), tuning=W.EngineTuning(packed=True), devices=[0])
for thr in [int(x) for x in (sys.argv[1:] or ["-1", "0"])]:
    os.environ["WSB_HOST_PACK_THREADS"] = str(thr)
    from paper_2205_07610_b200.engine import get_context
    get_context(0).set_host_pack_threads(thr)
    import paper_2205_07610_b200.batch as B
    B._host_pack_policy = lambda thr=thr: thr
    rep = W.run_batch(job); rep = W.run_batch(job)
    ts = []
    for i in range(6):
        t0 = time.perf_counter(); rep = W.run_batch(job); ts.append((time.perf_counter() - t0) * 1e3)
    print(f"threads {thr}: ms per call {[round(t, 1) for t in ts]} h2d {rep.h2d_bytes}", flush=True)
