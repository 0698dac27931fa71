#!/usr/bin/env python
"""Benchmark of the batched pairwise-alignment hot path (BASELINE.json metric: GCUPS).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--impl reference]

A step is one pass of the score kernels over one synthetic batch.  At N = 1 the workload is cfg2, the configuration the
metric is quoted on: 4 M pairs of 150 bp reads, local alignment, affine gaps (2/-1/2/1), score-only, packed half2
kernel.  With N > 1 (torchrun, one rank per GPU) every rank aligns its own batch of the same size (weak scaling, no
data-path collective; gloo carries the barrier and the max-over-ranks of the step time).

value   whole-job GCUPS with the pools resident in HBM, timed with CUDA events on the launching stream (C ABI).
e2e     the same metric through the public API (run_batch on host buffers): H2D of the pools + kernels + D2H of the
        results inside the timed region.
roofline ALU-issue roofline of the dominant kernel: N_SM * 128 thread-instr/clk * f * W / I_cell.
cpu_baseline / --impl reference: the oracle port of the reference's DP (oracle/wsoracle.c, OpenMP, all host cores) on a
        bounded sample of the same workload.
"""
import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # before torch / the library initialise CUDA (see _native.load)
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs.  i_cell = the reference's instrumented score ops per cell; width = cells per
    # thread instruction of the dominant kernel (2 = packed half2, 1 = int32).
    "cfg1": dict(pairs=10_000, length=150, align_type="global", gap_model="linear", scheme=(2, -1, 1, 1), i_cell=5, variant="auto"),
    "cfg2": dict(pairs=4_000_000, length=150, align_type="local", gap_model="affine", scheme=(2, -1, 2, 1), i_cell=8, variant="auto"),
    "cfg2_i32": dict(pairs=1_000_000, length=150, align_type="local", gap_model="affine", scheme=(2, -1, 2, 1), i_cell=8,
                     variant="i32"),
    "cfg3": dict(pairs=1_000_000, length=250, align_type="semiglobal", gap_model="affine", scheme=(2, -1, 2, 1), i_cell=8,
                 variant="auto", traceback=True, related=0.5),
    "cfg4": dict(pairs=10_000, length=10_000, align_type="global", gap_model="affine", scheme=(2, -1, 2, 1), i_cell=7,
                 variant="auto"),
    # cfg5: 100 000 pairs in total (strong scaling: sharded over the ranks by cell count), truncated-Pareto lengths
    "cfg5": dict(pairs=100_000, length=None, align_type="local", gap_model="affine", scheme=(2, -1, 2, 1), i_cell=8,
                 variant="auto", pareto=True),
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def make_batch(cfg, seed):
    """Synthetic random-ACGT pools (uniform symbols, no flags), pair i = (query i, subject i)."""
    rng = np.random.default_rng(seed)
    n, L = cfg["pairs"], cfg["length"]
    q = rng.integers(0, 4, (n, L), dtype=np.uint8)
    s = rng.integers(0, 4, (n, L), dtype=np.uint8)
    if cfg.get("related"):  # cfg3: every second subject is a mutated copy of its query (3 % sub, 1 % ins, 1 % del)
        k = np.arange(0, n, 2)
        sub = rng.random((len(k), L)) < 0.03
        s[k] = np.where(sub, (q[k] + rng.integers(1, 4, (len(k), L), dtype=np.uint8)) % 4, q[k])
        shift = rng.random(len(k)) < 0.8   # one indel somewhere: shift the tail by one symbol either way
        pos = rng.integers(20, L - 20, len(k))
        for row, p_, left in zip(k[shift][:50_000], pos[shift][:50_000], rng.random(int(shift.sum()))[:50_000] < 0.5):
            s[row, p_:] = np.roll(s[row, p_:], 1 if left else -1)
    return q, s


def make_pareto(n, seed, cap=100_000):
    """cfg5: L = min(cap, floor(100/(1-u))), n = clip(round(L*v), 100, cap), v ~ U[0.8, 1.25]."""
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    L = np.minimum(cap, np.floor(100.0 / (1.0 - u))).astype(np.int64)
    M = np.clip(np.rint(L * rng.uniform(0.8, 1.25, n)), 100, cap).astype(np.int64)

    def pool(lens):
        off = np.zeros(n, np.int64)
        off[1:] = np.cumsum(lens[:-1])
        return rng.integers(0, 4, int(lens.sum()), dtype=np.uint8), off, lens.astype(np.int32)
    return pool(L), pool(M)


def pinned(arr):
    """Copy into page-locked host memory (torch is plumbing here: it owns the pinned allocation)."""
    import torch
    t = torch.empty(arr.shape, dtype=torch.uint8, pin_memory=torch.cuda.is_available())
    out = t.numpy()
    out[...] = arr
    out_t = (out, t)  # keep the tensor alive with the view
    return out_t


class ClockSampler(threading.Thread):
    """SM clock + throttle reasons during the timed region (nvidia-ml-py)."""

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index, self.samples, self.reasons, self.max_mhz = index, [], set(), None
        self._stop_evt = threading.Event()
        self._sampled = threading.Event()

    def run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {nv.nvmlClocksThrottleReasonHwSlowdown: "hw_slowdown",
                     nv.nvmlClocksThrottleReasonHwThermalSlowdown: "hw_thermal_slowdown",
                     nv.nvmlClocksThrottleReasonSwThermalSlowdown: "sw_thermal_slowdown",
                     nv.nvmlClocksThrottleReasonSwPowerCap: "sw_power_cap"}
            while not self._stop_evt.is_set():
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for bit, name in names.items():
                    if mask & bit:
                        self.reasons.add(name)
                self._sampled.set()
                time.sleep(0.02)
        except Exception as exc:  # no NVML: report nothing rather than guess
            self.reasons.add(f"nvml_unavailable:{type(exc).__name__}")
            self._sampled.set()

    def stop(self):
        self._sampled.wait(timeout=2)   # a timed region of a few hundred microseconds (cfg1) ends before NVML is up
        self._stop_evt.set()
        self.join(timeout=2)
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return rank, local, world


def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def dist_max(x, world):
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])
    return x


def dist_sum(x, world):
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t[0])
    return x


def cpu_sample(cfg, seconds_target=12.0, seed=7):
    """Oracle port (plain C restatement of refdp, OpenMP over pairs) on a bounded sample of the workload."""
    import oracle
    # all host cores, whatever OMP_NUM_THREADS says (torchrun sets it to 1 for its workers)
    threads = max(oracle.max_threads(), len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    L = cfg["length"]
    sch = cfg["scheme"]
    if cfg.get("pareto"):  # bounded sample of the length distribution: cap 6000 bp keeps a pair under ~0.1 s of one core
        (qc, qo, ql), (sc, so, sl) = make_pareto(3000, seed, cap=6000)
        idx = np.arange(3000, dtype=np.int32)
        t0 = time.perf_counter()
        oracle.score_batch(qc, qo, ql, sc, so, sl, idx, idx, cfg["align_type"], cfg["gap_model"] == "affine", *sch, threads=threads)
        dt = time.perf_counter() - t0
        return float((ql.astype(np.int64) * sl).sum()) / dt / 1e9, threads, 3000, dt

    def run(npairs):
        q, s = make_batch(dict(pairs=npairs, length=L), seed)
        off = np.arange(npairs, dtype=np.int64) * L
        ln = np.full(npairs, L, np.int32)
        idx = np.arange(npairs, dtype=np.int32)
        t0 = time.perf_counter()
        if cfg.get("traceback"):
            oracle.traceback_batch(q.reshape(-1), off, ln, s.reshape(-1), off, ln, idx, idx, cfg["align_type"],
                                   cfg["gap_model"] == "affine", *sch, threads=threads)
        else:
            oracle.score_batch(q.reshape(-1), off, ln, s.reshape(-1), off, ln, idx, idx, cfg["align_type"],
                               cfg["gap_model"] == "affine", *sch, threads=threads)
        dt = time.perf_counter() - t0
        return npairs * L * L / dt / 1e9, dt

    probe_pairs = max(64, int(2e8 / (L * L)))
    rate, dt = run(probe_pairs)
    pairs = int(min(cfg["pairs"], max(probe_pairs, rate * 1e9 * seconds_target / (L * L))))
    rate, dt = run(pairs)
    return rate, threads, pairs, dt


def workload_config(args, cfg, n_pairs):
    """The `config` object of the JSON line: identical for the GPU arm and the reference arm (what differs between them --
    kernel variant, host format, the CPU arm's bounded sample -- lives outside it)."""
    L = cfg["length"]
    traceback = bool(cfg.get("traceback"))
    input_bytes = 2 * n_pairs * L if L else 0   # (the Pareto batch of cfg5: ~0.2 GB, described in words below)
    return {"workload": args.workload, "pairs_per_gpu": n_pairs, "read_length": L if L else "pareto 100..%d" % args.cap,
            "align_type": cfg["align_type"], "gap_model": cfg["gap_model"], "scheme": list(cfg["scheme"]),
            "result_mode": "traceback" if traceback else "score_only",
            "statistic": "median of the timed steps, mean of the two middle values (reference bench.py:35-43, PAPER.md:454)",
            "l2": (f"inputs {input_bytes / 1e6:.0f} MB per GPU vs 126 MB L2 " if L else "inputs ~200 MB per batch vs 126 MB L2 ")
                  + ("(no flush needed)" if input_bytes > 252e6 else
                     "(inputs re-read from L2/HBM each step; per-cell DRAM traffic is ~0 either way)"),
            "sharding": "independent pairs per rank, no collective; gloo for barrier/max only"}


def median_rule(values):
    """Median; even count: mean of the two middle values (reference bench.py:35-43)."""
    v = sorted(values)
    mid = len(v) // 2
    return v[mid] if len(v) % 2 else 0.5 * (v[mid - 1] + v[mid])


def run_reference(args, cfg, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port, all host threads); rank 0 only."""
    if rank != 0:
        return
    rates = []
    info = None
    for step in range(args.warmup + args.steps):
        rate, threads, pairs, dt = cpu_sample(cfg, seconds_target=max(2.0, 20.0 / max(args.steps + args.warmup, 1)), seed=11 + step)
        info = (threads, pairs, dt)
        if step >= args.warmup:
            rates.append(rate)
    value = float(median_rule(rates))
    threads, pairs, dt = info
    length = cfg["length"] if cfg["length"] else "pareto(cap 6000)"
    sample = (f"every step scores {pairs} pairs of {length} bp of the workload ({dt:.2f} s; GCUPS does not depend on the batch "
              f"size), {cfg['align_type']}/{cfg['gap_model']}")
    line = {"impl": "reference", "metric": "GCUPS", "value": value, "unit": "GCUPS", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": workload_config(args, cfg, cfg["pairs"]),
            "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pairs", type=int, default=0, help="override pairs per GPU (debug)")
    ap.add_argument("--cap", type=int, default=100_000, help="cfg5: length cap of the truncated Pareto distribution")
    ap.add_argument("--host-format", default="bytes", choices=["bytes", "packed2"],
                    help="e2e leg: host pools as one byte per symbol, or in the reference's 2-bit Sequence.data layout")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard-api", type=int, default=0,
                    help="also time ONE process calling run_batch(devices=[0..N-1]) (the product's own multi-GPU path; devices wrap "
                         "around the GPUs present, so N > 1 works on a one-GPU box and then measures the sharding overhead)")
    args = ap.parse_args()
    cfg = dict(WORKLOADS[args.workload])
    if args.pairs:
        cfg["pairs"] = args.pairs
    rank, local, world = dist_setup()

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import paper_2205_07610_b200 as W
    from paper_2205_07610_b200 import _native as N

    ndev = N.device_count()
    if ndev < 1:
        raise SystemExit("bench.py needs a CUDA device: the alignment path has no CPU fallback")
    device = local % ndev
    scheme = W.ScoringScheme(*cfg["scheme"], cfg["gap_model"])
    variant = cfg.get("variant", "f16x2")
    strong = bool(cfg.get("pareto"))
    seed = 220507610 + int("".join(ch for ch in args.workload if ch.isdigit())[:1] or 0)
    if cfg.get("pareto"):   # strong scaling: one batch, sharded over the ranks by cell count (wsb_plan_shards)
        (qc, qo, ql), (sc, so, sl) = make_pareto(cfg["pairs"], seed, cap=args.cap)
        all_idx = np.arange(cfg["pairs"], dtype=np.int32)
        if world > 1:
            shard_of, _ = N.plan_shards(ql, sl, all_idx, all_idx, world)
            idx = all_idx[shard_of == rank]
        else:
            idx = all_idx
        q_keep = s_keep = None
        pool_q, pool_s = (qc, qo, ql), (sc, so, sl)
        L = None
    else:
        q, s = make_batch(cfg, seed + rank)
        L = cfg["length"]
        (q_pin, q_keep), (s_pin, s_keep) = pinned(q), pinned(s)
        off = np.arange(cfg["pairs"], dtype=np.int64) * L
        ln = np.full(cfg["pairs"], L, np.int32)
        idx = np.arange(cfg["pairs"], dtype=np.int32)
        pool_q, pool_s = (q_pin.reshape(-1), off, ln), (s_pin.reshape(-1), off, ln)
    n = len(idx)
    ctx = W.get_context(device)
    batch = N.Batch(ctx, *pool_q, *pool_s, idx, idx)
    cells = batch.total_cells
    traceback = bool(cfg.get("traceback"))

    def step():
        if traceback:
            return batch.traceback(scheme, cfg["align_type"])
        return batch.score(scheme, cfg["align_type"], variant)

    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(device)
    sampler.start()
    dist_barrier(world)
    step_ms, launches = [], 0
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        ms, nl = step()          # CUDA events on the launching stream bracket the kernels; synchronised before return
        step_ms.append(ms)
        launches += nl
    dist_barrier(world)
    wall = time.perf_counter() - t_wall0
    clocks = sampler.stop()
    total_ms = dist_max(float(np.sum(step_ms)), world)      # slowest rank
    median_ms = dist_max(float(median_rule(step_ms)), world)
    total_cells = dist_sum(float(cells), world) * args.steps   # weak: every rank its own batch; strong (cfg5): the shards add up to the one batch
    value = total_cells / args.steps / (median_ms * 1e-3) / 1e9   # the reference's statistic: median step, not the mean
    value_mean = total_cells / (total_ms * 1e-3) / 1e9
    # SM cycles of the last packed int16 short-read launch: only where that kernel IS the step (cfg1 / cfg2 under AUTO)
    kernel_cycles = batch.kernel_cycles if (args.workload in ("cfg1", "cfg2") and variant == "auto" and not traceback) else 0
    launches = int(dist_sum(float(launches), world))

    # end to end through the public API: host buffers in, host results out, every step
    pair_arr = np.stack([idx, idx], 1)
    if cfg.get("pareto"):
        host_q, host_s = W.SequencePool(*pool_q), W.SequencePool(*pool_s)
    else:   # a reads matrix: one row per read (run_batch then needs no offset / length / pair arrays on the device side)
        host_q, host_s = W.SequencePool.from_uniform(q_pin), W.SequencePool.from_uniform(s_pin)
    if args.host_format == "packed2":   # packed once, outside the timed region: the host format of the input, not a step
        host_q, host_s = host_q.to_packed(), host_s.to_packed()
        keep_packed = [pinned(hp.packed) for hp in (host_q, host_s)]
        host_q.packed, host_s.packed = keep_packed[0][0], keep_packed[1][0]
    job = W.BatchJob(host_q, host_s, pair_arr, W.AlignConfig(cfg["align_type"], cfg["gap_model"],
                                                           "traceback" if traceback else "score_only"),
                     scheme, tuning=W.EngineTuning(packed=(variant != "i32")), devices=[device])
    if variant == "i32":
        os.environ["WSB_VARIANT"] = "i32"
    e2e_steps = max(1, min(args.steps, 5))
    rep = W.run_batch(job)  # warm-up (twice: the previous result set is still referenced while the next one is
    rep = W.run_batch(job)  # fetched, so the pinned-buffer cache needs two sets before it stops allocating)
    dist_barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        rep = W.run_batch(job)
        _ = int(rep.results.score[0]) if isinstance(rep.results, W.ResultArray) else rep.results[0].score
    e2e_time = dist_max(time.perf_counter() - t0, world)
    e2e_value = total_cells / args.steps * e2e_steps / e2e_time / 1e9

    # the same end-to-end step from the reference's own in-memory layout (2-bit Sequence.data, core.py:78-87): a quarter of
    # the bytes on the bus.  Reported beside `e2e` (which stays on byte pools, the conservative figure) for uniform workloads.
    e2e_packed = None
    if args.host_format == "bytes" and not cfg.get("pareto") and not traceback and world == 1:
        pq2, ps2 = host_q.to_packed(), host_s.to_packed()
        keep2 = [pinned(hp.packed) for hp in (pq2, ps2)]
        pq2.packed, ps2.packed = keep2[0][0], keep2[1][0]
        job_p = W.BatchJob(pq2, ps2, pair_arr, job.cfg, scheme, tuning=job.tuning, devices=[device])
        rep_p = W.run_batch(job_p)  # two result sets must exist before the timed loop (see the warm-up above)
        rep_p = W.run_batch(job_p)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            rep_p = W.run_batch(job_p)
            _ = int(rep_p.results.score[0]) if isinstance(rep_p.results, W.ResultArray) else rep_p.results[0].score
        dt = time.perf_counter() - t0
        e2e_packed = {"value": cells * e2e_steps / dt / 1e9, "unit": "GCUPS", "h2d_bytes_per_step": int(rep_p.h2d_bytes),
                      "d2h_bytes_per_step": int(rep_p.d2h_bytes), "steps": e2e_steps, "run_batch_wall_ms": rep_p.wall_time * 1e3,
                      "host_format": "2-bit packed pools (the reference's Sequence.data layout), packed outside the timed region"}

    sharded = None
    if args.shard_api > 0 and world == 1:   # the product's own sharding: one process, one host thread + context + stream per shard
        devs = [d % ndev for d in range(args.shard_api)]
        job_s = W.BatchJob(host_q, host_s, pair_arr, job.cfg, scheme, tuning=job.tuning, devices=devs)
        rep_s = W.run_batch(job_s)
        rep_s = W.run_batch(job_s)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            rep_s = W.run_batch(job_s)
            _ = int(rep_s.results.score[0]) if isinstance(rep_s.results, W.ResultArray) else rep_s.results[0].score
        dt = time.perf_counter() - t0
        same = bool(np.array_equal(np.asarray(rep_s.results.score), np.asarray(rep.results.score))) if isinstance(rep.results, W.ResultArray) else None
        sharded = {"value": cells * e2e_steps / dt / 1e9, "unit": "GCUPS", "shards": args.shard_api, "devices": sorted(set(devs)),
                   "h2d_bytes_per_step": int(rep_s.h2d_bytes), "d2h_bytes_per_step": int(rep_s.d2h_bytes),
                   "scores_equal_single_device": same}

    # roofline: ALU-issue bound of the dominant kernel
    peaks = measured_peaks()
    f_ghz = float(peaks.get("sm_max_mhz", 1965.0)) / 1e3
    n_sm = ctx.sm_count
    # dominant kernel: cfg3 int32 fill, cfg5 int32 long-read kernel; cfg4's equal-shape pairs run two per block in packed int16
    # cfg3: the direction-code fill of a uniform batch runs packed int16 (two alignments per thread) unless switched off
    tb16 = args.workload == "cfg3" and not os.environ.get("WSB_TB_NO16")
    width = 1 if (variant == "i32" or args.workload == "cfg5" or (args.workload == "cfg3" and not tb16)) else 2
    dtype = "i32" if width == 1 else ("f16x2" if variant == "f16x2" else "s16x2")
    peak = n_sm * 128 * f_ghz * width / cfg["i_cell"]
    per_gpu = value / world
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(args.workload)
    except OSError:
        pass
    roofline = {"bound": "alu_issue", "achieved": per_gpu, "peak": peak, "unit": "GCUPS", "frac": per_gpu / peak,
                "traffic": traffic, "traffic_source": "static: profiles/ncu_traffic.json (dram__bytes_read + dram__bytes_write of one "
                "ncu --set full capture of this workload's dominant kernel, scaled to the launch size); not re-measured per run",
                "peak_source": "N_SM*128*f_SM*W/I_cell with f_SM = " + ("sm_max_mhz of MEASURED_PEAKS.json" if "sm_max_mhz" in peaks
                                                                          else "1965 MHz (fallback: MEASURED_PEAKS.json absent)"),
                "i_cell": cfg["i_cell"], "cells_per_thread_instr": width, "n_sm": n_sm, "f_ghz": f_ghz}
    if clocks.get("sm_mhz"):
        cyc_peak = n_sm * 128 * clocks["sm_mhz"] / 1e3 * width / cfg["i_cell"]
        roofline["frac_at_measured_clock"] = per_gpu / cyc_peak
    if kernel_cycles > 0:   # cycle-based fraction: algorithmic thread-instructions / issue slots the launch had
        roofline["frac_cycle_based"] = (cells * cfg["i_cell"] / width) / (float(kernel_cycles) * n_sm * 128)
        roofline["kernel_sm_cycles"] = int(kernel_cycles)

    if rank == 0:
        line = {"metric": "GCUPS", "value": value, "unit": "GCUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": median_ms, "ms_per_step_mean": total_ms / args.steps, "value_mean": value_mean, "higher_is_better": True, "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": workload_config(args, cfg, n if not strong else cfg["pairs"]),
                "variant": variant, "e2e_host_format": args.host_format,
                "roofline": roofline,
                # h2d_bytes_per_step: what crossed the bus (library counter); host_input_bytes_per_step: the host arrays handed to
                # run_batch.  They differ when the library packs large byte pools into the 2-bit layout on the host, inside the
                # timed call (hostpack.cpp: single-device jobs, off under torchrun)
                "e2e": {"value": e2e_value, "unit": "GCUPS", "h2d_bytes_per_step": int(rep.h2d_bytes) * world,
                        "d2h_bytes_per_step": int(rep.d2h_bytes) * world, "steps": e2e_steps,
                        "host_input_bytes_per_step": int(sum((hp.packed if hp.packed is not None else hp.codes).nbytes for hp in (host_q, host_s))) * world,
                        "host_pack": W.host_pack_info()},
                "gpu_launches": launches, "clocks": clocks, "wall_s_timed_region": wall}
        if e2e_packed:
            line["e2e_packed2_host"] = e2e_packed
        if sharded:
            line["e2e_shard_api"] = sharded
        if not args.no_cpu_baseline and world == 1:   # the CPU baseline is timed on rank 0 at N = 1 only
            rate, threads, pairs, dt = cpu_sample(cfg)
            line["cpu_baseline"] = {"value": rate, "unit": "GCUPS", "cores": threads, "kind": "port",
                                    "sample": f"{pairs} pairs of {L if L else 'pareto(cap 6000)'} bp ({dt:.1f} s), oracle/wsoracle.c with OpenMP"}
        print(json.dumps(line))
    batch.close()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
