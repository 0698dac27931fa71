"""CPU-only tests: the C-ABI library loads and exports what include/wsb200.h declares, host-side helpers, API types,
the shard planner, and the multi-rank (gloo, world_size 2) sharding logic.  No kernel is launched here."""
import os
import re
import sys

import numpy as np
import pytest

import paper_2205_07610_b200 as W
from paper_2205_07610_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "wsb200.h")).read()
    declared = set(re.findall(r"^(?:const char\*|int|int64_t|void)\s+(wsb_[a-z0-9_]+)\(", header, re.M))
    assert len(declared) >= 19
    lib = N.load()
    missing = [name for name in declared if not hasattr(lib, name)]
    assert not missing, missing
    assert set(N.EXPORTED_SYMBOLS) == declared
    assert b"sm_100a" in lib.wsb_version()
    assert lib.wsb_strerror(0) == b"ok" and b"range" in lib.wsb_strerror(N.WSB_E_RANGE)


def test_no_cpu_fallback_without_device():
    if N.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(W.DeviceError):
        N.Context(0)
    q = W.encode_sequence("q", "ACGT")
    with pytest.raises(W.DeviceError):
        W.engine_score(q, q, W.AlignConfig("global", "affine"), W.ScoringScheme())


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2205_07610_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".inl", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "wsoracle" not in text, f


def test_merged_state_exact_matches_reference_rule():
    # pkg/tests/test_engine.py:66-69 and engine.py:71-94
    assert W.merged_state_exact(W.ScoringScheme(2, -1, 2, 1, "affine"))
    assert not W.merged_state_exact(W.ScoringScheme(2, -9, 2, 1, "affine"))
    for ma, mi, a, b in [(3, -2, 4, 1), (1, -3, 2, 2), (5, -4, 10, 1), (2, -1, 1, 3), (1, -1, 0, 0), (1, 2, 1, 1)]:
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            sch = W.ScoringScheme(ma, mi, a, b, "affine")
        worst = min(mi, ma)
        want = not (ma < mi or a + b < -worst or 2 * b < -worst)
        assert W.merged_state_exact(sch) == want, (ma, mi, a, b)


def test_range_predicates():
    sch = W.ScoringScheme(2, -1, 2, 1, "affine")
    assert W.f16_range_ok(sch, 150, 150) and W.f16_range_ok(sch, 250, 250) and W.f16_range_ok(sch, 510, 510)
    assert not W.f16_range_ok(sch, 600, 600)
    assert W.packed_range_ok(sch, 4000, 4000) and not W.packed_range_ok(sch, 5000, 5000)
    with pytest.raises(W.LengthOverflow):
        W.check_length_bounds(2 ** 28, 2 ** 28, sch)


def test_core_types_follow_the_reference():
    s = W.encode_sequence("x", "acgtNn-A")
    assert s.codes.tolist() == [0, 1, 2, 3, 0, 0, 0, 0] and s.flags.tolist() == [False] * 4 + [True] * 3 + [False]
    assert s.device_codes().tolist() == [0, 1, 2, 3, 4, 4, 4, 0]
    assert W.decode_sequence(s) == "ACGTNNNA" and s.has_ambiguous
    # 2-bit packing, low bits first (pkg/tests/test_core.py:59-62)
    assert W.encode_sequence("y", "ACGT").data == bytes([0b11100100])
    assert W.encode_sequence("y", "TA").data == bytes([0b0011])
    with pytest.raises(W.EmptySequence):
        W.encode_sequence("e", "")
    assert W.validate_config(W.AlignConfig("local", "affine"), W.ScoringScheme()).nu == 0
    assert W.validate_config(W.AlignConfig("global", "affine"), W.ScoringScheme()).nu == W.NEG_INF
    with pytest.raises(W.ConfigMismatch):
        W.validate_config(W.AlignConfig("global", "linear"), W.ScoringScheme())
    with pytest.raises(W.ConfigMismatch):
        W.ScoringScheme(2, -1, -1, 1)
    assert W.merge_ops([("M", 2), ("M", 1), ("I", 0), ("D", 3)]) == [("M", 3), ("D", 3)]
    assert W.gap_cost(W.ScoringScheme(), 3) == 4 and W.gap_cost(W.ScoringScheme(2, -1, 2, 2, "linear"), 3) == 6
    q, t = W.encode_sequence("q", "ACGT"), W.encode_sequence("t", "AGT")
    res = W.AlignmentResult(5, 0, 4, 0, 3, [("M", 1), ("I", 1), ("M", 2)])
    assert W.rescore_alignment(res, q, t, W.ScoringScheme(2, -1, 1, 1, "linear")) == 5
    assert W.cigar_string(res) == "1M1I2M"
    assert W.auto_tuning(150) == W.EngineTuning(32, 8) and W.auto_tuning(10_000).cols_per_lane == 16
    with pytest.raises(ValueError):
        W.EngineTuning(lanes=5)


def test_resolve_workers_and_devices(monkeypatch):
    monkeypatch.delenv("WAVESEQ_WORKERS", raising=False)
    assert W.resolve_workers(3) == 3 and W.resolve_workers(0) == (os.cpu_count() or 1)
    monkeypatch.setenv("WAVESEQ_WORKERS", "5")
    assert W.resolve_workers(3) == 5
    monkeypatch.setenv("WAVESEQ_WORKERS", "x")
    with pytest.raises(ValueError):
        W.resolve_workers()
    monkeypatch.delenv("WAVESEQ_DEVICES", raising=False)
    assert W.resolve_devices() == [0] and W.resolve_devices(4) == [0, 1, 2, 3] and W.resolve_devices([2, 5]) == [2, 5]
    monkeypatch.setenv("WAVESEQ_DEVICES", "8")
    assert W.resolve_devices() == list(range(8))


def _skewed_lengths(rng, n):
    u = rng.random(n)
    L = np.minimum(100_000, np.floor(100 / (1 - u))).astype(np.int32)
    v = rng.uniform(0.8, 1.25, n)
    return L, np.clip(np.round(L * v), 100, 100_000).astype(np.int32)


def test_plan_shards_balances_cells():
    rng = np.random.default_rng(220507615)
    n = 20_000
    m, nn = _skewed_lengths(rng, n)     # cfg5 length law
    idx = np.arange(n, dtype=np.int32)
    shard_of, cells = N.plan_shards(m, nn, idx, idx, 8)
    total = (m.astype(np.int64) * nn).sum()
    assert cells.sum() == total and set(np.unique(shard_of)) <= set(range(8))
    biggest = int((m.astype(np.int64) * nn).max())
    assert cells.max() - cells.min() <= biggest          # LPT: spread bounded by the largest item
    assert cells.max() <= total / 8 + biggest
    # uniform batches split into contiguous equal blocks
    shard_of, cells = N.plan_shards(np.full(10, 150, np.int32), np.full(10, 150, np.int32), np.arange(10, dtype=np.int32),
                                    np.arange(10, dtype=np.int32), 2)
    assert shard_of.tolist() == [0] * 5 + [1] * 5 and cells.tolist() == [5 * 22500] * 2
    # determinism: the plan is a pure function of the job
    again, _ = N.plan_shards(m, nn, idx, idx, 8)
    shard_of8, _ = N.plan_shards(m, nn, idx, idx, 8)
    assert (again == shard_of8).all()


def test_batch_job_validation_and_pool():
    qs = [W.encode_sequence("a", "ACGT"), W.encode_sequence("b", "GGN")]
    pool = W.SequencePool.from_sequences(qs)
    assert pool.codes.tolist() == [0, 1, 2, 3, 2, 2, 4] and pool.off.tolist() == [0, 4] and pool.len.tolist() == [4, 3]
    assert W.decode_sequence(pool[1]) == "GGN"
    assert W.all_pairs(qs, qs) == [(0, 0), (0, 1), (1, 0), (1, 1)]
    with pytest.raises(ValueError):
        W.all_pairs([], qs)
    cfg, sch = W.AlignConfig("global", "affine"), W.ScoringScheme()
    with pytest.raises(ValueError):
        W.BatchJob(qs, qs, [], cfg, sch)
    with pytest.raises(ValueError):
        W.BatchJob(qs, qs, [(0, 2)], cfg, sch)
    job = W.BatchJob(qs, qs, [(1, 0)], cfg, sch)
    assert job._pair_array.tolist() == [[1, 0]]
    u = W.SequencePool.from_uniform(np.zeros((3, 5), np.uint8))
    assert len(u) == 3 and u.off.tolist() == [0, 5, 10]


def _rank_main(rank, world, port, out_dir):
    """One rank of the multi-GPU sharding protocol on CPU: plan -> own shard -> gather of shard summaries (gloo)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)                       # every rank builds the same job
    m, nn = _skewed_lengths(rng, 4000)
    idx = np.arange(4000, dtype=np.int32)
    shard_of, cells = N.plan_shards(m, nn, idx, idx, world)
    mine = np.nonzero(shard_of == rank)[0]
    my_cells = int((m[mine].astype(np.int64) * nn[mine]).sum())
    assert my_cells == int(cells[rank])
    # stand-in for the per-rank GPU results: a checksum per pair, scattered back by pair index after the gather
    local = torch.zeros(4000, dtype=torch.int64)
    local[torch.from_numpy(mine)] = torch.from_numpy((m[mine].astype(np.int64) * 31 + nn[mine]))
    dist.all_reduce(local, op=dist.ReduceOp.SUM)         # disjoint shards: the sum is the gather
    want = torch.from_numpy(m.astype(np.int64) * 31 + nn)
    assert torch.equal(local, want)
    t = torch.tensor([float(my_cells)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        total = int((m.astype(np.int64) * nn).sum())
        with open(os.path.join(out_dir, "ok"), "w") as fh:
            fh.write(f"{t.item() / (total / world):.4f}")
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_over_gloo(tmp_path):
    import torch.multiprocessing as mp
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    imbalance = float(open(tmp_path / "ok").read())
    assert 1.0 <= imbalance < 1.6   # the skewed law has a few 10^10-cell pairs; LPT keeps the max shard near the mean


def test_pinned_result_buffers_fall_back_to_pageable_memory_without_a_device():
    from paper_2205_07610_b200 import _native as N
    a = N.pinned_empty(1000)
    assert a.shape == (1000,) and a.dtype == np.int32
    a[:] = 7                      # writable either way
    assert int(a.sum()) == 7000


def test_bench_workload_generators_are_seeded_and_shaped():
    import bench
    (qc, qo, ql), (sc, so, sl) = bench.make_pareto(5000, 1)
    assert ql.min() >= 100 and ql.max() <= 100_000 and sl.min() >= 100 and sl.max() <= 100_000
    assert len(qc) == int(ql.sum()) and qo[-1] + ql[-1] == len(qc) and qc.max() <= 3
    (qc2, _, ql2), _ = bench.make_pareto(5000, 1)
    assert (ql == ql2).all() and (qc == qc2).all()
    q, s = bench.make_batch(dict(pairs=64, length=250, related=0.5), 3)
    assert q.shape == s.shape == (64, 250)
    assert (q[::2] == s[::2]).mean() > 0.5 and (q[1::2] == s[1::2]).mean() < 0.4


def test_packed_pool_round_trip_matches_reference_layout():
    """2-bit pool layout = the reference's Sequence.data (core.py:78-87): low bits first, flagged symbols stored as 0."""
    from paper_2205_07610_b200.pool import SequencePool
    rng = np.random.default_rng(9)
    lens = rng.integers(1, 40, 50).astype(np.int32)
    off = np.zeros(50, np.int64); off[1:] = np.cumsum(lens[:-1])
    codes = rng.integers(0, 4, int(lens.sum())).astype(np.uint8)
    codes[[3, 17, 100]] = 4
    pool = SequencePool(codes, off, lens)
    packed = pool.to_packed()
    assert packed.packed.nbytes == (len(codes) + 3) // 4 and list(packed.flag_pos) == [3, 17, 100]
    assert packed.packed[0] == (codes[0] | (codes[1] << 2) | (codes[2] << 4) | (0 << 6))   # symbol 3 is flagged -> 0
    assert (packed.codes == codes).all()
    seq = packed[5]
    assert len(seq) == lens[5]


def test_wire_formats_and_bench_conventions(tmp_path):
    """cigar_string / write_results_tsv (io.py:80-110) and median_rate / theoretical_peak (bench.py:30-43) conventions."""
    import paper_2205_07610_b200 as W
    r = W.AlignmentResult(score=5, q_start=0, q_end=4, s_start=0, s_end=3, ops=[("M", 1), ("I", 1), ("M", 1), ("M", 1)],
                          cells_computed=12)
    assert W.cigar_string(r) == "1M1I2M"
    assert W.cigar_string(W.AlignmentResult(3, 1, 1, 2, 2, None, 4)) == ""
    path = tmp_path / "out.tsv"
    W.write_results_tsv([("q0", "s0", r)], path)
    lines = path.read_text().splitlines()
    assert lines[0].split("\t") == list(W.TSV_HEADER) and lines[1] == "q0\ts0\t5\t0\t4\t0\t3\t1M1I2M"
    assert W.median_rate([3.0, 1.0, 2.0]) == 2.0 and W.median_rate([4.0, 1.0, 2.0, 3.0]) == 2.5
    with pytest.raises(ValueError):
        W.median_rate([])
    hw = W.HardwareModel.b200(ops_per_cell=8, cells_per_instruction=2)
    assert abs(W.theoretical_peak(hw) - 9306.24) < 0.01
    with pytest.raises(ValueError):
        W.HardwareModel(0, 1.0, 1.0)


def test_packed_traceback_fill_keeps_its_max_operand_order():
    """max_mark2 (traceback_fill16.cuh) relies on VIMNMX.S16x2's per-half "first operand won" predicates.  ptxas 12.9
    moves an immediate operand into second place WITHOUT adjusting the predicate uses (seen with the local stop test's
    zero), so the built library must not contain a predicated packed max with an immediate operand."""
    import shutil, subprocess
    lib = N.library_path() if hasattr(N, "library_path") else os.path.join(os.path.dirname(N.__file__), "libwsb200.so")
    dump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(lib) or not os.path.exists(dump):
        pytest.skip("library or cuobjdump not available")
    names = subprocess.run([dump, "-elf", lib], capture_output=True, text=True).stdout
    funcs = sorted(set(re.findall(r"_ZN3wsb16tb_fill16_kernel\w+", names)))
    assert funcs, "packed fill kernels missing from the library"
    sass = subprocess.run([dump, "-sass", *sum((["-fun", f] for f in funcs), []), lib], capture_output=True, text=True).stdout
    maxes = [ln for ln in sass.splitlines() if "VIMNMX.S16x2" in ln]
    assert len(maxes) > 100
    bad = [ln for ln in maxes if re.search(r"VIMNMX\.S16x2 R\d+, P[0-6], P[0-6], R\d+, (0x|-0x|c\[)", ln)]
    assert not bad, bad[:3]


def test_plan_stats_instruction_mix_matches_the_built_kernels():
    """EngineStats.ops_* come from a per-kernel instruction mix (csrc/wsb200.cu: op_mix_q).  Pin the packed int16 rows of
    that table to the SASS of the built library: per trip of 19 columns x 2 alignments the hot loops must hold the modelled
    number of packed max / add / lookup instructions (plus the few the hand-over and the record add)."""
    import shutil, subprocess, collections
    lib = os.path.join(os.path.dirname(N.__file__), "libwsb200.so")
    dump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(lib) or not os.path.exists(dump):
        pytest.skip("library or cuobjdump not available")

    def hot_loop(pattern, op, min_hits):
        names = subprocess.run([dump, "-elf", lib], capture_output=True, text=True).stdout
        fn = sorted(f for f in set(re.findall(r"_ZN3wsb\w+", names)) if pattern in f)[0]
        sass = subprocess.run([dump, "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
        ins = [(int(m.group(1), 16), m.group(2), m.group(0)) for m in
               re.finditer(r"/\*([0-9a-f]{4,5})\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_.]+)[^;]*;", sass)]
        best = None
        for a, o, l in ins:
            t = re.search(r"BRA\S*\s+(?:\S+,\s*)?0x([0-9a-f]+)", l) if o.startswith("BRA") else None
            if t and int(t.group(1), 16) < a:
                body = [x for x in ins if int(t.group(1), 16) <= x[0] <= a]
                if sum(1 for x in body if x[1].startswith(op)) >= min_hits and (best is None or len(body) < len(best)):
                    best = body
        assert best, pattern
        return collections.Counter(o for _, o, _ in best)

    cells = 2 * 19
    c = hot_loop("s16_local_short_kernelILi8ELi19ELi1ELi4ELi2ELi1E", "VIMNMX3", 40)       # local, merged affine: 5 / 6 / 2 quarters
    n_max = sum(v for k, v in c.items() if k.startswith(("VIMNMX", "VIADDMNMX")))
    n_add = sum(v for k, v in c.items() if k.startswith("VIADD.16"))
    assert cells * 5 / 4 <= n_max <= cells * 5 / 4 + 4, c
    assert cells * 6 / 4 <= n_add <= cells * 6 / 4 + 2, c
    assert c["PRMT"] == cells * 2 // 4
    c = hot_loop("s16_global_short_kernelILi8ELi19ELi0ELb0ELi1ELi1E", "VIMNMX3", 15)      # global, linear: 2 / 4 / 2 quarters
    n_max = sum(v for k, v in c.items() if k.startswith(("VIMNMX", "VIADDMNMX")))
    n_add = sum(v for k, v in c.items() if k.startswith("VIADD.16"))
    assert cells * 2 / 4 <= n_max <= cells * 2 / 4 + 3, c
    assert cells * 4 / 4 <= n_add <= cells * 4 / 4 + 3, c
    assert c["PRMT"] == cells * 2 // 4
