"""Multi-rank (world_size 2, gloo, CPU) coverage of the sequence-sharded
path: the partition, the per-rank synthetic inputs, the stats gather and the
max-over-ranks timing rule, and -- through the oracle -- that sharding
sequences across ranks leaves every sequence's results unchanged (units of
different sequences never interact)."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2510_01290_b200 import shard
from paper_2510_01290_b200.synth import band_script

SEED = 0x71534B56


def test_seq_range_partitions():
    for n in (1, 5, 32, 33):
        for w in (1, 2, 3, 8):
            got = [shard.seq_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(e - b for b, e in got) - min(e - b for b, e in got) <= 1
    with pytest.raises(ValueError):
        shard.seq_range(4, 2, 2)


def _cfg(num_seqs, script):
    return O.RunConfig(num_seqs=num_seqs, units_per_seq=2, num_q_heads=4, head_dim=32, tau=16,
                       group_size=8, block_size=4, budget=24, levels=(8, 4, 2), psi_bits=(4, 8, 2),
                       max_gen_len=80, script=script)


def _run_oracle(cfg, unit0, steps):
    run = O.OracleRun(cfg)
    outs = []
    for t in range(steps):
        q, k, v = O.synth_step(SEED, cfg.units_per_seq, cfg.tau, cfg.num_seqs * cfg.units_per_seq,
                               cfg.num_q_heads, cfg.head_dim, t, unit0=unit0)
        out, _ = run.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
        outs.append(out)
    run.finish()
    dumps = [{w: run.dump(s, w) for w in ("tables", "segments", "events", "metrics")}
             for s in range(cfg.num_seqs)]
    return np.stack(outs), dumps


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        global_seqs = 4
        script = band_script(SEED, global_seqs, 8, 3, 300)
        b, e = shard.seq_range(global_seqs, rank, world)
        cfg = _cfg(e - b, shard.shard_script(script, rank, world))
        unit0 = shard.unit_offset(global_seqs, cfg.units_per_seq, rank, world)
        out, dumps = _run_oracle(cfg, unit0, 80)
        stats = shard.gather_stats([float(rank), float(e - b), float(out.sum())])
        tmax = shard.max_over_ranks(1.5 + rank)
        with open(os.path.join(result_dir, f"rank{rank}.json"), "w") as f:
            json.dump({"range": [b, e], "stats": stats, "tmax": tmax, "dumps": dumps,
                       "out": out.tolist()}, f)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_sharding_matches_single_rank(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    # stats gather: every rank sees every rank's vector, in rank order
    for r in res:
        assert [s[0] for s in r["stats"]] == [0.0, 1.0]
        assert sum(s[1] for s in r["stats"]) == 4
        assert r["tmax"] == 2.5
    # the whole batch on one rank
    script = band_script(SEED, 4, 8, 3, 300)
    full_out, full_dumps = _run_oracle(_cfg(4, script), 0, 80)
    sharded_dumps = res[0]["dumps"] + res[1]["dumps"]
    assert sharded_dumps == full_dumps
    sharded_out = np.concatenate([np.array(r["out"]) for r in res], axis=1)
    assert np.array_equal(sharded_out, full_out)


def test_bench_workload_weak_and_strong_split():
    """bench.py's per-rank workload: weak scaling gives every rank --seqs
    sequences of a world * seqs global batch; strong scaling splits --seqs
    over the ranks; in both the ranks' scripts tile the global script."""
    import argparse
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    for mode, world in (("weak", 2), ("strong", 2), ("strong", 8)):
        a = argparse.Namespace(seqs=32, layers=2, kv_heads=2, q_per_kv=4, head_dim=64, tau=128, block_size=16,
                               budget=1024, max_gen=1024, psi=(4, 4, 2), pT_permille=100, scaling=mode)
        cfgs = [bench.workload(a, r, world) for r in range(world)]
        gs = bench.global_seqs(a, world)
        assert gs == (32 * world if mode == "weak" else 32)
        assert sum(c.num_seqs for c in cfgs) == gs
        full = band_script(bench.SEED, gs, 1024 // 128 + 2, 3, 100)
        assert [s for c in cfgs for s in c.script] == [list(s) for s in full]
