"""The sequence-sharded CUDA path at world size 2 on one GPU:
two gloo ranks each decode their contiguous block of sequences on cuda:0
(synthetic inputs of their own global units, tkv_synth_inputs' unit0), the
verify-mode gather (shard.gather_outputs) assembles the global outputs, and
every output and every sequence's cache state is bit-identical to a 1-rank
run of the whole batch."""
import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2510_01290_b200 import DecodeRun, ThinkvConfig, shard  # noqa: E402
from paper_2510_01290_b200.synth import band_script  # noqa: E402

SEED = 0x71534B56
GLOBAL_SEQS, UPS, G, D, STEPS = 5, 4, 4, 128, 300


def _cfg(seqs, script):
    return ThinkvConfig(num_seqs=seqs, units_per_seq=UPS, num_q_heads=G, head_dim=D, tau=32, group_size=16,
                        block_size=16, budget=64, levels=(16, 8, 4), max_gen_len=STEPS, script=script,
                        record_events=True)


def _decode(cfg, unit0):
    run = DecodeRun(cfg)
    dev = torch.device("cuda:0")
    q = torch.empty((cfg.units, G, D), dtype=torch.bfloat16, device=dev)
    k = torch.empty((cfg.units, D), dtype=torch.bfloat16, device=dev)
    v = torch.empty((cfg.units, D), dtype=torch.bfloat16, device=dev)
    out = torch.empty((cfg.units, G, D), device=dev)
    outs = []
    for t in range(STEPS):
        run.synth_inputs(SEED, t, q, k, v, unit0=unit0)
        run.step(q, k, v, out)
        if t % 37 == 0 or t == STEPS - 1:
            outs.append(out.clone())
    run.finish()
    return run, outs


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        script = band_script(SEED, GLOBAL_SEQS, STEPS // 32 + 2, 3, 300)
        b, e = shard.seq_range(GLOBAL_SEQS, rank, world)
        cfg = _cfg(e - b, shard.shard_script(script, rank, world))
        run, outs = _decode(cfg, shard.unit_offset(GLOBAL_SEQS, UPS, rank, world))
        gathered = [shard.gather_outputs(o, GLOBAL_SEQS, UPS).cpu() for o in outs]
        if rank == 0:
            torch.save(gathered, os.path.join(result_dir, "outs.pt"))
        state = {str(b + s): {w: run.tables(s) if w == "tables" else (run.events(s) if w == "events" else
                                                                       (run.segments(s) if w == "segments"
                                                                        else run.metrics(s)))
                              for w in ("tables", "segments", "events", "metrics")} for s in range(e - b)}
        with open(os.path.join(result_dir, f"state{rank}.json"), "w") as f:
            json.dump(state, f)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_the_single_rank_run(tmp_path):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    script = band_script(SEED, GLOBAL_SEQS, STEPS // 32 + 2, 3, 300)
    run, outs = _decode(_cfg(GLOBAL_SEQS, script), 0)
    got = torch.load(os.path.join(tmp_path, "outs.pt"))
    assert len(got) == len(outs)
    for a, b in zip(got, outs):
        assert torch.equal(a, b.cpu())
    state = {}
    for r in range(2):
        state.update(json.load(open(os.path.join(tmp_path, f"state{r}.json"))))
    assert sorted(state, key=int) == [str(s) for s in range(GLOBAL_SEQS)]
    for s in range(GLOBAL_SEQS):
        assert state[str(s)]["tables"] == run.tables(s)
        assert state[str(s)]["segments"] == run.segments(s)
        assert state[str(s)]["events"] == run.events(s)
        assert state[str(s)]["metrics"] == run.metrics(s)
