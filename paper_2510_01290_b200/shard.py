"""Sequence sharding across ranks.

Units are independent but a sequence's units must stay
together: its thought label averages sparsity over its own units
(sim.cpp:717-722).  So the batch is cut into contiguous blocks of whole
sequences, one block per rank, with no collective on the data path.  The only
collectives are end-of-run gathers of per-rank statistics and the max-over-
ranks of timings; both go through torch.distributed (NCCL over NVLink on the
GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def seq_range(global_seqs: int, rank: int, world: int) -> Tuple[int, int]:
    """[begin, end) of the global sequences owned by `rank` (contiguous blocks;
    the first global_seqs % world ranks get one extra sequence)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(global_seqs, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def unit_offset(global_seqs: int, units_per_seq: int, rank: int, world: int) -> int:
    """Global index of the rank's first unit (feeds tkv_synth_inputs' unit0)."""
    return seq_range(global_seqs, rank, world)[0] * units_per_seq


def shard_script(script: Sequence[Sequence[int]], rank: int, world: int) -> List[List[int]]:
    """The scripted thought bands of the rank's sequences."""
    b, e = seq_range(len(script), rank, world)
    return [list(s) for s in script[b:e]]


def gather_stats(values: Sequence[float], device=None) -> List[List[float]]:
    """All-gather one fixed-length float vector per rank (rank order)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [t.tolist()]
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over ranks (the bench's timing rule)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_outputs(out, global_seqs: int, units_per_seq: int):
    """Verify mode: all-gather every rank's attention outputs
    [its units, rows, d] into the global batch [global_seqs * units_per_seq,
    rows, d] on every rank (NCCL over NVLink on the GPU box; gloo needs host
    tensors, so the gather goes through the CPU there).  Ranks hold
    contiguous sequence blocks (seq_range), padded to the largest block for
    the collective."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return out
    world = dist.get_world_size()
    sizes = [(e - b) * units_per_seq for b, e in (seq_range(global_seqs, r, world) for r in range(world))]
    width = max(sizes)
    dev = out.device if dist.get_backend() == "nccl" else torch.device("cpu")
    pad = torch.zeros((width,) + tuple(out.shape[1:]), dtype=out.dtype, device=dev)
    pad[: out.shape[0]] = out.to(dev)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:n] for p, n in zip(parts, sizes)]).to(out.device)
