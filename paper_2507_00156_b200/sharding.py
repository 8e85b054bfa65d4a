"""Multi-GPU target sharding.

Targets are independent (the paper's own parallelism is a
loop over targets), so one process per GPU evaluates a contiguous range of
the targets against all sources.  There is no data-path collective; the only
collectives are an optional all-gather of the outputs and the max-over-ranks
timing reduction of bench.py.
"""
from __future__ import annotations

from typing import Callable, Optional


def shard_bounds(M: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) target range of `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world) or M < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(M, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def slice_targets(tgt_xyz, tgt_b, tgt_x0_density, start: int, stop: int):
    """Contiguous copies of one target range (SoA rows keep their layout)."""
    return (tgt_xyz[:, start:stop].contiguous(), tgt_b[start:stop].contiguous(),
            tgt_x0_density[:, start:stop].contiguous())


def gather_columns(local, M: int, group=None):
    """All-gather per-rank (R, m_r) column blocks into the full (R, M) array (rank order)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_bounds(M, r, world) for r in range(world)]
    mmax = max(b - a for a, b in sizes)
    buf = torch.zeros((local.shape[0], mmax), dtype=local.dtype, device=local.device)
    buf[:, :local.shape[1]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:, :b - a] for p, (a, b) in zip(parts, sizes)], dim=1)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (bench.py's device time), 1 collective outside the data path."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def evaluate_sharded(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho, mode=3,
                     group=None, gather: bool = True, evaluate_fn: Optional[Callable] = None):
    """Evaluate this rank's target range against all sources; optionally all-gather.

    `evaluate_fn` defaults to the CUDA path (paper_2507_00156_b200.evaluate); it
    receives the same arguments with the local target arrays."""
    import torch.distributed as dist

    if evaluate_fn is None:
        from . import evaluate as evaluate_fn
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    M = int(tgt_b.shape[0])
    a, b = shard_bounds(M, rank, world)
    ty, tb, tx = slice_targets(tgt_xyz, tgt_b, tgt_x0_density, a, b)
    u, v = evaluate_fn(src_xyz, src_normal, src_weight, f, q, ty, tb, tx, h, rho, mode=mode)
    if not gather or world == 1:
        return u, v
    return (None if u is None else gather_columns(u, M, group)), (None if v is None else gather_columns(v, M, group))
