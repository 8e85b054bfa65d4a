"""Multi-GPU sharding.

General targets are independent (the paper's own parallelism
is a loop over targets), so one process per GPU evaluates a contiguous range
of the Morton-sorted targets against all sources, and an optional all-gather
assembles the field (evaluate_sharded).  Node targets (evaluate_nodes_sharded)
split the symmetric kernel's block-pair items instead, and one all-reduce sums
the ranks' partial fields.  bench.py adds a max-over-ranks timing reduction.
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


def morton_order(tgt_xyz):
    """Permutation sorting the targets by a 30-bit Morton key of their box-normalised
    coordinates (10 bits per axis), so contiguous ranges of it are spatially compact
    (contiguous ranges of Morton-sorted targets).  Index bookkeeping
    only; ties keep input order (stable sort)."""
    import torch

    x = tgt_xyz
    lo = x.min(dim=1, keepdim=True).values
    ext = (x.max(dim=1, keepdim=True).values - lo).clamp_min(1e-300)
    q = ((x - lo) / ext * 1023.0).clamp(0, 1023).to(torch.int64)

    def spread(v):  # 10 bits -> every third bit
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        return (v | (v << 2)) & 0x09249249

    key = spread(q[0]) | (spread(q[1]) << 1) | (spread(q[2]) << 2)
    return torch.sort(key, stable=True).indices


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
                     group=None, gather: bool = True, evaluate_fn: Optional[Callable] = None,
                     morton: bool = True):
    """Evaluate this rank's target range against all sources; optionally all-gather.

    With `morton` the ranges are contiguous in Morton order of the targets (each rank gets
    a spatially compact set, so its 32-target warps keep tight boxes); the gathered result
    is returned in the caller's order.  Without `gather`, a rank returns its own columns
    (in Morton order when `morton`; `morton_order` gives the permutation).
    `evaluate_fn` defaults to the CUDA path (paper_2507_00156_b200.evaluate); it
    receives the same arguments with the local target arrays."""
    import torch
    import torch.distributed as dist

    if evaluate_fn is None:
        from . import evaluate as evaluate_fn
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    M = int(tgt_b.shape[0])
    a, b = shard_bounds(M, rank, world)
    if morton and world > 1:
        perm = morton_order(tgt_xyz)
        idx = perm[a:b]
        ty, tb, tx = (tgt_xyz[:, idx].contiguous(), tgt_b[idx].contiguous(), tgt_x0_density[:, idx].contiguous())
    else:
        perm = None
        ty, tb, tx = slice_targets(tgt_xyz, tgt_b, tgt_x0_density, a, b)
    u, v = evaluate_fn(src_xyz, src_normal, src_weight, f, q, ty, tb, tx, h, rho, mode=mode)
    if not gather or world == 1:
        return u, v

    def full(local):
        if local is None:
            return None
        g = gather_columns(local, M, group)
        if perm is None:
            return g
        out = torch.empty_like(g)
        out[:, perm.to(g.device)] = g
        return out

    return full(u), full(v)


def evaluate_nodes_sharded(src_xyz, src_normal, src_weight, f, q, h, rho, mode=3, group=None,
                           evaluate_fn: Optional[Callable] = None, options=None, workspace=None, stream=None):
    """The node-target evaluation (stokes_er_eval_nodes) split across the ranks of `group`.

    Node targets make the far sum symmetric: one block-pair item adds to the
    nodes of BOTH blocks, so the work does not split by target ranges.  Rank r computes shard r
    of the evaluation -- a contiguous 1/world of the symmetric kernel's items and of the
    neighbour units' target groups (options.shard_index / shard_count) -- whose partial u, v
    (chi q0 only on rank 0) sum over the ranks to the evaluation: ONE all-reduce (sum) of the
    48 N bytes, the path's exchange step.  Every rank returns the full u, v.
    `evaluate_fn(src_xyz, src_normal, src_weight, f, q, h, rho, mode, shard_index, shard_count)`
    defaults to the CUDA path (paper_2507_00156_b200.evaluate_nodes)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if evaluate_fn is None:
        from . import Options, evaluate_nodes

        def evaluate_fn(sx, sn, sw, ff, qq, hh, rr, md, si, sc):
            opt = options if options is not None else Options()
            opt.shard_index, opt.shard_count = si, sc
            return evaluate_nodes(sx, sn, sw, ff, qq, hh, rr, mode=md, workspace=workspace, stream=stream,
                                  options=opt)
    u, v = evaluate_fn(src_xyz, src_normal, src_weight, f, q, h, rho, mode, rank, world)
    if world > 1:
        for t in (u, v):
            if t is not None:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return u, v
