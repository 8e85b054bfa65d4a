"""N > 1 host logic on CPU: world_size-2 gloo processes shard the targets, evaluate
their range (the CPU oracle stands in for the CUDA evaluator: no GPU here) and
all-gather; the result must equal the single-process evaluation bit for bit."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

from paper_2507_00156_b200.sharding import shard_bounds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_bounds_partition():
    for M in (0, 1, 7, 504, 1001):
        for world in (1, 2, 3, 8):
            rngs = [shard_bounds(M, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
            sizes = [b - a for a, b in rngs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2507_00156_b200.sharding import evaluate_sharded, max_over_ranks
    from workloads.configs import config1

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    blk = config1(inv_h=8, per_class=11)  # M = 77: uneven shards

    def oracle_fn(sx, sn, sw, f, q, ty, tb, tx, h, rho, mode=3):
        u, v = oracle.evaluate(*(a.numpy() for a in (sx, sn, sw, f, q, ty, tb, tx)), h, rho, mode=mode)
        return torch.from_numpy(u), torch.from_numpy(v)

    arrs = [torch.from_numpy(a) for a in blk.arrays()]
    u, v = evaluate_sharded(*arrs, blk.h, blk.rho, evaluate_fn=oracle_fn)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        np.save(os.path.join(out_dir, "u.npy"), u.numpy())
        np.save(os.path.join(out_dir, "v.npy"), v.numpy())
        np.save(os.path.join(out_dir, "t.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shard_and_gather(tmp_path):
    import torch.multiprocessing as mp

    import oracle
    from workloads.configs import config1

    oracle.build()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    blk = config1(inv_h=8, per_class=11)
    u_ref, v_ref = oracle.evaluate_block(blk)
    np.testing.assert_array_equal(np.load(tmp_path / "u.npy"), u_ref)
    np.testing.assert_array_equal(np.load(tmp_path / "v.npy"), v_ref)
    assert float(np.load(tmp_path / "t.npy")[0]) == 2.0  # max over ranks


def test_morton_order_is_a_local_permutation():
    """ranks take contiguous ranges of Morton-sorted targets.  The order is a
    permutation, and consecutive targets in it are far closer than in a random order."""
    import torch

    from paper_2507_00156_b200.sharding import morton_order
    from workloads.configs import config2

    blk = config2(inv_h=16)
    x = torch.from_numpy(blk.tgt_xyz)
    p = morton_order(x)
    assert sorted(p.tolist()) == list(range(blk.M))
    step = lambda perm: float((x[:, perm[1:]] - x[:, perm[:-1]]).norm(dim=0).mean())
    assert step(p) < 0.25 * step(torch.arange(blk.M))  # config 2 lists nodes, then a random shell


def _bench_worker(rank, world, port, out_dir):
    """bench.py's multi-rank arm: its step goes through sharding.evaluate_sharded on ONE
    target set (the rank-0 seed on every rank) and gathers the full field."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench
    import oracle
    from paper_2507_00156_b200 import sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    calls = []
    real = sharding.evaluate_sharded

    def spy(*a, **kw):
        calls.append(kw.get("gather"))
        return real(*a, **kw)

    sharding.evaluate_sharded = spy
    blk = bench.make_workload(1, 16, 0)  # what run_eval builds on every rank (strong scaling)
    seen = []

    def oracle_fn(sx, sn, sw, f, q, ty, tb, tx, h, rho, mode=3):
        seen.append(int(tb.shape[0]))
        u, v = oracle.evaluate(*(a.numpy() for a in (sx, sn, sw, f, q, ty, tb, tx)), h, rho, mode=mode)
        return torch.from_numpy(u), torch.from_numpy(v)

    u, v = bench.sharded_step([torch.from_numpy(a) for a in blk.arrays()], blk, oracle_fn)
    assert calls == [True] and seen == [sharding.shard_bounds(blk.M, rank, world)[1]
                                        - sharding.shard_bounds(blk.M, rank, world)[0]]
    if rank == 0:
        np.save(os.path.join(out_dir, "bu.npy"), u.numpy())
        np.save(os.path.join(out_dir, "bv.npy"), v.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_bench_multirank_arm_goes_through_evaluate_sharded(tmp_path):
    import torch.multiprocessing as mp

    import oracle
    sys.path.insert(0, ROOT)
    import bench

    oracle.build()
    port = _free_port()
    mp.spawn(_bench_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    blk = bench.make_workload(1, 16, 0)
    u_ref, v_ref = oracle.evaluate_block(blk)
    np.testing.assert_array_equal(np.load(tmp_path / "bu.npy"), u_ref)
    np.testing.assert_array_equal(np.load(tmp_path / "bv.npy"), v_ref)


def _nodes_worker(rank, world, port, out_dir):
    """sharding.evaluate_nodes_sharded: each rank's partial (here a stand-in: the oracle over this
    rank's share of the sources, chi q0 only on rank 0 -- the same linearity the CUDA shards use)
    is all-reduced into the full field on every rank."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2507_00156_b200.sharding import evaluate_nodes_sharded, shard_bounds
    from workloads.configs import config5, node_block

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    blk = node_block(config5(inv_h=8))
    calls = []

    def partial_fn(sx, sn, sw, f, q, h, rho, mode, si, sc):
        calls.append((si, sc))
        a, b = shard_bounds(blk.N, si, sc)
        w = np.zeros(blk.N)
        w[a:b] = blk.src_weight[a:b]  # this shard's sources (the rest weigh 0: add exactly 0)
        u, v = oracle.evaluate(blk.src_xyz, blk.src_normal, w, blk.f, blk.q, blk.tgt_xyz, blk.tgt_b,
                               blk.tgt_x0_density, h, rho, mode=mode, localized=True)
        if si != 0:
            v = v - 0.5 * blk.q  # chi q0 once, on shard 0
        return torch.from_numpy(u), torch.from_numpy(v)

    t = lambda a: torch.from_numpy(a)
    u, v = evaluate_nodes_sharded(t(blk.src_xyz), t(blk.src_normal), t(blk.src_weight), t(blk.f), t(blk.q), blk.h,
                                  blk.rho, evaluate_fn=partial_fn)
    assert calls == [(rank, world)]
    np.save(os.path.join(out_dir, f"nu{rank}.npy"), u.numpy())
    np.save(os.path.join(out_dir, f"nv{rank}.npy"), v.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_nodes_allreduce(tmp_path):
    import torch.multiprocessing as mp

    import oracle
    from workloads.configs import config5, node_block

    oracle.build()
    port = _free_port()
    mp.spawn(_nodes_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    blk = node_block(config5(inv_h=8))
    u_ref, v_ref = oracle.evaluate_block(blk, localized=True)
    for r in range(2):  # every rank holds the full field
        u, v = np.load(tmp_path / f"nu{r}.npy"), np.load(tmp_path / f"nv{r}.npy")
        assert np.abs(u - u_ref).max() <= 1e-13 * np.abs(u_ref).max()
        assert np.abs(v - v_ref).max() <= 1e-13 * np.abs(v_ref).max()
