"""GPU parity of the node-target path (stokes_er_eval_nodes, csrc/sym.cuh) against the CPU oracle.

The oracle evaluates the same argument set through its general entry point: targets = the
nodes, b = 0, x0d = [n; f; q] (workloads.configs.node_block).  Tolerance as in
test_gpu_parity.py (north_star): max-norm relative <= 1e-12 per field.  The symmetric far
kernel shares each far pair's geometry between (i <- j) and (j <- i); the neighbour units own
every pair of a block pair that is not all-far.  These tests cover both owners, their
boundary (96-node block boxes), padding, ragged N, degenerate delta and determinism.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

import oracle
from workloads.configs import config2, config3, config5, node_block
from workloads.densities import ConstField, RigidField

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def ser():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2507_00156_b200 as ser

    ser._lib.load()
    return ser


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def gpu_nodes(ser, blk, mode=3, **kw):
    u, v = ser.evaluate_nodes_block(blk, mode=mode, **kw)
    return (None if u is None else u.cpu().numpy()), (None if v is None else v.cpu().numpy())


def check_nodes(ser, blk, mode=3, localized=False, idx=None, tol=TOL):
    """GPU node path on the whole node set; oracle on all nodes or on the sample `idx`."""
    u, v = gpu_nodes(ser, blk, mode=mode)
    nb = node_block(blk)
    if idx is not None:
        nb = nb.take_targets(idx)
        u = None if u is None else u[:, idx]
        v = None if v is None else v[:, idx]
    ur, vr = oracle.evaluate_block(nb, mode=mode, localized=localized)
    out = {}
    if mode & 1:
        out["u"] = rel(u, ur)
    if mode & 2:
        out["v"] = rel(v, vr)
    assert all(e <= tol for e in out.values()), out
    return out


def sample(n, k, seed=3):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, n - 1], rng.choice(n, min(k, n), replace=False)]))


@pytest.mark.parametrize("mode", [3, 1, 2])
def test_sphere_h16_full(ser, mode):
    """Config 5 at 1/h = 16 (N = 4,302): every node, every mode, against definition mode."""
    check_nodes(ser, config5(inv_h=16), mode=mode)


def test_sphere_h32_full(ser):
    """N = 17,070 (267 blocks: most block pairs are all-far, so the symmetric kernel does
    most of the work), every node against the oracle's localized mode (definition mode
    agrees with it to 6e-16, test_oracle_pins)."""
    check_nodes(ser, config5(inv_h=32), localized=True)


def test_closed_form_densities(ser):
    for f, q in ((ConstField((1.0, 0.0, 0.0)), ConstField((1.0, -2.0, 0.5))),
                 (RigidField(Omega=(0.3, -0.5, 0.7)), RigidField(U=(0.2, 0.1, -0.4), Omega=(1.0, 0.5, -0.25)))):
        blk = config5(inv_h=16)
        from workloads.configs import make_block
        from workloads.quadrature import sphere
        x, n, w = blk.src_xyz, blk.src_normal, blk.src_weight
        b2 = make_block(sphere(), blk.h, x, np.zeros(x.shape[1]), x, n, f, q, blk.rho, src=(x, n, w))
        check_nodes(ser, b2)


def test_ellipsoid_nodes_sampled(ser):
    """The ellipsoid of config 3 (trigonometric densities) at 1/h = 64: node path vs oracle on a
    sample and vs the general path (stokes_er_eval with the same node targets) everywhere."""
    blk = config3(inv_h=64)
    idx = sample(blk.N, 256)
    check_nodes(ser, blk, idx=idx)
    u, v = gpu_nodes(ser, blk)
    ug, vg = ser.evaluate_block(node_block(blk))
    assert rel(u, ug.cpu().numpy()) <= 1e-13 and rel(v, vg.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("inv_h", [64, 128])
def test_sphere_sampled_and_vs_general_path(ser, inv_h):
    blk = config5(inv_h=inv_h)
    check_nodes(ser, blk, idx=sample(blk.N, 128 if inv_h == 64 else 64))
    u, v = gpu_nodes(ser, blk)
    ug, vg = ser.evaluate_block(blk)  # config 5's own targets are its nodes
    assert rel(u, ug.cpu().numpy()) <= 1e-13 and rel(v, vg.cpu().numpy()) <= 1e-13


def test_max_size_sampled(ser):
    """BASELINE.json config 5 at 1/h = 256 (N = 1,090,854: the bench workload) in the bench's
    launch configuration; 48 sampled nodes against the definition-mode oracle."""
    blk = config5(inv_h=256)
    check_nodes(ser, blk, idx=sample(blk.N, 46, seed=7))


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 95, 96, 97, 127, 129, 383, 384, 385, 1000, 3001])
def test_ragged_node_counts(ser, n):
    """Node subsets of the 1/h = 16 sphere: partial 96-node blocks, zero-weight padding in the
    last block, a single node (the self pair only)."""
    blk = config5(inv_h=16)
    idx = np.arange(n) * 7 % blk.N
    cut = lambda a: np.ascontiguousarray(a[..., idx])
    sub = dataclasses.replace(blk, src_xyz=cut(blk.src_xyz), src_normal=cut(blk.src_normal),
                              src_weight=cut(blk.src_weight), f=cut(blk.f), q=cut(blk.q))
    check_nodes(ser, sub)


@pytest.mark.parametrize("scale", [0.02, 6.0])
def test_degenerate_delta_scales(ser, scale):
    """delta far below the node spacing (every block pair but the diagonal is all-far: the
    symmetric kernel does everything except self pairs) and far above it (no block pair is
    all-far: the neighbour units do everything)."""
    blk = config5(inv_h=16)
    check_nodes(ser, dataclasses.replace(blk, h=blk.h * scale))


@pytest.mark.parametrize("rho", [(1.0, 2.0, 5.0), (2.0, 3.5, 4.0)])
def test_other_rho(ser, rho):
    check_nodes(ser, dataclasses.replace(config5(inv_h=16), rho=tuple(rho)))


def test_duplicate_and_zero_weight_nodes(ser):
    """Coincident nodes (r = 0 between DISTINCT nodes, possibly in different blocks) and
    zero-weight nodes."""
    blk = config5(inv_h=8)
    k = 40
    cat = lambda a, b: np.ascontiguousarray(np.concatenate([a, b], axis=-1))
    dup = dataclasses.replace(blk, src_xyz=cat(blk.src_xyz, blk.src_xyz[:, :k]),
                              src_normal=cat(blk.src_normal, blk.src_normal[:, :k]),
                              src_weight=cat(blk.src_weight, 0.5 * blk.src_weight[:k]),
                              f=cat(blk.f, -blk.f[:, :k]), q=cat(blk.q, 2.0 * blk.q[:, :k]))
    w = dup.src_weight.copy()
    w[::13] = 0.0
    check_nodes(ser, dataclasses.replace(dup, src_weight=w))


def test_deterministic_and_host_entry(ser):
    """Bitwise reproducible (static CTA assignment, per-CTA accumulators, fixed-order sums), and
    the host entry point returns the device result exactly."""
    blk = config5(inv_h=32)
    a = gpu_nodes(ser, blk)
    b = gpu_nodes(ser, blk)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    uh, vh = ser.evaluate_nodes_host(blk.src_xyz, blk.src_normal, blk.src_weight, blk.f, blk.q, blk.h, blk.rho)
    np.testing.assert_array_equal(uh.numpy(), a[0])
    np.testing.assert_array_equal(vh.numpy(), a[1])


def test_modes_compose(ser):
    blk = config5(inv_h=32)
    u3, v3 = gpu_nodes(ser, blk, mode=3)
    u1, _ = gpu_nodes(ser, blk, mode=1)
    _, v2 = gpu_nodes(ser, blk, mode=2)
    assert rel(u1, u3) <= 1e-14 and rel(v2, v3) <= 1e-14


def test_errors(ser):
    import torch

    blk = config5(inv_h=8)
    arrs = [torch.from_numpy(a).cuda() for a in (blk.src_xyz, blk.src_normal, blk.src_weight, blk.f, blk.q)]
    with pytest.raises(ser.StokesERError) as ei:
        ser.evaluate_nodes(*arrs, -1.0, blk.rho)
    assert ei.value.status == 1
    with pytest.raises(ser.StokesERError) as ei:
        ser.evaluate_nodes(*arrs, blk.h, (3.0, 2.0, 4.0))
    assert ei.value.status == 1
    ws = torch.empty(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(ser.StokesERError) as ei:
        ser.evaluate_nodes(*arrs, blk.h, blk.rho, workspace=ws)
    assert ei.value.status == 3


def test_cuda_graph_capture_and_replay(ser):
    """stokes_er_eval_nodes only enqueues (memsets, kernels, CUB sort): capturable, and a
    replay equals the eager result bitwise."""
    import torch

    blk = config5(inv_h=32)
    arrs = [torch.from_numpy(a).cuda() for a in (blk.src_xyz, blk.src_normal, blk.src_weight, blk.f, blk.q)]
    N = blk.N
    out_u = torch.empty((3, N), dtype=torch.float64, device="cuda")
    out_v = torch.empty((3, N), dtype=torch.float64, device="cuda")
    ws = torch.empty(ser.nodes_workspace_bytes(N), dtype=torch.uint8, device="cuda")
    ref = ser.evaluate_nodes(*arrs, blk.h, blk.rho)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ser.evaluate_nodes(*arrs, blk.h, blk.rho, out_u=out_u, out_v=out_v, workspace=ws, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ser.evaluate_nodes(*arrs, blk.h, blk.rho, out_u=out_u, out_v=out_v, workspace=ws,
                           stream=torch.cuda.current_stream())
    out_u.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_u, ref[0]) and torch.equal(out_v, ref[1])


@pytest.mark.parametrize("inv_h,mode", [(16, 3), (32, 3), (32, 2), (16, 1)])
def test_onsurface_sharp_at_nodes(ser, inv_h, mode):
    """NEXT-1 at the nodes (stokes_er_eval_nodes_onsurface: s#, delta = 3h, cutoff 7 --
    the two-drop self block) against the oracle's sharp mode with node targets (definition:
    every pair regularized), and against the general stokes_er_eval_onsurface."""
    import torch

    blk = config5(inv_h=inv_h)
    delta = 3 * blk.h
    arrs = [torch.from_numpy(a).cuda() for a in (blk.src_xyz, blk.src_normal, blk.src_weight, blk.f, blk.q)]
    u, v = ser.evaluate_nodes_onsurface(*arrs, delta, mode=mode)
    idx = None if inv_h == 16 else sample(blk.N, 300)
    nb = node_block(blk) if idx is None else node_block(blk).take_targets(idx)
    ur, vr = oracle.evaluate_sharp(*nb.arrays(), delta, mode=mode, localized=False, cutoff=7.0)
    pick = (lambda a: a.cpu().numpy()) if idx is None else (lambda a: a.cpu().numpy()[:, idx])
    if mode & 1:
        assert rel(pick(u), ur) <= TOL
    if mode & 2:
        assert rel(pick(v), vr) <= TOL
    ug, vg = ser.evaluate_onsurface(*ser.to_device(node_block(blk)), delta, mode=mode)
    if mode & 1:
        assert rel(u.cpu().numpy(), ug.cpu().numpy()) <= 1e-13
    if mode & 2:
        assert rel(v.cpu().numpy(), vg.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("count", [2, 3])
def test_shards_sum_to_the_evaluation(ser, count):
    """options.shard_index / shard_count (the multi-GPU split of the node path, one all-reduce):
    the shards' partial u, v, computed one after another on this GPU, sum to the evaluation."""
    import torch

    blk = config5(inv_h=32)
    arrs = [torch.from_numpy(a).cuda() for a in (blk.src_xyz, blk.src_normal, blk.src_weight, blk.f, blk.q)]
    u, v = ser.evaluate_nodes(*arrs, blk.h, blk.rho)
    su = torch.zeros_like(u)
    sv = torch.zeros_like(v)
    for r in range(count):
        o = ser.Options()
        o.shard_index, o.shard_count = r, count
        pu, pv = ser.evaluate_nodes(*arrs, blk.h, blk.rho, options=o)
        su += pu
        sv += pv
    assert rel(su.cpu().numpy(), u.cpu().numpy()) <= 1e-13 and rel(sv.cpu().numpy(), v.cpu().numpy()) <= 1e-13
    o = ser.Options()
    o.shard_index, o.shard_count = count, count
    with pytest.raises(ser.StokesERError):
        ser.evaluate_nodes(*arrs, blk.h, blk.rho, options=o)
