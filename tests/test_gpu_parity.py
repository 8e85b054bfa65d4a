"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle (-m gpu).

Tolerance (BASELINE.json north_star): max-norm relative error
    max_i |gpu_i - oracle_i| / max_i |oracle_i|  <= 1e-12
separately for u and v, and <= 1e-13 for the extrapolation solve alone.
The oracle runs in definition mode (every pair regularized) unless noted; the
GPU path localizes, which moves totals by <= 6e-16 relative.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from workloads.configs import config1, config2, config3, config4, config5, subsample
from workloads.densities import ConstField, RigidField

pytestmark = pytest.mark.gpu

TOL = 1e-12
TOL_SOLVE = 1e-13


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


def run_gpu(ser, block, mode=3, **kw):
    u, v = ser.evaluate_block(block, mode=mode, **kw)
    return (None if u is None else u.cpu().numpy()), (None if v is None else v.cpu().numpy())


def check_block(ser, block, localized=False, mode=3, tol=TOL, **kw):
    u, v = run_gpu(ser, block, mode=mode, **kw)
    ur, vr = oracle.evaluate_block(block, mode=mode, localized=localized)
    out = {}
    if mode & 1:
        out["u"] = rel(u, ur)
        assert out["u"] <= tol, out
    if mode & 2:
        out["v"] = rel(v, vr)
        assert out["v"] <= tol, out
    return out


def test_config1_full_parity(ser):
    """Config 1 (sphere 1/h = 16, 504 targets at b/h in {0,+-1,+-2,+-3}) vs definition-mode oracle."""
    blk = config1()
    check_block(ser, blk, localized=False)
    check_block(ser, blk, localized=True)


@pytest.mark.parametrize("mode", [1, 2])
def test_config1_single_modes(ser, mode):
    check_block(ser, config1(), mode=mode)


def test_config1_closed_form_densities(ser):
    for f, q in ((ConstField((1.0, 0.0, 0.0)), ConstField((1.0, -2.0, 0.5))),
                 (RigidField(Omega=(0.3, -0.5, 0.7)), RigidField(U=(0.2, 0.1, -0.4), Omega=(1.0, 0.5, -0.25)))):
        check_block(ser, config1(f_field=f, q_field=q))


def test_per_delta_sums(ser):
    """stokes_er_eval_deltas vs the oracle's per-delta values (localized)."""
    blk = config1()
    arrs = ser.to_device(blk)
    ud, vd = ser.eval_deltas(*arrs, blk.h, blk.rho)
    ur, vr = oracle.eval_deltas_block(blk, localized=True)
    for k in range(3):
        assert rel(ud[k].cpu().numpy(), ur[k]) <= TOL
        assert rel(vd[k].cpu().numpy(), vr[k]) <= TOL


def test_extrapolation_solve(ser):
    """stokes_er_extrapolate (closed-form cofactor weights) vs the oracle's pivoted elimination."""
    import torch

    rng = np.random.default_rng(5)
    M, C, h = 4096, 6, 1 / 64
    b = np.concatenate([np.zeros(64), rng.uniform(-4 * h, 4 * h, M - 128), rng.uniform(-30 * h, 30 * h, 64)])
    ind = rng.standard_normal((3, C, M))
    ref = oracle.extrapolate(b, h, (2, 3, 4), ind)
    got = ser.extrapolate(torch.from_numpy(b).cuda(), h, (2, 3, 4), torch.from_numpy(ind).cuda()).cpu().numpy()
    assert rel(got, ref) <= TOL_SOLVE


def test_config2_h32_full(ser):
    blk = config2(inv_h=32)
    check_block(ser, blk, localized=True)


def _sampled(ser, block, k=512, seed=1, mode=3, **kw):
    """Full-size GPU run (the bench launch configuration), oracle on a target sample."""
    u, v = run_gpu(ser, block, mode=mode, **kw)
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, block.M - 1], rng.choice(block.M, k, replace=False)]))
    sub = block.take_targets(idx)
    ur, vr = oracle.evaluate_block(sub, mode=mode, localized=False)
    return rel(u[:, idx], ur), rel(v[:, idx], vr)


def test_config2_h64_sampled(ser):
    eu, ev = _sampled(ser, config2(inv_h=64))
    assert eu <= TOL and ev <= TOL


def test_config3_ellipsoid_sampled(ser):
    eu, ev = _sampled(ser, config3(inv_h=64), k=384)
    assert eu <= TOL and ev <= TOL


def test_config4_two_spheres_sampled(ser):
    for blk in config4(eps=0.02, inv_h=32):
        eu, ev = _sampled(ser, blk, k=256)
        assert eu <= TOL and ev <= TOL, blk.name


def test_config5_h128_sampled(ser):
    eu, ev = _sampled(ser, config5(inv_h=128), k=96)
    assert eu <= TOL and ev <= TOL


def test_config5_h256_max_size_sampled(ser):
    """The largest configuration (BASELINE.json config 5 at 1/h = 256: N = M = 1,090,854),
    full GPU evaluation, 48 sampled targets against the definition-mode oracle."""
    eu, ev = _sampled(ser, config5(inv_h=256), k=48)
    assert eu <= TOL and ev <= TOL


def test_config3_h128_and_config4_h64_sampled(ser):
    """BASELINE.json configs 3 and 4 at their full sizes (ellipsoid 1/h = 128; two spheres
    at 1/h = 64, eps = 0.05, all four blocks)."""
    eu, ev = _sampled(ser, config3(inv_h=128), k=96)
    assert eu <= TOL and ev <= TOL
    for blk in config4(eps=0.05, inv_h=64):
        eu, ev = _sampled(ser, blk, k=64)
        assert eu <= TOL and ev <= TOL, blk.name


def test_tunings_agree(ser):
    """targets/thread 2 vs 4 and different source chunkings: same sums up to rounding order."""
    blk = config2(inv_h=32)
    base = run_gpu(ser, blk)
    for T, ch in ((4, 0), (2, 1), (4, 7)):
        o = ser.Options()
        o.targets_per_thread = T
        o.source_chunk_tiles = ch
        u, v = run_gpu(ser, blk, options=o)
        assert rel(u, base[0]) <= 1e-13 and rel(v, base[1]) <= 1e-13


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_schedules_agree(ser, mode):
    """Fused (default) vs separate far/near kernels: the same pair sums (same
    per-slot partials, same fixed-order finalize), so bitwise equal; both vs oracle."""
    blk = config2(inv_h=32)
    o = ser.Options()
    o.schedule = 1
    fu = run_gpu(ser, blk, mode=mode)
    se = run_gpu(ser, blk, mode=mode, options=o)
    for a, b in zip(fu, se):
        if a is not None:
            assert rel(a, b) <= 1e-14
    check_block(ser, config1(), mode=mode)
    check_block(ser, config1(), mode=mode, options=o)


def test_deterministic(ser):
    blk = config2(inv_h=32)
    a = run_gpu(ser, blk)
    b = run_gpu(ser, blk)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_source_permutation_invariance(ser):
    import dataclasses

    blk = config2(inv_h=32)
    perm = np.random.default_rng(2).permutation(blk.N)
    pb = dataclasses.replace(blk, src_xyz=np.ascontiguousarray(blk.src_xyz[:, perm]),
                             src_normal=np.ascontiguousarray(blk.src_normal[:, perm]),
                             src_weight=np.ascontiguousarray(blk.src_weight[perm]),
                             f=np.ascontiguousarray(blk.f[:, perm]), q=np.ascontiguousarray(blk.q[:, perm]))
    a = run_gpu(ser, blk)
    b = run_gpu(ser, pb)
    assert rel(b[0], a[0]) <= 1e-13 and rel(b[1], a[1]) <= 1e-13


def test_small_path_permutation_invariance(ser):
    """N, M <= 8192 (the counting-rank Morton prologue): the sums do not depend on the input order of
    the sources or of the targets (each order gives the same stable Morton order up to equal keys, so
    equal results to rounding), including a duplicated node (equal keys: ties broken by index)."""
    import dataclasses

    blk = config1()
    k = 5
    cat = lambda a, b: np.ascontiguousarray(np.concatenate([a, b], axis=-1))
    blk = dataclasses.replace(blk, src_xyz=cat(blk.src_xyz, blk.src_xyz[:, :k]),
                              src_normal=cat(blk.src_normal, blk.src_normal[:, :k]),
                              src_weight=cat(blk.src_weight, 0.25 * blk.src_weight[:k]),
                              f=cat(blk.f, blk.f[:, :k]), q=cat(blk.q, blk.q[:, :k]))
    rng = np.random.default_rng(5)
    ps, pt = rng.permutation(blk.N), rng.permutation(blk.M)
    pb = dataclasses.replace(blk, src_xyz=np.ascontiguousarray(blk.src_xyz[:, ps]),
                             src_normal=np.ascontiguousarray(blk.src_normal[:, ps]),
                             src_weight=np.ascontiguousarray(blk.src_weight[ps]),
                             f=np.ascontiguousarray(blk.f[:, ps]), q=np.ascontiguousarray(blk.q[:, ps]))
    pb = pb.take_targets(pt)
    assert ser.launch_count(blk.M, blk.N) == 4
    a = run_gpu(ser, blk)
    b = run_gpu(ser, pb)
    assert rel(b[0], a[0][:, pt]) <= 1e-13 and rel(b[1], a[1][:, pt]) <= 1e-13
    check_block(ser, pb, localized=False)


def test_host_entry_point_matches_device(ser):
    blk = config1()
    ud, vd = run_gpu(ser, blk)
    uh, vh = ser.evaluate_host(*blk.arrays(), blk.h, blk.rho)
    np.testing.assert_array_equal(uh.numpy(), ud)
    np.testing.assert_array_equal(vh.numpy(), vd)


@pytest.mark.parametrize("m", [1, 7, 255, 256, 257, 1000])
def test_ragged_target_counts(ser, m):
    blk = config2(inv_h=16)
    sub = blk.take_targets(np.arange(m) * 3 % blk.M)
    check_block(ser, sub, localized=True)


def test_single_source_and_tiny(ser):
    blk = config1(inv_h=4, per_class=2)
    check_block(ser, blk)
    import dataclasses
    one = dataclasses.replace(blk, src_xyz=blk.src_xyz[:, :1].copy(), src_normal=blk.src_normal[:, :1].copy(),
                              src_weight=blk.src_weight[:1].copy(), f=blk.f[:, :1].copy(), q=blk.q[:, :1].copy())
    check_block(ser, one)


def test_empty_targets_and_errors(ser):
    import torch

    blk = config1(inv_h=8, per_class=1)
    arrs = list(ser.to_device(blk))
    e = [a[..., :0].contiguous() for a in arrs[5:]]
    u, v = ser.evaluate(*arrs[:5], *e, blk.h, blk.rho)
    assert u.shape == (3, 0) and v.shape == (3, 0)
    with pytest.raises(ser.StokesERError) as ei:
        ser.evaluate(*arrs, -1.0, blk.rho)
    assert ei.value.status == 1
    with pytest.raises(ser.StokesERError):
        ser.evaluate(*arrs, blk.h, (2.0, 2.0, 4.0))
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(ser.StokesERError) as ei:
        ser.evaluate(*arrs, blk.h, blk.rho, workspace=ws)
    assert ei.value.status == 3


def test_far_targets_pass_through(ser):
    """|b| > 6 delta_max: no near pairs, weights (1,0,0); compare with the oracle."""
    from workloads.configs import pure_far
    blk = pure_far(inv_h=32, b=0.9)
    blk = blk.take_targets(np.arange(0, blk.M, 11))
    check_block(ser, blk, localized=False)


# ---------------------------------------------------------------- NEXT-1
def _onsurface(ser, block, delta, mode=3):
    arrs = ser.to_device(block)
    u, v = ser.evaluate_onsurface(*arrs, delta, mode=mode)
    return (None if u is None else u.cpu().numpy()), (None if v is None else v.cpu().numpy())


@pytest.mark.parametrize("inv_h", [16, 32])
def test_onsurface_sharp_parity(ser, inv_h):
    """stokes_er_eval_onsurface (s#, delta = 3h) vs the oracle's
    sharp mode (definition: every pair regularized) on all sphere nodes."""
    blk = config5(inv_h=inv_h)
    if inv_h == 32:
        blk = blk.take_targets(np.arange(0, blk.M, 7))
    delta = 3 * blk.h
    u, v = _onsurface(ser, blk, delta)
    ur, vr = oracle.evaluate_sharp(*blk.arrays(), delta, localized=False, cutoff=7.0)
    assert rel(u, ur) <= TOL and rel(v, vr) <= TOL


def test_onsurface_two_sphere_self_block(ser):
    blk = config4(eps=0.05, inv_h=32)[0]
    blk = blk.take_targets(np.arange(0, blk.M, 5))
    delta = 3 * blk.h
    for mode in (1, 2, 3):
        u, v = _onsurface(ser, blk, delta, mode=mode)
        ur, vr = oracle.evaluate_sharp(*blk.arrays(), delta, mode=mode, localized=True, cutoff=7.0)
        if mode & 1:
            assert rel(u, ur) <= TOL
        if mode & 2:
            assert rel(v, vr) <= TOL


def test_delta_power_schedule_parity(ser):
    """NEXT-4 (delta ~ h^q): the call with h_eff = C h^q (q = 0.8) matches
    the oracle at the same h_eff, on config 2 at 1/h = 32."""
    import dataclasses

    blk = config2(inv_h=32)
    h_eff = blk.h ** 0.8 * (1.0 / 16) ** 0.2
    b2 = dataclasses.replace(blk, h=h_eff)
    check_block(ser, b2.take_targets(np.arange(0, b2.M, 7)), localized=True)


def test_mode_composition_and_linearity(ser):
    """Properties: the SL-only and DL-only calls give the BOTH call's u and
    v; the map (f, q) -> (u, v) is linear (the subtraction terms use f(x0), q(x0) of
    the same fields)."""
    import dataclasses

    blk = config2(inv_h=32)
    u3, v3 = run_gpu(ser, blk, mode=3)
    u1, _ = run_gpu(ser, blk, mode=1)
    _, v2 = run_gpu(ser, blk, mode=2)
    assert rel(u1, u3) <= 1e-14 and rel(v2, v3) <= 1e-14
    from workloads.densities import PolyField

    rng = np.random.default_rng(77)  # same geometry, other seeded cubic densities
    F, Q = PolyField(rng), PolyField(rng)
    x0d = np.concatenate([blk.tgt_x0_density[:3], F(blk.tgt_x0), Q(blk.tgt_x0)])
    other = dataclasses.replace(blk, f=np.ascontiguousarray(F(blk.src_xyz)), q=np.ascontiguousarray(Q(blk.src_xyz)),
                                tgt_x0_density=np.ascontiguousarray(x0d))
    a, b = 0.7, -1.3
    mix = dataclasses.replace(blk, f=a * blk.f + b * other.f, q=a * blk.q + b * other.q,
                              tgt_x0_density=np.ascontiguousarray(np.concatenate(
                                  [blk.tgt_x0_density[:3], a * blk.tgt_x0_density[3:] + b * other.tgt_x0_density[3:]])))
    um, vm = run_gpu(ser, mix)
    uo, vo = run_gpu(ser, other)
    assert rel(um, a * u3 + b * uo) <= 1e-13 and rel(vm, a * v3 + b * vo) <= 1e-13


def test_target_shards_concatenate(ser):
    """Multi-GPU sharding simulated on one GPU: the contiguous target ranges
    of paper_2507_00156_b200.sharding evaluated separately concatenate to the full run."""
    from paper_2507_00156_b200.sharding import shard_bounds

    blk = config2(inv_h=32)
    u, v = run_gpu(ser, blk)
    parts = []
    for r in range(3):
        a, b = shard_bounds(blk.M, r, 3)
        parts.append(run_gpu(ser, blk.take_targets(np.arange(a, b))))
    us = np.concatenate([p[0] for p in parts], axis=1)
    vs = np.concatenate([p[1] for p in parts], axis=1)
    assert rel(us, u) <= 1e-13 and rel(vs, v) <= 1e-13


def test_cuda_graph_capture_and_replay(ser):
    """stokes_er_eval only enqueues work (no host sync, no allocation), so a whole
    evaluation can be captured in a CUDA graph and replayed: the replay reproduces the
    eager result bitwise, also after the inputs change in place."""
    import torch

    blk = config2(inv_h=16)
    arrs = ser.to_device(blk)
    M, N = blk.M, blk.N
    out_u = torch.empty((3, M), dtype=torch.float64, device="cuda")
    out_v = torch.empty((3, M), dtype=torch.float64, device="cuda")
    ws = ser.alloc_workspace(M, N)
    ref = ser.evaluate(*arrs, blk.h, blk.rho)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up on the side stream (sets kernel attributes)
        ser.evaluate(*arrs, blk.h, blk.rho, out_u=out_u, out_v=out_v, workspace=ws, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ser.evaluate(*arrs, blk.h, blk.rho, out_u=out_u, out_v=out_v, workspace=ws,
                     stream=torch.cuda.current_stream())
    out_u.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_u, ref[0]) and torch.equal(out_v, ref[1])
    arrs[3].mul_(2.0)  # f -> 2 f in place (and f(x0) with it): u doubles exactly
    arrs[7][3:6].mul_(2.0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_u, 2.0 * ref[0])


@pytest.mark.parametrize("scale", [0.01, 8.0])
def test_degenerate_delta_scales(ser, scale):
    """delta far below the node spacing (only r = 0 self pairs are near: the far path does
    everything else) and far above it (every pair is near: the far path skips every
    sub-tile as all-near and the near units do all the work); against the oracle."""
    import dataclasses

    blk = config2(inv_h=16)
    blk = dataclasses.replace(blk, h=blk.h * scale).take_targets(np.arange(0, blk.M, 3))
    check_block(ser, blk, localized=False)


def test_duplicate_and_zero_weight_sources(ser):
    """Two nodes at the same position with different densities, and zero-weight nodes
    (the angular cutoff of the quadrature, reading R10), against the oracle."""
    import dataclasses

    blk = config1(inv_h=8, per_class=4)
    k = 17
    cat = lambda a, b: np.ascontiguousarray(np.concatenate([a, b], axis=-1))
    dup = dataclasses.replace(blk, src_xyz=cat(blk.src_xyz, blk.src_xyz[:, :k]),
                              src_normal=cat(blk.src_normal, blk.src_normal[:, :k]),
                              src_weight=cat(blk.src_weight, 0.5 * blk.src_weight[:k]),
                              f=cat(blk.f, -blk.f[:, :k]), q=cat(blk.q, 2.0 * blk.q[:, :k]))
    w = dup.src_weight.copy()
    w[::11] = 0.0
    dup = dataclasses.replace(dup, src_weight=w)
    check_block(ser, dup, localized=False)


@pytest.mark.parametrize("r_over_h", [5.0, 11.9, 12.03, 17.98, 18.02, 23.9])
def test_near_pair_exact_s_factors(ser, r_over_h):
    """Reading R1 on the GPU, pair by pair: just inside / just past 6 delta_1 and
    6 delta_2 (rho = (2, 3, 4)) a near pair uses the exact s-factors of every
    delta (a per-delta s = 1 rule would miss by ~1e-13 here).  The per-delta
    values match the oracle to rounding (2e-15; the extrapolated ones, which
    carry the weights w_k, to 1e-14), far tighter than the general tolerance."""
    from pair_blocks import one_pair_block

    blk = one_pair_block(r_over_h)
    u, v = run_gpu(ser, blk)
    ur, vr = oracle.evaluate_block(blk, localized=True)
    assert rel(u, ur) <= 1e-14 and rel(v, vr) <= 1e-14
    ud, vd = ser.eval_deltas(*ser.to_device(blk), blk.h, blk.rho)
    udr, vdr = oracle.eval_deltas_block(blk, localized=True)
    for k in range(3):
        assert rel(ud[k].cpu().numpy(), udr[k]) <= 2e-15
        assert rel(vd[k].cpu().numpy(), vdr[k]) <= 2e-15


def test_randomized_parity_sweep(ser, tmp_path):
    """40 seeded random cases (tools/parity_sweep.py: sphere or ellipsoid with a random centre and
    semi-axes, 1/h in {8, 12, 16, 24}, a random increasing rho in [1.5, 6], SL / DL / both,
    polynomial or trigonometric densities, node + shell + far targets; every 5th case also the
    s# variant) all within the 1e-12 bar of the oracle's localized mode."""
    import importlib.util
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "parity_sweep.py")
    spec = importlib.util.spec_from_file_location("parity_sweep", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.main(str(tmp_path / "sweep.json"), 40) == 0


@pytest.mark.parametrize("rho", [(1.0, 2.0, 5.0), (1.0, 3.0, 8.0)])
def test_wide_rho_ratio(ser, rho):
    """rho_3 / rho_1 > 4.4: a near pair (r <= 6 delta_3) reaches t_1 = r/delta_1 = 6 rho_3/rho_1
    > 26.6, where t_1^2 > 700 would overflow the CUDA path's exp unless its argument is clamped
    (device_math.cuh sfactor_s).  Every pair of config 2 at 1/h = 16 is compared with the
    oracle's definition mode (libm exp underflows to 0 there)."""
    import dataclasses

    blk = config2(inv_h=16)
    blk = dataclasses.replace(blk, rho=tuple(rho)).take_targets(np.arange(0, blk.M, 2))
    check_block(ser, blk, localized=False)


@pytest.mark.parametrize("n", [8192, 8193])
def test_small_sort_prologue_boundary(ser, n):
    """N, M <= 8192 take the one-launch Morton prologue (small_rank_kernel: ranks by counting,
    + pack_both), larger problems bbox + morton + the CUB device sorts: both sides of the boundary
    against the oracle (the first n nodes of the 1/h = 32 sphere as sources, a target sample of
    config 2)."""
    import dataclasses

    blk = config2(inv_h=32)
    cut = lambda a: np.ascontiguousarray(a[..., :n])
    sub = dataclasses.replace(blk, src_xyz=cut(blk.src_xyz), src_normal=cut(blk.src_normal),
                              src_weight=cut(blk.src_weight), f=cut(blk.f), q=cut(blk.q))
    sub = sub.take_targets(np.arange(0, blk.M, 37))
    check_block(ser, sub, localized=True)
    assert ser.launch_count(sub.M, n) == (4 if n <= 8192 else 7)
