"""B200-native hot path of arXiv 2507.00156 (localized extrapolated regularization
of nearly singular Stokes single/double layer potentials).

Thin Python layer over the C ABI of include/stokes_er.h (libstokes_er.so):
PyTorch provides device memory and streams only; every arithmetic step runs in
the library's sm_100a kernels.  No CPU fallback exists: without the built
library or a CUDA device the calls raise.

    u, v = evaluate(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho)

All tensors float64 CUDA, SoA [rows][count] contiguous (see include/stokes_er.h).
"""
from __future__ import annotations

import ctypes

from . import _lib

SL, DL, BOTH = 1, 2, 3
CUTOFF = 6.0  # STOKES_ER_CUTOFF
CUTOFF_SURFACE = 7.0  # STOKES_ER_CUTOFF_SURFACE (R15)


def _torch():
    import torch

    return torch


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check_dev(name, t, shape):
    torch = _torch()
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError(f"{name}: expected a contiguous float64 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def _stream_handle(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def workspace_bytes(M: int, N: int, mode: int = BOTH) -> int:
    return int(_lib.load().stokes_er_workspace_bytes(M, N, mode))


def host_workspace_bytes(M: int, N: int, mode: int = BOTH) -> int:
    return int(_lib.load().stokes_er_host_workspace_bytes(M, N, mode))


def launch_count(M: int, N: int, mode: int = BOTH) -> int:
    return int(_lib.load().stokes_er_launch_count(M, N, mode))


def alloc_workspace(M: int, N: int, mode: int = BOTH, device="cuda", host=False):
    torch = _torch()
    nbytes = host_workspace_bytes(M, N, mode) if host else workspace_bytes(M, N, mode)
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)


def _scratch(nbytes, dev, stream):
    """Temporary device buffer for one call, allocated on `dev` and tied to `stream`:
    the caching allocator must not hand it out again while the call's kernels run
    on a stream other than torch's current one."""
    torch = _torch()
    with torch.cuda.device(dev):
        t = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)
    if stream is not None:
        t.record_stream(stream)
    return t


def _out(shape, dev, stream):
    torch = _torch()
    with torch.cuda.device(dev):
        t = torch.empty(shape, dtype=torch.float64, device=dev)
    if stream is not None:
        t.record_stream(stream)
    return t


def _check_inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, mode):
    """Shapes/dtypes/devices of the hot-path inputs (raises before any launch)."""
    M, N = _shapes(src_xyz, tgt_b)
    _check_dev("src_xyz", src_xyz, (3, N))
    _check_dev("src_normal", src_normal, (3, N))
    _check_dev("src_weight", src_weight, (N,))
    _check_dev("f", f if mode & SL else None, (3, N))
    _check_dev("q", q if mode & DL else None, (3, N))
    _check_dev("tgt_xyz", tgt_xyz, (3, M))
    _check_dev("tgt_b", tgt_b, (M,))
    _check_dev("tgt_x0_density", tgt_x0_density, (9, M))
    dev = src_xyz.device
    for name, t in (("src_normal", src_normal), ("src_weight", src_weight), ("f", f if mode & SL else None),
                    ("q", q if mode & DL else None), ("tgt_xyz", tgt_xyz), ("tgt_b", tgt_b),
                    ("tgt_x0_density", tgt_x0_density)):
        if t is not None and t.device != dev:
            raise ValueError(f"{name}: on {t.device}, expected {dev} (all inputs on one device)")
    return M, N, dev


def _shapes(src_xyz, tgt_b):
    return int(tgt_b.shape[0]), int(src_xyz.shape[1])


def evaluate(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho, mode=BOTH,
             out_u=None, out_v=None, workspace=None, stream=None, options: "_lib.Options | None" = None):
    """stokes_er_eval on device tensors; returns (u (3,M) or None, v (3,M) or None).
    Asynchronous on `stream` (default: torch's current stream)."""
    M, N, dev = _check_inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, mode)
    _check_dev("out_u", out_u if mode & SL else None, (3, M))
    _check_dev("out_v", out_v if mode & DL else None, (3, M))
    if mode & SL and out_u is None:
        out_u = _out((3, M), dev, stream)
    if mode & DL and out_v is None:
        out_v = _out((3, M), dev, stream)
    L = _lib.load()
    if workspace is None:
        if options is None:
            workspace = _scratch(workspace_bytes(M, N, mode), dev, stream)
        else:
            workspace = _scratch(L.stokes_er_workspace_bytes_ex(M, N, mode, ctypes.byref(options)), dev, stream)
    args = [_ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
            _ptr(q if mode & DL else None), _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M, N, float(h),
            _lib.rho_arg(rho), int(mode), _ptr(out_u if mode & SL else None), _ptr(out_v if mode & DL else None),
            _ptr(workspace), int(workspace.numel()), _stream_handle(stream)]
    if options is None:
        _lib.check("stokes_er_eval", L.stokes_er_eval(*args))
    else:
        _lib.check("stokes_er_eval_ex", L.stokes_er_eval_ex(*args, ctypes.byref(options)))
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def evaluate_host(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho, mode=BOTH,
                  out_u=None, out_v=None, workspace=None, stream=None):
    """stokes_er_eval_host: HOST float64 tensors/arrays in and out (pinned memory
    recommended); the library copies in, evaluates, copies out and synchronizes."""
    torch = _torch()
    import numpy as np

    def host(a):
        if a is None:
            return None
        if isinstance(a, np.ndarray):
            a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        if a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError("evaluate_host expects contiguous float64 host tensors")
        return a

    src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density = map(
        host, (src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density))
    M, N = _shapes(src_xyz, tgt_b)
    if mode & SL and out_u is None:
        out_u = torch.empty((3, M), dtype=torch.float64).pin_memory()
    if mode & DL and out_v is None:
        out_v = torch.empty((3, M), dtype=torch.float64).pin_memory()
    if workspace is None:
        workspace = alloc_workspace(M, N, mode, "cuda", host=True)
    L = _lib.load()
    _lib.check("stokes_er_eval_host", L.stokes_er_eval_host(
        _ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
        _ptr(q if mode & DL else None), _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M, N, float(h),
        _lib.rho_arg(rho), int(mode), _ptr(out_u if mode & SL else None), _ptr(out_v if mode & DL else None),
        _ptr(workspace), int(workspace.numel()), _stream_handle(stream)))
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def evaluate_onsurface(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, delta, mode=BOTH,
                       out_u=None, out_v=None, workspace=None, stream=None):
    """stokes_er_eval_onsurface (NEXT-1): single delta, s# factors, no extrapolation."""
    M, N, dev = _check_inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, mode)
    _check_dev("out_u", out_u if mode & SL else None, (3, M))
    _check_dev("out_v", out_v if mode & DL else None, (3, M))
    if mode & SL and out_u is None:
        out_u = _out((3, M), dev, stream)
    if mode & DL and out_v is None:
        out_v = _out((3, M), dev, stream)
    if workspace is None:
        workspace = _scratch(workspace_bytes(M, N, mode), dev, stream)
    L = _lib.load()
    _lib.check("stokes_er_eval_onsurface", L.stokes_er_eval_onsurface(
        _ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
        _ptr(q if mode & DL else None), _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M, N, float(delta),
        int(mode), _ptr(out_u if mode & SL else None), _ptr(out_v if mode & DL else None), _ptr(workspace),
        int(workspace.numel()), _stream_handle(stream)))
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def nodes_workspace_bytes(N: int, mode: int = BOTH, options: "_lib.Options | None" = None) -> int:
    L = _lib.load()
    if options is None:
        return int(L.stokes_er_nodes_workspace_bytes(N, mode))
    return int(L.stokes_er_nodes_workspace_bytes_ex(N, mode, ctypes.byref(options)))


def nodes_launch_count(N: int, mode: int = BOTH) -> int:
    return int(_lib.load().stokes_er_nodes_launch_count(N, mode))


def evaluate_nodes(src_xyz, src_normal, src_weight, f, q, h, rho, mode=BOTH, out_u=None, out_v=None, workspace=None,
                   stream=None, options: "_lib.Options | None" = None):
    """stokes_er_eval_nodes: the same evaluation as `evaluate` with the targets = the N nodes
    (b = 0, x0 = node, n0 = its normal, f(x0) = f, q(x0) = q); returns (u (3,N), v (3,N))."""
    N = int(src_xyz.shape[1])
    _check_dev("src_xyz", src_xyz, (3, N))
    _check_dev("src_normal", src_normal, (3, N))
    _check_dev("src_weight", src_weight, (N,))
    _check_dev("f", f if mode & SL else None, (3, N))
    _check_dev("q", q if mode & DL else None, (3, N))
    _check_dev("out_u", out_u if mode & SL else None, (3, N))
    _check_dev("out_v", out_v if mode & DL else None, (3, N))
    dev = src_xyz.device
    for name, t in (("src_normal", src_normal), ("src_weight", src_weight), ("f", f if mode & SL else None),
                    ("q", q if mode & DL else None)):
        if t is not None and t.device != dev:
            raise ValueError(f"{name}: on {t.device}, expected {dev}")
    if mode & SL and out_u is None:
        out_u = _out((3, N), dev, stream)
    if mode & DL and out_v is None:
        out_v = _out((3, N), dev, stream)
    L = _lib.load()
    if workspace is None:
        workspace = _scratch(nodes_workspace_bytes(N, mode, options), dev, stream)
    args = [_ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
            _ptr(q if mode & DL else None), N, float(h), _lib.rho_arg(rho), int(mode),
            _ptr(out_u if mode & SL else None), _ptr(out_v if mode & DL else None), _ptr(workspace),
            int(workspace.numel()), _stream_handle(stream)]
    if options is None:
        _lib.check("stokes_er_eval_nodes", L.stokes_er_eval_nodes(*args))
    else:
        _lib.check("stokes_er_eval_nodes_ex", L.stokes_er_eval_nodes_ex(*args, ctypes.byref(options)))
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def evaluate_nodes_onsurface(src_xyz, src_normal, src_weight, f, q, delta, mode=BOTH, out_u=None, out_v=None,
                             workspace=None, stream=None):
    """stokes_er_eval_nodes_onsurface: NEXT-1's s# evaluation (one delta, cutoff 7) at the nodes."""
    N = int(src_xyz.shape[1])
    for name, t, shp in (("src_xyz", src_xyz, (3, N)), ("src_normal", src_normal, (3, N)),
                         ("src_weight", src_weight, (N,)), ("f", f if mode & SL else None, (3, N)),
                         ("q", q if mode & DL else None, (3, N)), ("out_u", out_u if mode & SL else None, (3, N)),
                         ("out_v", out_v if mode & DL else None, (3, N))):
        _check_dev(name, t, shp)
    dev = src_xyz.device
    if mode & SL and out_u is None:
        out_u = _out((3, N), dev, stream)
    if mode & DL and out_v is None:
        out_v = _out((3, N), dev, stream)
    if workspace is None:
        workspace = _scratch(nodes_workspace_bytes(N, mode), dev, stream)
    _lib.check("stokes_er_eval_nodes_onsurface", _lib.load().stokes_er_eval_nodes_onsurface(
        _ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
        _ptr(q if mode & DL else None), N, float(delta), int(mode), _ptr(out_u if mode & SL else None),
        _ptr(out_v if mode & DL else None), _ptr(workspace), int(workspace.numel()), _stream_handle(stream)))
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def nodes_pair_counts(N: int, h, rho, workspace, mode: int = BOTH, stream=None):
    """(directed pairs summed by the symmetric far kernel, pairs owned by the neighbour kernel)
    of the last evaluate_nodes with this workspace (synchronizes; statistics only)."""
    c = (ctypes.c_int64 * 2)()
    _lib.check("stokes_er_nodes_pair_counts", _lib.load().stokes_er_nodes_pair_counts(
        N, int(mode), float(h), _lib.rho_arg(rho), _ptr(workspace), int(workspace.numel()), c,
        _stream_handle(stream)))
    return int(c[0]), int(c[1])


def evaluate_nodes_host(src_xyz, src_normal, src_weight, f, q, h, rho, mode=BOTH, out_u=None, out_v=None,
                        workspace=None, stream=None):
    """stokes_er_eval_nodes_host: HOST float64 arrays in and out (pinned recommended)."""
    torch = _torch()
    import numpy as np

    def host(a):
        if a is None:
            return None
        if isinstance(a, np.ndarray):
            a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        if a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError("evaluate_nodes_host expects contiguous float64 host tensors")
        return a

    src_xyz, src_normal, src_weight, f, q = map(host, (src_xyz, src_normal, src_weight, f, q))
    N = int(src_xyz.shape[1])
    if mode & SL and out_u is None:
        out_u = torch.empty((3, N), dtype=torch.float64).pin_memory()
    if mode & DL and out_v is None:
        out_v = torch.empty((3, N), dtype=torch.float64).pin_memory()
    L = _lib.load()
    if workspace is None:
        workspace = torch.empty(max(int(L.stokes_er_nodes_host_workspace_bytes(N, mode)), 1), dtype=torch.uint8,
                                device="cuda")
    _lib.check("stokes_er_eval_nodes_host", L.stokes_er_eval_nodes_host(
        _ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
        _ptr(q if mode & DL else None), N, float(h), _lib.rho_arg(rho), int(mode), _ptr(out_u if mode & SL else None),
        _ptr(out_v if mode & DL else None), _ptr(workspace), int(workspace.numel()), _stream_handle(stream)))
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def evaluate_nodes_block(block, mode=BOTH, device="cuda", **kw):
    """Convenience for tests/bench: the node-target evaluation of a Block's SOURCES (its
    own targets are ignored; `node_block` in workloads.configs builds the equivalent
    general-path Block)."""
    torch = _torch()
    arrs = [torch.from_numpy(a).to(device) for a in (block.src_xyz, block.src_normal, block.src_weight, block.f,
                                                     block.q)]
    return evaluate_nodes(*arrs, block.h, block.rho, mode=mode, **kw)


def eval_deltas(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho, mode=BOTH,
                stream=None):
    """stokes_er_eval_deltas: per-delta u^{delta_k}, v^{delta_k} as (3,3,M) tensors [k][i][m]."""
    M, N, dev = _check_inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, mode)
    ud = _out((3, 3, M), dev, stream) if mode & SL else None
    vd = _out((3, 3, M), dev, stream) if mode & DL else None
    L = _lib.load()
    _lib.check("stokes_er_eval_deltas", L.stokes_er_eval_deltas(
        _ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
        _ptr(q if mode & DL else None), _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M, N, float(h),
        _lib.rho_arg(rho), int(mode), _ptr(ud), _ptr(vd), None, 0, _stream_handle(stream)))
    return ud, vd


def extrapolate(tgt_b, h, rho, in_delta, stream=None):
    """stokes_er_extrapolate: in_delta (3, C, M) device -> (C, M)."""
    _, C, M = in_delta.shape
    _check_dev("tgt_b", tgt_b, (M,))
    in_delta = in_delta.contiguous()
    _check_dev("in_delta", in_delta, (3, C, M))
    out = _out((C, M), in_delta.device, stream)
    L = _lib.load()
    _lib.check("stokes_er_extrapolate", L.stokes_er_extrapolate(
        _ptr(tgt_b), M, float(h), _lib.rho_arg(rho), _ptr(in_delta), int(C), _ptr(out),
        _stream_handle(stream)))
    return out


def to_device(block, device="cuda"):
    """Copy a workloads.configs.Block's arrays to device tensors (tuple in API order)."""
    torch = _torch()
    return tuple(torch.from_numpy(a).to(device) for a in block.arrays())


def evaluate_block(block, mode=BOTH, device="cuda", **kw):
    """Convenience for tests/bench: device-resident evaluation of a Block."""
    arrs = to_device(block, device)
    return evaluate(*arrs, block.h, block.rho, mode=mode, **kw)


Options = _lib.Options
StokesERError = _lib.StokesERError


class TwoDropSolver:
    """NEXT-2 (Sec. 4.3): IE (35) on two drops through the C ABI
    (stokes_er_twodrop_*).  Holds the device inputs and the workspace in which
    stokes_er_twodrop_setup leaves the interpolation stencils.

    drops: two dicts with device tensors xyz (3,N), normal (3,N), weight (N,), f (3,N)
    and float lam; cross: two dicts with b (N_b,) and x0d (6,N_b) (n0, [f](x0)) of
    drop b's nodes seen from drop 1-b (include/stokes_er.h)."""

    def __init__(self, drops, cross, h, rho, delta_self, mu0=1.0, tol=1e-10, max_iter=100, stream=None,
                 tree=None):
        """tree: None (direct sums) or (leaf_size, degree, theta): every block through the
        treecode (NEXT-3), with one TreePlan per drop."""
        torch = _torch()
        self.L = _lib.load()
        self._keep = (drops, cross)
        self.N = [int(d["xyz"].shape[1]) for d in drops]
        self.n = 3 * sum(self.N)
        self.device = drops[0]["xyz"].device
        for b, d in enumerate(drops):
            N = self.N[b]
            for k, shp in (("xyz", (3, N)), ("normal", (3, N)), ("weight", (N,)), ("f", (3, N))):
                _check_dev(f"drops[{b}].{k}", d[k], shp)
            _check_dev(f"cross[{b}].b", cross[b]["b"], (N,))
            _check_dev(f"cross[{b}].x0d", cross[b]["x0d"], (6, N))
        self.drops = (_lib.Drop * 2)(*[_lib.Drop(self.N[b], _ptr(d["xyz"]), _ptr(d["normal"]), _ptr(d["weight"]),
                                                 _ptr(d["f"]), float(d["lam"])) for b, d in enumerate(drops)])
        self.cross = (_lib.Cross * 2)(*[_lib.Cross(_ptr(c["b"]), _ptr(c["x0d"])) for c in cross])
        self.params = _lib.TwoDropParams(float(h), (ctypes.c_double * 3)(*[float(r) for r in rho]),
                                         float(delta_self), float(mu0), float(tol), int(max_iter))
        self.plans = None
        if tree is not None:
            self.plans = [TreePlan(d["xyz"].cpu().numpy(), *tree) for d in drops]
            self.tree_params = _lib.TreeParams(int(tree[0]), int(tree[1]), float(tree[2]))
            self.params.use_tree = 1
            self.params.tree_plan[0] = self.plans[0].buf.ctypes.data
            self.params.tree_plan[1] = self.plans[1].buf.ctypes.data
            self.params.tree = ctypes.pointer(self.tree_params)
        nbytes = int(self.L.stokes_er_twodrop_workspace_bytes_ex(self.N[0], self.N[1], ctypes.byref(self.params)))
        if nbytes == 0:
            raise ValueError("stokes_er_twodrop_workspace_bytes: invalid sizes")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.stream = stream
        _lib.check("stokes_er_twodrop_setup",
                   self.L.stokes_er_twodrop_setup(self.drops, self.cross, ctypes.byref(self.params), _ptr(self.ws),
                                                  nbytes, _stream_handle(stream)))

    def _common(self):
        return self.drops, self.cross, ctypes.byref(self.params)

    def rhs(self, out=None):
        torch = _torch()
        out = out if out is not None else torch.empty(self.n, dtype=torch.float64, device=self.device)
        _lib.check("stokes_er_twodrop_rhs", self.L.stokes_er_twodrop_rhs(
            *self._common(), _ptr(out), _ptr(self.ws), int(self.ws.numel()), _stream_handle(self.stream)))
        return out

    def apply(self, u, out=None):
        torch = _torch()
        _check_dev("u", u, (self.n,))
        out = out if out is not None else torch.empty(self.n, dtype=torch.float64, device=self.device)
        _lib.check("stokes_er_twodrop_apply", self.L.stokes_er_twodrop_apply(
            *self._common(), _ptr(u), _ptr(out), _ptr(self.ws), int(self.ws.numel()), _stream_handle(self.stream)))
        return out

    def solve(self, out=None):
        """Returns (u (n,), iterations, residual history list)."""
        torch = _torch()
        out = out if out is not None else torch.empty(self.n, dtype=torch.float64, device=self.device)
        iters = ctypes.c_int(0)
        hist = (ctypes.c_double * self.params.max_iter)()
        st = self.L.stokes_er_twodrop_solve(*self._common(), _ptr(out), ctypes.byref(iters), hist, _ptr(self.ws),
                                            int(self.ws.numel()), _stream_handle(self.stream))
        _lib.check("stokes_er_twodrop_solve", st)
        return out, int(iters.value), [float(hist[i]) for i in range(iters.value)]


def twodrop_solver(td, device="cuda", max_iter=100, stream=None, tree=None):
    """TwoDropSolver from a workloads.twodrop.TwoDrop input set (numpy arrays -> device)."""
    import numpy as np

    torch = _torch()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
    drops = [dict(xyz=dev(d.x), normal=dev(d.n), weight=dev(d.w), f=dev(d.f), lam=d.lam) for d in td.drops]
    cross = [dict(b=dev(c.b), x0d=dev(np.concatenate([c.n0, c.f0], axis=0))) for c in td.cross]
    return TwoDropSolver(drops, cross, td.h, td.rho, td.delta_self, 1.0, td.tol, max_iter, stream, tree)


class TreePlan:
    """NEXT-3 octree over HOST node positions (stokes_er_tree_build, Sec. 3.4).
    leaf_size = N0, degree = p, theta = MAC parameter (eq. (28))."""

    def __init__(self, src_xyz_host, leaf_size=2000, degree=6, theta=0.6):
        import numpy as np

        L = _lib.load()
        x = np.ascontiguousarray(src_xyz_host, dtype=np.float64)
        if x.ndim != 2 or x.shape[0] != 3:
            raise ValueError("src_xyz_host: expected (3, N) float64")
        self.N = int(x.shape[1])
        self.params = _lib.TreeParams(int(leaf_size), int(degree), float(theta))
        nbytes = int(L.stokes_er_tree_plan_bytes(self.N, ctypes.byref(self.params)))
        if nbytes == 0:
            raise ValueError("stokes_er_tree_plan_bytes: invalid parameters")
        self.buf = np.zeros(nbytes, dtype=np.uint8)
        _lib.check("stokes_er_tree_build", L.stokes_er_tree_build(
            x.ctypes.data_as(ctypes.c_void_p), self.N, ctypes.byref(self.params),
            self.buf.ctypes.data_as(ctypes.c_void_p), nbytes))
        n, d = ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check("stokes_er_tree_info", L.stokes_er_tree_info(self.ptr(), self.N, ctypes.byref(n), ctypes.byref(d)))
        self.nodes, self.depth = int(n.value), int(d.value)

    def ptr(self):
        return self.buf.ctypes.data_as(ctypes.c_void_p)


def evaluate_tree(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho, plan: TreePlan,
                  mode=BOTH, out_u=None, out_v=None, workspace=None, stream=None):
    """stokes_er_eval_tree on device tensors with a TreePlan over the same nodes."""
    M, N, dev = _check_inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, mode)
    _check_dev("out_u", out_u if mode & SL else None, (3, M))
    _check_dev("out_v", out_v if mode & DL else None, (3, M))
    if plan.N != N:
        raise ValueError("plan built for another node count")
    L = _lib.load()
    if mode & SL and out_u is None:
        out_u = _out((3, M), dev, stream)
    if mode & DL and out_v is None:
        out_v = _out((3, M), dev, stream)
    if workspace is None:
        workspace = _scratch(L.stokes_er_tree_workspace_bytes(M, N, mode, ctypes.byref(plan.params), plan.ptr()),
                             dev, stream)
    st = L.stokes_er_eval_tree(_ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
                               _ptr(q if mode & DL else None), _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M,
                               N, float(h), _lib.rho_arg(rho), int(mode), ctypes.byref(plan.params), plan.ptr(),
                               _ptr(out_u if mode & SL else None), _ptr(out_v if mode & DL else None),
                               _ptr(workspace), int(workspace.numel()), _stream_handle(stream))
    _lib.check("stokes_er_eval_tree", st)
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def evaluate_tree_block(block, plan=None, mode=BOTH, device="cuda", leaf_size=2000, degree=6, theta=0.6, **kw):
    if plan is None:
        plan = TreePlan(block.src_xyz, leaf_size, degree, theta)
    return evaluate_tree(*to_device(block, device), block.h, block.rho, plan, mode=mode, **kw)


def evaluate_tree_onsurface(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, delta,
                            plan: TreePlan, mode=BOTH, out_u=None, out_v=None, workspace=None, stream=None):
    """stokes_er_eval_tree_onsurface: NEXT-1's s# evaluation with the treecode far part."""
    M, N, dev = _check_inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, mode)
    _check_dev("out_u", out_u if mode & SL else None, (3, M))
    _check_dev("out_v", out_v if mode & DL else None, (3, M))
    if plan.N != N:
        raise ValueError("plan built for another node count")
    L = _lib.load()
    if mode & SL and out_u is None:
        out_u = _out((3, M), dev, stream)
    if mode & DL and out_v is None:
        out_v = _out((3, M), dev, stream)
    if workspace is None:
        workspace = _scratch(L.stokes_er_tree_workspace_bytes(M, N, mode, ctypes.byref(plan.params), plan.ptr()),
                             dev, stream)
    st = L.stokes_er_eval_tree_onsurface(_ptr(src_xyz), _ptr(src_normal), _ptr(src_weight),
                                         _ptr(f if mode & SL else None), _ptr(q if mode & DL else None),
                                         _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M, N, float(delta),
                                         int(mode), ctypes.byref(plan.params), plan.ptr(),
                                         _ptr(out_u if mode & SL else None), _ptr(out_v if mode & DL else None),
                                         _ptr(workspace), int(workspace.numel()), _stream_handle(stream))
    _lib.check("stokes_er_eval_tree_onsurface", st)
    return (out_u if mode & SL else None), (out_v if mode & DL else None)
