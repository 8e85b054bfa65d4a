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


def _shapes(src_xyz, tgt_b):
    return int(tgt_b.shape[0]), int(src_xyz.shape[1])


def evaluate(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho, mode=BOTH,
             out_u=None, out_v=None, workspace=None, stream=None, options: "_lib.Options | None" = None):
    """stokes_er_eval on device tensors; returns (u (3,M) or None, v (3,M) or None).
    Asynchronous on `stream` (default: torch's current stream)."""
    torch = _torch()
    M, N = _shapes(src_xyz, tgt_b)
    dev = src_xyz.device
    _check_dev("src_xyz", src_xyz, (3, N))
    _check_dev("src_normal", src_normal, (3, N))
    _check_dev("src_weight", src_weight, (N,))
    _check_dev("f", f if mode & SL else None, (3, N))
    _check_dev("q", q if mode & DL else None, (3, N))
    _check_dev("tgt_xyz", tgt_xyz, (3, M))
    _check_dev("tgt_b", tgt_b, (M,))
    _check_dev("tgt_x0_density", tgt_x0_density, (9, M))
    if mode & SL and out_u is None:
        out_u = torch.empty((3, M), dtype=torch.float64, device=dev)
    if mode & DL and out_v is None:
        out_v = torch.empty((3, M), dtype=torch.float64, device=dev)
    L = _lib.load()
    if workspace is None:
        if options is None:
            workspace = alloc_workspace(M, N, mode, dev)
        else:
            nbytes = int(L.stokes_er_workspace_bytes_ex(M, N, mode, ctypes.byref(options)))
            workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
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
    torch = _torch()
    M, N = _shapes(src_xyz, tgt_b)
    dev = src_xyz.device
    if mode & SL and out_u is None:
        out_u = torch.empty((3, M), dtype=torch.float64, device=dev)
    if mode & DL and out_v is None:
        out_v = torch.empty((3, M), dtype=torch.float64, device=dev)
    if workspace is None:
        workspace = alloc_workspace(M, N, mode, dev)
    L = _lib.load()
    _lib.check("stokes_er_eval_onsurface", L.stokes_er_eval_onsurface(
        _ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
        _ptr(q if mode & DL else None), _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M, N, float(delta),
        int(mode), _ptr(out_u if mode & SL else None), _ptr(out_v if mode & DL else None), _ptr(workspace),
        int(workspace.numel()), _stream_handle(stream)))
    return (out_u if mode & SL else None), (out_v if mode & DL else None)


def eval_deltas(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho, mode=BOTH,
                stream=None):
    """stokes_er_eval_deltas: per-delta u^{delta_k}, v^{delta_k} as (3,3,M) tensors [k][i][m]."""
    torch = _torch()
    M, N = _shapes(src_xyz, tgt_b)
    dev = src_xyz.device
    ud = torch.empty((3, 3, M), dtype=torch.float64, device=dev) if mode & SL else None
    vd = torch.empty((3, 3, M), dtype=torch.float64, device=dev) if mode & DL else None
    L = _lib.load()
    _lib.check("stokes_er_eval_deltas", L.stokes_er_eval_deltas(
        _ptr(src_xyz), _ptr(src_normal), _ptr(src_weight), _ptr(f if mode & SL else None),
        _ptr(q if mode & DL else None), _ptr(tgt_xyz), _ptr(tgt_b), _ptr(tgt_x0_density), M, N, float(h),
        _lib.rho_arg(rho), int(mode), _ptr(ud), _ptr(vd), None, 0, _stream_handle(stream)))
    return ud, vd


def extrapolate(tgt_b, h, rho, in_delta, stream=None):
    """stokes_er_extrapolate: in_delta (3, C, M) device -> (C, M)."""
    torch = _torch()
    _, C, M = in_delta.shape
    out = torch.empty((C, M), dtype=torch.float64, device=in_delta.device)
    L = _lib.load()
    _lib.check("stokes_er_extrapolate", L.stokes_er_extrapolate(
        _ptr(tgt_b), M, float(h), _lib.rho_arg(rho), _ptr(in_delta.contiguous()), int(C), _ptr(out),
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
