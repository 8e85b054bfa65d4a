"""ctypes binding of include/stokes_er.h (argument marshalling only).

Every step of the evaluation runs in libstokes_er.so's CUDA kernels.  There is
no CPU fallback: a missing library or a missing GPU raises.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STOKES_ER_LIB") or os.path.join(PKG, "libstokes_er.so")

STATUS = {0: "ok", 1: "EINVAL", 2: "ECUDA", 3: "EWORKSPACE", 4: "EARCH", 5: "ENOCONV"}

_dp = ctypes.c_void_p  # device or host pointers are passed as raw addresses
_i64 = ctypes.c_int64


class StokesERError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed: status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("pair_kernel_start_event", ctypes.c_void_p), ("pair_kernel_end_event", ctypes.c_void_p),
                ("targets_per_thread", ctypes.c_int), ("source_chunk_tiles", ctypes.c_int),
                ("stats", ctypes.c_int64 * 4), ("near_kernel_start_event", ctypes.c_void_p),
                ("near_kernel_end_event", ctypes.c_void_p), ("near_phases", ctypes.c_int),
                ("schedule", ctypes.c_int), ("shard_index", ctypes.c_int), ("shard_count", ctypes.c_int)]


class Drop(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("xyz", ctypes.c_void_p), ("normal", ctypes.c_void_p),
                ("weight", ctypes.c_void_p), ("f", ctypes.c_void_p), ("lam", ctypes.c_double)]


class Cross(ctypes.Structure):
    _fields_ = [("b", ctypes.c_void_p), ("x0d", ctypes.c_void_p)]


class TreeParams(ctypes.Structure):
    _fields_ = [("leaf_size", ctypes.c_int), ("degree", ctypes.c_int), ("theta", ctypes.c_double)]


class TwoDropParams(ctypes.Structure):
    _fields_ = [("h", ctypes.c_double), ("rho", ctypes.c_double * 3), ("delta_self", ctypes.c_double),
                ("mu0", ctypes.c_double), ("tol", ctypes.c_double), ("max_iter", ctypes.c_int),
                ("use_tree", ctypes.c_int), ("tree_plan", ctypes.c_void_p * 2), ("tree", ctypes.POINTER(TreeParams))]


EXPORTS = ["stokes_er_workspace_bytes", "stokes_er_workspace_bytes_ex", "stokes_er_eval", "stokes_er_eval_ex", "stokes_er_host_workspace_bytes",
           "stokes_er_eval_host", "stokes_er_eval_deltas", "stokes_er_eval_onsurface", "stokes_er_extrapolate", "stokes_er_launch_count",
           "stokes_er_status_string", "stokes_er_abi_version", "stokes_er_twodrop_workspace_bytes",
           "stokes_er_twodrop_workspace_bytes_ex", "stokes_er_twodrop_setup", "stokes_er_twodrop_rhs", "stokes_er_twodrop_apply", "stokes_er_twodrop_solve",
           "stokes_er_tree_plan_bytes", "stokes_er_tree_build", "stokes_er_tree_info", "stokes_er_tree_workspace_bytes",
           "stokes_er_eval_tree", "stokes_er_eval_tree_onsurface", "stokes_er_nodes_workspace_bytes",
           "stokes_er_nodes_workspace_bytes_ex", "stokes_er_eval_nodes", "stokes_er_eval_nodes_ex",
           "stokes_er_nodes_host_workspace_bytes", "stokes_er_eval_nodes_host", "stokes_er_nodes_launch_count",
           "stokes_er_nodes_pair_counts", "stokes_er_eval_nodes_onsurface"]

_lib = None


def load():
    """Load libstokes_er.so (built by paper_2507_00156_b200.build / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: the CUDA extension is not built "
                          "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    eval_args = [_dp] * 8 + [_i64, _i64, ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                             _dp, _dp, _dp, ctypes.c_size_t, _dp]
    L.stokes_er_workspace_bytes.argtypes = [_i64, _i64, ctypes.c_int]
    L.stokes_er_workspace_bytes.restype = ctypes.c_size_t
    L.stokes_er_workspace_bytes_ex.argtypes = [_i64, _i64, ctypes.c_int, ctypes.POINTER(Options)]
    L.stokes_er_workspace_bytes_ex.restype = ctypes.c_size_t
    L.stokes_er_host_workspace_bytes.argtypes = [_i64, _i64, ctypes.c_int]
    L.stokes_er_host_workspace_bytes.restype = ctypes.c_size_t
    L.stokes_er_eval.argtypes = eval_args
    L.stokes_er_eval.restype = ctypes.c_int
    L.stokes_er_eval_ex.argtypes = eval_args + [ctypes.POINTER(Options)]
    L.stokes_er_eval_ex.restype = ctypes.c_int
    L.stokes_er_eval_host.argtypes = eval_args
    L.stokes_er_eval_host.restype = ctypes.c_int
    L.stokes_er_eval_onsurface.argtypes = [_dp] * 8 + [_i64, _i64, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp,
                                                      ctypes.c_size_t, _dp]
    L.stokes_er_eval_onsurface.restype = ctypes.c_int
    L.stokes_er_eval_deltas.argtypes = eval_args
    L.stokes_er_eval_deltas.restype = ctypes.c_int
    L.stokes_er_extrapolate.argtypes = [_dp, _i64, ctypes.c_double, ctypes.POINTER(ctypes.c_double), _dp,
                                        ctypes.c_int, _dp, _dp]
    L.stokes_er_extrapolate.restype = ctypes.c_int
    L.stokes_er_launch_count.argtypes = [_i64, _i64, ctypes.c_int]
    L.stokes_er_launch_count.restype = ctypes.c_int
    L.stokes_er_status_string.argtypes = [ctypes.c_int]
    L.stokes_er_status_string.restype = ctypes.c_char_p
    L.stokes_er_abi_version.restype = ctypes.c_int
    td = [ctypes.POINTER(Drop), ctypes.POINTER(Cross), ctypes.POINTER(TwoDropParams)]
    L.stokes_er_twodrop_workspace_bytes.argtypes = [_i64, _i64, ctypes.c_int]
    L.stokes_er_twodrop_workspace_bytes.restype = ctypes.c_size_t
    L.stokes_er_twodrop_workspace_bytes_ex.argtypes = [_i64, _i64, ctypes.POINTER(TwoDropParams)]
    L.stokes_er_twodrop_workspace_bytes_ex.restype = ctypes.c_size_t
    L.stokes_er_twodrop_setup.argtypes = td + [_dp, ctypes.c_size_t, _dp]
    L.stokes_er_twodrop_setup.restype = ctypes.c_int
    L.stokes_er_twodrop_rhs.argtypes = td + [_dp, _dp, ctypes.c_size_t, _dp]
    L.stokes_er_twodrop_rhs.restype = ctypes.c_int
    L.stokes_er_twodrop_apply.argtypes = td + [_dp, _dp, _dp, ctypes.c_size_t, _dp]
    L.stokes_er_twodrop_apply.restype = ctypes.c_int
    L.stokes_er_twodrop_solve.argtypes = td + [_dp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                               _dp, ctypes.c_size_t, _dp]
    L.stokes_er_twodrop_solve.restype = ctypes.c_int
    tp = ctypes.POINTER(TreeParams)
    L.stokes_er_tree_plan_bytes.argtypes = [_i64, tp]
    L.stokes_er_tree_plan_bytes.restype = ctypes.c_size_t
    L.stokes_er_tree_build.argtypes = [_dp, _i64, tp, _dp, ctypes.c_size_t]
    L.stokes_er_tree_build.restype = ctypes.c_int
    L.stokes_er_tree_info.argtypes = [_dp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
    L.stokes_er_tree_info.restype = ctypes.c_int
    L.stokes_er_tree_workspace_bytes.argtypes = [_i64, _i64, ctypes.c_int, tp, _dp]
    L.stokes_er_tree_workspace_bytes.restype = ctypes.c_size_t
    L.stokes_er_eval_tree.argtypes = [_dp] * 8 + [_i64, _i64, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                                                  ctypes.c_int, tp, _dp, _dp, _dp, _dp, ctypes.c_size_t, _dp]
    L.stokes_er_eval_tree.restype = ctypes.c_int
    L.stokes_er_eval_tree_onsurface.argtypes = [_dp] * 8 + [_i64, _i64, ctypes.c_double, ctypes.c_int, tp, _dp, _dp,
                                                            _dp, _dp, ctypes.c_size_t, _dp]
    L.stokes_er_eval_tree_onsurface.restype = ctypes.c_int
    nodes_args = [_dp] * 5 + [_i64, ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.c_int, _dp, _dp, _dp,
                              ctypes.c_size_t, _dp]
    L.stokes_er_nodes_workspace_bytes.argtypes = [_i64, ctypes.c_int]
    L.stokes_er_nodes_workspace_bytes.restype = ctypes.c_size_t
    L.stokes_er_nodes_workspace_bytes_ex.argtypes = [_i64, ctypes.c_int, ctypes.POINTER(Options)]
    L.stokes_er_nodes_workspace_bytes_ex.restype = ctypes.c_size_t
    L.stokes_er_nodes_host_workspace_bytes.argtypes = [_i64, ctypes.c_int]
    L.stokes_er_nodes_host_workspace_bytes.restype = ctypes.c_size_t
    L.stokes_er_eval_nodes.argtypes = nodes_args
    L.stokes_er_eval_nodes.restype = ctypes.c_int
    L.stokes_er_eval_nodes_ex.argtypes = nodes_args + [ctypes.POINTER(Options)]
    L.stokes_er_eval_nodes_ex.restype = ctypes.c_int
    L.stokes_er_eval_nodes_host.argtypes = nodes_args
    L.stokes_er_eval_nodes_host.restype = ctypes.c_int
    L.stokes_er_nodes_launch_count.argtypes = [_i64, ctypes.c_int]
    L.stokes_er_nodes_launch_count.restype = ctypes.c_int
    L.stokes_er_eval_nodes_onsurface.argtypes = [_dp] * 5 + [_i64, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp,
                                                 ctypes.c_size_t, _dp]
    L.stokes_er_eval_nodes_onsurface.restype = ctypes.c_int
    L.stokes_er_nodes_pair_counts.argtypes = [_i64, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_double), _dp,
                                              ctypes.c_size_t, ctypes.POINTER(_i64), _dp]
    L.stokes_er_nodes_pair_counts.restype = ctypes.c_int
    _lib = L
    return L


def check(fn: str, status: int):
    if status != 0:
        raise StokesERError(fn, status, load().stokes_er_status_string(status).decode())


def rho_arg(rho):
    return (ctypes.c_double * 3)(*[float(r) for r in rho])
