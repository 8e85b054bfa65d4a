"""CPU oracle for the extrapolated-regularization Stokes layer potentials.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package.  The product
package paper_2507_00156_b200 never imports it, and it never imports the
product package.  See stokes_er_oracle.c for the formulas and PAPER.md
citations; every function here only marshals numpy arrays to that C code.

Pins (tests/test_oracle_*.py) tie it to closed forms, exact rational
extrapolation weights, paper-printed counts and a 50-digit mpmath brute
force, not to itself.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stokes_er_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

SL, DL, BOTH = 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_dp = ctypes.POINTER(ctypes.c_double)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_s_factors.argtypes = [ctypes.c_double, _dp]
        L.oracle_s_sharp_factors.argtypes = [ctypes.c_double, _dp]
        L.oracle_I0.argtypes = [ctypes.c_double]
        L.oracle_I0.restype = ctypes.c_double
        L.oracle_I2.argtypes = [ctypes.c_double]
        L.oracle_I2.restype = ctypes.c_double
        common = [_dp] * 8 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]
        L.oracle_eval_deltas.argtypes = common + [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.oracle_eval.argtypes = common + [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.oracle_eval_sharp.argtypes = common + [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                                 _dp, _dp]
        L.oracle_extrapolate.argtypes = [_dp, ctypes.c_int64, ctypes.c_double, _dp, _dp, ctypes.c_int, _dp]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_eval_tree.argtypes = common + [_dp, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                                ctypes.c_int, _dp, _dp, _dp]
        L.oracle_eval_tree_sharp.argtypes = common + [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                                      ctypes.c_int, _dp, _dp, _dp]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def s_factors(t: float):
    out = np.zeros(3)
    lib().oracle_s_factors(float(t), _p(out))
    return out


def s_sharp_factors(t: float):
    out = np.zeros(3)
    lib().oracle_s_sharp_factors(float(t), _p(out))
    return out


def I0(lam: float) -> float:
    return lib().oracle_I0(float(lam))


def I2(lam: float) -> float:
    return lib().oracle_I2(float(lam))


def max_threads() -> int:
    return lib().oracle_max_threads()


def _inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density):
    arrs = [_f64(a) for a in (src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density)]
    N = arrs[2].shape[0]
    M = arrs[6].shape[0]
    return arrs, M, N


def eval_deltas(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho,
                mode=BOTH, localized=False, nthreads=0):
    """Per-delta values: returns (u_delta (3,3,M) or None, v_delta (3,3,M) or None), index [k][i][m]."""
    arrs, M, N = _inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density)
    ud = np.zeros((3, 3, M)) if mode & SL else None
    vd = np.zeros((3, 3, M)) if mode & DL else None
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    rc = lib().oracle_eval_deltas(*[_p(a) for a in arrs], M, N, float(h), _p(rho), int(mode), int(localized),
                                  int(nthreads), _p(ud), _p(vd))
    if rc:
        raise ValueError("oracle_eval_deltas: invalid arguments")
    return ud, vd


def extrapolate(tgt_b, h, rho, in_delta):
    """in_delta: (3, C, M) -> (C, M); pivoted Gaussian elimination per target."""
    in_delta = _f64(in_delta)
    tgt_b = _f64(tgt_b)
    _, C, M = in_delta.shape
    out = np.zeros((C, M))
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    rc = lib().oracle_extrapolate(_p(tgt_b), M, float(h), _p(rho), _p(in_delta), C, _p(out))
    if rc:
        raise ValueError("oracle_extrapolate: invalid arguments")
    return out


def evaluate(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho,
             mode=BOTH, localized=False, nthreads=0):
    """Extrapolated u (3,M) and v (3,M) (None for a field the mode does not produce)."""
    arrs, M, N = _inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density)
    u = np.zeros((3, M)) if mode & SL else None
    v = np.zeros((3, M)) if mode & DL else None
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    rc = lib().oracle_eval(*[_p(a) for a in arrs], M, N, float(h), _p(rho), int(mode), int(localized),
                           int(nthreads), _p(u), _p(v))
    if rc:
        raise ValueError("oracle_eval: invalid arguments")
    return u, v


def evaluate_sharp(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, delta,
                   mode=BOTH, localized=False, cutoff=7.0, nthreads=0):
    """NEXT-1: single-delta on-surface evaluation with the s# factors."""
    arrs, M, N = _inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density)
    u = np.zeros((3, M)) if mode & SL else None
    v = np.zeros((3, M)) if mode & DL else None
    rc = lib().oracle_eval_sharp(*[_p(a) for a in arrs], M, N, float(delta), int(mode), int(localized),
                                 float(cutoff), int(nthreads), _p(u), _p(v))
    if rc:
        raise ValueError("oracle_eval_sharp: invalid arguments")
    return u, v


def evaluate_block(block, mode=BOTH, localized=False, nthreads=0):
    return evaluate(*block.arrays(), block.h, block.rho, mode=mode, localized=localized, nthreads=nthreads)


def eval_deltas_block(block, mode=BOTH, localized=False, nthreads=0):
    return eval_deltas(*block.arrays(), block.h, block.rho, mode=mode, localized=localized, nthreads=nthreads)


def evaluate_tree(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, h, rho,
                  leaf_size=2000, degree=6, theta=0.6, mode=BOTH, nthreads=0, stats=False):
    """NEXT-3: the treecode of PAPER.md Sec. 3.4 for the far part (readings R22-R25 in
    stokes_er_oracle.c).  Returns (u, v) or (u, v, stats) with stats =
    (nodes, accepted target-cluster pairs, directly summed target-source pairs)."""
    arrs, M, N = _inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density)
    u = np.zeros((3, M)) if mode & SL else None
    v = np.zeros((3, M)) if mode & DL else None
    st = np.zeros(3)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    rc = lib().oracle_eval_tree(*[_p(a) for a in arrs], M, N, float(h), _p(rho), int(mode), int(leaf_size),
                                int(degree), float(theta), int(nthreads), _p(u), _p(v), _p(st))
    if rc:
        raise ValueError(f"oracle_eval_tree: status {rc}")
    return (u, v, tuple(int(x) for x in st)) if stats else (u, v)


def evaluate_tree_block(block, mode=BOTH, nthreads=0, **kw):
    return evaluate_tree(*block.arrays(), block.h, block.rho, mode=mode, nthreads=nthreads, **kw)


def evaluate_tree_sharp(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, delta,
                        leaf_size=2000, degree=6, theta=0.6, mode=BOTH, nthreads=0):
    """NEXT-1's on-surface s# evaluation (single delta, cutoff 7) with the treecode far part."""
    arrs, M, N = _inputs(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density)
    u = np.zeros((3, M)) if mode & SL else None
    v = np.zeros((3, M)) if mode & DL else None
    rc = lib().oracle_eval_tree_sharp(*[_p(a) for a in arrs], M, N, float(delta), int(mode), int(leaf_size),
                                      int(degree), float(theta), int(nthreads), _p(u), _p(v), None)
    if rc:
        raise ValueError(f"oracle_eval_tree_sharp: status {rc}")
    return u, v
