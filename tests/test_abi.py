"""The C-ABI library loads and exports every symbol include/stokes_er.h declares (CPU only: no compute calls)."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "stokes_er.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stokes_er_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_00156_b200 import build
    build.build()
    from paper_2507_00156_b200 import _lib
    return _lib.load()


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ["stokes_er_eval", "stokes_er_workspace_bytes", "stokes_er_eval_deltas", "stokes_er_extrapolate",
              "stokes_er_eval_host", "stokes_er_status_string"]:
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2507_00156_b200 import _lib
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == set(declared_functions())


def test_pure_host_queries(lib):
    assert lib.stokes_er_abi_version() == 4
    assert lib.stokes_er_nodes_launch_count(0, 3) == 0 and lib.stokes_er_nodes_launch_count(10, 3) == 8
    assert lib.stokes_er_status_string(5) == b"GMRES reached max_iter above the tolerance"
    assert lib.stokes_er_status_string(3) == b"workspace too small"
    assert lib.stokes_er_launch_count(0, 10, 3) == 0


def test_sm100a_only_cubin():
    """The library carries sm_100a SASS (no PTX JIT fallback for other archs)."""
    import subprocess
    from paper_2507_00156_b200 import build
    path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass or "UBLKPF" in sass or "BLKCP" in sass  # TMA bulk copy in the pair kernel
    assert "DFMA" in sass and "MUFU.RSQ64H" in sass


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2507_00156_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in text and "from oracle" not in text and "liboracle" not in text, fn


def _build_c_demo(tmp_path):
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "c_api_demo")
    pkg = os.path.join(root, "paper_2507_00156_b200")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(root, "examples", "c_api_demo.c"), "-L", pkg, "-lstokes_er",
                           "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{pkg}", "-o", exe])
    return exe


def test_c_demo_compiles_against_the_header(tmp_path):
    """The boundary is usable from plain C: examples/c_api_demo.c compiles and links
    against include/stokes_er.h and libstokes_er.so (no torch, no Python)."""
    assert os.path.exists(_build_c_demo(tmp_path))


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    import subprocess

    out = subprocess.run([_build_c_demo(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
