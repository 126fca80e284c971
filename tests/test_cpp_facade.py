"""The header-only C++ facade (include/superneuro_mat.hpp) compiles against the
C ABI with a plain g++ (CPU) and reproduces two reference KATs (GPU)."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "facade_example.cpp")
LIBDIR = os.path.join(ROOT, "paper_2305_02510_b200")


def _build(tmp_path):
    exe = str(tmp_path / "facade_example")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lsnmat", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                   check=True, capture_output=True, text=True)
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_facade_runs_reference_kats(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade ok" in out.stdout
