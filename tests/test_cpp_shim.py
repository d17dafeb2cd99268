"""The C++ drop-in shim (include/vdfcg.hpp) compiles and links against libvdfcg.so (CPU);
on a GPU it fits and rethrows the reference's exception types."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2504_14897_b200")


def _build(tmp_path):
    exe = str(tmp_path / "abi_smoke")
    subprocess.run(["g++", "-std=c++17", "-O2", os.path.join(ROOT, "tests", "cpp", "abi_smoke.cpp"),
                    "-L" + PKG, "-lvdfcg", "-Wl,-rpath," + PKG, "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "invalid_argument: fit: degenerate data: axis 0 has zero spread" in r.stdout
    assert "cells ok=64 records=64" in r.stdout
    assert "generate T=(0.850,0.850)" in r.stdout
    assert "invalid_argument: fractions must sum to 1" in r.stdout
