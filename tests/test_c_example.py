"""The C ABI used from plain C: examples/heat1d_c_example.c compiles against include/heat1d.h
and links libheat1d.so (CPU), and runs the paper's model problem on the GPU (-m gpu)."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2307_01117_b200")


def build_example(tmp_path):
    from paper_2307_01117_b200 import _build
    _build.build()
    exe = str(tmp_path / "heat1d_c_example")
    subprocess.run(["cc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "heat1d_c_example.c"), "-L", PKG, "-l:libheat1d.so",
                    "-Wl,-rpath," + PKG, "-o", exe], check=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    assert os.path.exists(build_example(tmp_path))


@pytest.mark.gpu
def test_c_example_runs_paper_problem(tmp_path):
    exe = build_example(tmp_path)
    p = subprocess.run([exe, "1000000", "1000"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "solve_host==run:yes" in p.stdout
