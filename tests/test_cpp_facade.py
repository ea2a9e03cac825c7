"""The C++ facade (include/batchheap_b200.hpp) compiles against the C ABI
library here (CPU) and runs the reference-shaped test cases on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
LIBDIR = os.path.join(ROOT, "paper_1906_06504_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_facade")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lbatchheap_b200", f"-Wl,-rpath,{LIBDIR}", "-lpthread", "-o", exe],
                   check=True)
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_facade_runs_reference_cases(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
