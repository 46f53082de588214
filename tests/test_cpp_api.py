"""The drop-in C++ API (include/sof_b200/sof.hpp) compiled against the Eigen/GTest shims,
running the reference's own test cases (tests/cpp/test_api.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "test_api")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "oracle", "eigen_shim"), "-I", os.path.join(ROOT, "oracle", "gtest_shim"),
           os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-L", os.path.join(ROOT, "paper_2506_19139_b200"),
           "-lsof_cuda", "-Wl,-rpath," + os.path.join(ROOT, "paper_2506_19139_b200"), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return exe


def test_cpp_api_compiles(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_cpp_api_reference_cases(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
