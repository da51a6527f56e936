# SPDX-License-Identifier: Apache-2.0
"""The C++ rankformer::gpu binding (include/rankformer/sort_gpu.hpp) compiles against the C ABI
and behaves like the reference API: host-only planner calls on CPU, scoring on the GPU."""
import os
import subprocess

import pytest

from paper_2603_03988_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "sort_gpu_example")


def _compile():
    B.build()
    src = os.path.join(ROOT, "tests", "cpp", "sort_gpu_example.cpp")
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(
            os.path.getmtime(src), os.path.getmtime(B.LIB),
            os.path.getmtime(os.path.join(ROOT, "include", "rankformer", "sort_gpu.hpp"))):
        subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                               "-I", "/usr/local/cuda/include", src, "-o", EXE,
                               "-L", os.path.dirname(B.LIB), "-lsort_b200",
                               "-Wl,-rpath," + os.path.dirname(B.LIB)])
    return EXE


def test_cpp_binding_host_rules():
    out = subprocess.run([_compile()], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "host ok" in out.stdout


@pytest.mark.gpu
def test_cpp_binding_scores_on_gpu():
    out = subprocess.run([_compile(), "--gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "gpu ok" in out.stdout
