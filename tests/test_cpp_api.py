"""The C++ host API (include/denseplan_b200/block.hpp) compiled against
libdpb.so and exercised by tests/cpp/block_api_test.cpp."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "block_api_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_1707_06990_b200", "_build")
EXE = os.path.join(LIBDIR, "block_api_test")


@pytest.fixture(scope="module")
def exe():
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", f"-I{ROOT}/include", "-I/usr/local/cuda/include", SRC,
           f"-L{LIBDIR}", "-ldpb", f"-Wl,-rpath,{LIBDIR}", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", EXE]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_cpp_api_host(exe):
    r = subprocess.run([exe, "--host"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_device(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
