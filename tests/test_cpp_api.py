"""The C++ host API (include/ldpc_b200.hpp) compiled with g++ against the
in-tree libldpc_b200.so and run: host cases on CPU, decoding cases on GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_1202_1060_b200")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "test_api")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", f"-I{os.path.join(ROOT, 'include')}", SRC, "-o", out,
           f"-L{LIBDIR}", "-lldpc_b200", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_host_api(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


@pytest.mark.gpu
def test_cpp_decode_api(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
