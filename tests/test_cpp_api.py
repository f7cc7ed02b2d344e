"""The C++ host layer (include/flexattn_b200.hpp): compiles on CPU; its test program
(tests/cpp/test_cpp_api.cpp) runs on the GPU and checks BlockMask, forward, backward and the
error taxonomy against the oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "test_cpp_api")
PKG = os.path.join(ROOT, "paper_2412_05496_b200")
ORACLE = os.path.join(ROOT, "oracle")


def build():
    cmd = ["g++", "-std=c++17", "-O2", SRC, "-o", EXE, f"-I{ROOT}/include", f"-I{ORACLE}",
           "-I/usr/local/cuda/include", f"-L{PKG}", f"-L{ORACLE}", "-L/usr/local/cuda/lib64",
           "-lflexattn_b200", "-lflex_oracle", "-lcudart", f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{ORACLE}"]
    subprocess.run(cmd, check=True)


def test_cpp_header_compiles():
    build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_api_on_gpu(dev):
    if not os.path.exists(EXE):
        build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
