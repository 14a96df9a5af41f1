"""The C++ mirror of the reference API (include/rbd/<name>.hpp): compile the
port of the reference's own C++ tests (tests/cpp/test_rbd_api.cpp) against
librbd_b200.so (CPU: must compile cleanly), and run it on the GPU."""
import os
import shutil
import subprocess

import pytest

from paper_1503_05947_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_rbd_api.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "build", "test_rbd_api")


def compile_test():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    cmd = [cxx, "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", _build.PKG, "-lrbd_b200", f"-Wl,-rpath,{_build.PKG}", "-o", OUT]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return OUT


def test_cpp_mirror_compiles():
    assert os.path.exists(compile_test())


@pytest.mark.gpu
def test_cpp_mirror_reference_tests_pass(cuda):
    exe = compile_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
