"""The header-only C++ host layer (include/bht_b200.hpp) compiled with g++ and linked against the C-ABI library:
host-side checks here on CPU, the full build / find / error-behaviour program on the GPU box."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "wrapper_check.cpp")
LIBDIR = os.path.join(ROOT, "paper_2108_07232_b200", "lib")


def build_exe(tmpdir):
    exe = os.path.join(tmpdir, "wrapper_check")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(cuda, "include"),
                           SRC, "-o", exe, "-L" + LIBDIR, "-lbht_b200", "-L" + os.path.join(cuda, "lib64"), "-lcudart",
                           "-Wl,-rpath," + LIBDIR, "-Wl,-rpath," + os.path.join(cuda, "lib64")])
    return exe


def test_cpp_wrapper_host_side(tmp_path, bht):
    exe = build_exe(str(tmp_path))
    r = subprocess.run([exe, "nogpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_c_header_is_plain_c(tmp_path):
    """include/bht_b200.h is a C header: plain pointers and PODs only, compiles as C11."""
    c = tmp_path / "t.c"
    c.write_text('#include "bht_b200.h"\nint main(void){ bht_config c; (void)c; return (int)sizeof(bht_insert_result) == 0; }\n')
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"), "-c", str(c), "-o",
                           str(tmp_path / "t.o")])


@pytest.mark.gpu
def test_cpp_wrapper_on_gpu(tmp_path):
    exe = build_exe(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "wrapper checks ok" in r.stdout
