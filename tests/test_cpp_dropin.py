"""The C++ drop-in (include/radial/*.hpp over libradial_cuda.so): reference-style caller
code compiles unchanged (CPU) and passes its parity program on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_2506_19852_b200", "lib")


def _compile(out):
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", "-o", out, SRC, f"-L{LIBDIR}",
           "-lradial_cuda", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_dropin_headers_compile_and_link(tmp_path):
    _compile(str(tmp_path / "dropin_test"))


@pytest.mark.gpu
def test_dropin_parity_program_on_gpu(tmp_path):
    exe = str(tmp_path / "dropin_test")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
