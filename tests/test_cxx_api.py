"""The C++ drop-in headers (include/intergrams/) compiled against the library
with g++ -std=c++20: header-only host logic runs everywhere; the GPU cases run
on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cxx_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2511_14955_b200", "_lib")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cxx") / "test_cxx_api")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", LIBDIR, "-lintergrams_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    subprocess.run(cmd, check=True)
    return out


def test_cxx_api_host_paths(binary):
    r = subprocess.run([binary, "--no-gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout


@pytest.mark.gpu
def test_cxx_api_on_gpu(binary, gpu_lib):
    r = subprocess.run([binary], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
