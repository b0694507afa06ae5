"""The drop-in C++ API (include/fourierbf/*.hpp + libfourierbf_b200.so) compiled
against and exercised like the reference's own suites (tests/cpp/test_api.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1603_08081_b200", "_lib")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "test_api")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-L", LIBDIR, "-lfourierbf_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def test_cpp_api_host_checks(binary):
    r = subprocess.run([binary, "--host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_full(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
