"""Builds tests/cpp/test_api.cpp against the reference-compatible C++ library
(libtrioalign.so) and runs it on the GPU: the reference's own public-API test
cases, checked against the C oracle."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
PKG = os.path.join(ROOT, "paper_2605_28400_b200")


def build_test_binary(tmp_path):
    exe = os.path.join(str(tmp_path), "test_api")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    subprocess.run(["g++", "-O1", "-std=c++20", "-I", os.path.join(PKG, "csrc", "include"),
                    "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "test_api.cpp"),
                    os.path.join(ROOT, "oracle", "trio_oracle.c"), "-x", "none",
                    "-L", PKG, "-ltrioalign", "-ltrioalign_b200", f"-Wl,-rpath,{PKG}", "-lpthread", "-o", exe],
                   check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    build_test_binary(tmp_path)


@pytest.mark.gpu
def test_cpp_api_reference_cases(tmp_path):
    exe = build_test_binary(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(out.stdout[-2000:], out.stderr[-4000:])
    assert out.returncode == 0
    assert "failed: 0" in out.stdout
