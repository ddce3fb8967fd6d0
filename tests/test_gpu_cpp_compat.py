"""Builds and runs tests/cpp/test_compat.cpp: the reference's C++ batch API surface
(include/gecc/sm2batch_compat.hpp) exercised the way the reference's own
tests/test_batch_point.cpp does, on the GPU, checked against the C oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(out, source="test_compat.cpp"):
    from oracle import coracle
    coracle.lib()  # makes sure oracle/_build/libgecc_oracle.so exists
    lib = os.path.join(ROOT, "paper_2501_03245_b200", "lib")
    orc = os.path.join(ROOT, "oracle", "_build")
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                           "-I" + os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "cpp", source),
                           "-o", out, "-L" + lib, "-lgecc_b200", "-L" + orc, "-lgecc_oracle",
                           "-Wl,-rpath," + lib, "-Wl,-rpath," + orc])


def test_compat_header_compiles(tmp_path):
    """CPU-side: the header is valid C++20 and links against the library."""
    _compile(str(tmp_path / "test_compat"))


@pytest.mark.gpu
def test_compat_cpp_suite(tmp_path):
    exe = str(tmp_path / "test_compat")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "compat tests passed" in r.stdout


def test_protocol_compat_compiles(tmp_path):
    _compile(str(tmp_path / "test_protocol_compat"), "test_protocol_compat.cpp")


@pytest.mark.gpu
def test_protocol_compat_cpp_suite(tmp_path):
    """protocol.hpp:14-124 mirrored over the C ABI: the scenarios of the reference's
    test_protocol.cpp:40-228 and test_batch_point.cpp:160-208 on the GPU, both curves."""
    exe = str(tmp_path / "test_protocol_compat")
    _compile(exe, "test_protocol_compat.cpp")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "protocol compat tests passed" in r.stdout
