"""The C++ drop-in (include/agq_b200/*.hpp: the reference's agq:: API on the
GPU via libagq_cuda.so) builds here, and on the B200 passes the reference's
hot-path test cases re-expressed in tests/cpp/dropin_tests.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_00539_b200")


def build(out):
    subprocess.run(["g++", "-std=c++20", "-O2", "-o", out,
                    os.path.join(ROOT, "tests", "cpp", "dropin_tests.cpp"),
                    "-L" + PKG, "-lagq_cuda", "-Wl,-rpath," + PKG,
                    "-L" + os.path.join(ROOT, "oracle"), "-loracle",
                    "-Wl,-rpath," + os.path.join(ROOT, "oracle")], check=True)


def test_dropin_headers_compile_and_link(tmp_path):
    build(str(tmp_path / "dropin_tests"))


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(tmp_path, cuda):
    exe = str(tmp_path / "dropin_tests")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert " 0 failures" in r.stdout
