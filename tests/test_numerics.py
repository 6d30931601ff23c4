"""The device element functions (paper_2605_00539_b200/csrc/agq_numerics.cuh),
compiled for the host from the SAME source, against the oracle: exhaustive
over the BF16 activation domain and every (code, BF16 scale) pair, random +
adversarial near-boundary FP32 inputs, extreme block scales.
tests/test_gpu_codec.py repeats the exhaustive classes on the B200 itself."""
import os
import subprocess

import oracle_ffi as O

ROOT = O.ROOT


def test_numerics_exhaustive_host(tmp_path):
    exe = tmp_path / "numerics_check"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tests", "cpp", "numerics_check.cpp"),
                    "-L" + os.path.join(ROOT, "oracle"), "-loracle",
                    "-Wl,-rpath," + os.path.join(ROOT, "oracle")], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    assert "TOTAL mismatches=0" in r.stdout
