"""The bench's reference arm (`bench.py --impl reference`) runs the reference
compiled from /root/reference (oracle/_ref) on host cores only: keep it
working, its JSON line complete, and free of this repo's own library (CPU
test)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_stage_bits_literal_is_the_plan():
    sys.path.insert(0, ROOT)
    import bench
    import oracle_ffi as O
    import paper_2605_00539_b200 as A
    assert list(bench.STAGE_BITS) == A.plan_bit_widths(A.PipelineConfig(8, 16, 2)).assigned()
    counts, raw, bits = np.zeros(8, np.int32), np.zeros(8), np.zeros(8, np.int32)
    O.orc.oracle_plan_bit_widths(8, 16, 2, O._p(counts), O._p(raw), O._p(bits))
    assert list(bench.STAGE_BITS) == bits.tolist()


def test_reference_arm_line_and_no_repo_library():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libagq_ref.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    code = ("import runpy, sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1',"
            " '--warmup', '1']; runpy.run_path('bench.py', run_name='__main__');"
            " maps = open('/proc/self/maps').read();"
            " print(json.dumps({'libagq_cuda': 'libagq_cuda' in maps,"
            " 'libagq_ref': 'libagq_ref' in maps}))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    line, maps = json.loads(lines[-2]), json.loads(lines[-1])
    assert maps == {"libagq_cuda": False, "libagq_ref": True}
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    cb = line["cpu_baseline"]
    assert line["value"] > 0 and cb["kind"] == "reference"
    assert cb["single_core"]["cores"] == 1 and cb["single_core"]["value"] > 0
    assert cb["nproc"] >= 1 and cb["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
