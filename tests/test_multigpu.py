"""Multi-GPU decomposed all-reduce parity (needs >= 2 GPUs on one box):
launches tests/mp_allreduce_check.py under torchrun with every visible GPU,
once per fused-kernel shape (16 elements per thread, the default, and 8)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("ept", ["16", "8"])
def test_allreduce_multigpu_bitexact(ept):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    n = torch.cuda.device_count()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29533 + int(ept)}",
           os.path.join(HERE, "mp_allreduce_check.py")]
    env = dict(os.environ, AGQ_P2P_EPT=ept)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert "failures=0" in r.stdout
