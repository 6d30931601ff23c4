"""Real-rank decomposed all-reduce parity: launches tests/mp_allreduce_check.py
under torchrun with one process per visible GPU — also on a 1-GPU box, where
P = 1 still runs NCCL communicator init, the IPC export/open of the symmetric
buffer, the epoch flags and the fused kernel k_fused_allreduce<1>."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = os.path.dirname(os.path.abspath(__file__))


def test_allreduce_real_ranks_bitexact():
    n = torch.cuda.device_count()
    assert n >= 1, "needs a GPU"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29541",
           os.path.join(HERE, "mp_allreduce_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:], r.stderr[-6000:])
    assert r.returncode == 0
    assert "failures=0" in r.stdout
