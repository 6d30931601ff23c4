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


def test_allreduce_p2p_more_ranks_than_gpus():
    """P2P-only communicators with two ranks per GPU (time-sliced): the fused
    and push kernels at up to P = 8 on a 4-GPU box (P = 2 on one GPU)."""
    g = torch.cuda.device_count()
    assert g >= 1, "needs a GPU"
    n = min(8, 2 * g)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29543",
           os.path.join(HERE, "mp_p2p_oversubscribed.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    print(r.stdout[-6000:], r.stderr[-6000:])
    assert r.returncode == 0
    assert "failures=0" in r.stdout
