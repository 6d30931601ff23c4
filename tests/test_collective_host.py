"""Host-side choices of the real-rank all-reduce (CPU, no communicator):
algo="auto" must depend only on state every rank shares (capacity, n, block,
world size), so all ranks run the same algorithm."""
import pytest
import torch

import paper_2605_00539_b200 as A
from paper_2605_00539_b200 import _lib as L
from paper_2605_00539_b200.collective import Communicator


def comm(world, capacity, nccl=True):
    c = Communicator.__new__(Communicator)  # the selection logic only
    c.world, c.p2p_capacity, c.nccl = world, capacity, nccl
    return c


def grad(n, block=128):
    return A.QuantizedTensor(torch.empty(n, dtype=torch.uint8),
                             torch.empty((n + block - 1) // block), 8, block, (n,),
                             A.CodecKind.Fp8E4M3, packed=False)


@pytest.mark.parametrize("world,n,want", [
    (2, 64 << 10, "oneshot"), (2, 1 << 20, "oneshot"), (2, (1 << 20) + 128, "p2p"),
    (4, 512 << 10, "oneshot"), (4, (512 << 10) + 128, "p2p"),
    (8, 200 << 10, "oneshot"), (8, 256 << 10, "p2p"),
    (9, 64 << 10, "p2p"), (1, 1 << 20, "oneshot"),
])
def test_auto_picks_oneshot_for_small_messages(world, n, want):
    assert comm(world, 1 << 30)._auto_algo(grad(n)) == want


def test_auto_without_peer_buffers_or_other_blocks():
    assert comm(4, 0)._auto_algo(grad(1 << 20)) == "nccl"
    assert comm(4, 1 << 20)._auto_algo(grad((1 << 20) + 128)) == "nccl"  # beyond capacity
    assert comm(4, 1 << 30)._auto_algo(grad(4096, block=64)) == "nccl"   # P2P kernels: block 128
    with pytest.raises(L.InvalidArgument):
        comm(4, 0, nccl=False)._auto_algo(grad(4096))


def test_algorithm_ids_match_the_c_abi():
    assert Communicator.ALGOS == {"nccl": L.AGQ_AR_NCCL, "p2p": L.AGQ_AR_FUSED_P2P,
                                  "push": L.AGQ_AR_PUSH_P2P, "oneshot": L.AGQ_AR_ONESHOT_P2P}
    hdr = open(L.LIB_PATH.replace("paper_2605_00539_b200/libagq_cuda.so",
                                  "include/agq_cuda.h")).read()
    assert "AGQ_AR_ONESHOT_P2P = 3" in hdr
