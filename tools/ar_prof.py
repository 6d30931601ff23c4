"""Experiment (library built with -DAGQ_AR_PROFILE, AGQ_LIB pointing at it):
globaltimer stamps inside back-to-back fused all-reduces, per rank.
0 kernel start (CTA 0), 1 CTA 0 past the start barrier, 2 CTA 0 done with
its groups, 3 last CTA enters the end section, 4 errors shared + done
published, 5 every done seen, 6 call complete. Launch with torchrun."""
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200.collective import Communicator  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("gloo")
lib = A._lib.lib
lib.agq_ar_profile.argtypes = [C.c_void_p]
comm = Communicator(device=rank)
comm.enable_p2p(1 << 22)
for n in (1 << 16, 1 << 20, 1 << 22):
    pc, ps = comm.p2p_buffers(n)
    src = A.quantize_blockwise(torch.randn(n, device=dev) * 1e-3, 8, 128, A.CodecKind.Fp8E4M3,
                               packed=False)
    pc.copy_(src.codes)
    ps.copy_(src.scales)
    q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
    err = A.ErrorRecord(dev)
    prev_end = None
    rows = []
    for it in range(8):
        comm.allreduce_fp8(q, algo=os.environ.get("AR_ALGO", "p2p"), check=False, errors=err)
        buf = (C.c_ulonglong * 8)()
        lib.agq_ar_profile(buf)
        t = list(buf)
        rows.append([round((t[i] - t[0]) / 1e3, 2) for i in range(1, 7)])
    torch.cuda.synchronize()
    dist.barrier()
    for r in range(world):
        if r == rank:
            print(f"n={n} rank {rank} stamps us (1..6 rel. to 0), last 3 calls:", rows[-3:], flush=True)
        dist.barrier()
comm.close()
