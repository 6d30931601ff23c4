"""Latency floor of the decomposed 8-bit all-reduce (fused NVLink vs NCCL v1 vs
BF16 ncclAllReduce) at small messages. Launch with torchrun, N >= 2."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200 import _lib as L  # noqa: E402
from paper_2605_00539_b200.collective import Communicator  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("gloo")
    comm = Communicator(device=rank)
    nmax = 1 << 22
    comm.enable_p2p(nmax)
    pc, ps = comm.p2p_buffers(nmax)
    sp = torch.cuda.current_stream().cuda_stream
    err = A.ErrorRecord(dev).reset()
    src = torch.randn(nmax, device=dev) * 1e-3
    q = A.quantize_blockwise(src, 8, 128, A.CodecKind.Fp8E4M3, packed=False)
    gb = torch.randn(nmax, device=dev).to(torch.bfloat16)
    wc, ws = q.codes.clone(), q.scales.clone()
    out = []
    for n in (128, 1 << 14, 1 << 17, 1 << 20, 1 << 22):
        nb = (n + 127) // 128
        row = {"elements": n}
        for algo, (cb, sb) in (("p2p", (pc, ps)), ("nccl", (wc, ws))):
            def fn():
                # restore inputs each call (values would grow x P per call)
                cb[:n].copy_(q.codes[:n])
                sb[:nb].copy_(q.scales[:nb])
                L.check(L.lib.agq_allreduce_fp8(comm._h, cb.data_ptr(), sb.data_ptr(), n, 128,
                                                comm.ALGOS[algo], err.ptr, sp))
            def copies():
                cb[:n].copy_(q.codes[:n])
                sb[:nb].copy_(q.scales[:nb])
            for f in (fn, copies):
                for _ in range(5):
                    f()
            ts = {}
            for label, f in (("with_restore", fn), ("restore_only", copies)):
                torch.cuda.synchronize()
                dist.barrier()
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record()
                for _ in range(50):
                    f()
                e.record()
                torch.cuda.synchronize()
                t = torch.tensor([s.elapsed_time(e) / 50 * 1e3])
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ts[label] = t.item()
            row[algo + "_us"] = round(ts["with_restore"] - ts["restore_only"], 2)
        def bf():
            L.check(L.lib.agq_allreduce_bf16_nccl(comm._h, gb.data_ptr(), n, sp))
        for _ in range(5):
            bf()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(50):
            bf()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / 50 * 1e3])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        row["bf16_nccl_us"] = round(t.item(), 2)
        L.errors_message(err.read(), L.AGQ_OP_ALLREDUCE)
        out.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
