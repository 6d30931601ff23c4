"""allreduce_naive_fp8 (the FP8 ring strawman, collective.hpp:338-431) vs the
decomposed all-reduce (collective.hpp:226-333, NCCL v1 and the fused NVLink
kernel) on real ranks: device time (max over ranks), overflow counts and the
relative L2 error against the exact FP32 sum of the dequantized inputs.
Launch with torchrun, N >= 2. Inputs: rank r's gradient = FP8 quantize of
N(0, 1e-3) from torch.Generator seed r (every rank regenerates all of them)."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200.collective import Communicator  # noqa: E402


def grad(r, n, dev):
    g = torch.Generator(device=dev).manual_seed(r)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    return A.quantize_blockwise(x, 8, 128, A.CodecKind.Fp8E4M3, packed=False)


def timed(fn, restore, iters=20):
    for f in (fn, restore):
        for _ in range(3):
            f()
    ts = []
    for f in (fn, restore):
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(iters):
            f()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / iters])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ts.append(t.item())
    return ts[0] - ts[1]


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("gloo")
    comm = Communicator(device=rank)
    sizes = [1 << 20, 1 << 24, 1 << 27]
    comm.enable_p2p(max(sizes))
    for n in sizes:
        qs = [grad(r, n, dev) for r in range(world)]
        exact = torch.zeros(n, device=dev)
        for q in qs:
            exact += A.dequantize_blockwise(q, out_dtype=torch.float32)
        mine = qs[rank]
        nb = (n + 127) // 128
        pc, ps = comm.p2p_buffers(n)
        wc, ws = mine.codes.clone(), mine.scales.clone()
        row = {"world": world, "elements": n}
        for algo in ("naive", "nccl", "p2p"):
            cb, sb = (pc, ps) if algo == "p2p" else (wc, ws)
            work = A.QuantizedTensor(cb[:n], sb[:nb], 8, 128, (n,), A.CodecKind.Fp8E4M3,
                                     packed=False)

            def restore():
                cb[:n].copy_(mine.codes)
                sb[:nb].copy_(mine.scales)

            def run():
                restore()
                if algo == "naive":
                    return comm.allreduce_naive_fp8(work)
                return comm.allreduce_fp8(work, algo=algo, check=False)

            ms = timed(run, restore)
            res = run()
            got = A.dequantize_blockwise(work, out_dtype=torch.float32)
            rel = ((got - exact).norm() / exact.norm()).item()
            row[algo + "_ms"] = round(ms, 4)
            row[algo + "_rel_l2"] = round(rel, 5)
            row[algo + "_wire_busbw_GBs"] = round(2 * (world - 1) / world * n * (1 + 4 / 128)
                                                  / (ms * 1e-3) / 1e9, 1)
            if algo == "naive":
                row["naive_overflow_elements"] = res[1]
        if rank == 0:
            print(json.dumps(row), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
