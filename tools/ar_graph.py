"""Small-message all-reduce latency: 50 back-to-back in-place calls issued
eagerly (through the Python API, or the C-ABI entry alone) vs the same 50
calls captured once in a CUDA graph and replayed (the P2P epoch lives on the
device, so the fused and push all-reduces are capturable). Device time per
call, max over ranks. Launch with torchrun."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200.collective import Communicator  # noqa: E402

CALLS = 50


def timed(fn, world):
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) * 1e3 / CALLS])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("gloo")
    comm = Communicator(device=rank)
    nmax = 1 << 24
    comm.enable_p2p(nmax)
    pc, ps = comm.p2p_buffers(nmax)
    src = A.quantize_blockwise(torch.randn(nmax, device=dev) * 1e-3, 8, 128, A.CodecKind.Fp8E4M3,
                               packed=False)
    err = A.ErrorRecord(dev)
    sp = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    L = A._lib
    rows = []
    for n in (1 << 16, 1 << 18, 1 << 19, 3 << 18, 1 << 20, 1 << 22):
        nb = n // 128
        q = A.QuantizedTensor(pc[:n], ps[:nb], 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)

        def restore():  # back-to-back calls grow the values x P per call:
            pc[:n].copy_(src.codes[:n])  # 50 calls stay far below FP32 range
            ps[:nb].copy_(src.scales[:nb])
            torch.cuda.synchronize()
        row = {"elements": n, "fp8_bytes": n}
        algos = ("p2p", "push", "oneshot") if world > 1 else ("p2p", "oneshot")
        for algo in algos:
            if algo == "oneshot" and n > comm.ONESHOT_MAX:
                continue
            def api():  # the Python API (validate, error record reset)
                for _ in range(CALLS):
                    comm.allreduce_fp8(q, algo=algo, check=False, errors=err)

            def abi():  # the C-ABI entry alone
                for _ in range(CALLS):
                    L.check(L.lib.agq_allreduce_fp8(comm._h, q.codes.data_ptr(), q.scales.data_ptr(),
                                                    n, 128, comm.ALGOS[algo], err.ptr, sp()))
            restore()
            api()  # warm up
            restore()
            row[f"{algo}_eager_api_us"] = round(timed(api, world), 2)
            restore()
            row[f"{algo}_eager_abi_us"] = round(timed(abi, world), 2)
            g = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                api()
            restore()
            g.replay()
            restore()
            row[f"{algo}_graph_us"] = round(timed(g.replay, world), 2)
            err.raise_if_any(L.AGQ_OP_ALLREDUCE)
            del g
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
