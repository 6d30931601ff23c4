"""Randomised multi-rank soak of the all-reduce algorithms against the CPU
oracle's allreduce_decomposed: random sizes (ragged tails), magnitudes with
zero blocks and extreme scales, every algorithm (NCCL, fused, push,
one-shot, auto) in random order, in place and through copies. Launch with
torchrun; argv[1] = seconds. Prints a summary on rank 0, exit 1 on a mismatch."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_ffi as O  # noqa: E402
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200.collective import Communicator  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    cap = 1 << 20
    comm = Communicator(device=local, p2p_capacity=cap)
    algos = ["nccl", "p2p", "push", "oneshot", "auto"] if world > 1 else ["nccl", "p2p", "oneshot"]
    seed0 = torch.tensor([int(time.time())], device=dev)
    dist.broadcast(seed0, 0)  # every rank draws the same case sequence
    rng = np.random.default_rng(int(seed0.item()))
    cases = fails = 0
    t0 = time.time()
    while True:
        go = torch.tensor([1 if time.time() - t0 < budget else 0], device=dev)
        dist.all_reduce(go, op=dist.ReduceOp.MIN)
        if not go.item():
            break
        n = int(rng.choice([rng.integers(1, 3000), rng.integers(3000, 300000), 128 * rng.integers(1, 8192)]))
        nb = (n + 127) // 128
        algo = algos[int(rng.integers(0, len(algos)))]
        inplace = bool(rng.integers(0, 2))
        g = []
        for r in range(world):
            mag = np.repeat(10.0 ** rng.uniform(-20, 20, nb), 128)[:n]
            x = (rng.standard_normal(n) * mag).astype(np.float32)
            if nb > 2:
                z = int(rng.integers(0, nb))
                x[z * 128:(z + 1) * 128] = 0.0
            g.append(O.quantize(x, 8, 128, O.FP8))
        want_c, want_s = O.allreduce_decomposed([c for c, _ in g], [s for _, s in g])
        c, s = g[rank]
        if inplace and algo != "nccl":
            pc, ps = comm.p2p_buffers(n)
            pc.copy_(torch.from_numpy(c))
            ps.copy_(torch.from_numpy(s))
            q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
        else:
            q = A.QuantizedTensor(torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev), 8, 128,
                                  (n,), A.CodecKind.Fp8E4M3, packed=False)
        err = None
        try:
            comm.allreduce_fp8(q, algo=algo)
        except A.ProtocolError as e:  # an fp32 overflow is a legitimate outcome
            err = str(e)
        if err is None:
            ok = np.array_equal(q.codes.cpu().numpy(), want_c) and \
                np.array_equal(q.scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))
        else:
            ok = "overflow" in err and not np.isfinite(want_s).all()
        if not ok:
            fails += 1
            print(f"rank {rank}: MISMATCH algo={algo} n={n} inplace={inplace} err={err}", flush=True)
        cases += 1
    t = torch.tensor([fails], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_soak world={world} cases={cases} failures={int(t.item())}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
