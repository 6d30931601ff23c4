"""Real-rank P2P all-reduce with more ranks than GPUs (torchrun, gloo for
the handle exchange, P2P-only communicators: NCCL refuses two ranks on one
GPU). Ranks r and r + G share GPU r % G, their kernels time-sliced by the
driver; the system-scope flag protocol must still complete. This is what runs
the P = 5..8 instances of the fused and push kernels (k_fused_allreduce<NP>,
k_push_reduce<NP>) on hardware on a 4-GPU box. Each rank checks its result
against the CPU oracle's allreduce_decomposed bit for bit, the gathered
message trace against the reference's, and the shared bad-scale abort."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
import oracle_ffi as O  # noqa: E402
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200.collective import Communicator  # noqa: E402


ALGOS = ("p2p", "push")


def grads(world, n, seed):
    out = []
    for r in range(world):
        rng = np.random.default_rng(seed * 100 + r)
        mag = np.repeat(10.0 ** rng.uniform(-6, 2, (n + 127) // 128), 128)[:n]
        out.append(O.quantize((rng.standard_normal(n) * mag).astype(np.float32), 8, 128, O.FP8))
    return out


def main():
    local = int(os.environ["LOCAL_RANK"])
    ngpu = torch.cuda.device_count()
    dev_i = local % ngpu
    torch.cuda.set_device(dev_i)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", dev_i)
    cap = 8192 * 5 + 300
    global ALGOS
    # the push and one-shot kernels cover 2..8 ranks
    ALGOS = ("p2p", "push", "oneshot") if world <= 8 else ("p2p",)
    comm = Communicator(device=dev_i, p2p_capacity=cap, timeout_s=240.0, nccl=False)
    fails = 0
    for seed, n in enumerate([128 * 3, 8192 * 2 + 77, cap]):
        g = grads(world, n, seed)
        want_c, want_s = O.allreduce_decomposed([c for c, _ in g], [s for _, s in g])
        for algo in ALGOS:
            c, s = g[rank]
            pc, ps = comm.p2p_buffers(n)
            pc.copy_(torch.from_numpy(c))
            ps.copy_(torch.from_numpy(s))
            q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
            comm.allreduce_fp8(q, algo=algo)
            if not (np.array_equal(q.codes.cpu().numpy(), want_c) and
                    np.array_equal(q.scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))):
                fails += 1
                print(f"rank {rank}: MISMATCH algo={algo} n={n}", flush=True)
            if algo == "oneshot":  # its own messages: the whole tensor to every peer
                mine, _ = comm.last_trace()
                if [(e.receiver, e.chunk_len) for e in mine] != \
                        [(q, n) for q in range(world) if q != rank]:
                    fails += 1
                    print(f"rank {rank}: ONESHOT TRACE n={n}", flush=True)
                continue
            full = comm.gather_trace()
            want_t = A.decomposed_trace(n, 128, world)
            if [tuple(e.__dict__.values()) for e in full] != \
                    [tuple(e.__dict__.values()) for e in want_t]:
                fails += 1
                print(f"rank {rank}: TRACE MISMATCH algo={algo} n={n}", flush=True)
    # a bad scale on the last two workers: every rank raises the lowest one's
    n = 8192 * 2
    c, s = grads(world, n, 9)[rank]
    s = s.copy()
    if rank >= world - 2:
        s[rank] = -1.0
    for algo in ALGOS:
        pc, ps = comm.p2p_buffers(n)
        pc.copy_(torch.from_numpy(c))
        ps.copy_(torch.from_numpy(s))
        q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
        try:
            comm.allreduce_fp8(q, algo=algo)
            fails += 1
            print(f"rank {rank}: no bad-scale error algo={algo}", flush=True)
        except A.InvalidArgument as e:
            if str(e) != f"quantized tensor: bad scale at block {world - 2}":
                fails += 1
                print(f"rank {rank}: wrong error {e}", flush=True)
    t = torch.tensor([fails])
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_p2p_oversubscribed world={world} gpus={ngpu} failures={int(t.item())}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
