"""Multi-GPU parity of the decomposed 8-bit all-reduce (run under torchrun,
one process per GPU). Every rank regenerates every rank's FP8 gradient from
its seed, so each rank checks its result against the CPU oracle's
allreduce_decomposed bit for bit, for both algorithms (NCCL grouped
send/recv + reduce kernel; fused NVLink peer-memory kernel), ragged sizes,
P=1..world, the overflow and bad-scale aborts on every rank
(collective.hpp:158-168, :278-281), the message trace each algorithm
records against the reference's MessageTrace (collective.hpp:195-206), and
the barrier timeout (a rank that never arrives fails every rank)."""
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


def grads(world, n, seed, big_rank=-1):
    out = []
    for r in range(world):
        rng = np.random.default_rng(seed * 100 + r)
        mag = np.repeat(10.0 ** rng.uniform(-6, 2, (n + 127) // 128), 128)[:n]
        x = (rng.standard_normal(n) * mag).astype(np.float32)
        if r == big_rank:
            x[:256] = 3e38
        out.append(O.quantize(x, 8, 128, O.FP8))
    return out


VALID = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], np.uint8)
SCALES = np.array([0.0, 2.0 ** -60, 2.0 ** 60, 2.0 ** -61, 2.0 ** 61, 1e-40, 1e-30, 1e30, 1e37,
                   3.0, 0.125], np.float32)


def every_code_grads(world, nblk, seed):
    """Every non-NaN E4M3 code per block, block scales on both sides of the
    block-table decode's fast range: the fused kernels' table and fallback
    paths on real ranks."""
    out = []
    for r in range(world):
        rng = np.random.default_rng(seed * 100 + r)
        c = np.concatenate([rng.permutation(VALID)[:128] for _ in range(nblk)])
        out.append((c, rng.choice(SCALES, nblk).astype(np.float32)))
    return out


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    comm = Communicator(device=local)
    cap = 8192 * 9 + 300
    comm.enable_p2p(cap)
    fails = 0
    cases = [(seed, n, None) for seed, n in enumerate([128, 1000, 8192 * 3 + 300, 8192 * 9 + 300, 77])]
    cases.append((50, 128 * 160, "every_code"))
    for seed, n, kind in cases:
        g = every_code_grads(world, n // 128, seed) if kind else grads(world, n, seed)
        want_c, want_s = O.allreduce_decomposed([c for c, _ in g], [s for _, s in g])
        for algo in ("nccl", "p2p", "push", "oneshot", "auto", "auto-copy"):
            c, s = g[rank]
            if algo in ("p2p", "push", "oneshot", "auto"):
                pc, ps = comm.p2p_buffers(n)
                pc.copy_(torch.from_numpy(c))
                ps.copy_(torch.from_numpy(s))
                q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
            else:
                q = A.QuantizedTensor(torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev), 8, 128,
                                      (n,), A.CodecKind.Fp8E4M3, packed=False)
            # "auto-copy": auto on a tensor outside the symmetric buffers -> the
            # fused kernel with the copy in / copy out path
            comm.allreduce_fp8(q, algo="auto" if algo == "auto-copy" else algo)
            ok = np.array_equal(q.codes.cpu().numpy(), want_c) and \
                np.array_equal(q.scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))
            if not ok:
                fails += 1
                print(f"rank {rank}: MISMATCH algo={algo} n={n}", flush=True)
            if algo == "auto-copy":
                continue
            mine, moved = comm.last_trace()
            alg = comm._auto_algo(q) if algo == "auto" else algo
            if alg == "oneshot":  # not the reference protocol: its own messages
                want_mine = [(q, n) for q in range(world) if q != rank]
                got_mine = [(e.receiver, e.chunk_len) for e in mine
                            if e.phase == "all_to_all" and e.sender == rank]
                nb = (n + 127) // 128
                if got_mine != want_mine or moved != (n * (world - 1), nb * (world - 1)):
                    fails += 1
                    print(f"rank {rank}: ONESHOT TRACE {got_mine} {moved} n={n}", flush=True)
                continue
            # trace of what the real collective issued == the reference's trace
            full = comm.gather_trace()
            want_t = A.decomposed_trace(n, 128, world)
            if [tuple(e.__dict__.values()) for e in full] != \
                    [tuple(e.__dict__.values()) for e in want_t]:
                fails += 1
                print(f"rank {rank}: TRACE MISMATCH algo={algo} n={n} {full[:3]} vs {want_t[:3]}",
                      flush=True)
            if alg in ("p2p", "push") and world > 1:
                # the kernel's own counters of the phase-1 traffic
                if alg == "p2p":
                    a2a = [e for e in mine if e.phase == "all_to_all" and e.receiver == rank]
                else:
                    a2a = [e for e in mine if e.phase == "all_to_all" and e.sender == rank]
                want_m = (sum(e.chunk_len for e in a2a), sum((e.chunk_len + 127) // 128 for e in a2a))
                if moved != want_m:
                    fails += 1
                    print(f"rank {rank}: MOVED {moved} != {want_m} algo={algo} n={n}", flush=True)
    # the NCCL algorithm at other block sizes (receive slots sized per block):
    # any block >= 1 is valid in the reference (quantize.hpp:64-74)
    for blk, n in ((32, 70000), (64, 131072 + 77), (1000, 50000)):
        g = []
        for r in range(world):
            rng = np.random.default_rng(7000 + 10 * blk + r)
            g.append(O.quantize((rng.standard_normal(n) * 1e-2).astype(np.float32), 8, blk, O.FP8))
        want_c, want_s = O.allreduce_decomposed([c for c, _ in g], [s for _, s in g], block=blk)
        c, s = g[rank]
        q = A.QuantizedTensor(torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev), 8, blk, (n,),
                              A.CodecKind.Fp8E4M3, packed=False)
        comm.allreduce_fp8(q, algo="nccl")
        if not (np.array_equal(q.codes.cpu().numpy(), want_c) and
                np.array_equal(q.scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))):
            fails += 1
            print(f"rank {rank}: MISMATCH nccl block={blk} n={n}", flush=True)
    # allreduce_naive_fp8 (collective.hpp:338-431) on real ranks: codes,
    # scales and overflow_elements against the oracle; this rank's
    # overflow_events against the one-device simulation.
    naive_cases = [(seed, n, None) for seed, n in enumerate([128, 1000, 8192 * 3 + 300, 77, 5000])]
    naive_cases += [(60, 128 * 40, "every_code"), (61, 4096, "const64")]
    for seed, n, kind in naive_cases:
        if kind == "every_code":
            g = every_code_grads(world, n // 128, seed)
        elif kind == "const64":  # test_collective.cpp:160-181: naive pins at 64
            g = [O.quantize(np.full(n, 64.0, np.float32), 8, 128, O.FP8) for _ in range(world)]
        else:
            g = grads(world, n, seed)
        want_c, want_s, want_ov = O.allreduce_naive([c for c, _ in g], [s for _, s in g])
        mains = [A.QuantizedTensor(torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev), 8, 128,
                                   (n,), A.CodecKind.Fp8E4M3, packed=False) for c, s in g]
        _, _, sim_ev = A.allreduce_naive_simulated(mains, events=True)
        q = mains[rank]
        _, ov, ev = comm.allreduce_naive_fp8(q)
        ok = np.array_equal(q.codes.cpu().numpy(), want_c) and \
            np.array_equal(q.scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32)) and \
            ov == want_ov and ev == sim_ev[rank]
        if kind == "const64" and world > 1:
            nb = n // 128
            mine = 128 * (nb // world + (rank < nb % world))
            ok = ok and ov == n and ev == n - mine and bool((q.codes.cpu().numpy() == want_c[0]).all())
        if not ok:
            fails += 1
            print(f"rank {rank}: NAIVE MISMATCH n={n} kind={kind} ov={ov}/{want_ov} "
                  f"ev={ev}/{sim_ev[rank]}", flush=True)
    # an fp32 overflow in ONE owner's local reduce aborts the protocol on
    # every rank (collective.hpp:278-281): block 0 (owned by rank 0) holds
    # 3e38 on every rank, so only rank 0's reduce overflows.
    if world > 1:
        for algo in ("nccl", "p2p", "push", "oneshot"):
            n = 8192 * 2
            g = grads(world, n, 99, big_rank=-1)
            c, s = g[rank]
            big_c, big_s = O.quantize(np.full(128, 3e38, np.float32), 8, 128, O.FP8)
            c = c.copy()
            s = s.copy()
            c[:128], s[0] = big_c, big_s[0]
            if algo in ("p2p", "push", "oneshot"):
                pc, ps = comm.p2p_buffers(n)
                pc.copy_(torch.from_numpy(c))
                ps.copy_(torch.from_numpy(s))
                q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
            else:
                q = A.QuantizedTensor(torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev), 8,
                                      128, (n,), A.CodecKind.Fp8E4M3, packed=False)
            try:
                comm.allreduce_fp8(q, algo=algo)
                fails += 1
                print(f"rank {rank}: no overflow raised algo={algo}", flush=True)
            except A.ProtocolError as e:
                if "fp32 overflow" not in str(e):
                    fails += 1
                    print(f"rank {rank}: wrong error {e}", flush=True)
    # a bad (negative) block scale on some workers aborts every rank with
    # the reference's error: the lowest worker's lowest bad block
    # (collective.hpp:158-168 check_workers -> validate, quantize.hpp:170-175)
    n = 8192 * 3 + 300
    nb = (n + 127) // 128
    bad = {min(1, world - 1): [150, 40], world - 1: [7]}
    want_blk = min(bad[min(bad)])
    for algo in ("nccl", "p2p", "push", "oneshot"):
        c, s = grads(world, n, 123)[rank]
        s = s.copy()
        for b in bad.get(rank, []):
            s[b % nb] = -1.0
        if algo in ("p2p", "push", "oneshot"):
            pc, ps = comm.p2p_buffers(n)
            pc.copy_(torch.from_numpy(c))
            ps.copy_(torch.from_numpy(s))
            q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
        else:
            q = A.QuantizedTensor(torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev), 8, 128,
                                  (n,), A.CodecKind.Fp8E4M3, packed=False)
        try:
            comm.allreduce_fp8(q, algo=algo)
            fails += 1
            print(f"rank {rank}: no bad-scale error algo={algo}", flush=True)
        except A.InvalidArgument as e:
            if str(e) != f"quantized tensor: bad scale at block {want_blk}":
                fails += 1
                print(f"rank {rank}: wrong bad-scale error algo={algo}: {e}", flush=True)
    # CUDA graphs: the P2P all-reduces captured once and replayed on fresh
    # inputs, interleaved with eager calls. The epoch lives on the device
    # (each call's last CTA stores it), so replays stay in step with peers.
    n = 8192 * 3 + 300
    for algo in ("p2p", "push", "oneshot") if world > 1 else ("p2p", "oneshot"):
        pc, ps = comm.p2p_buffers(n)
        q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
        err = A.ErrorRecord(dev)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            comm.allreduce_fp8(q, algo=algo, check=False, errors=err)
        for it in range(4):
            g = grads(world, n, 300 + it)
            want_c, want_s = O.allreduce_decomposed([c for c, _ in g], [s for _, s in g])
            pc.copy_(torch.from_numpy(g[rank][0]))
            ps.copy_(torch.from_numpy(g[rank][1]))
            if it == 2:  # an eager call between replays
                comm.allreduce_fp8(q, algo=algo)
            else:
                graph.replay()
                torch.cuda.synchronize()
                err.raise_if_any(A._lib.AGQ_OP_ALLREDUCE)
            if not (np.array_equal(q.codes.cpu().numpy(), want_c) and
                    np.array_equal(q.scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))):
                fails += 1
                print(f"rank {rank}: GRAPH MISMATCH algo={algo} it={it}", flush=True)
        del graph
    # the barrier timeout: the last rank never calls; every other rank's call
    # times out, and the failure is sticky on ALL ranks (later calls fail fast)
    if world > 1:
        comm2 = Communicator(device=local, p2p_capacity=4096, timeout_s=3.0)
        pc, ps = comm2.p2p_buffers(4096)
        q = A.QuantizedTensor(pc, ps, 8, 128, (4096,), A.CodecKind.Fp8E4M3, packed=False)
        q.codes.zero_()
        q.scales.zero_()
        if rank != world - 1:
            try:
                comm2.allreduce_fp8(q, algo="p2p")
                fails += 1
                print(f"rank {rank}: no timeout raised", flush=True)
            except A.ProtocolError as e:
                if "did not arrive" not in str(e):
                    fails += 1
                    print(f"rank {rank}: wrong timeout error {e}", flush=True)
        dist.barrier()
        import time
        t0 = time.time()
        try:
            comm2.allreduce_fp8(q, algo="p2p")
            fails += 1
            print(f"rank {rank}: failed communicator did not raise", flush=True)
        except A.ProtocolError:
            if time.time() - t0 > 2.5:
                fails += 1
                print(f"rank {rank}: failed communicator waited {time.time() - t0:.1f} s", flush=True)
        comm2.close()
    t = torch.tensor([fails], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_allreduce_check world={world} failures={int(t.item())}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
