"""Multi-rank host logic of the decomposed all-reduce on CPU (gloo, world
size 2, one process per rank): each rank owns ChunkAssignment chunk r (from
the C ABI), ships chunk q of its FP8 gradient ([codes|scales]) to rank q with
the same message schedule the NCCL path uses, reduces its chunk in ascending
sender rank (here with the CPU oracle as the reducer), and all-gathers the
reduced chunks into place. The result must equal the reference's
allreduce_decomposed bit for bit, and the bytes moved must equal the
reference trace's payload."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ffi as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(world, n, seed):
    out = []
    for r in range(world):
        rng = np.random.default_rng(seed * 10 + r)
        x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 1)).astype(np.float32)
        out.append(O.quantize(x, 8, 128, O.FP8))
    return out


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2605_00539_b200 as A
    try:
        g = _grads(world, n, 5)
        codes, scales = g[rank]
        codes, scales = codes.copy(), scales.copy()
        rng = A.ChunkAssignment.block_aligned(n, 128, world).ranges
        moved = 0
        # 1) all-to-all: chunk q -> rank q
        recv_c = {}
        recv_s = {}
        reqs = []
        b_r, e_r = rng[rank]
        for peer in range(world):
            if peer == rank:
                continue
            b, e = rng[peer]
            if e > b:
                t_c = torch.from_numpy(codes[b:e].copy())
                t_s = torch.from_numpy(scales[b // 128:(e + 127) // 128].copy())
                reqs += [dist.isend(t_c, peer, tag=0), dist.isend(t_s, peer, tag=1)]
                moved += t_c.numel() + 4 * t_s.numel()
            if e_r > b_r:
                recv_c[peer] = torch.empty(e_r - b_r, dtype=torch.uint8)
                recv_s[peer] = torch.empty((e_r - b_r + 127) // 128, dtype=torch.float32)
                reqs += [dist.irecv(recv_c[peer], peer, tag=0), dist.irecv(recv_s[peer], peer, tag=1)]
        for r_ in reqs:
            r_.wait()
        # 2) reduce own chunk, pieces in ascending sender rank
        if e_r > b_r:
            pc = [codes[b_r:e_r] if s == rank else recv_c[s].numpy() for s in range(world)]
            ps = [scales[b_r // 128:(e_r + 127) // 128] if s == rank else recv_s[s].numpy()
                  for s in range(world)]
            rc, rs = O.allreduce_decomposed(pc, ps)
            codes[b_r:e_r] = rc
            scales[b_r // 128:(e_r + 127) // 128] = rs
        # 3) all-gather: reduced chunk r -> every rank, into place
        reqs = []
        got = {}
        for peer in range(world):
            if peer == rank:
                continue
            if e_r > b_r:
                t_c = torch.from_numpy(codes[b_r:e_r].copy())
                t_s = torch.from_numpy(scales[b_r // 128:(e_r + 127) // 128].copy())
                reqs += [dist.isend(t_c, peer, tag=2), dist.isend(t_s, peer, tag=3)]
                moved += t_c.numel() + 4 * t_s.numel()
            b, e = rng[peer]
            if e > b:
                got[peer] = (torch.empty(e - b, dtype=torch.uint8),
                             torch.empty((e - b + 127) // 128, dtype=torch.float32))
                reqs += [dist.irecv(got[peer][0], peer, tag=2), dist.irecv(got[peer][1], peer, tag=3)]
        for r_ in reqs:
            r_.wait()
        for peer, (c_, s_) in got.items():
            b, e = rng[peer]
            codes[b:e] = c_.numpy()
            scales[b // 128:(e + 127) // 128] = s_.numpy()
        want_c, want_s = O.allreduce_decomposed([c for c, _ in g], [s for _, s in g])
        trace = A.decomposed_trace(n, 128, world)
        sent_trace = sum(e.payload_bytes for e in trace if e.sender == rank)
        q.put((rank, bool(np.array_equal(codes, want_c) and np.array_equal(scales, want_s)),
               moved, sent_trace))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [4096, 8192 * 3 + 300, 77])
def test_decomposed_protocol_two_ranks_gloo(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, moved, sent in res:
        assert ok, f"rank {rank} result differs from allreduce_decomposed"
        assert moved == sent, (moved, sent)
