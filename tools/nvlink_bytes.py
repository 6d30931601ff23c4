"""NVLink traffic of one all-reduce, from the GPU's own NVLink data counters
(NVML field NVLINK_THROUGHPUT_DATA_TX/RX, summed over links, KiB), per rank
per call, against the decomposed algorithm's wire bytes 2(P-1)/P * N * (1 +
4/128) per direction and BF16 ncclAllReduce's 2(P-1)/P * 2N (ring).
Run under torchrun, one process per GPU:
  python -m torch.distributed.run --nproc-per-node 2 tools/nvlink_bytes.py [N]"""
import json
import os
import sys

import pynvml
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200.collective import Communicator  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local)
try:
    h = pynvml.nvmlDeviceGetHandleByPciBusId(
        pynvml.nvmlDeviceGetPciInfo(h).busId)
except Exception:
    pass
LINKS = 18


def counters():
    ids = []
    for link in range(LINKS):
        ids.append((pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link))
        ids.append((pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link))
    vals = pynvml.nvmlDeviceGetFieldValues(h, ids)
    tx = rx = 0
    for i, v in enumerate(vals):
        if v.nvmlReturn != 0:
            continue
        x = v.value.ullVal
        if i % 2 == 0:
            tx += x
        else:
            rx += x
    return tx * 1024, rx * 1024


comm = Communicator(p2p_capacity=n)
dev = torch.device("cuda", local)
src_c = torch.randint(0, 0x7e, (n,), dtype=torch.uint8, device=dev)
src_s = torch.full(((n + 127) // 128,), 1e-3, dtype=torch.float32, device=dev)
pc, ps = comm.p2p_buffers(n)
res = {"rank": rank, "world": world, "elements": n,
       "expected_fp8_bytes_per_direction": 2 * (world - 1) / world * n * (1 + 4 / 128),
       "expected_bf16_ring_bytes_per_direction": 2 * (world - 1) / world * 2 * n}
K = 5
for algo in ("p2p", "push", "nccl"):
    q = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
    tot_tx = tot_rx = 0
    for _ in range(K):
        pc.copy_(src_c)
        ps.copy_(src_s)
        torch.cuda.synchronize()
        dist.barrier()
        t0, r0 = counters()
        comm.allreduce_fp8(q, algo=algo)
        torch.cuda.synchronize()
        dist.barrier()
        t1, r1 = counters()
        tot_tx += t1 - t0
        tot_rx += r1 - r0
    res[algo] = {"tx_bytes_per_call": tot_tx / K, "rx_bytes_per_call": tot_rx / K,
                 "tx_over_expected": round(tot_tx / K / res["expected_fp8_bytes_per_direction"], 4),
                 "rx_over_expected": round(tot_rx / K / res["expected_fp8_bytes_per_direction"], 4)}
gb = torch.randn(n, device=dev).to(torch.bfloat16)
tot_tx = tot_rx = 0
for _ in range(K):
    torch.cuda.synchronize()
    dist.barrier()
    t0, r0 = counters()
    comm.allreduce_bf16(gb)
    torch.cuda.synchronize()
    dist.barrier()
    t1, r1 = counters()
    tot_tx += t1 - t0
    tot_rx += r1 - r0
res["bf16_nccl"] = {"tx_bytes_per_call": tot_tx / K, "rx_bytes_per_call": tot_rx / K,
                    "tx_over_ring_expected": round(tot_tx / K / res["expected_bf16_ring_bytes_per_direction"], 4),
                    "nccl_algo": os.environ.get("NCCL_ALGO", "default")}
out = [None] * world
dist.all_gather_object(out, res)
if rank == 0:
    for r in out:
        print(json.dumps(r), flush=True)
comm.close()
dist.destroy_process_group()
