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
h = pynvml.nvmlDeviceGetHandleByIndex(local)  # CUDA and NVML order agree on this box
# The NVLink data counters (NVML field values) are not exposed on this VM;
# GPU Performance Monitoring (GPM) is: NVLINK_TOTAL_{TX,RX}_PER_SEC averaged
# between two samples, times the interval between them = bytes.
import time  # noqa: E402

_s1 = pynvml.nvmlGpmSampleAlloc()
_s2 = pynvml.nvmlGpmSampleAlloc()


def gpm_begin():
    pynvml.nvmlGpmSampleGet(h, _s1)
    return time.perf_counter()


def gpm_end(t0):
    pynvml.nvmlGpmSampleGet(h, _s2)
    dt = time.perf_counter() - t0
    mg = pynvml.c_nvmlGpmMetricsGet_t()
    mg.version = pynvml.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = 2
    mg.sample1 = _s1
    mg.sample2 = _s2
    mg.metrics[0].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
    mg.metrics[1].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
    pynvml.nvmlGpmMetricsGet(mg)
    return mg.metrics[0].value * dt, mg.metrics[1].value * dt, dt


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
        t0 = gpm_begin()
        comm.allreduce_fp8(q, algo=algo)
        torch.cuda.synchronize()
        tx, rx, _ = gpm_end(t0)
        dist.barrier()
        tot_tx += tx
        tot_rx += rx
    res[algo] = {"tx_bytes_per_call": tot_tx / K, "rx_bytes_per_call": tot_rx / K,
                 "tx_over_expected": round(tot_tx / K / res["expected_fp8_bytes_per_direction"], 4),
                 "rx_over_expected": round(tot_rx / K / res["expected_fp8_bytes_per_direction"], 4)}
gb = torch.randn(n, device=dev).to(torch.bfloat16)
tot_tx = tot_rx = 0
for _ in range(K):
    torch.cuda.synchronize()
    dist.barrier()
    t0 = gpm_begin()
    comm.allreduce_bf16(gb)
    torch.cuda.synchronize()
    tx, rx, _ = gpm_end(t0)
    dist.barrier()
    tot_tx += tx
    tot_rx += rx
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
