"""Benchmark of the AGoQ quantization hot path on B200 (bench contract).

Metric (BASELINE.json): activation quant+dequant GB/s vs HBM peak; 8-bit
gradient all-reduce bus GB/s at 1/2/4/8 GPUs.

Workload of `value` (config C2): one LLaMA-8B transformer block's stored
activations at seq 4096 x micro-batch 4 (T = 16384 tokens; norm1/norm2/out-proj
inputs T x 4096, SiLU gate/value T x 14336 = 671,088,640 BF16 elements), stored
under EVERY stage policy of an 8-stage DBCA pipeline (dbca.hpp plan_bit_widths
-> widths 4,4,5,5,6,7,8,8): per stage one grouped quantize launch (BF16 ->
packed codes + FP32 block scales) and one grouped dequantize launch (-> BF16).
A step = all 8 stages. value = algorithmic bytes / device time:
  per element quant 2 + b/8 + 4/128 B, dequant b/8 + 4/128 + 2 B.
Inputs (1.34 GB) and outputs are far larger than L2 (126 MB).

Also reported on the same line:
  accumulate : config C3, FP8 local_accumulate over 8,030,261,248 params
               (LLaMA-8B), FP32 local gradient, in place, 6.0625 B/param.
  allreduce  : (N > 1) config C4, decomposed 8-bit all-reduce of the
               LLaMA-8B FP8 gradient, NCCL and fused-NVLink algorithms, vs a
               BF16 ncclAllReduce of the same gradient.
  e2e        : the activation metric through the host-buffer path: pinned
               host BF16 activations -> device every step, dequantized outputs
               of every stage -> host.
  roofline, cpu_baseline, clocks, gpu_launches: see the bench contract.

Inputs: the activations are the reference's own bytes — make_rng(seed,
0x1D, index = tensor) + std::normal_distribution<float> (tools/agq.cpp:47-65,
rng.hpp:9-28; inputs.materialize), BF16-rounded; the reference arm draws the
same stream through oracle/_ref, so both arms quantize identical values. The
8e9-element gradient configs (C3/C4) are generated on the device
(torch.Generator; SURVEY 8d allows counter-based generation at full size)
and checked against the oracle on sampled blocks.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref, the unmodified reference headers compiled as-is) of the same
workload on a bounded sample, on all host threads, plus one pinned core. It
imports nothing from the package (the stage widths are the literal
STAGE_BITS, pinned by tests/test_bench_reference.py).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T_TOKENS = 4 * 4096
HIDDEN, FFN = 4096, 14336
TENSORS = [("norm1_input", HIDDEN), ("norm2_input", HIDDEN), ("outproj_input", HIDDEN),
           ("silu_gate", FFN), ("silu_value", FFN)]
LLAMA8B_PARAMS = 8_030_261_248
METRIC = "act quant+dequant GB/s vs HBM peak; INT8 grad all-reduce bus GB/s @1/2/4/8 GPU"


# dbca.hpp:63-78 plan_bit_widths for 8 stages (= A.plan_bit_widths and the
# oracle's; tests/test_bench_reference.py pins it)
STAGE_BITS = (4, 4, 5, 5, 6, 7, 8, 8)
TENSOR_SCALES = (1.0, 1.0, 0.5, 4.0, 1.0)  # per-tensor std
SEED = 0


def stage_bits():
    return list(STAGE_BITS)


def act_bytes_per_elem(bits):
    q = 2 + bits / 8 + 4 / 128
    return q, q  # quant, dequant (bf16 in / bf16 out)


NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (nominal)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/agq_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows]
        load = [float(r[0]) for r in rows if float(r[2]) > 150.0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl != "reference":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------
class ActWorkload:
    def __init__(self, dev, seed=0):
        import torch
        import paper_2605_00539_b200 as A
        from paper_2605_00539_b200 import _lib as L
        self.A, self.L, self.torch = A, L, torch
        self.dev = dev
        from paper_2605_00539_b200.inputs import materialize_parallel
        host = materialize_parallel([T_TOKENS * w for _, w in TENSORS], seed, torch.bfloat16,
                                    scales=TENSOR_SCALES)
        self.x = [h.to(dev) for h in host]
        del host
        self.n = [t.numel() for t in self.x]
        self.N = sum(self.n)
        self.bits = stage_bits()
        self.out = [torch.empty_like(t) for t in self.x]
        self.q = {}
        for b in sorted(set(self.bits)):
            self.q[b] = [(torch.empty(int(L.lib.agq_packed_bytes(n, b)), dtype=torch.uint8, device=dev),
                          torch.empty((n + 127) // 128, dtype=torch.float32, device=dev)) for n in self.n]
        self.err = A.ErrorRecord(dev).reset()
        self.segq, self.segd = {}, {}
        for b in self.q:
            sq = (L.AgqSegment * 5)()
            sd = (L.AgqSegment * 5)()
            for i in range(5):
                c, s = self.q[b][i]
                sq[i] = L.AgqSegment(self.x[i].data_ptr(), c.data_ptr(), s.data_ptr(), self.n[i])
                sd[i] = L.AgqSegment(self.out[i].data_ptr(), c.data_ptr(), s.data_ptr(), self.n[i])
            self.segq[b], self.segd[b] = sq, sd

    def bytes_per_step(self):
        return sum(self.N * sum(act_bytes_per_elem(b)) for b in self.bits)

    def quant(self, b, stream):
        self.L.check(self.L.lib.agq_quantize_grouped(self.segq[b], 5, self.L.AGQ_BF16, b, 0,
                                                     self.err.ptr, stream))

    def dequant(self, b, stream):
        # with the reference's validate checks (quantize.hpp:157-179)
        self.L.check(self.L.lib.agq_dequantize_grouped(self.segd[b], 5, self.L.AGQ_BF16, b, 0, 1,
                                                       self.err.ptr, stream))

    def step(self, stream, ev=None):
        for i, b in enumerate(self.bits):
            if ev is not None:
                ev[4 * i].record()
            self.quant(b, stream)
            if ev is not None:
                ev[4 * i + 1].record()
                ev[4 * i + 2].record()
            self.dequant(b, stream)
            if ev is not None:
                ev[4 * i + 3].record()

    def verify_sample(self, nblk=16):
        """Bit-exact check of `nblk` random blocks of every tensor at every
        stage width against the oracle: packed codes, scales and the BF16
        reconstruction (the full-size comparison is
        tests/test_gpu_r02.py::test_c2_full_tensors_every_width)."""
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import numpy as np
        import oracle_ffi as O
        sp = self.torch.cuda.current_stream().cuda_stream
        rng = np.random.default_rng(3)
        ok = True
        for b in sorted(set(self.bits)):
            self.quant(b, sp)
            self.dequant(b, sp)
            self.torch.cuda.synchronize()
            for i in range(5):
                codes, scales = self.q[b][i]
                for blk in rng.integers(0, self.n[i] // 128, nblk):
                    x = self.x[i][blk * 128:(blk + 1) * 128].float().cpu().numpy()
                    c, sc = O.quantize(x, b, 128, 0)
                    got = codes[blk * 16 * b:(blk + 1) * 16 * b].cpu().numpy()
                    ok &= bool(np.array_equal(got, O.pack(c, b))) and float(scales[blk]) == float(sc[0])
                    y = self.out[i][blk * 128:(blk + 1) * 128].float().cpu().numpy()
                    ok &= bool(np.array_equal(y.view(np.uint32),
                                              O.bf16_round(O.dequantize(c, sc, b)).view(np.uint32)))
        return bool(ok)


def bench_act(wl, args, world):
    import torch
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    for _ in range(args.warmup):
        wl.step(sp)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4 * len(wl.bits) * args.steps)]
    launches0 = wl.A.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for k in range(args.steps):
        wl.step(sp, ev[4 * len(wl.bits) * k: 4 * len(wl.bits) * (k + 1)])
    t1.record()
    torch.cuda.synchronize()
    launches = wl.A.launch_count() - launches0
    sec = t0.elapsed_time(t1) * 1e-3
    barrier(world)
    sec = max_over_ranks(sec, world)
    # per-kernel durations on the launching stream
    qt, dt = [], []
    qb, db = [], []
    for k in range(args.steps):
        for i, b in enumerate(wl.bits):
            base = 4 * len(wl.bits) * k + 4 * i
            qt.append(ev[base].elapsed_time(ev[base + 1]) * 1e-3)
            dt.append(ev[base + 2].elapsed_time(ev[base + 3]) * 1e-3)
            qb.append(wl.N * act_bytes_per_elem(b)[0])
            db.append(wl.N * act_bytes_per_elem(b)[1])
    h = wl.err.read()
    wl.L.errors_message(h, wl.L.AGQ_OP_QUANTIZE)
    wl.L.errors_message(h, wl.L.AGQ_OP_DEQUANTIZE)
    return sec, launches, (sum(qb) / sum(qt) / 1e9, sum(qt)), (sum(db) / sum(dt) / 1e9, sum(dt))


def bench_e2e(wl, args, world, steps, chunks=16, nstreams=4):
    """Host-buffer path: pinned BF16 activations H2D every step, all stage
    policies quantize+dequantize on device, each stage's BF16 reconstruction
    D2H (what dequantize_blockwise returns to a host caller).

    The step is split into `chunks` block-aligned slices of every tensor,
    issued round-robin on `nstreams` streams, so the H2D of one slice, the
    kernels of another and the D2H of a third overlap (the two copy directions
    run on separate copy engines). Block-aligned slices quantize exactly like
    the whole tensor (no block straddles a slice boundary)."""
    import torch
    L = wl.L
    host_in = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for n in wl.n]
    for h, x in zip(host_in, wl.x):
        h.copy_(x)
    host_out = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for n in wl.n]
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    # per chunk: element range of every tensor, and grouped segment tables
    plan = []
    for k in range(chunks):
        rng = []
        for n in wl.n:
            nb = (n + 127) // 128
            b0, b1 = nb * k // chunks, nb * (k + 1) // chunks
            rng.append((b0 * 128, min(b1 * 128, n)))
        segq, segd = {}, {}
        for b in wl.q:
            sq, sd = (L.AgqSegment * 5)(), (L.AgqSegment * 5)()
            for i, (e0, e1) in enumerate(rng):
                c, sc = wl.q[b][i]
                cp = c.data_ptr() + e0 * b // 8
                spp = sc.data_ptr() + (e0 // 128) * 4
                sq[i] = L.AgqSegment(wl.x[i].data_ptr() + 2 * e0, cp, spp, e1 - e0)
                sd[i] = L.AgqSegment(wl.out[i].data_ptr() + 2 * e0, cp, spp, e1 - e0)
            segq[b], segd[b] = sq, sd
        plan.append((rng, segq, segd))

    def one():
        main = torch.cuda.current_stream()
        for st in streams:
            st.wait_stream(main)
        for k, (rng, segq, segd) in enumerate(plan):
            st = streams[k % nstreams]
            with torch.cuda.stream(st):
                sp = st.cuda_stream
                for i, (e0, e1) in enumerate(rng):
                    wl.x[i][e0:e1].copy_(host_in[i][e0:e1], non_blocking=True)
                for b in wl.bits:
                    L.check(L.lib.agq_quantize_grouped(segq[b], 5, L.AGQ_BF16, b, 0, wl.err.ptr, sp))
                    L.check(L.lib.agq_dequantize_grouped(segd[b], 5, L.AGQ_BF16, b, 0, 1,
                                                         wl.err.ptr, sp))
                    for i, (e0, e1) in enumerate(rng):
                        host_out[i][e0:e1].copy_(wl.out[i][e0:e1], non_blocking=True)
        for st in streams:
            main.wait_stream(st)

    one()
    torch.cuda.synchronize()
    barrier(world)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        one()
    e.record()
    torch.cuda.synchronize()
    sec = max_over_ranks(s.elapsed_time(e) * 1e-3, world)
    h = wl.err.read()
    wl.L.errors_message(h, wl.L.AGQ_OP_QUANTIZE)
    wl.L.errors_message(h, wl.L.AGQ_OP_DEQUANTIZE)
    # the result read back must equal the device result of the last stage
    last = wl.bits[-1]
    ok = all(torch.equal(h[:4096], o[:4096].cpu()) for h, o in zip(host_out, wl.out))
    if not ok:
        raise RuntimeError(f"e2e: host copy of stage {last} differs from the device result")
    bi = sum(wl.n) * 2
    bo = sum(wl.n) * 2 * len(wl.bits)
    return wl.bytes_per_step() * steps * world / sec / 1e9, bi, bo


def bench_c2_stage(wl, args, layers=4, widths=(4, 8)):
    """A whole pipeline stage in ONE grouped call: LLaMA-8B at 8 stages holds
    4 layers per stage, each storing the five C2 tensors (layers.hpp:266-301)
    under the stage policy (dbca.hpp:172-177) -> 20 tensors (2.68e9
    elements) per quantize call and per dequantize call (validate on)."""
    import torch
    L = wl.L
    xs = [x.clone() for _ in range(layers) for x in wl.x]
    outs = [torch.empty_like(x) for x in xs]
    sp = torch.cuda.current_stream().cuda_stream
    res = {"config": f"C2 stage: {layers} layers x 5 stored tensors = {5 * layers} tensors per "
                     f"grouped call", "elements": sum(x.numel() for x in xs)}
    for b in widths:
        qs = [(torch.empty(int(L.lib.agq_packed_bytes(x.numel(), b)), dtype=torch.uint8,
                           device=x.device),
               torch.empty((x.numel() + 127) // 128, dtype=torch.float32, device=x.device))
              for x in xs]
        sq = (L.AgqSegment * len(xs))()
        sd = (L.AgqSegment * len(xs))()
        for i, (x, o, (c, sc)) in enumerate(zip(xs, outs, qs)):
            sq[i] = L.AgqSegment(x.data_ptr(), c.data_ptr(), sc.data_ptr(), x.numel())
            sd[i] = L.AgqSegment(o.data_ptr(), c.data_ptr(), sc.data_ptr(), x.numel())

        def run():
            L.check(L.lib.agq_quantize_grouped(sq, len(xs), L.AGQ_BF16, b, 0, wl.err.ptr, sp))
            L.check(L.lib.agq_dequantize_grouped(sd, len(xs), L.AGQ_BF16, b, 0, 1, wl.err.ptr, sp))
        run()
        torch.cuda.synchronize()
        n0 = wl.A.launch_count()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 5
        s.record()
        for _ in range(iters):
            run()
        e.record()
        torch.cuda.synchronize()
        sec = s.elapsed_time(e) * 1e-3 / iters
        h = wl.err.read()
        L.errors_message(h, L.AGQ_OP_QUANTIZE)
        L.errors_message(h, L.AGQ_OP_DEQUANTIZE)
        nbytes = res["elements"] * sum(act_bytes_per_elem(b))
        res[f"b{b}"] = {"ms": round(sec * 1e3, 3), "GBs": round(nbytes / sec / 1e9, 1),
                        "launches_per_call_pair": (wl.A.launch_count() - n0) // iters}
        del qs
    res["GBs"] = min(res[f"b{b}"]["GBs"] for b in widths)
    del xs, outs
    torch.cuda.empty_cache()
    return res


def pcie_rates(dev, mb=256, reps=3):
    """Pinned-host <-> device copy rates (GB/s) of this box, one direction at
    a time: the bound the host-buffer API runs against."""
    import torch
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) * 1e-3)
        out[name] = n / best / 1e9
    del h, d
    return out


def bench_dropin(dev):
    """e2e through the C++ drop-in API (tools/dropin_bench.cpp): host
    std::vector in/out, as a reference-side C++ caller, beside the reference's
    own single-threaded calls; against this box's pinned PCIe rates."""
    exe = os.path.join(ROOT, "paper_2605_00539_b200", "build", "dropin_bench")
    ref = os.path.join(ROOT, "oracle", "_ref", "libagq_ref.so")
    if not os.path.exists(exe):
        return {"error": "dropin_bench not built"}
    pc = pcie_rates(dev)
    r = subprocess.run([exe, ref], capture_output=True, text=True, timeout=600)
    try:
        j = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": (r.stdout + r.stderr)[-300:]}
    # lower bound of each call on this box: its larger direction at the
    # pinned rate (the pipeline overlaps the two directions)
    bq = max(j["quantize_h2d_bytes"] / pc["h2d"], j["quantize_d2h_bytes"] / pc["d2h"]) / 1e9
    bd = max(j["dequantize_h2d_bytes"] / pc["h2d"], j["dequantize_d2h_bytes"] / pc["d2h"]) / 1e9
    ba = max(j["accumulate_h2d_bytes"] / pc["h2d"], j["accumulate_d2h_bytes"] / pc["d2h"]) / 1e9
    # every API byte also passes once through the host staging copy
    # (caller memory <-> pinned slots) at the measured host copy rate
    hc = j["host_copy_GBs"] * 1e9
    hq = (j["quantize_h2d_bytes"] + j["quantize_d2h_bytes"]) / hc
    hd = (j["dequantize_h2d_bytes"] + j["dequantize_d2h_bytes"]) / hc
    ha = (j["accumulate_h2d_bytes"] + j["accumulate_d2h_bytes"]) / hc
    rt = j["roundtrip_ms"] * 1e-3
    moved = (j["quantize_h2d_bytes"] + j["quantize_d2h_bytes"] + j["dequantize_h2d_bytes"] +
             j["dequantize_d2h_bytes"])
    n = j["elements"]
    res = {"config": j["config"], "pinned_pcie_GBs": {k: round(v, 1) for k, v in pc.items()},
           "roundtrip_ms": j["roundtrip_ms"], "quantize_ms": j["quantize_ms"],
           "dequantize_ms": j["dequantize_ms"],
           "api_bytes_per_roundtrip": int(moved),
           "GBs_api_bytes": round(moved / rt / 1e9, 1),
           "frac_of_pinned_pcie_bound": round((bq + bd) / rt, 3),
           # the metric's algorithmic bytes for FP32 in/out, b = 4
           "GBs_algorithmic": round(2 * n * (4 + 0.5 + 4 / 128) / rt / 1e9, 2),
           "abi_host_entry_ms": {"quantize": j["abi_quantize_host_ms"],
                                 "dequantize": j["abi_dequantize_host_ms"],
                                 "frac_of_pinned_pcie_bound": round(
                                     (bq + bd) / ((j["abi_quantize_host_ms"] +
                                                   j["abi_dequantize_host_ms"]) * 1e-3), 3),
                                 "frac_of_bound": round(
                                     (max(bq, hq) + max(bd, hd)) / ((j["abi_quantize_host_ms"] +
                                                                     j["abi_dequantize_host_ms"]) * 1e-3), 3),
                                 "note": "agq_*_host into caller-owned buffers: the library's "
                                         "path without the API's value-initialised result "
                                         "vectors"},
           # the bound of a pageable-buffer API: per call the slower of PCIe
           # (pinned rate) and the host staging copy of the same bytes
           "host_copy_GBs": j["host_copy_GBs"],
           "bound_ms": {"quantize": round(max(bq, hq) * 1e3, 3),
                        "dequantize": round(max(bd, hd) * 1e3, 3),
                        "accumulate": round(max(ba, ha) * 1e3, 3)},
           "frac_of_bound": round((max(bq, hq) + max(bd, hd)) / rt, 3),
           # where the API's time goes: the split entry (begin; the caller's
           # single-threaded value-initialisation of the result vectors,
           # overlapping the transfers and kernels; finish = result copy)
           "api_quantize_job_parts_ms": j["api_quantize_job_parts_ms"],
           "api_dequantize_job_parts_ms": j["api_dequantize_job_parts_ms"],
           "accumulate_ms": j["accumulate_ms"],
           "accumulate_frac_of_pinned_pcie_bound": round(ba / (j["accumulate_ms"] * 1e-3), 3),
           "reference_1thread": {"roundtrip_ms": round(j["ref_quantize_ms"] + j["ref_dequantize_ms"], 2),
                                 "accumulate_ms": j["ref_accumulate_ms"]},
           "speedup_vs_reference_1thread": round((j["ref_quantize_ms"] + j["ref_dequantize_ms"]) /
                                                 j["roundtrip_ms"], 1),
           "bitexact_vs_reference": j["bitexact_vs_ref"] and j["accumulate_bitexact_vs_ref"]}
    return res


def bench_c1(dev, args):
    """C1: INT4 block-128 quantize/dequantize round trip of a 4096x4096 BF16
    activation (the reference's CPU-runnable config). 16 rotating copies
    (1.6 GB) so every launch streams from HBM, not the 126 MB L2."""
    import torch
    from paper_2605_00539_b200 import _lib as L
    from paper_2605_00539_b200.inputs import materialize_parallel
    n, R = 4096 * 4096, 16
    # copy 0 = the reference CLI's `--seed 1 --normal 16777216` bytes (BF16)
    xs = [h.to(dev) for h in materialize_parallel([n] * R, 1, torch.bfloat16)]
    cs = [torch.empty(n // 2, dtype=torch.uint8, device=dev) for _ in range(R)]
    ss = [torch.empty(n // 128, dtype=torch.float32, device=dev) for _ in range(R)]
    ys = [torch.empty_like(xs[0]) for _ in range(R)]
    sp = torch.cuda.current_stream().cuda_stream

    def rt(i):
        L.check(L.lib.agq_quantize(xs[i].data_ptr(), L.AGQ_BF16, n, 4, 128, 0, cs[i].data_ptr(),
                                   L.AGQ_CODES_PACKED, ss[i].data_ptr(), None, sp))
        L.check(L.lib.agq_dequantize(cs[i].data_ptr(), L.AGQ_CODES_PACKED, ss[i].data_ptr(), n, 4,
                                     128, 0, ys[i].data_ptr(), L.AGQ_BF16, 0, None, sp))
    for i in range(R):
        rt(i)
    torch.cuda.synchronize()
    iters = 5 * R
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        rt(i % R)
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) * 1e-3 / iters
    nbytes = 2 * n * (2 + 0.5 + 4 / 128)

    def fused(i):  # the same round trip through the fused entry point
        L.check(L.lib.agq_quantize_roundtrip(xs[i].data_ptr(), L.AGQ_BF16, n, 4, 128, 0,
                                             cs[i].data_ptr(), L.AGQ_CODES_PACKED, ss[i].data_ptr(),
                                             ys[i].data_ptr(), L.AGQ_BF16, None, sp))
    for i in range(R):
        fused(i)
    torch.cuda.synchronize()
    s.record()
    for i in range(iters):
        fused(i % R)
    e.record()
    torch.cuda.synchronize()
    fsec = s.elapsed_time(e) * 1e-3 / iters
    # the practical floor at this size: two back-to-back device copies moving
    # the same bytes (each kernel of the round trip moves half of nbytes)
    half = int(nbytes / 4)
    cx = [torch.empty(half, dtype=torch.uint8, device=dev).fill_(1) for _ in range(R)]
    cy = [torch.empty(half, dtype=torch.uint8, device=dev) for _ in range(R)]
    for i in range(R):
        cy[i].copy_(cx[i])
    torch.cuda.synchronize()
    s.record()
    for i in range(2 * iters):
        cy[i % R].copy_(cx[i % R])
    e.record()
    torch.cuda.synchronize()
    floor = s.elapsed_time(e) * 1e-3 / iters
    del cx, cy
    return {"config": "C1 INT4 block-128 quantize+dequantize, 4096x4096 BF16",
            "us_per_roundtrip": round(sec * 1e6, 2), "GBs": round(nbytes / sec / 1e9, 1),
            "copy_floor_us": round(floor * 1e6, 2),
            "fused_roundtrip_us": round(fsec * 1e6, 2),
            "fused_roundtrip_GBs_moved": round(n * (2 + 0.5 + 4 / 128 + 2) / fsec / 1e9, 1),
            "fused_note": "agq_quantize_roundtrip: one kernel pass (x read once, codes + scales + "
                          "reconstruction written), bit-identical to the two calls",
            "copy_floor_note": "two back-to-back torch device copies of nbytes/4 each (same "
                               "total traffic as the round trip), 16 rotating buffers"}


def bench_reduce_local(dev, args, P=8):
    """K4 on one GPU: the local reduce one rank performs in the decomposed
    all-reduce of the LLaMA-8B gradient at P=8 (its 1/8 chunk, 8 pieces)."""
    import torch
    import paper_2605_00539_b200 as A
    from paper_2605_00539_b200 import _lib as L
    n = (LLAMA8B_PARAMS // P + 127) // 128 * 128
    g = torch.Generator(device=dev).manual_seed(12)
    pieces = []
    for _ in range(P):
        x = torch.randn(n, device=dev, generator=g) * 1e-3
        pieces.append(A.quantize_blockwise(x, 8, 128, A.CodecKind.Fp8E4M3, packed=False, check=False))
        del x
    oc = torch.empty(n, dtype=torch.uint8, device=dev)
    osc = torch.empty(n // 128, dtype=torch.float32, device=dev)
    err = A.ErrorRecord(dev).reset()
    pc = L.ptr_array([q.codes.data_ptr() for q in pieces])
    ps = L.ptr_array([q.scales.data_ptr() for q in pieces])
    po, pso = L.ptr_array([oc.data_ptr()]), L.ptr_array([osc.data_ptr()])
    sp = torch.cuda.current_stream().cuda_stream

    def run():
        L.check(L.lib.agq_fp8_reduce_requant(P, pc, ps, n, 128, 1, po, pso, err.ptr, sp))
    run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        run()
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) * 1e-3 / 3
    L.errors_message(err.read(), L.AGQ_OP_ALLREDUCE)
    del pieces
    torch.cuda.empty_cache()
    return {"config": f"K4 local reduce-requant, LLaMA-8B chunk at P={P} ({n} elems, {P} pieces)",
            "ms": round(sec * 1e3, 3), "GBs": round(n * (P + 1) * (1 + 4 / 128) / sec / 1e9, 1)}


def bench_accumulate(dev, args, n_params):
    """C3: FP8 local_accumulate over an 8B-param gradient, in place. Headline:
    FP32 local gradient, FP32 sum (6.0625 B/param). Variants on the same
    buffers: BF16 / FP16-rounded sums (collective.hpp:141-142) and a BF16
    local gradient (4.0625 B/param)."""
    import torch
    import paper_2605_00539_b200 as A
    from paper_2605_00539_b200 import _lib as L
    codes = torch.empty(n_params, dtype=torch.uint8, device=dev)
    scales = torch.empty((n_params + 127) // 128, dtype=torch.float32, device=dev)
    local = torch.empty(n_params, dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev).manual_seed(1)
    chunk = 1 << 28
    for off in range(0, n_params, chunk):
        m = min(chunk, n_params - off)
        x = torch.randn(m, device=dev, generator=g) * 1e-3
        L.check(L.lib.agq_quantize(x.data_ptr(), L.AGQ_F32, m, 8, 128, 2, codes[off:].data_ptr(),
                                   L.AGQ_CODES_BYTES, scales[off // 128:].data_ptr(), None,
                                   torch.cuda.current_stream().cuda_stream))
        local[off:off + m].normal_(0.0, 1e-3, generator=g)
        del x
    local16 = local.to(torch.bfloat16)
    err = A.ErrorRecord(dev).reset()
    sp = torch.cuda.current_stream().cuda_stream

    def timed(loc, ldt, prec):
        def run():
            L.check(L.lib.agq_fp8_accumulate(codes.data_ptr(), scales.data_ptr(), loc.data_ptr(),
                                             ldt, n_params, 128, prec, codes.data_ptr(),
                                             scales.data_ptr(), err.ptr, sp))
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = max(3, min(args.steps, 10))
        s.record()
        for _ in range(iters):
            run()
        e.record()
        torch.cuda.synchronize()
        L.errors_message(err.read(), L.AGQ_OP_ACCUMULATE)
        sec = s.elapsed_time(e) * 1e-3 / iters
        bpp = 2 * (1 + 4 / 128) + loc.element_size()
        return {"ms": round(sec * 1e3, 3), "GBs": round(n_params * bpp / sec / 1e9, 1),
                "bytes_per_param": bpp}

    res = {"config": "C3 FP8 local_accumulate, LLaMA-8B params, fp32 local, in place",
           "params": n_params, **timed(local, L.AGQ_F32, 0)}
    res["variants"] = {"fp32_local_bf16_sum": timed(local, L.AGQ_F32, 1),
                       "fp32_local_fp16_sum": timed(local, L.AGQ_F32, 2),
                       "bf16_local": timed(local16, L.AGQ_BF16, 0),
                       "bf16_local_bf16_sum": timed(local16, L.AGQ_BF16, 1)}
    del codes, scales, local, local16
    torch.cuda.empty_cache()
    return res


def allreduce_oracle_sample(src_codes, src_scales, result, world, rank, nsample=64, seed=5):
    """Check `nsample` random whole blocks of the real-rank all-reduce result
    against the CPU oracle's allreduce_decomposed (collective.hpp:226-333)
    over every rank's input blocks (gathered to every rank). Blocks are
    reduced independently, so the sampled blocks form a valid all-reduce of
    their own."""
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as O
    nfull = src_codes.numel() // 128
    blks = torch.from_numpy(np.sort(np.random.default_rng(seed).choice(nfull, nsample, False)))
    blks = blks.to(src_codes.device)
    idx = (blks[:, None] * 128 + torch.arange(128, device=blks.device)[None, :]).reshape(-1)
    mine_c, mine_s = src_codes[idx].contiguous(), src_scales[blks].contiguous()
    all_c = [torch.empty_like(mine_c) for _ in range(world)]
    all_s = [torch.empty_like(mine_s) for _ in range(world)]
    if world > 1:
        dist.all_gather(all_c, mine_c)
        dist.all_gather(all_s, mine_s)
    else:
        all_c, all_s = [mine_c], [mine_s]
    want_c, want_s = O.allreduce_decomposed([c.cpu().numpy() for c in all_c],
                                            [x.cpu().numpy() for x in all_s])
    got_c = result.codes[idx].cpu().numpy()
    got_s = result.scales[blks].cpu().numpy()
    return bool(np.array_equal(got_c, want_c) and
                np.array_equal(got_s.view(np.uint32), want_s.view(np.uint32)))


def bench_allreduce(dev, args, world, rank, n):
    """C4: decomposed 8-bit all-reduce vs BF16 ncclAllReduce, same gradient;
    64 sampled blocks of every algorithm's result checked against the CPU
    oracle over all ranks' inputs."""
    import torch
    import paper_2605_00539_b200 as A
    from paper_2605_00539_b200 import _lib as L
    from paper_2605_00539_b200.collective import Communicator
    comm = Communicator(device=dev.index)
    sp = torch.cuda.current_stream().cuda_stream
    nb = (n + 127) // 128
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    src_codes = torch.empty(n, dtype=torch.uint8, device=dev)
    src_scales = torch.empty(nb, dtype=torch.float32, device=dev)
    chunk = 1 << 28
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        x = torch.randn(m, device=dev, generator=g) * 1e-3
        L.check(L.lib.agq_quantize(x.data_ptr(), L.AGQ_F32, m, 8, 128, 2, src_codes[off:].data_ptr(),
                                   L.AGQ_CODES_BYTES, src_scales[off // 128:].data_ptr(), None, sp))
        del x
    q = A.QuantizedTensor(torch.empty_like(src_codes), torch.empty_like(src_scales), 8, 128, (n,),
                          A.CodecKind.Fp8E4M3, packed=False)
    err = A.ErrorRecord(dev).reset()
    res = {"config": f"C4 decomposed 8-bit all-reduce, {n} FP8 elements per rank",
           "elements": n, "world": world}
    iters = max(2, min(args.steps, 5))

    def timed(fn, reset):
        for _ in range(1):
            reset()
            fn()
        torch.cuda.synchronize()
        barrier(world)
        tot = 0.0
        for _ in range(iters):
            reset()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            tot += s.elapsed_time(e) * 1e-3
        return max_over_ranks(tot / iters, world)

    wire = n * (1 + 4 / 128)
    fac = 2 * (world - 1) / world
    for algo in args.algos:
        if algo == "oneshot":  # the small-message algorithm (<= 1 Mi elements)
            continue
        if algo in ("p2p", "push"):
            comm.enable_p2p(n)
            pc, ps = comm.p2p_buffers(n)
            qq = A.QuantizedTensor(pc, ps, 8, 128, (n,), A.CodecKind.Fp8E4M3, packed=False)
        else:
            qq = q

        def reset(qq=qq):
            qq.codes.copy_(src_codes)
            qq.scales.copy_(src_scales)

        def fn(qq=qq, algo=algo):
            L.check(L.lib.agq_allreduce_fp8(comm._h, qq.codes.data_ptr(), qq.scales.data_ptr(), n, 128,
                                            comm.ALGOS[algo], err.ptr, sp))
        err.reset()
        try:
            sec = timed(fn, reset)
            L.errors_message(err.read(), L.AGQ_OP_ALLREDUCE)
        except Exception as ex:  # recorded, not fatal: the act metric still prints
            # (the failure modes — flag timeout, NCCL error — hit every rank alike)
            res[algo] = {"error": str(ex)[:300]}
            print(f"rank {rank}: allreduce {algo} failed: {ex}", file=sys.stderr, flush=True)
            continue
        res[algo] = {"ms": round(sec * 1e3, 3), "bus_GBs_wire": round(fac * wire / sec / 1e9, 1),
                     "bus_GBs_bf16_equiv": round(fac * 2 * n / sec / 1e9, 1),
                     "frac_of_nvlink_900": round(fac * wire / sec / 1e9 / NVLINK_GBS, 4),
                     "oracle_64_blocks_bitexact": allreduce_oracle_sample(src_codes, src_scales, qq,
                                                                          world, rank)}
        if algo in ("p2p", "push") and "ms" in res.get("nccl", {}):
            ok = torch.equal(qq.codes, q.codes) and torch.equal(qq.scales, q.scales)
            res[algo + "_equals_nccl"] = bool(ok)
    del src_codes
    # BF16 baseline on the same element count
    gb = torch.empty(n, dtype=torch.bfloat16, device=dev)
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        gb[off:off + m] = (torch.randn(m, device=dev, generator=g) * 1e-3).to(torch.bfloat16)

    def bf16_with(c):
        def run():
            L.check(L.lib.agq_allreduce_bf16_nccl(c._h, gb.data_ptr(), n, sp))
        return run
    sec = timed(bf16_with(comm), lambda: None)
    res["bf16_nccl"] = {"ms": round(sec * 1e3, 3), "bus_GBs": round(fac * 2 * n / sec / 1e9, 1),
                        "frac_of_nvlink_900": round(fac * 2 * n / sec / 1e9 / NVLINK_GBS, 4),
                        "nccl_algo": "default (NCCL's tuner)"}
    best_bf16 = res["bf16_nccl"]["ms"]
    # the BF16 baseline under each forced NCCL algorithm (NVLS = in-switch
    # reduction on NVSwitch), on a dedicated communicator created while
    # NCCL_ALGO is set (NCCL reads it at communicator init)
    for algo in args.bf16_algos:
        old = os.environ.get("NCCL_ALGO")
        os.environ["NCCL_ALGO"] = algo
        try:
            c2 = Communicator(device=dev.index)
        except Exception as ex:  # NCCL refused the algorithm on this fabric
            res[f"bf16_nccl_{algo}"] = {"error": str(ex)[:200]}
            continue
        finally:
            if old is None:
                os.environ.pop("NCCL_ALGO", None)
            else:
                os.environ["NCCL_ALGO"] = old
        try:
            sec = timed(bf16_with(c2), lambda: None)
            res[f"bf16_nccl_{algo}"] = {"ms": round(sec * 1e3, 3),
                                        "bus_GBs": round(fac * 2 * n / sec / 1e9, 1)}
            best_bf16 = min(best_bf16, sec * 1e3)
        except Exception as ex:
            res[f"bf16_nccl_{algo}"] = {"error": str(ex)[:200]}
        c2.close()
    done = [res[a]["ms"] for a in args.algos if "ms" in res.get(a, {})]
    if done:
        res["speedup_vs_bf16_nccl"] = round(res["bf16_nccl"]["ms"] / min(done), 3)
        res["speedup_vs_best_bf16_nccl"] = round(best_bf16 / min(done), 3)
    del gb, q
    comm.close()
    torch.cuda.empty_cache()
    return res


def bench_sweep(dev, args, world, rank):
    """C5: message-size sweep (FP8 payload 2^20..2^32 bytes) plus LLaMA-32B
    gradient buckets, decomposed 8-bit all-reduce vs BF16 ncclAllReduce of the
    same element count. LLaMA-32B (hidden 5120, FFN 27648, 64 layers, GQA-8,
    vocab 152064): one bucket per transformer layer and 40M-param
    Megatron-style buckets."""
    import torch
    import paper_2605_00539_b200 as A
    from paper_2605_00539_b200 import _lib as L
    from paper_2605_00539_b200.collective import Communicator
    sizes = [1 << k for k in range(16, 33)]
    # q,o (5120^2) + k,v (GQA-8, head 128: 5120x1024) + gate/up/down + 2 norms = 487.6M
    layer = 5120 * 5120 * 2 + 2 * 5120 * 1024 + 3 * 5120 * 27648 + 2 * 5120
    buckets = {"llama32b_layer_bucket": layer, "megatron_40M_bucket": 40_000_000}
    nmax = max(max(sizes), layer)
    comm = Communicator(device=dev.index)
    if any(a in args.algos for a in ("p2p", "push", "oneshot")):
        comm.enable_p2p(nmax)
    sp = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    src_c = torch.empty(nmax, dtype=torch.uint8, device=dev)
    src_s = torch.empty((nmax + 127) // 128, dtype=torch.float32, device=dev)
    for off in range(0, nmax, 1 << 28):
        m = min(1 << 28, nmax - off)
        x = torch.randn(m, device=dev, generator=g) * 1e-3
        L.check(L.lib.agq_quantize(x.data_ptr(), L.AGQ_F32, m, 8, 128, 2, src_c[off:].data_ptr(),
                                   L.AGQ_CODES_BYTES, src_s[off // 128:].data_ptr(), None, sp))
    work_c, work_s = torch.empty_like(src_c), torch.empty_like(src_s)
    if any(a in args.algos for a in ("p2p", "push", "oneshot")):
        pc, ps = comm.p2p_buffers(nmax)
    gb = torch.empty(nmax, dtype=torch.bfloat16, device=dev)
    gb.normal_(0, 1e-3, generator=g)
    err = A.ErrorRecord(dev).reset()
    fac = 2 * (world - 1) / world

    def timeit(fn, n, restore=None):
        """Device time per call, max over ranks: back-to-back calls, as
        consecutive gradient buckets issue them. With `restore`, batches of
        at most 16 in-place calls (each call multiplies the values by up to
        P; 16 calls stay far inside FP32 range at P <= 8), the inputs
        restored between batches outside the timed region. (Round 2 first
        subtracted a restore-only loop instead; at small sizes that loop is
        host bound, which understated the per-call time by ~10 us.)"""
        iters = int(min(200, max(5, (2 << 30) // max(n, 1))))
        batch = iters if restore is None else min(iters, 16)
        nbatch = max(1, iters // batch)
        if restore is not None:
            restore()
        for _ in range(3):
            fn()
        total = 0.0
        for _ in range(nbatch):
            if restore is not None:
                restore()
            torch.cuda.synchronize()
            barrier(world)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(batch):
                fn()
            e.record()
            torch.cuda.synchronize()
            total += s.elapsed_time(e) * 1e-3
        return max_over_ranks(total / (nbatch * batch), world)

    rows = []
    cases = [(f"{n >> 20}MiB" if n >= 1 << 20 else f"{n >> 10}KiB", n) for n in sizes] + \
        list(buckets.items())
    for name, n in cases:
        row = {"case": name, "elements": n, "fp8_wire_bytes": int(n * (1 + 4 / 128))}
        for algo in args.algos:
            if algo == "oneshot" and (n > comm.ONESHOT_MAX or world > 8):
                continue
            cb, sb = (pc, ps) if algo in ("p2p", "push", "oneshot") else (work_c, work_s)
            nb = (n + 127) // 128

            def restore(cb=cb, sb=sb):
                cb[:n].copy_(src_c[:n])
                sb[:nb].copy_(src_s[:nb])

            def fn(cb=cb, sb=sb, algo=algo):
                L.check(L.lib.agq_allreduce_fp8(comm._h, cb.data_ptr(), sb.data_ptr(), n, 128,
                                                comm.ALGOS[algo], err.ptr, sp))
            err.reset()
            sec = timeit(fn, n, restore)
            L.errors_message(err.read(), L.AGQ_OP_ALLREDUCE)
            row[algo + "_us"] = round(sec * 1e6, 1)
            row[algo + "_busGBs_wire"] = round(fac * n * (1 + 4 / 128) / sec / 1e9, 1)

        def bf():
            L.check(L.lib.agq_allreduce_bf16_nccl(comm._h, gb.data_ptr(), n, sp))
        sec = timeit(bf, 2 * n)
        row["bf16_nccl_us"] = round(sec * 1e6, 1)
        row["bf16_nccl_busGBs"] = round(fac * 2 * n / sec / 1e9, 1)
        best = min(row[a + "_us"] for a in args.algos if a + "_us" in row)
        row["speedup_vs_bf16"] = round(row["bf16_nccl_us"] / best, 3)
        rows.append(row)
    comm.close()
    return rows


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# the reference's CPU implementation (oracle/_ref) on a bounded sample
# ---------------------------------------------------------------------------
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_reference_rate(sample_elems, threads, rounds=1, min_seconds=0.0, pin_core=None):
    """GB/s (same algorithmic bytes as the GPU arm) of quantize_blockwise +
    dequantize_blockwise of the reference over every stage width, on the
    first `sample_elems` values of the GPU arm's first C2 tensor (the same
    make_rng(SEED, 0x1D, 0) normal draws, BF16-rounded), `threads` host
    threads over disjoint block ranges (blocks are independent,
    quantize.hpp:103-136). pin_core: run on that one core only (taskset)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as O
    kind = "reference" if O.ref is not None else "port"
    lib = O.ref if O.ref is not None else None
    if lib is not None:
        x = O.bf16_round(O.ref_normal(SEED, 0x1D, 0, sample_elems))
    else:
        x = O.bf16_round(np.random.default_rng(SEED).standard_normal(sample_elems).astype(np.float32))
    codes = np.empty(sample_elems, np.uint8)
    scales = np.empty((sample_elems + 127) // 128, np.float32)
    out = np.empty(sample_elems, np.float32)
    old = None
    if pin_core is not None and hasattr(os, "sched_setaffinity"):
        old = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {pin_core})
    try:
        t0 = time.perf_counter()
        nbytes = 0.0
        r = 0
        while r < rounds or time.perf_counter() - t0 < min_seconds:
            r += 1
            for b in STAGE_BITS:
                if lib is not None:
                    st = lib.ref_quantize_mt(O._p(x), sample_elems, b, 128, 0, O._p(codes),
                                             O._p(scales), threads)
                    st |= lib.ref_dequantize_mt(O._p(codes), O._p(scales), sample_elems, b, 128, 0,
                                                O._p(out), threads)
                    assert st == 0
                else:
                    c, sc = O.quantize(x, b, 128, 0)
                    O.dequantize(c, sc, b, 128, 0)
                nbytes += sample_elems * sum(act_bytes_per_elem(b))
        sec = time.perf_counter() - t0
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    return nbytes / sec / 1e9, kind, sec


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, world, rank):
    """The reference arm: oracle/_ref (the unmodified reference headers) on
    the host cores; loads no library of this repo's package."""
    if rank != 0:
        return
    threads = host_threads()
    sample = 1 << 24
    for _ in range(args.warmup):
        cpu_reference_rate(sample, threads)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, kind, _ = cpu_reference_rate(sample, threads)
        vals.append(v)
    sec = time.perf_counter() - t0
    value = sum(vals) / len(vals)
    v1, _, s1 = cpu_reference_rate(1 << 22, 1, pin_core=sorted(os.sched_getaffinity(0))[0])
    line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sec / args.steps * 1e3, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8 codes / f32 scales (bf16-valued f32 in)",
            "data": "synthetic: make_rng(0, 0x1D) N(0,1) draws rounded to bf16 (the GPU arm's "
                    "first C2 tensor)", "impl": "reference",
            "config": {"workload": "C2: LLaMA-8B block stored activations (seq 4096 x mb 4), "
                                   "8-stage DBCA policies, quant+dequant",
                       "stage_bits": list(STAGE_BITS), "block": 128,
                       "sample_elements_per_stage": sample,
                       "sample": "each step quantizes+dequantizes a 2^24-element sample of the "
                                 "workload at every stage width (the full 671M-element step is "
                                 "~10 min of CPU time)"},
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": kind,
                             "sample": f"{sample} elements x 8 stage widths per step",
                             "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                             "single_core": {"value": round(v1, 4), "unit": "GB/s", "cores": 1,
                                             "pinned": "taskset core 0 (sched_setaffinity)",
                                             "sample": "2^22 elements x 8 stage widths",
                                             "seconds": round(s1, 2)}},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ar-elements", type=int, default=LLAMA8B_PARAMS)
    ap.add_argument("--acc-elements", type=int, default=LLAMA8B_PARAMS)
    ap.add_argument("--algos", default="nccl,p2p,push,oneshot")
    ap.add_argument("--bf16-algos", default="NVLS,Ring",
                    help="extra BF16 ncclAllReduce baselines with NCCL_ALGO forced (C4)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--e2e-streams", type=int, default=4)
    ap.add_argument("--no-accumulate", action="store_true")
    ap.add_argument("--no-allreduce", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", action="store_true",
                    help="C5: all-reduce message-size sweep + LLaMA-32B buckets (N > 1)")
    args = ap.parse_args()
    args.algos = [a for a in args.algos.split(",") if a]
    args.bf16_algos = [a for a in args.bf16_algos.split(",") if a]
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import torch
    import paper_2605_00539_b200 as A
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if not A.device_ok():
        raise SystemExit("not an sm_100 device: the AGoQ kernels have no other path")
    if args.sweep:
        rows = bench_sweep(dev, args, world, rank)
        if rank == 0:
            print(json.dumps({"metric": "8-bit all-reduce bus GB/s sweep (C5)", "n_gpus": world,
                              "unit": "GB/s", "sweep": rows}), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    peak, peak_kind = load_peaks()
    clocks = Clocks(local)

    wl = ActWorkload(dev)
    parity = wl.verify_sample()
    clocks.start()
    sec, launches, (q_gbs, q_time), (d_gbs, d_time) = bench_act(wl, args, world)
    step_bytes = wl.bytes_per_step()
    value = step_bytes * args.steps * world / sec / 1e9
    extra = {}
    if not args.no_e2e:
        e2e_val, bi, bo = bench_e2e(wl, args, world, steps=2, chunks=args.e2e_chunks,
                                     nstreams=args.e2e_streams)
        extra["e2e"] = {"value": round(e2e_val, 1), "unit": "GB/s", "h2d_bytes_per_step": bi,
                        "d2h_bytes_per_step": bo}
    extra["c2_stage"] = bench_c2_stage(wl, args)
    del wl
    torch.cuda.empty_cache()
    extra["c1"] = bench_c1(dev, args)
    if not args.no_e2e and rank == 0:  # host-path measurement: one process
        extra["e2e_dropin"] = bench_dropin(dev)
    if not args.no_accumulate:
        extra["accumulate"] = bench_accumulate(dev, args, args.acc_elements)
    if world == 1 and not args.no_allreduce:
        extra["reduce_local"] = bench_reduce_local(dev, args)
    if world > 1 and not args.no_allreduce:
        extra["allreduce"] = bench_allreduce(dev, args, world, rank, args.ar_elements)
    clk = clocks.stop()
    for k in ("c1", "accumulate", "reduce_local", "c2_stage"):  # share of the HBM peak
        if k in extra and "GBs" in extra[k]:
            extra[k]["frac_of_peak"] = round(extra[k]["GBs"] / peak, 4)
    for v in extra.get("accumulate", {}).get("variants", {}).values():
        v["frac_of_peak"] = round(v["GBs"] / peak, 4)

    dom_name, dom_gbs, other = ("k_quant_warp", q_gbs, {"k_dequant_warp_GBs": round(d_gbs, 1)}) \
        if q_time >= d_time else ("k_dequant_warp", d_gbs, {"k_quant_warp_GBs": round(q_gbs, 1)})
    traffic = load_traffic().get(dom_name)
    roofline = {"bound": "hbm", "achieved": round(dom_gbs, 1), "peak": peak, "unit": "GB/s",
                "frac": round(dom_gbs / peak, 4), "frac_of_nominal_8tbs": round(dom_gbs / 8000.0, 4),
                "traffic": traffic, "kernel": dom_name,
                "peak_kind": peak_kind, **other}
    line = {"metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sec / args.steps * 1e3, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 in/out, u4-u8 packed codes, f32 scales",
            "data": "synthetic: the reference RNG's N(0, s_i) draws (make_rng(0, 0x1D, i), "
                    "BF16-rounded; s = 1, 1, 0.5, 4, 1), same bytes as the reference arm",
            "config": {"workload": "C2: LLaMA-8B block stored activations (seq 4096 x mb 4), "
                                   "8-stage DBCA policies, quant+dequant",
                       "elements_per_stage": sum(T_TOKENS * w for _, w in TENSORS),
                       "stage_bits": stage_bits(), "block": 128,
                       "l2": "inputs/outputs 1.3 GB per pass >> 126 MB L2 (no flush needed)",
                       "parallelism": f"replicas x{world}"},
            "roofline": roofline, "gpu_launches": launches, "parity_sample_bitexact": parity,
            "clocks": clk, **extra}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        th = host_threads()
        v, kind, csec = cpu_reference_rate(1 << 24, th, min_seconds=8.0)
        v1, _, s1 = cpu_reference_rate(1 << 22, 1, pin_core=sorted(os.sched_getaffinity(0))[0])
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "GB/s", "cores": th,
                                "kind": kind, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                                "sample": f"2^24 elements of the first C2 tensor (same bytes) x 8 "
                                          f"stage widths, repeated for {csec:.1f} s of CPU time",
                                "single_core": {"value": round(v1, 4), "unit": "GB/s", "cores": 1,
                                                "pinned": "core 0 (sched_setaffinity)",
                                                "sample": "2^22 elements x 8 stage widths"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
