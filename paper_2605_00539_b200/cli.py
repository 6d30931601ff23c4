"""`agq`-shaped command line over the B200 path (reference harness:
/root/reference/proj/tools/agq.cpp:114-152 run_quantize, :240-272 run_dbca,
:274-324 run_allreduce). Same subcommands, flags and JSON keys; the compute
runs on the GPU. Inputs are the reference's own bytes (inputs.materialize:
make_rng(seed, 0x1D) + std::normal_distribution<float>, agq.cpp:47-65), and
the statistics are summed on the host in the reference's order, so the JSON
equals the reference CLI's bit for bit.

  python -m paper_2605_00539_b200.cli quantize --normal 4096 --bits 4 [--codec linear] [--dump f]
  python -m paper_2605_00539_b200.cli allreduce-sim --workers 8 --elements 4096 --protocol decomposed
  python -m paper_2605_00539_b200.cli dbca-plan 4 [--reuse-onto 8]
"""
from __future__ import annotations

import argparse
import json
import math
import sys

CODECS = {"linear": 0, "symmetric_linear": 0, "fp4": 1, "fp4_e2m1": 1, "fp8": 2, "fp8_e4m3": 2}
NAMES = {0: "symmetric_linear", 1: "fp4_e2m1", 2: "fp8_e4m3"}


def _input(args, seed, n_default):
    from paper_2605_00539_b200.inputs import materialize
    n = args.normal or args.elements or n_default
    if args.const is not None:
        x = materialize(n, seed, "const", float(args.const))
    elif args.uniform:
        a, b = args.uniform
        if not a <= b:
            raise ValueError("--uniform needs a <= b")
        x = materialize(n, seed, "uniform", a, b)
    else:
        x = materialize(n, seed, "normal", 0.0, 1.0)
    return x.cuda()


def _seq_sum(v):
    """Left-to-right double sum (the reference's loops, agq.cpp:123-128)."""
    import numpy as np
    return float(np.add.accumulate(np.asarray(v, np.float64))[-1]) if len(v) else 0.0


def run_quantize(args):
    import torch
    import paper_2605_00539_b200 as A
    from paper_2605_00539_b200 import tensor_io
    x = _input(args, args.seed, 4096)
    kind = A.CodecKind(CODECS[args.codec])
    q = A.quantize_blockwise(x, args.bits, args.block, kind)
    back = A.dequantize_blockwise(q).double().cpu().numpy()
    xd = x.double().cpu().numpy()
    err = abs(back - xd)  # exact in double (both are floats)
    nz = xd != 0
    stats = {"elements": x.numel(), "bit_width": args.bits, "block_size": args.block,
             "codec": NAMES[int(kind)], "mae": _seq_sum(err) / x.numel(),
             "max_abs_error": float(err.max()),
             "max_rel_error": float((err[nz] / abs(xd[nz])).max()) if bool(nz.any()) else 0.0,
             "compression_ratio": 4.0 * x.numel() / (math.ceil(x.numel() * args.bits / 8)
                                                     + 4.0 * q.num_blocks())}
    if args.dump:
        blob = tensor_io.dump_tensor(q)
        with open(args.dump, "wb") as f:
            f.write(blob)
        q2 = tensor_io.load_tensor(open(args.dump, "rb").read())
        stats["dump"] = args.dump
        stats["dump_roundtrip_exact"] = bool(torch.equal(q2.codes, q.codes) and
                                             torch.equal(q2.scales, q.scales))
    return stats


def run_allreduce(args):
    import torch
    import paper_2605_00539_b200 as A
    mains = []
    for r in range(args.workers):
        x = _input(args, args.seed + r, 4096)
        mains.append(A.quantize_blockwise(x, 8, 128, A.CodecKind.Fp8E4M3, packed=False))
    oracle = torch.zeros(mains[0].num_elements(), dtype=torch.float32, device="cuda")
    for m in mains:  # allreduce_oracle: fp32 sum in ascending rank from +0.0f
        oracle += A.dequantize_blockwise(m)
    j = {"protocol": args.protocol, "workers": args.workers, "elements": mains[0].num_elements()}
    if args.protocol == "oracle":
        o = oracle.double().cpu().numpy()
        j["oracle_l2"] = math.sqrt(_seq_sum(o * o))
        return j
    if args.protocol == "decomposed":
        out, overflow = A.allreduce_simulated(mains), 0
        trace = A.decomposed_trace(out.num_elements(), 128, args.workers)
    elif args.protocol == "naive":
        out, overflow = A.allreduce_naive_simulated(mains)
        trace = A.naive_trace(out.num_elements(), 128, args.workers)
    else:
        raise ValueError("--protocol: expected decomposed, naive or oracle")
    vals = A.dequantize_blockwise(out).double().cpu().numpy()
    j["max_abs_dev_vs_oracle"] = float(abs(vals - oracle.double().cpu().numpy()).max())
    j["result_l2"] = math.sqrt(_seq_sum(vals * vals))
    j["overflow_total"] = int(overflow)
    if trace is not None:
        j["message_count"] = len(trace)
        j["payload_bytes"] = sum(e.payload_bytes for e in trace)
        if args.trace:
            with open(args.trace, "w") as f:
                for e in trace:
                    f.write(json.dumps(e.__dict__, sort_keys=True) + "\n")
            j["trace"] = args.trace
    return j


def run_dbca(args):
    import paper_2605_00539_b200 as A
    cfg = A.PipelineConfig(args.n_stages, args.micro_batches or 2 * args.n_stages, 2)
    plan = A.plan_bit_widths(cfg)
    chk = A.peak_memory_check(plan, args.minibatch_bytes)
    j = {"n_stages": plan.n_stages, "counts": [s.stored_minibatches for s in plan.stages],
         "raw_bits": [s.raw_bits for s in plan.stages], "assigned_bits": plan.assigned(),
         "peak_check": {"pass": chk.passed, "budget_bytes": chk.budget_bytes,
                        "slack_bytes": chk.slack_bytes, "stages": chk.stages}}
    if args.reuse_onto:
        r = A.plan_reuse_check(cfg, A.PipelineConfig(args.reuse_onto, 2 * args.reuse_onto, 2))
        j["reuse"] = {"onto_stages": args.reuse_onto, **r}
    return j


def main(argv=None):
    ap = argparse.ArgumentParser(prog="agq-b200")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    sub = ap.add_subparsers(dest="cmd", required=True)
    q = sub.add_parser("quantize")
    a = sub.add_parser("allreduce-sim")
    for p in (q, a):
        p.add_argument("--normal", type=int)
        p.add_argument("--const", type=float)
        p.add_argument("--uniform", type=float, nargs=2)
        p.add_argument("--elements", type=int, default=4096)
    q.add_argument("--bits", type=int, default=4)
    q.add_argument("--block", type=int, default=128)
    q.add_argument("--codec", default="linear", choices=sorted(CODECS))
    q.add_argument("--dump", default="")
    a.add_argument("--workers", type=int, default=4)
    a.add_argument("--protocol", default="decomposed")
    a.add_argument("--trace", default="")
    d = sub.add_parser("dbca-plan")
    d.add_argument("n_stages", type=int)
    d.add_argument("--micro-batches", type=int, default=0)
    d.add_argument("--reuse-onto", type=int, default=0)
    d.add_argument("--minibatch-bytes", type=float, default=16.0)
    args = ap.parse_args(argv)
    try:
        res = {"quantize": run_quantize, "allreduce-sim": run_allreduce, "dbca-plan": run_dbca}[args.cmd](args)
    except Exception as e:  # agq.cpp:433-442: JSON error on stderr, non-zero exit
        print(json.dumps({"error": str(e)}), file=sys.stderr)
        return 1
    text = json.dumps(res, indent=2, sort_keys=True)  # nlohmann::json orders keys
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
    else:
        print(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
