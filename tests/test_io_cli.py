"""AGQT dump/load from device buffers (tensor_io.hpp) and the agq-shaped CLI
(tools/agq.cpp): dump bytes equal the reference's own dump; CLI subcommands
mirror the reference harness (proj/tests/CMakeLists.txt:39-52 smoke regexes)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle_ffi as O
import paper_2605_00539_b200 as A
from paper_2605_00539_b200 import cli, tensor_io

ROOT = O.ROOT


def test_cli_dbca_plan_cpu(capsys):
    assert cli.main(["dbca-plan", "4", "--reuse-onto", "8"]) == 0
    j = json.loads(capsys.readouterr().out)
    assert j["counts"] == [11, 9, 7, 5] and j["assigned_bits"] == [4, 5, 6, 8]
    assert j["peak_check"]["pass"] and j["reuse"]["applied_bits"] == [4, 4, 4, 4, 4, 5, 6, 8]


def test_cli_error_is_json_and_nonzero(capsys):
    assert cli.main(["dbca-plan", "4", "--micro-batches", "6"]) == 1
    err = json.loads(capsys.readouterr().err)
    assert "micro_batches >= 2 * n_stages" in err["error"]


@pytest.mark.gpu
def test_dump_matches_reference_bytes(cuda, golden):
    x = torch.tensor([1.0, -1.0, 0.5], device=cuda)
    q = A.quantize_blockwise(x, 4, 2)
    assert tensor_io.dump_tensor(q) == bytes(golden["dump_3_b4_k2"])
    x = torch.from_numpy(golden["x777"]).to(cuda)
    for packed in (True, False):
        q = A.quantize_blockwise(x, 6, 128, shape=(7, 111), packed=packed)
        blob = tensor_io.dump_tensor(q)
        assert blob == bytes(golden["dump_777_b6"])
        q2 = tensor_io.load_tensor(blob, cuda, packed=packed)
        assert torch.equal(q2.codes, q.codes) and torch.equal(q2.scales, q.scales)
        assert q2.shape == (7, 111) and q2.bit_width == 6
    with pytest.raises(A.ProtocolError, match="bad magic"):
        tensor_io.load_tensor(b"BAD!" + blob[4:], cuda)
    with pytest.raises(A.ProtocolError, match="truncated"):
        tensor_io.load_tensor(blob[:-3], cuda)


@pytest.mark.gpu
def test_cli_quantize_and_allreduce(cuda, tmp_path):
    run = lambda *a: json.loads(subprocess.run([sys.executable, "-m", "paper_2605_00539_b200.cli", *a],
                                               cwd=ROOT, capture_output=True, text=True,
                                               check=True).stdout)
    j = run("quantize", "--normal", "4096", "--bits", "4", "--dump", str(tmp_path / "t.agqt"))
    assert j["codec"] == "symmetric_linear" and j["dump_roundtrip_exact"] is True
    assert j["compression_ratio"] > 6.0
    j = run("allreduce-sim", "--workers", "8", "--const", "64", "--elements", "512",
            "--protocol", "naive")
    assert j["overflow_total"] == 512
    j = run("allreduce-sim", "--workers", "8", "--const", "64", "--elements", "512",
            "--protocol", "decomposed", "--trace", str(tmp_path / "tr.jsonl"))
    assert j["overflow_total"] == 0 and j["max_abs_dev_vs_oracle"] == 0.0
    assert j["message_count"] == len(open(tmp_path / "tr.jsonl").readlines())


def _seq(v):
    return float(np.add.accumulate(np.asarray(v, np.float64))[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("bits,codec", [(4, 0), (6, 0), (4, 1), (8, 2)])
def test_cli_quantize_stats_equal_reference(cuda, bits, codec):
    """`quantize --normal 4096 --bits b` JSON equals the reference CLI's
    (agq.cpp:114-152) bit for bit: the reference RNG's inputs, its quantizer
    (oracle/_ref) and its left-to-right double sums."""
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    name = {0: "linear", 1: "fp4", 2: "fp8"}[codec]
    out = subprocess.run([sys.executable, "-m", "paper_2605_00539_b200.cli", "--seed", "3",
                          "quantize", "--normal", "4096", "--bits", str(bits), "--codec", name],
                         cwd=ROOT, capture_output=True, text=True, check=True).stdout
    j = json.loads(out)
    x = O.ref_normal(3, 0x1D, 0, 4096)
    c, s = O.quantize(x, bits, 128, codec, lib=O.ref)
    back = O.dequantize(c, s, bits, 128, codec, lib=O.ref).astype(np.float64)
    err = np.abs(back - x.astype(np.float64))
    nz = x != 0
    want = {"elements": 4096, "bit_width": bits, "block_size": 128,
            "codec": {0: "symmetric_linear", 1: "fp4_e2m1", 2: "fp8_e4m3"}[codec],
            "mae": _seq(err) / 4096, "max_abs_error": float(err.max()),
            "max_rel_error": float((err[nz] / np.abs(x[nz].astype(np.float64))).max()),
            "compression_ratio": 4.0 * 4096 / (np.ceil(4096 * bits / 8.0) + 4.0 * s.size)}
    assert j == want
    assert list(j) == sorted(j)  # nlohmann::json key order


@pytest.mark.gpu
def test_cli_allreduce_stats_equal_reference(cuda):
    """`allreduce-sim --workers 4 --normal 1000` (agq.cpp:274-324): worker r
    from seed + r, the reference's all-reduce, oracle deviation and L2 in its
    summation order, its message trace totals."""
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "-m", "paper_2605_00539_b200.cli", "--seed", "5",
                          "allreduce-sim", "--workers", "4", "--normal", "1000"],
                         cwd=ROOT, capture_output=True, text=True, check=True).stdout
    j = json.loads(out)
    mains = [O.quantize(O.ref_normal(5 + r, 0x1D, 0, 1000), 8, 128, 2, lib=O.ref) for r in range(4)]
    oc, os_, ov, ev, _ = O.ref_allreduce(0, [m[0] for m in mains], [m[1] for m in mains])
    vals = O.dequantize(oc, os_, 8, 128, 2, lib=O.ref).astype(np.float64)
    orc = O.allreduce_oracle([m[0] for m in mains], [m[1] for m in mains]).astype(np.float64)
    assert j["result_l2"] == float(np.sqrt(_seq(vals * vals)))
    assert j["max_abs_dev_vs_oracle"] == float(np.abs(vals - orc).max())
    assert j["overflow_total"] == ov == 0
    assert j["message_count"] == len(ev) and j["payload_bytes"] == int(ev[:, 5].sum())
