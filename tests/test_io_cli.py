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
