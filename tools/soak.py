"""Randomized bit-exactness soak against the C oracle: random sizes
(ragged tails), block sizes, codecs, widths, input dtypes, magnitudes with
exact zeros, all-zero blocks and wide dynamic range; quantize, dequantize,
local_accumulate and the simulated all-reduce. Prints one line per failure
and a summary; exit 1 on any mismatch."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_ffi as O  # noqa: E402
import paper_2605_00539_b200 as A  # noqa: E402

dev = torch.device("cuda")
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(time.time()))
fails = cases = 0
t0 = time.time()
while time.time() - t0 < budget:
    n = int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 400000), 128 * rng.integers(1, 3000)]))
    block = int(rng.choice([128, 128, 128, 64, 32, 16, 256, 1000]))
    kind, bits = [(0, int(rng.integers(4, 9))), (1, 4), (2, 8)][int(rng.integers(0, 3))]
    nb = (n + block - 1) // block
    mag = np.repeat(10.0 ** rng.uniform(-30, 30, nb), block)[:n]
    x = (rng.standard_normal(n) * mag).astype(np.float32)
    x[rng.random(n) < 0.02] = 0.0
    if nb > 2:
        z = rng.integers(0, nb)
        x[z * block:(z + 1) * block] = 0.0
    bf16 = bool(rng.integers(0, 2))
    if bf16:
        x = O.bf16_round(x)
    xt = torch.from_numpy(x).to(dev)
    if bf16:
        xt = xt.to(torch.bfloat16)
    packed = bool(rng.integers(0, 2))
    cases += 1
    try:
        c, s = O.quantize(x, bits, block, kind)
        q = A.quantize_blockwise(xt, bits, block, A.CodecKind(kind), packed=packed)
        got = q.codes.cpu().numpy()
        want = O.pack(c, bits) if packed else c
        ok = np.array_equal(got, want) and np.array_equal(q.scales.cpu().numpy().view(np.uint32),
                                                          s.view(np.uint32))
        d = A.dequantize_blockwise(q).cpu().numpy()
        ok &= np.array_equal(d.view(np.uint32), O.dequantize(c, s, bits, block, kind).view(np.uint32))
        if kind == 2:
            loc = (rng.standard_normal(n) * mag * 0.1).astype(np.float32)
            oc, os_ = O.local_accumulate(c, s, loc, 0, block)
            acc = A.local_accumulate(A.QuantizedTensor(torch.from_numpy(c).to(dev),
                                                       torch.from_numpy(s).to(dev), 8, block, (n,),
                                                       A.CodecKind.Fp8E4M3, packed=False),
                                     torch.from_numpy(loc).to(dev))
            ok &= np.array_equal(acc.codes.cpu().numpy(), oc) and np.array_equal(
                acc.scales.cpu().numpy().view(np.uint32), os_.view(np.uint32))
            if block == 128:
                P = int(rng.integers(1, 9))
                pcs = []
                for _ in range(P):
                    xi = (rng.standard_normal(n) * mag).astype(np.float32)
                    pcs.append(O.quantize(xi, 8, 128, 2))
                wc, ws = O.allreduce_decomposed([a for a, _ in pcs], [b for _, b in pcs])
                out = A.allreduce_simulated([A.QuantizedTensor(torch.from_numpy(a).to(dev),
                                                               torch.from_numpy(b).to(dev), 8, 128,
                                                               (n,), A.CodecKind.Fp8E4M3,
                                                               packed=False) for a, b in pcs])
                ok &= np.array_equal(out.codes.cpu().numpy(), wc) and np.array_equal(
                    out.scales.cpu().numpy().view(np.uint32), ws.view(np.uint32))
    except Exception as e:  # inputs are finite and in range: no side may raise
        ok = False
        print(f"ERROR {type(e).__name__}: {e}", flush=True)
    if not ok:
        fails += 1
        print(f"MISMATCH n={n} block={block} kind={kind} bits={bits} bf16={bf16} packed={packed}",
              flush=True)
print(f"soak: {cases} cases in {time.time() - t0:.0f} s, {fails} mismatches", flush=True)
sys.exit(1 if fails else 0)
