"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU).

  python tools/ncu_summary.py report <file.ncu-rep> [label]   -> key metrics per kernel
  python tools/ncu_summary.py launches <launches.csv>         -> per-kernel share of time
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def report(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:120], "label": label}
        for k in KEYS:
            if k in d:
                rec[k] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[h])
                  for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued") and d[h] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1.0
        rec["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                                 for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        out.append(rec)
    return out


def launches(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rows = list(csv.DictReader(io.StringIO(txt)))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r.get("Metric Unit", "us"), 1.0)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    return [{"kernel": k, "launches": v[0], "total_us": round(v[1], 1), "share": round(v[1] / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    if sys.argv[1] == "report":
        print(json.dumps(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""), indent=1))
    else:
        print(json.dumps(launches(sys.argv[2]), indent=1))
