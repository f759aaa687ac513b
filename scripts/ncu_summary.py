"""Summarise ncu output into profiles/ (tracked).

  python scripts/ncu_summary.py launches <launches.csv> <out.json> [command]
  python scripts/ncu_summary.py full <report.ncu-rep> <out.json> [algorithmic_bytes]

`launches`: per-kernel launch count / mean / median duration and share of the
captured time (the --metrics gpu__time_duration.sum pass).
`full`: the metrics that explain an HBM-bound kernel, per captured launch,
from `ncu -i <rep> --page raw --csv` (dram bytes, duration, occupancy, stall
reasons, tensor pipe).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import statistics
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
]
UNITS_TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3,
                  "byte/block": 1}
UNITS_TO_NS = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}


def _csv_rows(text: str):
    lines = [l for l in text.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path: str, out: str, command: str | None):
    rows = _csv_rows(open(path).read())
    h = rows[0]
    ik, iname, ival = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    iunit = h.index("Metric Unit")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        if r[iname] == "gpu__time_duration.sum":
            d[r[ik]].append(float(r[ival].replace(",", "")) * UNITS_TO_NS.get(r[iunit], 1))
    total = sum(sum(v) for v in d.values())
    ks = [{"kernel": k[:120], "launches": len(v), "total_ns": sum(v), "mean_ns": statistics.mean(v),
           "median_ns": statistics.median(v), "min_ns": min(v), "max_ns": max(v),
           "share": sum(v) / total} for k, v in d.items()]
    ks.sort(key=lambda e: -e["total_ns"])
    json.dump({"command": command, "kernels": ks}, open(out, "w"), indent=1)
    print(json.dumps(ks[:4], indent=1))


def full(path: str, out: str, alg_bytes: float | None):
    text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                          text=True, check=True).stdout
    rows = _csv_rows(text)
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        e = {"kernel": r[h.index("Kernel Name")][:120]}
        for k in KEYS + [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_")
                         and not c.endswith("_not_issued")]:
            if k in h:
                v, u = r[h.index(k)], units[h.index(k)]
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if u in UNITS_TO_BYTES:
                    x, u = x * UNITS_TO_BYTES[u], "byte"
                if u in UNITS_TO_NS:
                    x, u = x * UNITS_TO_NS[u], "ns"
                e[k] = x
        if "dram__bytes_read.sum" in e and "gpu__time_duration.sum" in e:
            tb = e["dram__bytes_read.sum"] + e.get("dram__bytes_write.sum", 0.0)
            e["dram_bytes_per_launch"] = tb
            e["dram_gbs"] = tb / e["gpu__time_duration.sum"]  # bytes/ns = GB/s
            if alg_bytes:
                e["algorithmic_bytes"] = alg_bytes
                e["traffic_over_algorithmic"] = tb / alg_bytes
        stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: v for k, v in e.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_")}
        if stalls:
            tot = sum(stalls.values()) or 1
            e["top_stalls"] = {k: round(v / tot, 3) for k, v in
                               sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
            for k in list(e):
                if k.startswith("smsp__pcsamp_warps_issue_stalled_"):
                    del e[k]
        res.append(e)
    json.dump({"report": path.split("/")[-1], "launches": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    extra = sys.argv[4] if len(sys.argv) > 4 else None
    if mode == "launches":
        launches(src, dst, extra)
    else:
        full(src, dst, float(extra) if extra else None)
