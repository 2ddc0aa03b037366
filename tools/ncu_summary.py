"""Summarise ncu outputs for profiles/.

    python tools/ncu_summary.py launches <launch-list.csv>      # per-kernel count / total / share
    python tools/ncu_summary.py full <report.ncu-rep>            # key metrics per captured launch
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"]
            unit = d.get("Metric Unit", "ns")
            v = float(d["Metric Value"].replace(",", ""))
            v_us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
            agg.setdefault(name, []).append(v_us)
    total = sum(sum(v) for v in agg.values())
    out = [f"# kernels: {sum(len(v) for v in agg.values())} launches, {total / 1e3:.3f} ms total device time "
           "(ncu, serialised, cold-cache: compare shares, not absolutes)",
           f"{'share':>7} {'total_ms':>9} {'count':>6} {'avg_us':>9}  kernel"]
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{100 * sum(v) / total:6.2f}% {sum(v) / 1e3:9.3f} {len(v):6d} {sum(v) / len(v):9.2f}  {name[:110]}")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"== {d['Kernel Name'][:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"   {k} = {d[k]} {u.get(k, '')}")
        st = {k: float(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
              and v.replace(".", "").isdigit()}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
        out.append("   top stalls: " + ", ".join(f"{k.split('stalled_')[1]}={int(v)}" for k, v in top))
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
