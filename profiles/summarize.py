"""Summarise ncu output brought back by gpurun into committed, human-readable profiles.

    python profiles/summarize.py launches <launches.csv> [--skip-prefix at::]   -> per-kernel shares
    python profiles/summarize.py report <file.ncu-rep>                        -> key metrics per kernel
    python profiles/summarize.py traffic <file.ncu-rep> <config> [json]      -> DRAM bytes per launch

The launch list is cold-cache and serialised (ncu --metrics gpu__time_duration.sum
--clock-control none): compare SHARES, not absolute times.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEY_METRICS = [
    "Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
    "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active",
    "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
    "Avg. Active Threads Per Warp", "No Eligible", "Block Limit Registers", "Block Limit Shared Mem",
]
RAW_METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
               "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
               "smsp__issue_active.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_xu.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
               "gpu__time_duration.sum"]

_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}


def launches(path, skip_prefix=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        if "spin_kernel" in name:  # torch.cuda._sleep of the stage-profiled eager steps
            continue
        if skip_prefix and name.startswith(skip_prefix):
            name = "[torch] " + name
        v = float(d["Metric Value"].replace(",", "")) * _US.get(d["Metric Unit"], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |")
    return "\n".join(out)


def _ncu_csv(rep, page, extra=()):
    txt = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(txt)))


def report(rep):
    rows = _ncu_csv(rep, "details")
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] in KEY_METRICS:
            per.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = _ncu_csv(rep, "raw")
    rh = raw[0]
    rk = rh.index("Kernel Name")
    cols = {m: rh.index(m) for m in RAW_METRICS if m in rh}
    rawper = []
    for r in raw[2:]:
        rawper.append((r[rk].split("(")[0], {m: r[c] for m, c in cols.items()}))
    out = []
    for i, ((kid, name), m) in enumerate(per.items()):
        out.append(f"### {name} (launch {kid})\n")
        for k in KEY_METRICS:
            if k in m:
                out.append(f"- {k}: {m[k]}")
        if i < len(rawper):
            for k, v in rawper[i][1].items():
                out.append(f"- `{k}`: {v}")
        out.append("")
    return "\n".join(out)


def traffic(rep):
    raw = _ncu_csv(rep, "raw")
    rh = raw[0]
    units = raw[1]
    rk = rh.index("Kernel Name")
    cr, cw = rh.index("dram__bytes_read.sum"), rh.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.defaultdict(list)
    for r in raw[2:]:
        b = float(r[cr].replace(",", "")) * scale.get(units[cr], 1) + \
            float(r[cw].replace(",", "")) * scale.get(units[cw], 1)
        name = r[rk].split("(")[0].split("<")[0].split(" ")[-1].split("::")[-1].replace("_kernel", "")
        per[name].append(b)
    return {k: sum(v) / len(v) for k, v in per.items()}


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        print(launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "at::"))
    elif cmd == "report":
        print(report(sys.argv[2]))
    elif cmd == "traffic":
        t = traffic(sys.argv[2])
        if len(sys.argv) > 4:
            try:
                cur = json.load(open(sys.argv[4]))
            except Exception:
                cur = {}
            cur.setdefault(sys.argv[3], {}).update(t)
            json.dump(cur, open(sys.argv[4], "w"), indent=1)
        print(json.dumps(t, indent=1))
