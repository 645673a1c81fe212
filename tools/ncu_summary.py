"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep   > profiles/rNN_ncu_full.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.md

`full` reads a `--set full` capture (one row per profiled launch) and prints,
per launch: duration, DRAM bytes read/written (the `traffic` of the roofline),
DRAM throughput, tensor-pipe and SM utilisation, occupancy and resources.
`launches` reads a `--metrics gpu__time_duration.sum` launch list and prints
each kernel's count, mean duration and share of the profiled device time.
"""

from __future__ import annotations

import csv
import io
import re
import subprocess
import sys
from collections import OrderedDict

FULL = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("dram__bytes.sum.per_second", "dram_bw"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dsmem"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__t_bytes.sum", "l2_bytes"),
]


def short(name: str) -> str:
    name = re.sub(r"\(CUtensorMap_st.*", "", name)
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "")


def full(path: str) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    names = [m for m, _ in FULL if m in col]
    print(f"# ncu --set full summary: `{path.split('/')[-1]}`\n")
    print("| kernel | " + " | ".join(f"{lab} ({units[col[m]]})" for m, lab in FULL if m in col) + " |")
    print("|---" * (len(names) + 1) + "|")
    for r in data:
        vals = [r[col[m]] for m in names]
        print(f"| {short(r[col['Kernel Name']])} | " + " | ".join(vals) + " |")


def launches(path: str) -> None:
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Unit") == "us":
            ns *= 1e3
        elif r.get("Metric Unit") == "ms":
            ns *= 1e6
        agg.setdefault(short(r["Kernel Name"])[:90], []).append(ns)
    tot = sum(sum(v) for v in agg.values()) or 1.0
    print(f"# ncu launch list summary: `{path.split('/')[-1]}` ({sum(len(v) for v in agg.values())} launches)\n")
    print("| kernel | launches | mean us | share of profiled time |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")


def traffic(path: str, out: str) -> None:
    """profiles/ncu_traffic.json: dram read+write bytes per launch of each kernel
    (first capture of each name), the `traffic` term of bench.py's roofline."""
    import json

    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    import os

    res, seen = (json.load(open(out)) if os.path.exists(out) else {}), set()  # merge into the existing file
    for r in data:
        name = re.sub(r"<.*", "", short(r[col["Kernel Name"]])).split("::")[-1]
        if name in seen:
            continue
        b = sum(float(r[col[m]]) * scale[units[col[m]]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        seen.add(name)
        res[name] = {"dram_bytes": b, "us": float(r[col["gpu__time_duration.sum"]]), "capture": path.split("/")[-1]}
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1, sort_keys=True))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    else:
        {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
