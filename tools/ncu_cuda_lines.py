"""Warp-stall samples per CUDA source line of one kernel in an ncu report (needs -lineinfo):

    python tools/ncu_cuda_lines.py report.ncu-rep <kernel-regex> [top_n]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, si = None, None, None
agg, src = collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= si:
        continue
    try:
        ln, s = int(r[0]), int(r[si])
    except ValueError:
        continue
    agg[(fname, ln)] += s
    src[(fname, ln)] = r[1].strip()[:90]
tot = sum(agg.values()) or 1
for k, v in agg.most_common(top_n):
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]}  {src[k]}")
