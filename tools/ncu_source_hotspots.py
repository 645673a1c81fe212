"""Summarise `ncu --page source --csv --print-source=cuda,sass` output: stall samples per CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
stats = []
fname = None
h = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        si = h.index("Warp Stall Sampling (All Samples)")
        ii = h.index("Instructions Executed")
        continue
    if h is None or not r[0] or not r[0].isdigit():
        continue
    try:
        stats.append((int(r[si]), int(r[ii]), fname, int(r[0]), r[1].strip()))
    except ValueError:
        pass
tot = sum(s[0] for s in stats) or 1
for s, ins, f, ln, src in sorted(stats, reverse=True)[:top_n]:
    print("%5.1f%% inst=%9d %s:%d  %s" % (100 * s / tot, ins, f, ln, src[:80]))
