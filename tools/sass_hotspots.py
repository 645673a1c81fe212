"""Stall breakdown of one kernel from an ncu --set full report (SASS level).

    python tools/sass_hotspots.py gpurun_out/prof.ncu-rep k_causal_fwd [top]

Prints the kernel's warp-stall totals by reason and the top SASS instructions
by samples (with their dominant stall reason), with a window of the preceding
instructions so the hot spot can be mapped back to the source.
"""

import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"'))
# only the first kernel instance
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h, data = rows[0], rows[1:]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = {h[i]: 0 for i in stall_cols}
samples = []
for k, r in enumerate(data):
    try:
        s = int(r[si])
    except (ValueError, IndexError):
        continue
    per = {}
    for i in stall_cols:
        try:
            v = int(r[i])
        except ValueError:
            v = 0
        tot[h[i]] += v
        per[h[i]] = v
    samples.append((s, k, r[1].strip(), max(per, key=per.get) if s else ""))
allsum = sum(tot.values()) or 1
print(f"kernel {kern}: {allsum} stall samples")
for name, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {name:24s} {100 * v / allsum:5.1f}%")
print("\ntop instructions:")
for s, k, src, why in sorted(samples, reverse=True)[:top]:
    print(f"{100 * s / allsum:5.1f}%  [{k:5d}] {src[:70]:70s} {why}")
