"""Per-source-line global memory sectors of an ncu report (L1 -> L2 sectors requested, ideal and
excessive), the memory-workload breakdown of a kernel: `python scripts/ncu_mem_lines.py rep [units]`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
cur = None
h = None
agg = {}
for r in csv.reader(src):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        h = {k: i for i, k in enumerate(r)}
        continue
    if h is None or r[2] != "-" or not r[0]:
        continue
    try:
        sec = float(r[h["L2 Theoretical Sectors Global"]] or 0)
        ideal = float(r[h["L2 Theoretical Sectors Global Ideal"]] or 0)
        exc = float(r[h["L2 Theoretical Sectors Global Excessive"]] or 0)
    except (ValueError, KeyError):
        continue
    if sec:
        agg[(cur, int(r[0]))] = (sec, ideal, exc, r[h["Access Operation"]] if "Access Operation" in h else "", r[1].strip()[:90])
tot = sum(v[0] for v in agg.values())
print(f"L2 sectors requested: {tot:.4g} = {tot * 32 / 1e9:.2f} GB ({tot * 32 / units:.2f} B per unit)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{k[0]}:{k[1]:5d} {v[0] * 32 / 1e9:7.3f} GB ideal {v[1] * 32 / 1e9:7.3f} exc {v[2] * 32 / 1e9:6.3f}  {v[4]}")
