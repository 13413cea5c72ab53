"""Per-source-line stall samples / instructions / L2 sectors of one kernel in an ncu report:
`python scripts/ncu_src.py report.ncu-rep kernel_regex [top]`."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
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
    g = lambda k: float(r[h[k]] or 0) if k in h else 0.0
    agg[(cur, int(r[0]))] = (g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"),
                             g("L2 Theoretical Sectors Global"), r[1].strip()[:95])
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"stall samples {ts:.0f}, warp instructions {ti:.4g}, L2 sectors {sum(v[2] for v in agg.values()) * 32 / 1e9:.3f} GB")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / ts * 100:5.1f}% st {v[1] / ti * 100:5.1f}% in {v[2] * 32 / 1e9:6.3f} GB {k[0]}:{k[1]} {v[3]}")
