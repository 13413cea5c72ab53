"""Summarise an ncu report (raw metrics + per-source-line instructions / stall samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
ntiles = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ("gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_active.max", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active")
for i, h in enumerate(hdr):
    if h in want or ("average_warps_issue_stalled" in h and float(vals[i] or 0) > 0.2):
        print(h, units[i], vals[i])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
cur = None; h2 = None; agg = {}
for r in csv.reader(src):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": h2 = r; continue
    if h2 is None or len(r) < 8 or r[2] != "-": continue
    try: st = float(r[4] or 0); ex = float(r[7] or 0)
    except ValueError: continue
    agg[(cur, int(r[0]))] = (st, ex, r[1].strip()[:95])
ts = sum(v[0] for v in agg.values()); te = sum(v[1] for v in agg.values())
print(f"instructions per unit: {te / ntiles:.0f}")
print("-- by instructions")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{v[1] / ntiles:7.0f} {v[0] / ts * 100:5.1f}%st {k[0]}:{k[1]} {v[2]}")
print("-- by stall samples")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:15]:
    print(f"{v[1] / ntiles:7.0f} {v[0] / ts * 100:5.1f}%st {k[0]}:{k[1]} {v[2]}")
