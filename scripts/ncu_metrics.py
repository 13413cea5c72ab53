"""Parse `ncu --csv --metrics ...` output (stdin): one line per (kernel, metric) -> `tag kernel metric value`."""
import csv
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('"'))]
if rows:
    h = {k: i for i, k in enumerate(rows[0])}
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        print(tag, r[h["Kernel Name"]].split("(")[0][:40], r[h["Metric Name"]], r[h["Metric Value"]])
