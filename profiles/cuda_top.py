"""Summarise an `ncu --page source --csv --print-source cuda` export: the CUDA
source lines with the most warp-stall samples / L2 sectors (first kernel)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
data = []
for r in rows:
    if hdr is None and ("Source" in r or "# Line" in r):
        hdr = r
        continue
    if hdr is not None:
        if r and r[0] == "Kernel Name":
            if data:
                break
            continue
        if len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
num = lambda d, key: float((d.get(key) or "0").replace(",", "") or 0)
stall_key = next((h for h in (hdr or []) if h.startswith("Warp Stall Sampling (All")), None)
l2_key = next((h for h in (hdr or []) if h.startswith("L2 Theoretical Sectors Global") and "Excessive" not in h), None)
tot = sum(num(d, stall_key) for d in data) if stall_key else 0
print(f"lines {len(data)}  stall samples {tot:.0f}  columns: {stall_key} / {l2_key}")
for d in sorted(data, key=lambda d: -num(d, stall_key))[:k]:
    line = d.get("# Line", d.get("Line", "?"))
    print(f"{line:>6} {num(d, stall_key):9.0f} {100 * num(d, stall_key) / max(tot, 1):5.1f}% {num(d, l2_key):11.4g}  {d.get('Source', '').strip()[:100]}")
