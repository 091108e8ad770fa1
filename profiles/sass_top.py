"""Summarise an ncu --page source --print-source sass CSV: top instructions by
L2 sectors and by warp-stall samples (used to read profiles/ captures)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break  # first kernel of the capture only
    if len(r) == len(hdr) and r != hdr:
        data.append(dict(zip(hdr, r)))
num = lambda d, k: float(d.get(k, "0").replace(",", "") or 0)
tot_s = sum(num(d, "Warp Stall Sampling (All Samples)") for d in data)
tot_l2 = sum(num(d, "L2 Theoretical Sectors Global") for d in data)
print(f"instructions {len(data)}  stall samples {tot_s:.0f}  L2 theoretical sectors {tot_l2:.3e}")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("--- by L2 sectors")
for i, d in sorted(enumerate(data), key=lambda x: -num(x[1], "L2 Theoretical Sectors Global"))[:k]:
    print(f"{i:5d} {num(d,'L2 Theoretical Sectors Global'):12.4g} {num(d,'Warp Stall Sampling (All Samples)'):8.0f} {num(d,'Instructions Executed'):12.4g}  {d['Source'].strip()[:70]}")
print("--- by stall samples")
for i, d in sorted(enumerate(data), key=lambda x: -num(x[1], "Warp Stall Sampling (All Samples)"))[:k]:
    print(f"{i:5d} {num(d,'L2 Theoretical Sectors Global'):12.4g} {num(d,'Warp Stall Sampling (All Samples)'):8.0f} {num(d,'Instructions Executed'):12.4g}  {d['Source'].strip()[:70]}")
