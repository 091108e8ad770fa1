"""Stall / utilisation digest of one kernel capture: python profiles/stall_top.py raw.csv src.csv [n]
(raw.csv: ncu -i rep --page raw --csv; src.csv: ncu -i rep --page source --csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
b = {h: v for h, v in zip(rows[0], rows[2])}
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "lts__t_requests_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
          "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
          "lts__t_sectors_srcunit_tex_op_write.sum", "launch__registers_per_thread", "smsp__inst_executed.sum"]:
    print(f"{k:70s} {b.get(k)}")
rows = list(csv.reader(open(sys.argv[2])))
print(rows[0][1])
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
num = lambda d, k: float((d.get(k, "0") or "0").replace(",", "") or 0)
tot = sum(num(d, "Warp Stall Sampling (All Samples)") for d in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("samples", tot, " ".join(f"{s[6:]}={100 * sum(num(d, s) for d in data) / tot:.1f}%"
                               for s in sorted(stalls, key=lambda s: -sum(num(d, s) for d in data))[:5]))
n = int(sys.argv[3]) if len(sys.argv) > 3 else 14
for i, d in sorted(enumerate(data), key=lambda x: -num(x[1], "Warp Stall Sampling (All Samples)"))[:n]:
    print(f"{i:5d} {100 * num(d, 'Warp Stall Sampling (All Samples)') / tot:5.1f}% execs {num(d, 'Instructions Executed'):9.3g} "
          f"lanes {num(d, 'Avg. Threads Executed'):4.1f}  {d['Source'].strip()[:70]}")
print("avg lanes:", sum(num(d, "Thread Instructions Executed") for d in data) / sum(num(d, "Instructions Executed") for d in data))
