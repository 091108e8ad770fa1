"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel the launch count, total time and share (cold-cache, serialised
times: compare shares, not absolute values).

python profiles/launches.py <launches.csv> [title] > profiles/launches_<name>.md
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    agg = defaultdict(lambda: [0, 0.0])
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
                unit = d.get("Metric Unit", "nsecond")
                scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
                agg[k][0] += 1
                agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"# Launch list: {title}\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` over the bench command (cold-cache, "
          "serialised: compare shares)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k[:90]}` | {c} | {t:.3f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    main()
