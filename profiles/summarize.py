"""Summarise ncu captures into profiles/ (markdown + the per-launch DRAM
traffic JSON bench.py reports as roofline.traffic).

python profiles/summarize.py <report.ncu-rep> <config-name> [<launches.csv>]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sectors.sum", "L2 sectors (all)"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read"),
    ("lts__t_sectors_srcunit_tex_op_atom.sum", "L2 sectors atomic"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 sectors write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local-memory load sectors"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return x * scale


def main():
    rep, name = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    lines = [f"# ncu summary: {name} (`{os.path.basename(rep)}`, --set full, --clock-control none)", ""]
    traffic = {}
    for d in raw(rep):
        kname = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## `{kname[:90]}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in METRICS:
            if m in d:
                v, u = d[m]
                lines.append(f"| {label} (`{m}`) | {v} {u} |")
        lines.append("")
        if "dram__bytes_read.sum" in d:
            rd, wr = to_bytes(*d["dram__bytes_read.sum"]), to_bytes(*d["dram__bytes_write.sum"])
            dur = float(d["gpu__time_duration.sum"][0].replace(",", "")) if "gpu__time_duration.sum" in d else None
            if dur is not None:
                dur *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(
                    d["gpu__time_duration.sum"][1], 1.0)
            hit = float(d["lts__t_sector_hit_rate.pct"][0]) if "lts__t_sector_hit_rate.pct" in d else None
            traffic[kname] = {"total": rd + wr, "read": rd, "write": wr, "ms": dur, "l2_hit_pct": hit}
    if launches:
        rows = list(csv.reader(open(launches)))
        hdr = None
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows:
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                dd = dict(zip(hdr, r))
                if dd.get("Metric Name") == "gpu__time_duration.sum":
                    k = dd["Kernel Name"]
                    k = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
                    agg[k][0] += 1
                    agg[k][1] += float(dd["Metric Value"].replace(",", ""))
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (gpu__time_duration.sum, cold-cache serialised: compare shares)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k[:80]}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
        lines.append("")
    with open(os.path.join(HERE, f"ncu_{name}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    walk = [v for k, v in traffic.items() if "k_walk" in k]
    init = [v for k, v in traffic.items() if "k_init_all" in k]
    cfg = name.split("_")[0]
    if walk:
        commit = subprocess.run(["git", "-C", HERE, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                                text=True).stdout.strip() or None
        w = walk[0]
        with open(os.path.join(HERE, f"traffic_{cfg}.json"), "w") as f:
            json.dump({"kernel": "k_walk", "dram_bytes_per_launch": w["total"],
                       "dram_read_bytes_per_launch": w["read"], "dram_write_bytes_per_launch": w["write"],
                       "ncu_ms": w["ms"], "l2_hit_pct": w["l2_hit_pct"],
                       "init_kernel_dram_bytes_per_launch": init[0]["total"] if init else None,
                       "source": f"profiles/ncu_{name}.md", "tree": commit,
                       "env": {k: v for k, v in os.environ.items() if k.startswith("MHW_")}}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
