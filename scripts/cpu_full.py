"""One full reference generate_walks (oracle/_ref, unmodified engine.cpp:157-234)
on a BASELINE config with threads = all host cores; writes
gpurun_out/cpu_full_<cfg>.json (copied to profiles/ when committed).
bench.py reports it as cpu_baseline.full beside its bounded sample.

python scripts/cpu_full.py cfg2
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cfg = dict(bench.CONFIGS[name])
    cfg["name"] = name
    threads = bench.cpu_threads()
    t0 = time.time()
    hg, rg, rm, wc, _ = bench.reference_sample(cfg, threads, 1)
    setup = time.time() - t0
    _, _, st = rm.generate_walks(wc, threads=threads, n_nodes=hg.n, with_rows=False)
    cpu = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    out = {"config": name, "workload": cfg["workload"], "threads": threads, "cpu": cpu,
           "call": "generate_walks (engine.cpp:157-234), unmodified, one call, all walkers",
           "seconds": st["seconds"], "steps": st["steps"], "walks": st["walks"],
           "steps_per_sec": st["steps"] / st["seconds"], "reference_steps_per_sec": st["steps_per_sec"],
           "init_thread_seconds": st["init_seconds"], "host_graph_seconds": setup}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"cpu_full_{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
