"""Print the key fields of bench.py JSON lines found in the given logs."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        r = d.get("roofline") or {}
        c = d.get("config") or {}
        e = d.get("e2e") or {}
        print(f"{path}: value={d.get('value'):.4g} ms/step={d.get('ms_per_step'):.2f} "
              f"kernel_ms={r.get('kernel_ms', 0):.2f} frac={r.get('frac', 0):.3f} "
              f"e2e={e.get('value') or 0:.4g} inits={c.get('slot_inits')} retries={c.get('chain_retries')} "
              f"clocks={d.get('clocks')} cpu={d.get('cpu_baseline', {}).get('value')}")
