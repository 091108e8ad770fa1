"""Does a concurrent host<->device copy slow the walk kernel? (e2e diagnosis)

python scripts/copy_interference.py [cfg]   -- walk device time alone, beside a
2 GiB D2H copy, beside a 2 GiB H2D copy, and beside a kernel that streams a
2 GiB device buffer into pinned host memory (zero-copy writes)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2010_04895_b200 as mhw  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = dict(bench.CONFIGS[name])
cfg["name"] = name
g = bench.build_graph(cfg)
sess = mhw.Session(g, bench.make_model(cfg), bench.make_config(cfg))
main = torch.cuda.Stream()
side = torch.cuda.Stream()
dev = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
host = torch.empty(2 << 30, dtype=torch.uint8).pin_memory()


def walk_ms(side_op=None, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if side_op:
            with torch.cuda.stream(side):
                side_op()
        sess.run(main.cuda_stream)
        torch.cuda.synchronize()
        out.append(sess.stats().walk_seconds * 1e3)
    return min(out)


sess.run(main.cuda_stream)
torch.cuda.synchronize()
print(f"{name} walk alone          {walk_ms():.2f} ms")
print(f"{name} walk + 2 GiB D2H    {walk_ms(lambda: host.copy_(dev, non_blocking=True)):.2f} ms")
print(f"{name} walk + 2 GiB H2D    {walk_ms(lambda: dev.copy_(host, non_blocking=True)):.2f} ms")
hview = host.view(torch.int32)
print(f"{name} walk + zero-copy kernel writes {walk_ms(lambda: hview.copy_(dev.view(torch.int32), non_blocking=True)):.2f} ms")
