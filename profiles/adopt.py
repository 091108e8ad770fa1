"""Copy summaries brought back by gpurun (gpurun_out/profiles/) into profiles/,
stamping the traffic JSON with the local git tree they were measured at (the
GPU box's copy of the repo has no .git).

python profiles/adopt.py <tag> <name>   e.g.  python profiles/adopt.py cfg2_final cfg2_r02
  gpurun_out/profiles/ncu_<tag>.md      -> profiles/ncu_<name>.md
  gpurun_out/profiles/sass_<tag>.txt    -> profiles/sass_<name>.txt
  gpurun_out/profiles/traffic_<tag>.json -> profiles/traffic_<cfg>.json (tree stamped)
"""
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(os.path.dirname(HERE), "gpurun_out", "profiles")


def main():
    tag, name = sys.argv[1], sys.argv[2]
    cfg = tag.split("_")[0]
    tree = subprocess.run(["git", "-C", HERE, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                          text=True).stdout.strip()
    for src, dst in ((f"ncu_{tag}.md", f"ncu_{name}.md"), (f"sass_{tag}.txt", f"sass_{name}.txt")):
        if os.path.exists(os.path.join(SRC, src)):
            shutil.copy(os.path.join(SRC, src), os.path.join(HERE, dst))
    tj = os.path.join(SRC, f"traffic_{tag}.json")
    if os.path.exists(tj):
        d = json.load(open(tj))
        d["tree"] = tree
        d["source"] = f"profiles/ncu_{name}.md"
        variant = sys.argv[3] if len(sys.argv) > 3 else ""
        with open(os.path.join(HERE, f"traffic_{cfg}{variant}.json"), "w") as f:
            json.dump(d, f, indent=1)
    print("adopted", tag, "->", name, "tree", tree)


if __name__ == "__main__":
    main()
