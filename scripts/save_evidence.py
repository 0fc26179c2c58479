"""Copy the JSON results of scripts/gpu_evidence.sh (gpurun_out/, scratch) into profiles/ (tracked), tagged by round.
usage: python scripts/save_evidence.py <tag>"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
src, dst = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def last_json(path):
    if not os.path.exists(path):
        return None
    for line in reversed(open(path).read().strip().split("\n")):
        line = line.strip()
        if line.startswith("{"):
            try:
                return json.loads(line)
            except json.JSONDecodeError:
                continue
    return None


for name, out in [("bench_c1", "bench_c1"), ("bench_c2", "bench_c2"), ("bench_c4", "bench_c4"), ("bench_c6", "bench_c6"),
                  ("bench_c3s", "bench_c3s"), ("serving", "serving_c5"), ("saturation", "saturation")]:
    d = last_json(os.path.join(src, name + ".log"))
    if d is None:
        print("missing", name)
        continue
    if name == "saturation" and os.path.exists(os.path.join(src, "host_nproc.txt")):
        d["host"] = open(os.path.join(src, "host_nproc.txt")).read().strip()
    p = os.path.join(dst, f"{out}_{tag}.json")
    json.dump(d, open(p, "w"), indent=1)
    print("wrote", p)
