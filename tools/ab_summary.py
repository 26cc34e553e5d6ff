"""Summarise tools/gpu_ab.sh output: per variant and point, the ms per step of every rep."""
import glob
import json
import os
import sys

d = sys.argv[1]
res = {}
for f in sorted(glob.glob(os.path.join(d, "bench_*_*.json"))):
    v = os.path.basename(f)[6:-5].rsplit("_", 1)[0]
    try:
        line = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as ex:   # noqa: BLE001
        print(f, "unreadable", ex)
        continue
    for p, r in line.get("points", {}).items():
        res.setdefault(v, {}).setdefault(p, []).append(round(r["ms_per_step"] * 1e3, 1))
    if line.get("full_precision"):
        res.setdefault(v, {}).setdefault("full", []).append(round(line["full_precision"]["ms_per_step"] * 1e3, 1))
for v, pts in res.items():
    print(v, {p: (min(x), x) for p, x in pts.items()})
for f in sorted(glob.glob(os.path.join(d, "timeline_*.json"))):
    try:
        t = json.load(open(f))
    except Exception:   # noqa: BLE001
        continue
    for p, x in t.items():
        print(os.path.basename(f), p, "kernel", round(x["kernel_us"], 1), "fill", round(x["fill_us_mean"], 2),
              "core", x["smsp_warps_in_core_time_frac"], "zero", x["zero_core_time_split"])
