"""Whole-kernel durations (first block start -> last warp end, %globaltimer
trace probes) of every op in one replay, for split-K reduction modes side by
side: python scripts/op_durations.py MODEL DTYPE --modes push pull [--grids full]"""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2312_10351_b200 import engine

ap = argparse.ArgumentParser()
ap.add_argument("model")
ap.add_argument("dtype", nargs="?", default="bf16")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--grids", default="full")
ap.add_argument("--modes", nargs="+", default=["push", "pull"])
args = ap.parse_args()
model, _, x = bench.build_workload(args)
res = {}
for mode in args.modes:
    sg = engine.compile(model, x, device=0, dtype=args.dtype, bound_grids=args.grids == "bounded", splitk=mode)
    xd = tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda()
    sg.run(xd)
    per = defaultdict(list)
    for slot, name in ((engine.SLOT_SEQUENTIAL, "seq"), (engine.SLOT_PARALLEL, "par")):
        tr = sg.trace(slot)
        for nid, s, e in tr:
            op = sg.program.ops[nid - 1]
            key = (op.label.rstrip("_0123456789") or op.label, tuple(sorted(op.ints.items()))[:6])
            per[(name, op.label.split("_")[0], str(op.ints.get("Cin", "")) + "->" + str(op.ints.get("Cout", "")))].append((e - s) / 1e3)
    res[mode] = per
    print(mode, "par", sg.time(engine.SLOT_PARALLEL, iters=50).median_ms, "seq", sg.time(engine.SLOT_SEQUENTIAL, iters=50).median_ms)
keys = sorted(set(k for per in res.values() for k in per))
for k in keys:
    print(k, " ".join(f"{m}: {np.median(res[m][k]):6.2f} us (n={len(res[m][k])})" for m in args.modes if k in res[m]))
