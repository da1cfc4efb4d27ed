"""One traced replay of each slot: per-kernel [start, end] (globaltimer, ns)
printed in start order, for reading where a graph's latency goes.

    python scripts/trace_dump.py MODEL [DTYPE] [BATCH]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import argparse

import bench
from paper_2312_10351_b200 import engine

ap = argparse.ArgumentParser()
ap.add_argument("model")
ap.add_argument("dtype", nargs="?", default="f32")
ap.add_argument("batch", nargs="?", type=int, default=1)
args = ap.parse_args()
args.grids = "auto"
model, _, x = bench.build_workload(args)
sg = engine.compile(model, x, device=0, dtype=args.dtype, bound_grids="auto", profile_reps=5)
sg.run(tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda())
for slot, name in ((engine.SLOT_PARALLEL, "parallel"), (engine.SLOT_SEQUENTIAL, "sequential")):
    tr = sg.trace(slot)
    tr = sorted((s, e, nid) for nid, s, e in tr if sg.program.ops[nid - 1].kind != 0)
    print(f"== {name}: span {(max(e for _, e, _ in tr) - min(s for s, _, _ in tr)) / 1e3:.2f} us, "
          f"stream of node: plan {'opara' if slot == 0 else 'single'}")
    for s, e, nid in tr[:60]:
        op = sg.program.ops[nid - 1]
        print(f"  {s / 1e3:8.2f} {e / 1e3:8.2f} ({(e - s) / 1e3:6.2f})  node {nid:4d} {op.name:10s} "
              f"stream {sg.plan.assignment[nid] if slot == 0 else 0:3d} iso {sg.profile[nid - 1]['isolated_us']:.2f}")
