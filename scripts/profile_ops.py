"""Dump per-op profile (demand + isolated time) and one traced replay of each
slot for a model, as JSON under gpurun_out/profile_<model>_<dtype>.json.

    python scripts/profile_ops.py MODEL [DTYPE] [--batch B] [--grids auto|bounded|full]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2312_10351_b200 import engine

ap = argparse.ArgumentParser()
ap.add_argument("model")
ap.add_argument("dtype", nargs="?", default="f32")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--grids", default="auto")
args = ap.parse_args()
bench.resolve_dtype(args)
model, _, x = bench.build_workload(args)
sg = engine.compile(model, x, device=0, dtype=args.dtype,
                    bound_grids={"auto": "auto", "bounded": True, "full": False}[args.grids])
sg.run(tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda())
rows = []
for k, (op, p) in enumerate(zip(sg.program.ops, sg.profile)):
    rows.append({"id": k + 1, "kind": op.kind, "label": op.label, "ints": op.ints, "flops": op.flops,
                 "bytes": op.bytes_min, "engine": sg.engines.get(k), "tuning": sg.tuning.get(k), **p})
out = {"model": args.model, "dtype": args.dtype, "grids": "bounded" if sg.bound_grids else "full", "ops": rows,
       "edges": sg.program.edges, "trace_parallel": sg.trace(engine.SLOT_PARALLEL),
       "trace_sequential": sg.trace(engine.SLOT_SEQUENTIAL), "order": list(sg.schedule.order),
       "plan": {str(k): v for k, v in sg.plan.assignment.items()}, "critical_path_us": sg.critical_path_us(),
       "lat_par_ms": sg.time(engine.SLOT_PARALLEL, iters=50).median_ms,
       "lat_seq_ms": sg.time(engine.SLOT_SEQUENTIAL, iters=50).median_ms}
Path("gpurun_out").mkdir(exist_ok=True)
tag = f"{args.model}_{args.dtype}"
Path(f"gpurun_out/profile_{tag}.json").write_text(json.dumps(out))
print("ok", tag, out["grids"], "cp", round(sg.critical_path_us(), 1), "par", out["lat_par_ms"], "seq", out["lat_seq_ms"])
