"""Dump per-op profile (demand + isolated time) and one traced replay of each
slot for a model, as JSON under gpurun_out/.

    python scripts/profile_ops.py MODEL [f32|bf16] [--bounded]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2312_10351_b200 import engine, zoo

name = sys.argv[1] if len(sys.argv) > 1 else "googlenet"
dtype = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "f32"
bounded = "--bounded" in sys.argv
if name == "bert_base":
    model, _, x = zoo.build_bert()
    dtype = "bf16"
else:
    model, x = zoo.build(name)
sg = engine.compile(model, x, device=0, dtype=dtype, bound_grids=bounded)
sg.run(x.cuda())
rows = []
for k, (op, p) in enumerate(zip(sg.program.ops, sg.profile)):
    rows.append({"id": k + 1, "kind": op.kind, "label": op.label, "ints": op.ints, "flops": op.flops,
                 "bytes": op.bytes_min, **p})
out = {"model": name, "dtype": dtype, "ops": rows, "edges": sg.program.edges,
       "trace_parallel": sg.trace(engine.SLOT_PARALLEL),
       "trace_sequential": sg.trace(engine.SLOT_SEQUENTIAL),
       "order": list(sg.schedule.order), "plan": {str(k): v for k, v in sg.plan.assignment.items()},
       "critical_path_us": sg.critical_path_us(),
       "lat_par_ms": sg.time(engine.SLOT_PARALLEL, iters=50).median_ms,
       "lat_seq_ms": sg.time(engine.SLOT_SEQUENTIAL, iters=50).median_ms}
Path("gpurun_out").mkdir(exist_ok=True)
tag = f"{name}_{dtype}{'_bounded' if bounded else ''}"
Path(f"gpurun_out/profile_{tag}.json").write_text(json.dumps(out))
print("ok", tag, "cp", round(sg.critical_path_us(), 1), "par", out["lat_par_ms"], "seq", out["lat_seq_ms"])
