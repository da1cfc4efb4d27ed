"""Dump per-op profile (demand + isolated time) and one traced replay of each
slot for a model, as JSON under gpurun_out/."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2312_10351_b200 import engine, zoo

name = sys.argv[1] if len(sys.argv) > 1 else "googlenet"
model, x = zoo.build(name)
sg = engine.compile(model, x, device=0)
sg.run(x.cuda())
rows = []
for k, (op, p) in enumerate(zip(sg.program.ops, sg.profile)):
    rows.append({"id": k + 1, "kind": op.kind, "label": op.label, "ints": op.ints, "flops": op.flops,
                 "bytes": op.bytes_min, **p})
out = {"model": name, "ops": rows, "edges": sg.program.edges,
       "trace_parallel": sg.trace(engine.SLOT_PARALLEL),
       "trace_sequential": sg.trace(engine.SLOT_SEQUENTIAL),
       "order": list(sg.schedule.order), "plan": {str(k): v for k, v in sg.plan.assignment.items()},
       "critical_path_us": sg.critical_path_us()}
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/profile_{name}.json").write_text(json.dumps(out))
print("ok", name, sg.critical_path_us())
