"""Branch-overlap evidence (the nsys-timeline substitute: nsys is not in the
image): one traced replay of the Opara graph and of the sequential graph,
kernel start/end from %globaltimer, summarised into profiles/<tag>_timeline.md
(span, kernels running concurrently, busy time with >= 2 kernels in flight,
and an ASCII Gantt of the first kernels by plan stream).

    python scripts/timeline.py MODEL [DTYPE] [--batch B]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2312_10351_b200 import engine

ap = argparse.ArgumentParser()
ap.add_argument("model")
ap.add_argument("dtype", nargs="?", default="f32")
ap.add_argument("--batch", type=int, default=1)
args = ap.parse_args()
args.grids = "auto"
model, _, x = bench.build_workload(args)
sg = engine.compile(model, x, device=0, dtype=args.dtype, bound_grids="auto")
sg.run(tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda())


def stats(tr):
    ev = sorted((s, e) for _, s, e in tr)
    span = max(e for _, e in ev) - min(s for s, _ in ev)
    pts = sorted([(s, 1) for s, _ in ev] + [(e, -1) for _, e in ev])
    cur = peak = 0
    multi = 0
    last = pts[0][0]
    for t, d in pts:
        if cur >= 2:
            multi += t - last
        cur += d
        peak = max(peak, cur)
        last = t
    busy = sum(e - s for s, e in ev)
    return span, peak, multi, busy


lines = [f"# Kernel timeline — {args.model} {args.dtype} batch {args.batch}\n",
         "One replay of each captured graph with per-kernel `%globaltimer` probes (first block start "
         "after the PDL wait, last warp end; `opara_exec_trace`, warm replays first). "
         f"Grids: {'bounded' if sg.bound_grids else 'full'}, split-K: {sg.splitk}.\n",
         "| graph | span us | sum of kernel us | peak concurrent kernels | us with >= 2 kernels running |",
         "|---|---:|---:|---:|---:|"]
traces = {}
for slot, name in ((engine.SLOT_PARALLEL, "Opara (multi-stream)"), (engine.SLOT_SEQUENTIAL, "sequential")):
    tr = [t for t in sg.trace(slot) if sg.program.ops[t[0] - 1].kind != 0]
    traces[name] = tr
    span, peak, multi, busy = stats(tr)
    lines.append(f"| {name} | {span / 1e3:.1f} | {busy / 1e3:.1f} | {peak} | {multi / 1e3:.1f} |")
tr = sorted(traces["Opara (multi-stream)"], key=lambda t: t[1])[:48]
t0, t1 = tr[0][1], max(e for _, _, e in tr)
width = 100
lines.append(f"\nFirst {len(tr)} kernels of the Opara replay ({(t1 - t0) / 1e3:.1f} us, one column = "
             f"{(t1 - t0) / width / 1e3:.2f} us), one row per kernel, `s<stream>`:\n\n```")
for nid, s, e in tr:
    a = int((s - t0) / (t1 - t0) * width)
    b = max(a + 1, int((e - t0) / (t1 - t0) * width))
    lines.append(f"s{sg.plan.assignment[nid]:<3d} {sg.program.ops[nid - 1].name:10s} |" + " " * a + "#" * (b - a))
lines.append("```")
out = Path("gpurun_out") / f"{os.environ.get('OPARA_ROUND', 'r02')}_{args.model}_{args.dtype}_timeline.md"   # copied into profiles/
out.write_text("\n".join(lines) + "\n")
print("\n".join(lines[:8]))
