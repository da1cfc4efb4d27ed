"""A/B of the bounded-grid SM-share scale: python scripts/ab_scale.py MODEL:DTYPE:SPLITK ... -- S1 S2 ...
(same tune cache per model, Opara + sequential graph medians of 3 x 200 replays, L2 warm)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import argparse  # noqa: E402

import bench  # noqa: E402
from paper_2312_10351_b200 import engine  # noqa: E402

sep = sys.argv.index("--")
specs, scales = sys.argv[1:sep], [float(v) for v in sys.argv[sep + 1:]]
for spec in specs:
    name, dtype, splitk = spec.split(":")
    os.environ["OPARA_TUNE_CACHE"] = f"/tmp/ab_scale_{name}_{dtype}.json"
    m, _, x = bench.build_workload(argparse.Namespace(model=name, dtype=dtype, batch=1))
    xd = tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda()
    for rnd in range(2):
        for sc in scales:
            sg = engine.ScheduledGraph(engine.lower(m, x, dtype), 0, profile_reps=5, bound_grids=True,
                                       splitk=splitk, bound_scale=sc)
            sg.run(xd)
            par = sorted(sg.time(engine.SLOT_PARALLEL, iters=200).median_ms for _ in range(3))[1]
            print(f"{name} {dtype} {splitk} round {rnd} scale {sc}: par {par:.4f}", flush=True)
            sg.close()
