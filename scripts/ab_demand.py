"""A/B of the demand Alg. 2 sees: measured smem vs TMEM-folded co-resident smem
(OPARA_DEMAND=coresident).  Per model: one compile per mode (shared tune cache,
so the tiles match), then the Opara / dfs / wavefront orders of the same plan,
each as a real CUDA graph timed with L2 flushed (median of 3 x 200)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import argparse  # noqa: E402

import bench  # noqa: E402
from paper_2312_10351_b200 import engine  # noqa: E402
from paper_2312_10351_b200.order import LaunchSchedule, make_order  # noqa: E402

os.environ["OPARA_TUNE_CACHE"] = "/tmp/ab_demand_tune.json"
for spec in sys.argv[1:]:
    model_name, dtype = spec.split(":")
    a = argparse.Namespace(model=model_name, dtype=dtype, batch=1)
    m, _, x = bench.build_workload(a)
    for rnd in range(2):
        for mode in ("", "coresident"):
            os.environ["OPARA_DEMAND"] = mode
            sg = engine.compile(m, x, device=0, dtype=dtype, bound_grids=True, splitk="auto", profile_reps=5)
            xd = tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda()
            sg.run(xd)
            res = {}
            for slot, p in enumerate(("opara", "dfs", "wavefront")):
                sched = make_order(sg.graph, p, sg.gpu_config)
                sg.capture(10 + slot, sg.plan, LaunchSchedule(tuple(sched.order), p, None))
                res[p] = sorted(sg.time(10 + slot, warmup=10, iters=200, flush_l2=True).median_ms
                                for _ in range(3))[1]
            best = min(res["dfs"], res["wavefront"])
            print(f"{model_name} {dtype} round {rnd} demand={mode or 'measured':10s} " +
                  " ".join(f"{k} {v:.4f}" for k, v in res.items()) + f"  opara/best {res['opara'] / best:.3f}",
                  flush=True)
            sg.close()
