"""A/B of build-flag variants on one box: python scripts/ab_flags.py MODEL DTYPE
"bounded:pull" "full:push" -- "" "-DFOO" ... ; each flag set is built into its own
object dir, the model compiled with each (grids, split-K) config (shared tune
cache, so tile choices match) and timed (median of 3 x 200 replays)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
model, dtype = sys.argv[1], sys.argv[2]
sep = sys.argv.index("--")
configs, flags = sys.argv[3:sep], sys.argv[sep + 1:]
env0 = dict(os.environ, OPARA_TUNE_CACHE="/tmp/ab_tune.json")
snippet = r'''
import sys, torch
sys.path.insert(0, "%s")
import bench, argparse
from paper_2312_10351_b200 import engine
a = argparse.Namespace(model="%s", dtype="%s", batch=1)
m, _, x = bench.build_workload(a)
for cfg in %r:
    g, sk = cfg.split(":")
    sg = engine.compile(m, x, device=0, dtype=a.dtype, bound_grids=g == "bounded", splitk=sk)
    xd = tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda()
    sg.run(xd)
    par = sorted(sg.time(engine.SLOT_PARALLEL, iters=200).median_ms for _ in range(3))[1]
    seq = sorted(sg.time(engine.SLOT_SEQUENTIAL, iters=200).median_ms for _ in range(3))[1]
    print("   ", cfg, "par %%.4f seq %%.4f x %%.3f" %% (par, seq, seq / par), flush=True)
''' % (ROOT, model, dtype, configs)
for rnd in range(2):
    for f in flags:
        env = dict(env0, OPARA_NVCC_FLAGS=f)
        subprocess.run([sys.executable, "-m", "paper_2312_10351_b200.build"], env=env, cwd=ROOT, check=True,
                       capture_output=True)
        print(f"round {rnd} flags [{f}]", flush=True)
        subprocess.run([sys.executable, "-c", snippet], env=env, cwd=ROOT)
