"""A/B of whole source trees on one box: python scripts/ab_trees.py MODEL DTYPE TREE... -- CFG...
Each TREE (a directory holding a built copy of the package) compiles MODEL with
each "grids:splitk" CFG (own tune cache per tree) and times the Opara and
sequential graphs (median of 3 x 200 replays), two interleaved rounds."""
import os
import subprocess
import sys

model, dtype = sys.argv[1], sys.argv[2]
sep = sys.argv.index("--")
trees, configs = sys.argv[3:sep], sys.argv[sep + 1:]
snippet = r'''
import sys, torch
sys.path.insert(0, ".")
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
''' % (model, dtype, configs)
for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
    for t in trees:
        env = dict(os.environ, OPARA_TUNE_CACHE=f"/tmp/ab_tune_{os.path.basename(t.rstrip('/')) or 'head'}.json")
        print(f"round {rnd} tree {t}", flush=True)
        subprocess.run([sys.executable, "-c", snippet], env=env, cwd=t)
