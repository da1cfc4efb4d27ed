"""Per-phase timing of the bf16 tensor-core conv/GEMM kernel inside one graph
replay (diagnostic build: OPARA_NVCC_FLAGS=-DOPARA_PHASE_PROBE).  CTA (0,0,0)
of each launch records entry, post-griddepcontrol.wait, first/last MMA issue,
accumulator ready and exit; printed as deltas in us, grouped by GEMM shape.

    OPARA_NVCC_FLAGS=-DOPARA_PHASE_PROBE python -m paper_2312_10351_b200.build
    python scripts/phase_probe.py bert_base bf16 [--slot parallel|sequential]
"""
import argparse
import ctypes
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2312_10351_b200 import _lib, engine

ap = argparse.ArgumentParser()
ap.add_argument("model")
ap.add_argument("dtype", nargs="?", default="bf16")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--grids", default="full")
ap.add_argument("--slot", default="parallel")
ap.add_argument("--splitk", default=None)
args = ap.parse_args()
lib = _lib.lib()
fn = lib.opara_debug_phase_read
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros((4096, 12), dtype=np.uint64)
model, _, x = bench.build_workload(args)
sg = engine.compile(model, x, device=0, dtype=args.dtype, bound_grids=args.grids == "bounded", profile_reps=3,
                    splitk=args.splitk)
xd = tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda()
slot = engine.SLOT_PARALLEL if args.slot == "parallel" else engine.SLOT_SEQUENTIAL
for _ in range(3):
    sg.run(xd, slot=slot)
import torch
torch.cuda.synchronize()
fn(buf.ctypes.data, 4096, 1)
sg.run(xd, slot=slot)
torch.cuda.synchronize()
n = fn(buf.ctypes.data, 4096, 1)
rec = buf[:n].astype(np.int64)
groups = defaultdict(list)
for r in rec:
    m, cout, k = r[8] >> 40, (r[8] >> 20) & 0xFFFFF, r[8] & 0xFFFFF
    ctas, bn, nkb, flags = r[9] >> 32, (r[9] >> 24) & 0xFF, (r[9] >> 8) & 0xFFFF, r[9] & 0xFF
    mode = ("push" if flags & 0x80 else "l2" if flags & 0x40 else "pull") + \
        (" ln_in" if flags & 0x20 else "") + (" res_stats" if flags & 0x10 else "")
    t = r[:8].copy()
    for q in (5, 6):       # paths without the probe: carry the previous stamp
        if t[q] == 0:
            t[q] = t[q - 1]
    d = np.diff(t) / 1e3
    if r[10] and r[11]:   # staging split: TMEM->partials loop | CTA/cluster barrier | dealloc etc.
        d = np.concatenate([d, [(r[10] - t[4]) / 1e3, (r[11] - r[10]) / 1e3, (t[5] - r[11]) / 1e3]])
    else:
        d = np.concatenate([d, [0, 0, 0]])
    groups[(int(m), int(cout), int(k), int(ctas), int(bn), int(nkb), int(flags & 0x0F), mode)].append(d)
print(f"{n} launches; phases (us): wait | first stage | mma loop | accum | stage partials | peers ready | "
      "reduce+store || stage: loop | barrier | rest ")
for key, ds in sorted(groups.items(), key=lambda kv: -len(kv[1])):
    d = np.median(np.stack(ds), axis=0)
    print(f"M{key[0]} Cout{key[1]} K{key[2]} ctas{key[3]} BN{key[4]} nkb{key[5]} split{key[6]} {key[7]} x{len(ds)}: "
          + " | ".join(f"{v:5.2f}" for v in d[:7]) + f" | {d[1:7].sum():5.2f} || "
          + " | ".join(f"{v:5.2f}" for v in d[7:]))
