"""Per-stage timeline of the fp32 tensor-core conv (conv_tc.cu) inside one
graph replay: CTA (0,0,0) of every conv records (OPARA_CONV_DEBUG=1) its entry,
setup done, every stage's gather issue / landed / MMA issue, accumulator
ready, reduction and exit.  Prints deltas in us per conv.

    OPARA_CONV_DEBUG=1 python scripts/conv_stages.py inception_v3 [--slot sequential|parallel]
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("OPARA_CONV_DEBUG", "1")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_10351_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("model")
ap.add_argument("dtype", nargs="?", default="f32")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--grids", default="bounded")
ap.add_argument("--splitk", default=None)
ap.add_argument("--slot", default="sequential")
ap.add_argument("--limit", type=int, default=200)
args = ap.parse_args()
bench.resolve_dtype(args)
model, _, x = bench.build_workload(args)
sg = engine.compile(model, x, device=0, dtype=args.dtype, bound_grids={"auto": "auto", "bounded": True,
                                                                         "full": False}[args.grids],
                    profile_reps=3, splitk=args.splitk)
xd = tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda()
slot = engine.SLOT_PARALLEL if args.slot == "parallel" else engine.SLOT_SEQUENTIAL
for _ in range(3):
    sg.run(xd, slot=slot)
torch.cuda.synchronize()
for b in sg.debug_ts.values():
    b.zero_()
sg.run(xd, slot=slot)
torch.cuda.synchronize()
rows = []
for k, buf in sorted(sg.debug_ts.items()):
    d = buf.cpu().numpy().astype(np.int64)
    if sg.engines.get(k) != 1 or d[0] == 0:
        continue
    q = sg.program.ops[k].ints
    t0 = d[0]
    us = lambda t: (t - t0) / 1e3 if t else float("nan")  # noqa: E731
    gi = [d[768 + i] for i in range(64) if d[768 + i]]
    la = [d[256 + i] for i in range(64) if d[256 + i]]
    mm = [d[512 + i] for i in range(64) if d[512 + i]]
    exit_ = max(d[w * 8 + 7] for w in range(10))
    prof = sg.profile[k]
    rows.append((k, q, prof, len(mm), us(d[1]), us(gi[0]) if gi else 0, us(la[0]) if la else 0,
                 us(mm[0]) if mm else 0, us(mm[-1]) if mm else 0,
                 (mm[-1] - mm[0]) / 1e3 / max(1, len(mm) - 1) if len(mm) > 1 else 0,
                 us(d[4]), us(d[5]), us(d[6]), us(exit_), sg._recs[k].variant, sg._recs[k].i[19]))
print(f"{'op':>4} {'shape':30} {'grid':>5} {'nkb':>4} | {'setup':>6} {'gath0':>6} {'land0':>6} {'mma0':>6} "
      f"{'mmaN':>6} {'/stage':>6} {'accum':>6} {'sync':>6} {'store':>6} {'exit':>6} | {'iso':>6}")
for (k, q, p, n, su, g0, l0, m0, mN, per, acc, syn, st, ex, var, sp) in rows[: args.limit]:
    shape = f"{q.get('H')}x{q.get('W')} {q['Cin']}>{q['Cout']} {q['R']}x{q['S']}/{q.get('sh', 1)} v{var}s{sp}"
    print(f"{k:4d} {shape:30} {p['num_blocks']:5d} {n:4d} | {su:6.2f} {g0:6.2f} {l0:6.2f} {m0:6.2f} {mN:6.2f} "
          f"{per:6.3f} {acc:6.2f} {syn:6.2f} {st:6.2f} {ex:6.2f} | {p['isolated_us']:6.2f}")

# per-stage detail (us after the first gather issue): gather issue / landed / MMA issue
for k in [r[0] for r in rows][:: max(1, len(rows) // 6)]:
    d = sg.debug_ts[k].cpu().numpy().astype(np.int64)
    g0 = d[768]
    f = lambda t: f"{(t - g0) / 1e3:5.2f}" if t else "  -  "  # noqa: E731
    print(f"op {k}: issue  " + " ".join(f(d[768 + i]) for i in range(24) if d[768 + i]))
    print(f"op {k}: landed " + " ".join(f(d[256 + i]) for i in range(24) if d[256 + i]))
    print(f"op {k}: mma    " + " ".join(f(d[512 + i]) for i in range(24) if d[512 + i]))

# hand-off between consecutive convs of the (sequential) replay: the previous
# conv's last CTA exit (first 96 CTAs recorded) -> this conv's first CTA entry,
# its setup done, its first gather issue (after griddepcontrol.wait) and first landed stage
print("\nhand-off (us): prev last exit -> entry0 / setup0 / gather0 / land0   (negative = before the predecessor ended)")
prev = None
for k, buf in sorted(sg.debug_ts.items()):
    d = buf.cpu().numpy().astype(np.int64)
    if sg.engines.get(k) != 1 or d[0] == 0:
        continue
    ent = [d[64 + 2 * c] for c in range(96) if d[64 + 2 * c]]
    ext = [d[65 + 2 * c] for c in range(96) if d[65 + 2 * c]]
    if prev is not None and prev[0] == k - 1:
        pe = prev[1]
        print(f"{k:4d} {(min(ent) - pe) / 1e3:7.2f} {(d[1] - pe) / 1e3:7.2f} {(d[768] - pe) / 1e3:7.2f} "
              f"{(d[256] - pe) / 1e3:7.2f}   last-CTA exit spread {(max(ext) - min(ext)) / 1e3:6.2f}")
    prev = (k, max(ext) if ext else d[0])

# split-K rank skew inside cluster (0, 0): accumulator ready / partial drained /
# past the cluster barrier, per rank, relative to the earliest rank's accumulator
print("\nrank skew (us, cluster (0,0)): op splits | accum-ready spread | drain (rank max) | barrier exit - last accum")
for k, buf in sorted(sg.debug_ts.items()):
    d = buf.cpu().numpy().astype(np.int64)
    if sg.engines.get(k) != 1 or d[0] == 0:
        continue
    st = [(d[2048 + 4 * z], d[2049 + 4 * z], d[2050 + 4 * z]) for z in range(8) if d[2048 + 4 * z]]
    if len(st) < 2:
        continue
    acc = [t[0] for t in st]
    print(f"{k:4d} {len(st):2d} | {(max(acc) - min(acc)) / 1e3:6.2f} | {max(t[1] - t[0] for t in st) / 1e3:6.2f} | "
          f"{(max(t[2] for t in st) - max(acc)) / 1e3:6.2f}")
