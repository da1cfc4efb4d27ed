import signal
signal.signal(signal.SIGPIPE, signal.SIG_DFL)
"""Critical-path breakdown of a profiled model (gpurun_out/profile_<tag>.json
from scripts/profile_ops.py): per op kind, kernels and microseconds on the
longest isolated-time path, plus totals over all ops."""
import collections
import json
import sys

d = json.load(open(f"gpurun_out/profile_{sys.argv[1]}.json"))
ops = d["ops"]
n = len(ops)
preds = {i + 1: [] for i in range(n)}
for u, v in d["edges"]:
    preds[v + 1].append(u + 1)
dist, par = {}, {}
for v in range(1, n + 1):
    best, bp = 0.0, None
    for p in preds[v]:
        if dist[p] > best:
            best, bp = dist[p], p
    dist[v] = best + ops[v - 1]["isolated_us"]
    par[v] = bp
v = max(dist, key=dist.get)
path = []
while v:
    path.append(v)
    v = par[v]
names = {0: "nop", 1: "conv/gemm", 2: "maxpool", 3: "avgpool", 4: "gap", 5: "linear", 6: "add", 7: "layernorm",
         9: "embedding", 10: "attention", 11: "copy", 12: "fm", 13: "dwconv", 14: "relu", 16: "field_emb",
         17: "first_order", 18: "pack_input"}
cp = collections.defaultdict(lambda: [0, 0.0])
tot = collections.defaultdict(lambda: [0, 0.0])
for v in path:
    o = ops[v - 1]
    cp[names[o["kind"]]][0] += 1
    cp[names[o["kind"]]][1] += o["isolated_us"]
for o in ops:
    tot[names[o["kind"]]][0] += 1
    tot[names[o["kind"]]][1] += o["isolated_us"]
print(f"{sys.argv[1]}: critical path {dist[max(dist, key=dist.get)]:.1f} us over {len(path)} ops; "
      f"sum of all ops {sum(o['isolated_us'] for o in ops):.1f} us; par {d.get('lat_par_ms')} ms seq {d.get('lat_seq_ms')} ms")
print(f"{'kind':12s} {'cp n':>5s} {'cp us':>8s} {'cp avg':>7s} | {'all n':>6s} {'all us':>8s}")
for k in sorted(tot, key=lambda k: -cp[k][1]):
    c, t = cp[k], tot[k]
    print(f"{k:12s} {c[0]:5d} {c[1]:8.1f} {c[1] / max(1, c[0]):7.2f} | {t[0]:6d} {t[1]:8.1f}")
