import signal
signal.signal(signal.SIGPIPE, signal.SIG_DFL)
import json, sys
name = sys.argv[1]
d = json.load(open(f"gpurun_out/profile_{name}.json"))  # name = MODEL_DTYPE[_bounded]
ops = d["ops"]
print(name, "sum isolated", round(sum(o["isolated_us"] for o in ops), 1), "cp", round(d["critical_path_us"], 1))
n = len(ops); preds = {i + 1: [] for i in range(n)}
for u, v in d["edges"]: preds[v + 1].append(u + 1)
dist = {}; par = {}
for v in range(1, n + 1):
    best = 0; bp = None
    for p in preds[v]:
        if dist[p] > best: best = dist[p]; bp = p
    dist[v] = best + ops[v - 1]["isolated_us"]; par[v] = bp
v = max(dist, key=dist.get); path = []
while v: path.append(v); v = par[v]
path.reverse()
only_cp = len(sys.argv) < 3
for v in (path if only_cp else range(1, n + 1)):
    o = ops[v - 1]
    if o["kind"] == 0: continue
    q = o["ints"]
    desc = f'{q.get("H")}x{q.get("W")} {q.get("Cin", q.get("C"))}->{q.get("Cout", "")} k{q.get("R", q.get("kh"))}x{q.get("S", q.get("kw"))}' if o["kind"] in (1, 2, 3) else str(q)
    tf = o["flops"] / (o["isolated_us"] * 1e-6) / 1e12 if o["isolated_us"] else 0
    print(f'  {v:4d} k{o["kind"]} {o["isolated_us"]:7.2f}us blocks {o["num_blocks"]:4d} thr {o["threads_per_block"]} regs {o["registers_per_thread"]} smem {o["shared_mem_per_block"]} {desc} {tf:.2f}TF')
