import sys, torch
sys.path.insert(0, ".")
from paper_2312_10351_b200 import engine, zoo
model, ref_model, ids = zoo.build_bert()
sg = engine.compile(model, ids, device=0, profile_reps=2, dtype="bf16", fuse_layernorm=True)
h, p = sg.run(ids.cuda())
hf = model.hf
pd = hf.pooler.dense
mine = torch.tanh(torch.nn.functional.linear(h.float().reshape(128, 768)[:1], pd.weight.cuda(), pd.bias.cuda()))
print("pooled vs recompute from our hidden:", (p.float().reshape(-1) - mine.reshape(-1)).abs().max().item())
last = sg.program.ops[-1]
print("pooler op engine", sg.engines.get(len(sg.program.ops) - 1), "in dtype", last.inputs[0].root()[0].dtype, "out", last.output.dtype)
print([(k, o.kind, o.ints.get("ln"), o.output.dtype) for k, o in enumerate(sg.program.ops)][-4:])
h2, p2 = sg.run(ids.cuda(), slot=engine.SLOT_SEQUENTIAL)
print("seq slot pooled diff:", (p2.float().reshape(-1) - mine.reshape(-1)).abs().max().item())
y = sg.run_eager(ids.cuda())
import numpy as np
print("eager:", "n/a")
