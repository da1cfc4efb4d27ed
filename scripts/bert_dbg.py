import sys, torch
sys.path.insert(0, ".")
from paper_2312_10351_b200 import engine, zoo
torch.backends.cuda.matmul.allow_tf32 = False
model, ref_model, ids = zoo.build_bert()
sg = engine.compile(model, ids, device=0, profile_reps=2, dtype="bf16")
h, p = sg.run(ids.cuda())
with torch.no_grad():
    rh, rp = ref_model.cuda()(ids.cuda())
    bh, bp = ref_model.to(torch.bfloat16)(ids.cuda())
rel = lambda a, b: (torch.linalg.vector_norm(a.float().reshape(b.shape) - b) / torch.linalg.vector_norm(b)).item()
print("ours hidden", rel(h, rh), "pooled", rel(p, rp))
print("torch-bf16 hidden", rel(bh, rh), "pooled", rel(bp, rp))
print("pooled ours", p.flatten()[:8].tolist(), "\nref", rp.flatten()[:8].tolist())
