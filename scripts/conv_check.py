"""Compare one conv shape (tc vs simt vs fp64) and print error stats."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch
from test_gpu_kernels import Wrap
from paper_2312_10351_b200 import engine
cin, cout, k, s, p, hw = (int(v) for v in sys.argv[1:7])
torch.manual_seed(0)
m = Wrap(cin, cout, k, s, p, hw).eval()
x = torch.randn(1, 3, hw, hw)
with torch.no_grad():
    ref = m.double()(x.double()).float()
    refbody = m.body(m.stem(x.double())).float()
m = m.float()
for eng in ("tc", "simt"):
    sg = engine.compile(m, x, device=0, profile_reps=1, conv_engine=eng)
    y = sg.run(x.cuda()).permute(0, 3, 1, 2).cpu()
    rel = ((y - ref).norm() / ref.norm()).item()
    print(eng, "rel", rel, [ (o.kind, pr["num_blocks"]) for o, pr in zip(sg.program.ops, sg.profile)])
    # body conv output directly
    body_t = [t for t in sg.program.tensors if t.tid == sg.program.ops[1].output.tid][0]
    yb = sg._bufs[body_t.root()[0].tid].cpu().permute(0, 3, 1, 2)
    d = (yb - refbody).abs()
    print("  body max abs err", d.max().item(), "at", divmod(int(d.argmax()), yb.shape[2]*yb.shape[3]), "shape", tuple(yb.shape))
    bad = (d > 1e-3).nonzero()
    print("  #bad", bad.shape[0], "channels", sorted(set(bad[:, 1].tolist()))[:20], "pix", sorted(set((bad[:, 2]*yb.shape[3]+bad[:, 3]).tolist()))[:20])
