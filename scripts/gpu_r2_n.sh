# L2 split-K reduction (fp32 engine): parity vs pull, A/B in the Inception-v3 graph, phase stamps
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 900 python - <<'PY' 2>&1 | grep -v Warn
import torch, sys
sys.path.insert(0, ".")
from paper_2312_10351_b200 import engine, zoo
torch.backends.cudnn.allow_tf32 = False; torch.backends.cuda.matmul.allow_tf32 = False
m, x = zoo.build("inception_v3")
outs = {}
for sk in ("pull", "l2"):
    sg = engine.compile(m, x, device=0, bound_grids=True, splitk=sk, profile_reps=2)
    y = sg.run(x.cuda()); outs[sk] = y.clone()
    assert torch.equal(y, sg.run(x.cuda(), slot=engine.SLOT_SEQUENTIAL))
with torch.no_grad():
    ref = m.cuda()(x.cuda())
for sk, y in outs.items():
    print(sk, "rel", ((y - ref).norm() / ref.norm()).item())
PY
timeout 900 python scripts/ab_trees.py inception_v3 f32 . -- bounded:pull bounded:l2 full:push full:l2 2>&1 | grep -v Warn | tail -10
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded --splitk l2 --slot sequential > gpurun_out/stages_seq_l2.txt 2>&1; grep -E "^ +4[1-9] " gpurun_out/stages_seq_l2.txt
