# folded LayerNorm (BERT): parity tests, A/B folded vs unfolded
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k bert 2>&1 | tail -15
timeout 900 python - <<'PY' 2>&1 | grep -v Warn
import sys, torch
sys.path.insert(0, ".")
from paper_2312_10351_b200 import engine, frontend, zoo
m, ref, ids = zoo.build_bert()
for fold in (True, False):
    for b, sk in ((True, "auto"), (True, "l2"), (False, "l2")):
        sg = engine.ScheduledGraph(frontend.lower(m, ids, "bf16", fold_ln=fold), 0, profile_reps=3, bound_grids=b, splitk=sk)
        sg.run(ids.cuda())
        par = sorted(sg.time(engine.SLOT_PARALLEL, iters=200).median_ms for _ in range(3))[1]
        seq = sorted(sg.time(engine.SLOT_SEQUENTIAL, iters=200).median_ms for _ in range(3))[1]
        print("fold", fold, "bounded", b, sk, "par %.4f seq %.4f x %.3f" % (par, seq, seq / par), flush=True)
        sg.close()
PY
