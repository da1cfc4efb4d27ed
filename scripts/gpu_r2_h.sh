# TMA im2col activation loads: conv parity (TMA vs gather bit-equal, vs fp64), models, A/B TMA on/off
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider 2>&1 | tail -3
for m in "inception_v3 f32" "inception_v3 bf16" "bert_base bf16"; do set -- $m
  echo "== $1 $2 TMA on / off"
  OPARA_TMA=1 timeout 600 python scripts/ab_trees.py $1 $2 . -- bounded:pull bounded:push 2>&1 | grep -v Warn | tail -2
  OPARA_TMA=0 timeout 600 python scripts/ab_trees.py $1 $2 . -- bounded:pull bounded:push 2>&1 | grep -v Warn | tail -2
done
