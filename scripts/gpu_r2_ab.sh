# tensor-map prefetch before griddepcontrol.wait: A/B vs HEAD (ab_c)
python __graft_entry__.py > /dev/null 2>&1 || exit 1
for m in "inception_v3 f32" "inception_v3 bf16" "googlenet f32" "bert_base bf16"; do set -- $m
  echo "== $1 $2"
  timeout 1200 python scripts/ab_trees.py $1 $2 . ab_c -- bounded:auto full:l2 2>&1 | grep -v Warn | grep -E "par|tree"
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "tma or bf16" 2>&1 | tail -2
