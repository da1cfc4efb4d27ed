# L2 split-K reduction in both engines: kernel parity tests, then A/B of reductions per model
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k splitk 2>&1 | tail -2
for m in "inception_v3 f32" "googlenet f32" "inception_v3 bf16" "googlenet bf16" "bert_base bf16" "nasnet_large bf16"; do set -- $m
  echo "== $1 $2"
  AB_ROUNDS=1 timeout 1200 python scripts/ab_trees.py $1 $2 . -- bounded:pull bounded:l2 bounded:auto full:push full:l2 2>&1 | grep -v Warn | grep par
done
