# folded LayerNorm with 6 warps (gather warp 3 issues o + r tiles) vs 7 warps (ab_a): parity + A/B
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k bert 2>&1 | tail -2
for m in "bert_base bf16" "inception_v3 bf16" "googlenet bf16"; do set -- $m
  echo "== $1 $2"
  timeout 1200 python scripts/ab_trees.py $1 $2 . ab_a -- bounded:auto bounded:push full:push 2>&1 | grep -v Warn | grep -E "par|tree"
done
