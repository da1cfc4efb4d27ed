# gamma/beta prefetch before the PDL wait (folded LN consumers): BERT parity + A/B; sanitizer on the round-2 paths
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k bert 2>&1 | tail -2
timeout 900 python scripts/ab_trees.py bert_base bf16 . ab_a -- bounded:auto full:l2 2>&1 | grep -v Warn | grep -E "par|tree"
mkdir -p gpurun_out/sanitizer
for c in conv_f32_l2 conv_bf16_l2 bert_fold; do
  for t in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py $c > gpurun_out/sanitizer/${c}_$t.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok=' gpurun_out/sanitizer/${c}_$t.txt | tr '\n' ' ')"
  done
done
