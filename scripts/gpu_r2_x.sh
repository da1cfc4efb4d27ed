# synccheck of the folded-LayerNorm layer after replacing the named barrier with an mbarrier
python __graft_entry__.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/sanitizer
for t in synccheck racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 4 python scripts/sanitize.py bert_fold > gpurun_out/sanitizer/bert_fold_$t.txt 2>&1
  echo "bert_fold $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok=' gpurun_out/sanitizer/bert_fold_$t.txt | tr '\n' ' ')"
done
timeout 900 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k bert 2>&1 | tail -2
