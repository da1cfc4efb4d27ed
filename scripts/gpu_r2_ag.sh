# final verification of the committed tree: all GPU tests, smoke, sanitizer on the TMA attention (bert_layer)
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
mkdir -p gpurun_out/sanitizer
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 10 python scripts/sanitize.py bert_layer > gpurun_out/sanitizer/bert_layer_tma_$t.txt 2>&1
  echo "bert_layer $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok=' gpurun_out/sanitizer/bert_layer_tma_$t.txt | tr '\n' ' ')"
done
