# all GPU tests + compute-sanitizer (memcheck / racecheck / synccheck) per kernel family
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
mkdir -p gpurun_out/sanitizer
for c in conv_f32_push conv_f32_pull conv_bf16_push conv_bf16_pull bert_layer; do
  for t in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py $c > gpurun_out/sanitizer/${c}_$t.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok=' gpurun_out/sanitizer/${c}_$t.txt | tr '\n' ' ')"
  done
done
