# DeepFM GEMMs on the tensor-core engine + compute-sanitizer runs
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_new_ops.py -q -x -k deepfm -p no:cacheprovider 2>&1 | tail -2
for b in 1 8 32; do
  timeout 600 python bench.py --model deepfm --batch $b --steps 100 --warmup 10 --cpu-seconds 1 --cpu-model-seconds 0 > gpurun_out/c_deepfm_b$b.json 2>gpurun_out/c_deepfm_b$b.err
  python -c "import json;d=json.load(open('gpurun_out/c_deepfm_b$b.json'));print('deepfm b$b lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'engines',d['conv_engines'],'rel',d['rel_err_vs_torch_fp32'])" || tail -3 gpurun_out/c_deepfm_b$b.err
done
mkdir -p gpurun_out/sanitizer
for c in conv_f32_push conv_f32_pull conv_bf16_push conv_bf16_pull bert_layer; do
  for t in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py $c > gpurun_out/sanitizer/${c}_$t.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok=' gpurun_out/sanitizer/${c}_$t.txt | tr '\n' ' ')"
  done
done
