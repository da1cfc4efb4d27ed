python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py -x -q 2>&1 | tail -4
for dt in bf16 f32; do for m in googlenet inception_v3; do
  timeout 900 python bench.py --model $m --dtype $dt --steps 100 --warmup 10 --cpu-seconds 1 > gpurun_out/bench_${m}_$dt.json 2> gpurun_out/bench_$m.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${m}_$dt.json'));print('$dt $m', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'cp',d['dag_roofline']['critical_path_us'],'rel',d['rel_err_vs_torch_fp32'])" || tail -5 gpurun_out/bench_$m.err
done; done
