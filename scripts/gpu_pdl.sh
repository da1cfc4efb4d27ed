python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -2
for pdl in 1 0; do for m in googlenet inception_v3; do
  OPARA_PDL=$pdl timeout 900 python bench.py --model $m --steps 100 --warmup 10 --cpu-seconds 1 > gpurun_out/bench_${m}_pdl$pdl.json 2> gpurun_out/bench_$m.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${m}_pdl$pdl.json'));print('pdl=$pdl $m', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'warm',d['latency_warm_l2_ms'],'cp',d['dag_roofline']['critical_path_us'],'rel',d['rel_err_vs_torch_fp32'])" || tail -5 gpurun_out/bench_$m.err
done; done
