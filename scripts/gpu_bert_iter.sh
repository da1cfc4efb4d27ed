python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py tests/test_gpu_new_ops.py -x -q 2>&1 | tail -3
python scripts/bert_phases.py seq 2>&1 | head -40
python scripts/profile_ops.py bert_base && python scripts/show_profile.py bert_base_bf16 all | head -12
for m in bert_base inception_v3; do
timeout 900 python bench.py --model $m --dtype bf16 --steps 100 --warmup 10 --cpu-seconds 1 > gpurun_out/bench_${m}_bf16.json 2> gpurun_out/bench_${m}.err
python -c "import json;d=json.load(open('gpurun_out/bench_${m}_bf16.json'));print('$m', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'cp',d['dag_roofline']['critical_path_us'],'roof',d['dag_roofline']['frac'],'rel',d['rel_err_vs_torch_fp32'])" || tail -5 gpurun_out/bench_$m.err
done
