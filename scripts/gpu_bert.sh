python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_kernels.py -x -q -k "bert or layernorm or attention or embedding" 2>&1 | tail -3
python scripts/profile_ops.py bert_base > /dev/null && python scripts/show_profile.py bert_base_bf16 all | head -11
timeout 900 python bench.py --model bert_base --steps 100 --warmup 10 --cpu-seconds 1 > gpurun_out/bench_bert.json 2> gpurun_out/bench_bert.err
python -c "import json;d=json.load(open('gpurun_out/bench_bert.json'));print('lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'xbest',d['speedup_vs_best_sequential'],d['grids'],'cp',d['dag_roofline']['critical_path_us'],'rel',d['rel_err_vs_torch_fp32'])" || tail -5 gpurun_out/bench_bert.err
