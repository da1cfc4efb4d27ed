python __graft_entry__.py || exit 1
timeout 1200 python -m pytest tests/test_gpu_new_ops.py tests/test_gpu_models.py -x -q -k "separable or nasnet or relu" 2>&1 | tail -3
for spec in "nasnet_large bf16" "nasnet_large f32"; do
  set -- $spec
  timeout 900 python bench.py --model $1 --dtype $2 --steps 100 --warmup 10 --cpu-seconds 0.2 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$1 $2', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'xbest',d['speedup_vs_best_sequential'],d['grids'],d['splitk_reduction'],'cp',d['dag_roofline']['critical_path_us'],'rel',round(d['rel_err_vs_torch_fp32'],7))" || tail -3 /tmp/b.err
done
python scripts/profile_ops.py nasnet_large bf16 --grids full > /dev/null && python scripts/cp_breakdown.py nasnet_large_bf16
