python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_new_ops.py tests/test_gpu_models.py -q -x -k "separable or nasnet" 2>&1 | tail -2
for t in 0 1; do
  OPARA_DW_TILED=$t python scripts/profile_ops.py nasnet_large bf16 --grids full | tail -1 && python scripts/cp_breakdown.py nasnet_large_bf16 | head -5
done
for spec in "nasnet_large bf16" "nasnet_large f32"; do
  set -- $spec
  python bench.py --model $1 --dtype $2 --steps 200 --warmup 10 --cpu-seconds 0.2 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$1 $2', d['latency_ms'], d['sequential_latency_ms'], d['speedup_vs_sequential'], d['grids'], d['splitk_reduction'], d['rel_err_vs_torch_fp32'])" || tail -3 /tmp/b.err
done
