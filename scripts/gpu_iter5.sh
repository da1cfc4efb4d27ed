python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py -q -x 2>&1 | tail -2
python scripts/profile_ops.py bert_base bf16 --grids bounded | tail -1 && python scripts/cp_breakdown.py bert_base_bf16 && python scripts/show_profile.py bert_base_bf16 all | sed -n 2,10p
for spec in "bert_base bf16" "inception_v3 bf16" "googlenet bf16" "nasnet_large bf16"; do
  set -- $spec
  python bench.py --model $1 --dtype $2 --steps 200 --warmup 10 --cpu-seconds 0.2 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$1 $2', d['latency_ms'], d['sequential_latency_ms'], d['speedup_vs_sequential'], d['grids'], d['splitk_reduction'])" || tail -3 /tmp/b.err
done
