python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_models.py -q -x -k bert 2>&1 | tail -2
for mk in 0 1024 4096; do
  OPARA_LN_FUSE_MAX_K=$mk python scripts/profile_ops.py bert_base bf16 --grids bounded | tail -1
  python scripts/cp_breakdown.py bert_base_bf16 | head -4
  python scripts/show_profile.py bert_base_bf16 all | sed -n 2,9p
  OPARA_LN_FUSE_MAX_K=$mk python bench.py --model bert_base --steps 200 --warmup 10 --cpu-seconds 0.1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('maxk=$mk', d['latency_ms'], d['sequential_latency_ms'], d['speedup_vs_sequential'], d['speedup_vs_best_sequential'], d['grids'], d['splitk_reduction'], d['rel_err_vs_torch_fp32'])" || tail -3 /tmp/b.err
done
