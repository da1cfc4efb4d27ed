python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_models.py -q -x 2>&1 | tail -2
for r in 1 2; do for x in 0 1; do
  for spec in "inception_v3 f32 bounded" "bert_base bf16 bounded" "googlenet bf16 full" "nasnet_large bf16 full" "deepfm f32 full"; do
    set -- $spec
    OPARA_XSTREAM_PDL=$x timeout 600 python bench.py --model $1 --dtype $2 --grids $3 --steps 200 --warmup 10 --cpu-seconds 0.1 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('xpdl=$x $1 $2', d['latency_ms'], d['sequential_latency_ms'], d['speedup_vs_sequential'], d['rel_err_vs_torch_fp32'])" || tail -3 /tmp/b.err
  done
done; done
