python __graft_entry__.py || exit 1
for sc in 0.75 1.0 1.5 2.0; do
  for spec in "inception_v3 f32" "bert_base bf16" "googlenet f32" "nasnet_large f32"; do
    set -- $spec
    OPARA_BOUND_SCALE=$sc timeout 600 python bench.py --model $1 --dtype $2 --grids bounded --steps 200 --warmup 10 --cpu-seconds 0.1 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('scale=$sc $1 $2', d['latency_ms'], d['sequential_latency_ms'], d['splitk_reduction'])" || tail -3 /tmp/b.err
  done
done
