python __graft_entry__.py || exit 1
for spec in "bert_base bf16" "inception_v3 f32" "inception_v3 bf16" "googlenet f32" "googlenet bf16" "nasnet_large bf16"; do
  set -- $spec
  t0=$(date +%s)
  timeout 900 python bench.py --model $1 --dtype $2 --steps 100 --warmup 10 --cpu-seconds 0.2 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$1 $2', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'xbest',d['speedup_vs_best_sequential'],d['grids'],d['splitk_reduction'],'cp',d['dag_roofline']['critical_path_us']); print('   ', [(a['bounded'], a['splitk'], round(a['parallel_ms'],4), round(a['sequential_ms'],4)) for a in d['grid_autotune']])" || tail -3 /tmp/b.err
  echo "   $(( $(date +%s) - t0 )) s"
done
