# round 2: new parity tests (bench graphs, every autotune variant, edge safety,
# trace order, tightened bf16 gates, DeepFM sweep), measured order search on blocks
python __graft_entry__.py || exit 1
timeout 2400 python -m pytest tests/test_gpu_bench_graphs.py tests/test_gpu_search.py tests/test_gpu_new_ops.py tests/test_gpu_models.py -q -x -p no:cacheprovider 2>&1 | tail -15
for b in inception_v3_b googlenet_3a inception_v3_a; do
  timeout 900 python -m paper_2312_10351_b200 search $b --out gpurun_out/search_$b.json > gpurun_out/search_$b.log 2>&1; echo "search $b rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/search_$b.json'));print('$b', d['orders_examined'], d['latency_ms'], 'best', round(d['best_ms'],4), {k:(round(v['ms'],4),v['rank']) for k,v in d['policies'].items()}, 'simbest', d.get('simulated_best_order_measured_ms'))" || tail -5 gpurun_out/search_$b.log
done
