# build -> all GPU tests -> smoke -> bench across the configs
python __graft_entry__.py || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -3
for spec in "googlenet f32" "inception_v3 f32" "googlenet bf16" "inception_v3 bf16" "bert_base bf16"; do
  set -- $spec; m=$1; dt=$2
  timeout 900 python bench.py --model $m --dtype $dt --steps 100 --warmup 10 --cpu-seconds 1 > gpurun_out/bench_${m}_$dt.json 2> gpurun_out/bench_${m}_$dt.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${m}_$dt.json'));print('$dt $m', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'cp',d['dag_roofline']['critical_path_us'],'roof',d['dag_roofline']['frac'],'rel',d['rel_err_vs_torch_fp32'],'e2e',d['e2e']['value'],'dom',d['roofline']['kernel'],d['roofline']['frac'])" || tail -5 gpurun_out/bench_${m}_$dt.err
done
