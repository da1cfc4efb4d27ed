# build -> all GPU tests -> smoke -> bench across the configs
python __graft_entry__.py || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -2
for spec in ${SPECS:-"inception_v3 f32 1" "inception_v3 bf16 1" "googlenet f32 1" "googlenet bf16 1" "bert_base bf16 1" "nasnet_large f32 1" "nasnet_large bf16 1" "deepfm f32 1" "deepfm f32 32"}; do
  set -- $spec; m=$1; dt=$2; b=$3
  t0=$(date +%s)
  timeout 900 python bench.py --model $m --dtype $dt --batch $b --steps 100 --warmup 10 --cpu-seconds 1 > gpurun_out/bench_${m}_${dt}_b$b.json 2> gpurun_out/bench_${m}_${dt}_b$b.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${m}_${dt}_b$b.json'));print('$dt $m b$b', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'xbest',d['speedup_vs_best_sequential'],d['grids'],'cp',d['dag_roofline']['critical_path_us'],'roof',d['dag_roofline']['frac'],'rel',round(d['rel_err_vs_torch_fp32'],7),'val',d['value'],'e2e',d['e2e']['value'])" || tail -5 gpurun_out/bench_${m}_${dt}_b$b.err
  echo "   ($(( $(date +%s) - t0 )) s)"
done
