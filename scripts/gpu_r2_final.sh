# Round-end style run: all GPU tests, smoke, default bench, every config's bench line
python __graft_entry__.py || exit 1
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; tail -c 600 gpurun_out/r2_bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; tail -c 300 gpurun_out/r2_bench_reference.json
for spec in "inception_v3 f32 1" "inception_v3 bf16 1" "googlenet f32 1" "googlenet bf16 1" "bert_base bf16 1" "nasnet_large f32 1" "nasnet_large bf16 1" "deepfm f32 1" "deepfm f32 8" "deepfm f32 32"; do
  set -- $spec
  timeout 900 python bench.py --model $1 --dtype $2 --batch $3 --steps 200 --warmup 20 --cpu-seconds 2 > gpurun_out/r2final_$1_$2_b$3.json 2> gpurun_out/r2final_$1_$2_b$3.err
  python -c "import json;d=json.load(open('gpurun_out/r2final_$1_$2_b$3.json'));print('$1 $2 b$3', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'xbest',d['speedup_vs_best_sequential'],d['grids'],d['splitk_reduction'],'roof',d['dag_roofline']['frac'],'rel',d['rel_err_vs_torch_fp32'],'val',d['value'],'e2e',d['e2e']['value'],'cpu',d['cpu_baseline']['value'],'dom',d['roofline']['kernel'],d['roofline']['frac'],'clk',d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r2final_$1_$2_b$3.err
done
