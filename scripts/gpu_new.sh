# new operator families + DeepFM / NASNet parity and first bench lines
python __graft_entry__.py || exit 1
timeout 1200 python -m pytest tests/test_gpu_new_ops.py -x -q 2>&1 | tail -15
timeout 1200 python -m pytest tests/test_gpu_models.py -x -q -k nasnet 2>&1 | tail -15
for spec in "deepfm f32 1" "deepfm f32 32" "nasnet_large f32 1" "nasnet_large bf16 1"; do
  set -- $spec; m=$1; dt=$2; b=$3
  timeout 900 python bench.py --model $m --dtype $dt --batch $b --steps 50 --warmup 5 --cpu-seconds 1 --profile-reps 3 > gpurun_out/bench_${m}_${dt}_b$b.json 2> gpurun_out/bench_${m}_${dt}_b$b.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${m}_${dt}_b$b.json'));print('$dt $m b$b', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'cp',d['dag_roofline']['critical_path_us'],'roof',d['dag_roofline']['frac'],'rel',d['rel_err_vs_torch_fp32'],'val',d['value'],'e2e',d['e2e']['value'],'dom',d['roofline']['kernel'],d['roofline']['frac'])" || tail -5 gpurun_out/bench_${m}_${dt}_b$b.err
done
