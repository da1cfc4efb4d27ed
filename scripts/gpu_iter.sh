# quick iteration on the GPU box: build, conv stage timeline, kernel tests, default bench line
python __graft_entry__.py || exit 1
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded > gpurun_out/conv_stages.txt 2>&1; head -3 gpurun_out/conv_stages.txt; grep -E "^ +(59|60|61|62|79|80|103|104) " gpurun_out/conv_stages.txt; tail -12 gpurun_out/conv_stages.txt
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded --splitk push > gpurun_out/conv_stages_push.txt 2>&1; grep -E "^ +(59|60|61|62|79|80|103|104) " gpurun_out/conv_stages_push.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py -x -q 2>&1 | tail -2
for m in ${MODELS:-inception_v3}; do
timeout 900 python bench.py --model $m --steps 50 --warmup 5 --cpu-seconds 1 --cpu-model-seconds 0 > gpurun_out/iter_$m.json 2> gpurun_out/iter_$m.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/iter_$m.json'));print('$m lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],d['grids'],d['splitk_reduction'],d['bound_scale'],'cp',d['dag_roofline']['critical_path_us'],'rel',d['rel_err_vs_torch_fp32'],'dom',d['roofline']['avg_launch_us'],d['roofline']['frac'])" || tail -3 gpurun_out/iter_$m.err
done
