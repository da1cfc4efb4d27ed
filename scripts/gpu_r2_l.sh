# round-2 evidence: all GPU tests + smoke + default bench, then ncu launch lists (with DRAM bytes) + full captures
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/r2l_bench.json').read().strip().splitlines()[-1]);print({k:d.get(k) for k in ('value','ms_per_step','speedup_vs_sequential','speedup_vs_best_sequential','grids','splitk_reduction')}, d['roofline']['frac'], d['roofline']['avg_launch_us'], d['e2e']['value'], d['launch_order_latency_ms'])"
NCU_SPECS="inception_v3 f32 conv2d_tc_tf32x3|bert_base bf16 conv2d_tc_bf16" bash scripts/gpu_ncu_r02.sh 2>&1 | tail -12
