# final check of the committed tree: all GPU tests, smoke, default bench line
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2_last_bench.json 2> gpurun_out/r2_last_bench.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/r2_last_bench.json').read().strip().splitlines()[-1]);print({k:d.get(k) for k in ('value','ms_per_step','speedup_vs_sequential','speedup_vs_best_sequential','grids','splitk_reduction','gpu_launches_per_step')}, d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -c 300
