# re-entry check: build, all GPU tests, smoke, default bench line
python __graft_entry__.py > /dev/null 2>&1 || exit 1
cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo rc=$?; tail -c 3000 gpurun_out/r2e_bench.json; tail -3 gpurun_out/r2e_bench.err
timeout 900 python bench.py --model bert_base --steps 50 --warmup 5 > gpurun_out/r2e_bert.json 2> gpurun_out/r2e_bert.err; echo rc=$?; python -c "import json;d=json.loads(open('gpurun_out/r2e_bert.json').read().strip().splitlines()[-1]);print({k:d.get(k) for k in ('ms_per_step','speedup_vs_sequential','speedup_vs_best_sequential','rel_err')})"
