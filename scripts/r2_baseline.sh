python __graft_entry__.py || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 100 --warmup 10 --cpu-seconds 2 > gpurun_out/r2_base_default.json 2> gpurun_out/r2_base_default.err; tail -c 400 gpurun_out/r2_base_default.json
