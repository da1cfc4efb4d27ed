python __graft_entry__.py || exit 1
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded > gpurun_out/conv_stages_seq.txt 2>&1; tail -70 gpurun_out/conv_stages_seq.txt
timeout 900 python bench.py --steps 50 --warmup 5 --cpu-seconds 2 > gpurun_out/r2_bench_new.json 2> gpurun_out/r2_bench_new.err; echo rc=$?; tail -c 1500 gpurun_out/r2_bench_new.json; tail -3 gpurun_out/r2_bench_new.err
