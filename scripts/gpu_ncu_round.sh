# ncu evidence for profiles/: launch list of a short bench run + one full capture of the top kernel
python __graft_entry__.py || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_inception_v3.csv \
    python bench.py --model inception_v3 --steps 2 --warmup 3 --cpu-seconds 0.1 --profile-reps 1 > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:conv2d_tc_tf32x3 -s 300 -c 1 -o gpurun_out/conv_tc_full \
    python bench.py --model inception_v3 --steps 2 --warmup 3 --cpu-seconds 0.1 --profile-reps 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -n 2 gpurun_out/ncu_full.log
