# per-phase stamps of the TMA fp32 conv in the Opara and sequential graphs; bring back one full ncu report with source
python __graft_entry__.py > /dev/null 2>&1 || exit 1
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded --splitk pull --slot parallel > gpurun_out/stages_par.txt 2>&1; tail -5 gpurun_out/stages_par.txt
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded --splitk pull --slot sequential > gpurun_out/stages_seq.txt 2>&1; tail -5 gpurun_out/stages_seq.txt
export OPARA_TUNE_CACHE=/tmp/tune_incv3.json
python bench.py --steps 5 --warmup 3 --cpu-seconds 0.1 --grids bounded > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:conv2d_tc_tf32x3 -s 30 -c 1 \
   -o gpurun_out/conv_full python bench.py --grids bounded --steps 3 --warmup 3 --cpu-seconds 0.1 --profile-reps 2 --profile-region > /dev/null 2>&1; echo ncu rc=$?
ls -la gpurun_out/conv_full.ncu-rep
