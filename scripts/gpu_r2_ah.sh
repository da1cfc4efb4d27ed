# unsplit-tile store loop with four rows in flight (-DOPARA_UNSPLIT_UNROLL): stage stamps + A/B
python __graft_entry__.py > /dev/null 2>&1 || exit 1
export OPARA_NVCC_FLAGS=-DOPARA_UNSPLIT_UNROLL
python -m paper_2312_10351_b200.build > /dev/null 2>&1
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded --splitk l2 --slot sequential > gpurun_out/stages_unroll.txt 2>&1; grep -E "^ +(3|6|15) " gpurun_out/stages_unroll.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "matches_torch and tc" 2>&1 | tail -1
unset OPARA_NVCC_FLAGS
python -m paper_2312_10351_b200.build > /dev/null 2>&1
timeout 2000 python scripts/ab_flags.py inception_v3 f32 bounded:auto full:l2 -- "" "-DOPARA_UNSPLIT_UNROLL" 2>&1 | grep -v Warn | tail -12
python -m paper_2312_10351_b200.build > /dev/null 2>&1
