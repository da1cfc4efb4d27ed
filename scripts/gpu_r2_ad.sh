# two-accumulator 3xTF32 variant (-DOPARA_TC_ACC2) vs default: fp32 models
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 2400 python scripts/ab_flags.py inception_v3 f32 bounded:auto full:l2 -- "" "-DOPARA_TC_ACC2" 2>&1 | grep -v Warn | tail -12
timeout 1200 python scripts/ab_flags.py googlenet f32 bounded:auto full:l2 -- "" "-DOPARA_TC_ACC2" 2>&1 | grep -v Warn | tail -12
OPARA_NVCC_FLAGS=-DOPARA_TC_ACC2 python -m paper_2312_10351_b200.build > /dev/null 2>&1
OPARA_NVCC_FLAGS=-DOPARA_TC_ACC2 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "matches_torch and tc" 2>&1 | tail -2
python -m paper_2312_10351_b200.build > /dev/null 2>&1
