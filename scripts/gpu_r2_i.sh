# TMA im2col: corner probe (past-edge boxes), conv parity, all model tests
for i in 6 7 8; do timeout 60 ./scripts/micro/tma_im2col $i 2>&1 | tail -2; done
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 2400 python -m pytest tests/test_gpu_models.py tests/test_gpu_bench_graphs.py tests/test_gpu_new_ops.py -q -x -p no:cacheprovider 2>&1 | tail -3
