python __graft_entry__.py || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
OPARA_CONV_DEBUG=1 python scripts/one_conv.py 64 64 1 1 0 56
OPARA_CONV_DEBUG=1 python scripts/one_conv.py 64 192 3 1 1 56
OPARA_CONV_DEBUG=1 python scripts/one_conv.py 480 96 1 1 0 14
