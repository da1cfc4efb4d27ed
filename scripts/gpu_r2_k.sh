# attention: 16 warps, MN-major V; parity + BERT A/B + per-op durations
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k attention 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k bert 2>&1 | tail -2
timeout 600 python scripts/ab_trees.py bert_base bf16 . -- bounded:pull full:push 2>&1 | grep -v Warn | tail -4
timeout 600 python scripts/op_durations.py bert_base bf16 --grids bounded --modes pull 2>&1 | grep -v Warn | tail -30
