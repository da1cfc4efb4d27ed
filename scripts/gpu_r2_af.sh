# attention operands by TMA (2-D tiled, SW64): parity + BERT A/B vs HEAD (ab_c) + per-op durations
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py -q -x -p no:cacheprovider -k "attention or bert" 2>&1 | tail -2
timeout 900 python scripts/ab_trees.py bert_base bf16 . ab_c -- bounded:auto full:l2 2>&1 | grep -v Warn | grep -E "par|tree"
timeout 600 python scripts/op_durations.py bert_base bf16 --grids bounded --modes l2 2>&1 | grep -v Warn | grep self
