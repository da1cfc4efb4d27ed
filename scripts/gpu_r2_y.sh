# residual-slot ring (all tile widths eligible for LayerNorm on load): BERT parity, phases, A/B vs HEAD (ab_b)
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k bert 2>&1 | tail -2
timeout 900 python scripts/ab_trees.py bert_base bf16 . ab_b -- bounded:auto full:l2 2>&1 | grep -v Warn | grep -E "par|tree"
timeout 600 python scripts/op_durations.py bert_base bf16 --grids bounded --modes l2 2>&1 | grep -v Warn | tail -7
