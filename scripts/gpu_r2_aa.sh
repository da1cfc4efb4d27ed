# full GPU suite with the session tune cache (duration check) + SM-share scale A/B (2.0 vs 3.0)
python __graft_entry__.py > /dev/null 2>&1 || exit 1
start=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=8 2>&1 | tail -14
echo "suite seconds: $(( $(date +%s) - start ))"
timeout 900 python scripts/ab_scale.py inception_v3:bf16:auto nasnet_large:bf16:auto -- 2.0 3.0 2>&1 | grep -v Warn
