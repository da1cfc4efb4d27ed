python __graft_entry__.py || exit 1
for m in googlenet inception_v3; do timeout 600 python scripts/profile_ops.py $m; done
