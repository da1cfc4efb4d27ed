# bisect the fp32 conv regression: HEAD, A (single-row pull), B (57eab33 conv_tc.cu), old tree
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 1500 python scripts/ab_trees.py inception_v3 f32 . ab_a ab_b ab_old -- bounded:pull full:push 2>&1 | grep -v Warning | tee gpurun_out/ab_trees_incv3_g.txt
