# TMA im2col semantics probe + A/B of HEAD vs 57eab33 (run_a tree) on Inception-v3 fp32
./scripts/micro/tma_im2col > gpurun_out/tma_im2col.txt 2>&1; cat gpurun_out/tma_im2col.txt
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 1500 python scripts/ab_trees.py inception_v3 f32 . ab_old -- bounded:pull bounded:auto full:push 2>&1 | grep -v Warning | tee gpurun_out/ab_trees_incv3.txt
