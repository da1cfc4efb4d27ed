python __graft_entry__.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:conv2d_tc -s 4 -c 1 -o gpurun_out/conv_tc_3x3 python scripts/one_conv.py 64 192 3 1 1 56 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv2d_tc -s 4 -c 1 -o gpurun_out/conv_tc_1x1 python scripts/one_conv.py 64 64 1 1 0 56 > gpurun_out/ncu1.log 2>&1
tail -n 3 gpurun_out/ncu1.log gpurun_out/ncu2.log
