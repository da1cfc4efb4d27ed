# split-K rank skew (l2 vs pull) + A/B of the bulk-store L2 reduction build; torchrun path sanity
python __graft_entry__.py > /dev/null 2>&1 || exit 1
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded --splitk l2 --slot sequential > gpurun_out/stages_l2_skew.txt 2>&1; grep -A60 "rank skew" gpurun_out/stages_l2_skew.txt | head -40
OPARA_CONV_DEBUG=1 timeout 600 python scripts/conv_stages.py inception_v3 --grids bounded --splitk pull --slot sequential > gpurun_out/stages_pull_skew.txt 2>&1; grep -A60 "rank skew" gpurun_out/stages_pull_skew.txt | head -25
timeout 1500 python scripts/ab_flags.py inception_v3 f32 bounded:l2 full:l2 -- "" "-DOPARA_L2_BULK" 2>&1 | grep -v Warn | tail -12
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 --cpu-seconds 0.5 > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo torchrun rc=$?; tail -c 400 gpurun_out/torchrun1.json
