# Alg. 2 with TMEM-folded demands vs measured demands (launch-order A/B); torchrun sanity
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 2400 python scripts/ab_demand.py inception_v3:f32 inception_v3:bf16 googlenet:f32 googlenet:bf16 nasnet_large:bf16 2>&1 | grep -v Warn | tee gpurun_out/ab_demand.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 --cpu-seconds 0.5 > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo torchrun rc=$?; tail -c 300 gpurun_out/torchrun1.json
