set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_properties(0))"
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -30
