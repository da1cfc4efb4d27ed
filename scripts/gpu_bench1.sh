set -x
python __graft_entry__.py
timeout 900 python bench.py --model googlenet --steps 100 --warmup 10 --cpu-seconds 3 2>&1 | tail -5
timeout 900 python bench.py --steps 100 --warmup 10 --cpu-seconds 3 2>&1 | tail -5
