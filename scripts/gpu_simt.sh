python __graft_entry__.py || exit 1
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
for spec in "inception_v3 f32" "googlenet f32" "nasnet_large f32"; do
  set -- $spec
  t0=$(date +%s)
  timeout 900 python bench.py --model $1 --dtype $2 --steps 200 --warmup 10 --cpu-seconds 0.1 > /tmp/b.json 2>/tmp/b.err
  python -c "
import json;d=json.load(open('/tmp/b.json'));print('$1 $2', d['latency_ms'], d['sequential_latency_ms'], d['speedup_vs_sequential'], d['grids'], d['splitk_reduction'], d['bound_scale'], d['rel_err_vs_torch_fp32'], 'dom', d['roofline']['kernel'])" || tail -3 /tmp/b.err
  echo "  $(( $(date +%s) - t0 )) s"
done
python scripts/profile_ops.py inception_v3 f32 --grids bounded | tail -1
python -c "
import json; d=json.load(open('gpurun_out/profile_inception_v3_f32.json'))
import collections; print(collections.Counter((o['kind'], o['ints'].get('R')) for o in d['ops'] if o['kind']==1))
"
