# A/B: committed conv kernels vs working copy, on the same box (latency of par / seq graphs)
cp paper_2312_10351_b200/csrc/conv_tc.cu /tmp/new_tc.cu; cp paper_2312_10351_b200/csrc/conv_tc_bf16.cu /tmp/new_bf.cu
python __graft_entry__.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py tests/test_gpu_new_ops.py -x -q 2>&1 | tail -2
for v in orig new; do
  if [ $v = orig ]; then cp scripts/ab/conv_tc_orig.cu paper_2312_10351_b200/csrc/conv_tc.cu; cp scripts/ab/conv_tc_bf16_orig.cu paper_2312_10351_b200/csrc/conv_tc_bf16.cu;
  else cp /tmp/new_tc.cu paper_2312_10351_b200/csrc/conv_tc.cu; cp /tmp/new_bf.cu paper_2312_10351_b200/csrc/conv_tc_bf16.cu; fi
  python -m paper_2312_10351_b200.build > /dev/null || exit 1
  for spec in "bert_base bf16" "inception_v3 f32" "inception_v3 bf16" "googlenet f32" "nasnet_large bf16"; do
    set -- $spec
    for b in "" "--bounded"; do
      timeout 600 python bench.py --model $1 --dtype $2 --steps 50 --warmup 5 --cpu-seconds 0.2 --profile-reps 5 $b > /tmp/b.json 2>/tmp/b.err
      python -c "import json;d=json.load(open('/tmp/b.json'));print('$v $1 $2 $b', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'cp',d['dag_roofline']['critical_path_us'])" || tail -3 /tmp/b.err
    done
  done
done
