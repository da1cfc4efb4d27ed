# A/B: bias fetched before the PDL wait (default) vs in the epilogue (-DOPARA_BIAS_LATE)
for v in "" "-DOPARA_BIAS_LATE" ""; do
  OPARA_NVCC_FLAGS="$v" python -m paper_2312_10351_b200.build --clean > /dev/null || exit 1
  for spec in "bert_base bf16 bounded" "inception_v3 f32 bounded" "googlenet bf16 full"; do
    set -- $spec
    timeout 600 python bench.py --model $1 --dtype $2 --grids $3 --steps 200 --warmup 10 --cpu-seconds 0.1 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('[$v] $1 $2', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],d['splitk_reduction'],'cp',d['dag_roofline']['critical_path_us'])" || tail -3 /tmp/b.err
  done
done
