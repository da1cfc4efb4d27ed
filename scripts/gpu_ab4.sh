# A/B of two prebuilt libraries (scripts/ab/libopara_old.so vs the fresh build), same box, twice
cp paper_2312_10351_b200/libopara.so /tmp/new.so
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then cp scripts/ab/libopara_old.so paper_2312_10351_b200/libopara.so; else cp /tmp/new.so paper_2312_10351_b200/libopara.so; fi
  for spec in "bert_base bf16 bounded" "inception_v3 f32 bounded" "googlenet bf16 full" "nasnet_large bf16 full"; do
    set -- $spec
    timeout 600 python bench.py --model $1 --dtype $2 --grids $3 --steps 200 --warmup 10 --cpu-seconds 0.1 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('$v $1 $2', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],d['splitk_reduction'])" || tail -3 /tmp/b.err
  done
done; done
cp /tmp/new.so paper_2312_10351_b200/libopara.so
