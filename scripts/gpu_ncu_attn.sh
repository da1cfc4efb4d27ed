python __graft_entry__.py || exit 1
export OPARA_TUNE_CACHE=/tmp/tune_bert.json
python bench.py --model bert_base --grids bounded --steps 5 --warmup 3 --cpu-seconds 0.1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attention_tc -s 2 -c 1 \
   -o gpurun_out/full_attention python bench.py --model bert_base --grids bounded --steps 3 --warmup 3 \
   --cpu-seconds 0.1 --profile-reps 2 --profile-region > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:layernorm_rows_v -s 2 -c 1 \
   -o gpurun_out/full_layernorm python bench.py --model bert_base --grids bounded --steps 3 --warmup 3 \
   --cpu-seconds 0.1 --profile-reps 2 --profile-region > /dev/null 2>&1; echo "rc=$?"
