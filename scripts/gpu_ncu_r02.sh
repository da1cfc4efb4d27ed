# ncu evidence for profiles/: per workload, the launch list of the bench's timed
# region (cudaProfilerStart/Stop bracket) and one --set full capture of the
# dominant kernel family.  Autotune choices are cached first so ncu sees the
# bench's exact kernels without the tuning launches.
python __graft_entry__.py || exit 1
IFS="|"
for spec in ${NCU_SPECS:-"inception_v3 f32 conv2d_tc_tf32x3|bert_base bf16 conv2d_tc_bf16|nasnet_large bf16 conv2d_tc_bf16|googlenet f32 conv2d_tc_tf32x3"}; do
  IFS=" "; set -- $spec; m=$1; dt=$2; k=$3
  export OPARA_TUNE_CACHE=/tmp/tune_${m}_$dt.json
  python bench.py --model $m --dtype $dt --steps 20 --warmup 3 --cpu-seconds 0.1 > gpurun_out/pre_$m.json 2>/dev/null
  g=$(python -c "import json;print(json.load(open('gpurun_out/pre_$m.json'))['grids'])")
  echo "$m $dt grids=$g"
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/launches_${m}_$dt.csv python bench.py --model $m --dtype $dt --grids $g --steps 3 \
     --warmup 3 --cpu-seconds 0.1 --profile-reps 2 --profile-region > /dev/null 2>&1; echo "launch list rc=$?"
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 \
     -o gpurun_out/full_${m}_$dt python bench.py --model $m --dtype $dt --grids $g --steps 3 --warmup 3 \
     --cpu-seconds 0.1 --profile-reps 2 --profile-region > /dev/null 2>&1; echo "full rc=$?"
  timeout 300 python scripts/timeline.py $m $dt > /dev/null 2>&1; echo "timeline rc=$?"
  # summarise here: the raw reports and launch CSVs exceed what gpurun brings back
  mkdir -p gpurun_out/profiles
  python scripts/summarize_ncu.py r02_${m}_$dt gpurun_out/launches_${m}_$dt.csv gpurun_out/full_${m}_$dt.ncu-rep \
     gpurun_out/profiles > /dev/null 2>&1; echo "summary rc=$?"
  mv gpurun_out/r02_${m}_${dt}_timeline.md gpurun_out/profiles/ 2>/dev/null
  rm -f gpurun_out/launches_${m}_$dt.csv gpurun_out/full_${m}_$dt.ncu-rep gpurun_out/pre_$m.json
done
