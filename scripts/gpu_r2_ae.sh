# DeepFM batch sweep bench lines (1, 2, 4, 8, 16, 32)
python __graft_entry__.py > /dev/null 2>&1 || exit 1
for b in 1 2 4 8 16 32; do
  timeout 900 python bench.py --model deepfm --batch $b --steps 200 --warmup 20 --cpu-seconds 2 > gpurun_out/r2final_deepfm_f32_b$b.json 2> gpurun_out/deepfm_b$b.err
  python -c "import json;d=json.load(open('gpurun_out/r2final_deepfm_f32_b$b.json'));print('deepfm b$b', 'lat',d['latency_ms'],'seq',d['sequential_latency_ms'],'x',d['speedup_vs_sequential'],'xbest',d['speedup_vs_best_sequential'],'val',d['value'],'e2e',d['e2e']['value'],'rel',d['rel_err_vs_torch_fp32'],d['grids'],d['splitk_reduction'])" || tail -3 gpurun_out/deepfm_b$b.err
done
