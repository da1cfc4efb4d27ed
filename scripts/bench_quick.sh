# quick bench of SPECS ("model dtype batch|..."): one summary line each + the sizing search
IFS="|"; for spec in $SPECS; do IFS=" "; set -- $spec
  timeout 900 python bench.py --model $1 --dtype $2 --batch ${3:-1} --steps 100 --warmup 10 --cpu-seconds 1 > gpurun_out/bench_$1_$2_b${3:-1}.json 2>gpurun_out/bench_$1_$2_b${3:-1}.err
  python - "$1" "$2" "${3:-1}" <<'PY'
import json, sys
m, dt, b = sys.argv[1:4]
d = json.load(open(f"gpurun_out/bench_{m}_{dt}_b{b}.json"))
print(m, dt, "b" + b, "lat", d["latency_ms"], "seq", d["sequential_latency_ms"], "x", d["speedup_vs_sequential"],
      "xbest", d["speedup_vs_best_sequential"], d["grids"], d["splitk_reduction"], d.get("bound_scale"),
      "frac", d["dag_roofline"]["frac"], "rel", round(d["rel_err_vs_torch_fp32"], 7), "e2e", d["e2e"]["value"])
print("   ", [(t["bounded"], t["splitk"], t["scale"], round(t["parallel_ms"], 4), round(t["sequential_ms"], 4)) for t in d.get("grid_autotune", [])])
PY
done
