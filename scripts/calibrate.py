"""Calibrate the execution model (simulate) against the B200.

Inputs, per BASELINE config, from one bench run (scripts/gpu_round.sh):
  gpurun_out/bench_<model>_<dtype>_b<batch>.json   measured latencies per launch policy
  gpurun_out/schedules/<model>_<dtype>_b<batch>/    the profiled DAG (per-op demand + block
                                                    duration from in-graph kernel times)
For each config the model predicts the Opara (Alg. 1 plan + Alg. 2 order), dfs,
wavefront and sequential makespans with the b200 GpuConfig; the same-class
co-residency slowdown (the reference's only free parameter, simulator.py:62-79)
is fitted by grid search to minimise the mean |log(predicted / measured)| of
the multi-stream policies over all configs.  Writes a JSON + markdown table of
predicted vs measured speed-ups and the prediction error.

    python scripts/calibrate.py [--src gpurun_out] [--out profiles/r02_calibration]
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2312_10351_b200 as op  # noqa: E402

POLICIES = ("opara", "dfs", "wavefront")


def load(src: Path):
    rows = []
    for sdir in sorted((src / "schedules").iterdir()):
        bench = src / f"bench_{sdir.name}.json"
        if not bench.exists() or not (sdir / "graph.json").exists():
            continue
        b = json.loads(bench.read_text())
        g = op.load_graph(sdir / "graph.json")
        cfg = op.load_gpu_config(str(sdir / "gpu_config.json"))
        rows.append({"name": sdir.name, "graph": g, "cfg": cfg,
                     "measured": dict(b["launch_order_latency_ms"]),
                     "critical_path_us": b["dag_roofline"]["critical_path_us"]})
    return rows


def predict(row, slowdown: float) -> dict:
    g, cfg = row["graph"], replace(row["cfg"], same_class_slowdown=slowdown)
    plan = op.allocate_streams(g)
    out = {}
    for pol in POLICIES:
        out[pol] = op.simulate(g, plan, op.make_order(g, pol, cfg), cfg, blocks=False).makespan_ns / 1e6
    out["sequential"] = op.sequential_makespan_ns(g, cfg) / 1e6
    return out


def err(rows, preds) -> float:
    e = [abs(math.log(p[pol] / r["measured"][pol])) for r, p in zip(rows, preds) for pol in POLICIES]
    return sum(e) / len(e)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=str(ROOT / "gpurun_out"))
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_calibration"))
    args = ap.parse_args()
    rows = load(Path(args.src))
    if not rows:
        print("no bench + schedule pairs found", file=sys.stderr)
        return 1
    grid = [round(1.0 + 0.05 * i, 2) for i in range(61)]   # 1.00 .. 4.00
    # DeepFM's 30-odd sub-microsecond kernels are bound by the graph's launch
    # front end, which the reference model has no term for: fit on the
    # block-bound configs, report every config against that fit
    fit_rows = [r for r in rows if not r["name"].startswith("deepfm")] or rows
    fits = [(err(fit_rows, [predict(r, s) for r in fit_rows]), s) for s in grid]
    best_err, best_s = min(fits)
    default = [predict(r, 1.4) for r in rows]
    fitted = [predict(r, best_s) for r in rows]
    table = []
    for r, p0, p1 in zip(rows, default, fitted):
        m = r["measured"]
        table.append({
            "config": r["name"], "nodes": len(r["graph"]), "measured_ms": m,
            "simulated_ms_slowdown_1.4": {k: round(v, 4) for k, v in p0.items()},
            "simulated_ms_fitted": {k: round(v, 4) for k, v in p1.items()},
            "speedup_vs_sequential": {
                "measured": round(m["sequential"] / m["opara"], 3),
                "simulated_1.4": round(p0["sequential"] / p0["opara"], 3),
                "simulated_fitted": round(p1["sequential"] / p1["opara"], 3)},
            "opara_prediction_error_fitted": round(p1["opara"] / m["opara"] - 1, 4),
            "opara_vs_best_baseline": {
                "measured": round(m["opara"] / min(m["dfs"], m["wavefront"]), 4),
                "simulated_fitted": round(p1["opara"] / min(p1["dfs"], p1["wavefront"]), 4)},
        })
    res = {"fitted_same_class_slowdown": best_s, "fit_configs": [r["name"] for r in fit_rows],
           "mean_abs_log_error_fitted": round(best_err, 4),
           "mean_abs_log_error_1.4": round(err(fit_rows, [predict(r, 1.4) for r in fit_rows]), 4),
           "error_curve": [(s, round(e, 4)) for e, s in sorted(fits, key=lambda t: t[1])],
           "configs": table,
           "note": "block durations = each op's isolated in-graph time / its waves (engine.block_duration_us); "
                   "sequential makespan is calibrated by construction (sum of isolated times), so only the "
                   "multi-stream policies enter the fit"}
    out = Path(args.out)
    out.with_suffix(".json").write_text(json.dumps(res, indent=1) + "\n")
    lines = [f"# Execution-model calibration against the B200 ({Path(args.src).name})", "",
             f"Fitted `same_class_slowdown` = **{best_s}** (grid 1.00-4.00): mean |log(pred/meas)| over "
             f"opara/dfs/wavefront of the {len(fit_rows)} block-bound configs = {best_err:.3f} (reference default 1.4: "
             f"{err(fit_rows, [predict(r, 1.4) for r in fit_rows]):.3f}).  DeepFM is excluded from the fit: its "
             f"sub-microsecond kernels are bound by the graph launch front end, which the model has no term for.", "",
             "| config | V | measured opara / seq ms | sim@1.4 opara / seq | sim@fit opara / seq | "
             "speed-up meas / sim@1.4 / sim@fit | opara err @fit | opara/best(dfs,wf) meas / sim |",
             "|---|---:|---|---|---|---|---:|---|"]
    for t in table:
        m, a, b, s = (t["measured_ms"], t["simulated_ms_slowdown_1.4"], t["simulated_ms_fitted"],
                      t["speedup_vs_sequential"])
        lines.append(f"| {t['config']} | {t['nodes']} | {m['opara']:.4f} / {m['sequential']:.4f} | "
                     f"{a['opara']:.4f} / {a['sequential']:.4f} | {b['opara']:.4f} / {b['sequential']:.4f} | "
                     f"{s['measured']} / {s['simulated_1.4']} / {s['simulated_fitted']} | "
                     f"{t['opara_prediction_error_fitted']:+.1%} | {t['opara_vs_best_baseline']['measured']} / "
                     f"{t['opara_vs_best_baseline']['simulated_fitted']} |")
    lines += ["", res["note"] + "."]
    out.with_suffix(".md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    return 0


if __name__ == "__main__":
    sys.exit(main())
