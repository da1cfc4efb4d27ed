"""Benchmark: batch-1 inference through the Opara multi-stream CUDA Graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model inception_v3|googlenet]
    python bench.py --impl reference ...     # the reference's CPU path (oracle port)

A "step" is one batch-1 inference = one replay of the captured graph.  Every
rank (one per GPU, torchrun for N > 1) owns an independent replica — the path
does not shard, there is no collective on the data path; the
only cross-rank traffic is the max-over-ranks timing reduction.

The JSON line carries: value (whole-job inferences/s, device-timed, L2
flushed before every step), latency and the speed-up over the sequential
single-stream CUDA Graph of the same kernels, the DAG roofline fraction, the
dominant kernel's roofline, e2e (pinned host input -> H2D -> replay -> D2H of
the logits, through ScheduledGraph.run_host), clocks sampled during the timed
region, and cpu_baseline (the reference's CPU path: oracle port of
allocate_streams + order_opara + simulate on the same profiled DAG).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FP32_SIMT_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 TF/s FFMA, nominal


def _peaks():
    try:
        d = json.loads(PEAKS_FILE.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi sampled every 100 ms while the timed region (plus untimed
    replays around it, so short regions are covered) runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------ CPU baseline


def _cpu_sim_worker(args):
    """One process: oracle allocate_streams + order_opara + simulate, repeated
    until `budget_s` elapses.  Returns (runs, seconds)."""
    graph_dict, cfg, budget_s = args
    sys.path.insert(0, str(ROOT))
    from oracle import opsched_oracle as orc
    runs = 0
    t0 = time.perf_counter()
    while True:
        g = orc.Dag(graph_dict["nodes"], graph_dict["edges"])
        a, ns, sync = orc.allocate_streams(g)
        order = orc.order_opara(g, cfg)
        orc.simulate_makespan_ns(g, a, ns, sync, order, cfg)
        runs += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            return runs, el


def cpu_reference(graph_dict: dict, cfg: dict, budget_s: float, procs: int) -> dict:
    """The reference's CPU path on this host: `procs` processes in parallel."""
    if procs <= 1:
        runs, el = _cpu_sim_worker((graph_dict, cfg, budget_s))
        total = runs / el
    else:
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            res = pool.map(_cpu_sim_worker, [(graph_dict, cfg, budget_s)] * procs)
        total = sum(r / e for r, e in res)
        runs = sum(r for r, _ in res)
    return {"value": total, "runs": runs}


# ----------------------------------------------------------------- GPU arm


def build_workload(args):
    """(model, reference model, example input(s)) of the configured workload."""
    from paper_2312_10351_b200 import zoo
    if args.model == "bert_base":
        model, ref_model, x = zoo.build_bert()
        args.dtype = "bf16"  # BASELINE config: BERT-base seq 128 bf16
        return model, ref_model, x
    if args.model == "deepfm":
        model, x = zoo.build_deepfm(args.batch)
        args.dtype = "f32"   # fp32 recommendation model (the MLP runs on the exact-fp32 engine)
        return model, model, x
    model, x = zoo.build(args.model, batch=args.batch)
    return model, model, x


def workload_name(args, x) -> str:
    shape = "+".join("x".join(map(str, t.shape)) for t in (x if isinstance(x, tuple) else (x,)))
    return f"{args.model} batch={args.batch} {args.dtype} ({shape})"


def broadcast_value(dist, rank: int, compute):
    """compute() on rank 0, its (picklable) result on every rank."""
    box = [compute() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def run_gpu(args) -> dict | None:
    import torch
    import torch.distributed as dist

    world, rank, local = _dist()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False

    from paper_2312_10351_b200 import engine, zoo
    from paper_2312_10351_b200.dag import graph_to_dict

    model, ref_model, x = build_workload(args)
    bound = {"auto": "auto", "bounded": True, "full": False}[args.grids]
    if world > 1 and bound == "auto":
        # replicas run identical graphs: rank 0 searches the sizing variants and
        # tiles once, the other ranks compile its choice from the shared tuning cache
        import tempfile
        os.environ["OPARA_TUNE_CACHE"] = broadcast_value(dist, rank, lambda: os.environ.get("OPARA_TUNE_CACHE") or
                                                         os.path.join(tempfile.gettempdir(),
                                                                      f"opara_tune_{os.getpid()}.json"))
        sg = None
        if rank == 0:
            sg = engine.compile(model, x, device=local, bound_grids="auto", profile_reps=args.profile_reps,
                                dtype=args.dtype)
        bounded, splitk, scale = broadcast_value(dist, rank, lambda: (sg.bound_grids, sg.splitk, sg.bound_scale))
        if rank != 0:
            program = engine.lower(model, x, args.dtype)
            sg = engine.ScheduledGraph(program, local, profile_reps=args.profile_reps, bound_grids=bounded,
                                       splitk=splitk, bound_scale=scale)
    else:
        sg = engine.compile(model, x, device=local, bound_grids=bound, profile_reps=args.profile_reps,
                            dtype=args.dtype)
    xd = tuple(t.cuda(local) for t in x) if isinstance(x, tuple) else x.cuda(local)
    # correctness guard on every rank: a fast wrong answer is not a result
    y = sg.run(xd)
    y = y[0] if isinstance(y, tuple) else y
    with torch.no_grad():
        ref = ref_model.cuda(local)(*xd) if isinstance(xd, tuple) else ref_model.cuda(local)(xd)
    ref = ref[0] if isinstance(ref, tuple) else ref
    y = y.float().reshape(ref.shape)
    rel = (torch.linalg.vector_norm(y - ref) / torch.linalg.vector_norm(ref)).item()
    ref_model.cpu()
    del ref
    torch.cuda.synchronize()

    # device-timed K steps per slot, L2 flushed before every step (outside the bracket)
    for _ in range(args.warmup):
        sg.replay(engine.SLOT_PARALLEL)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        # keep the GPU busy with (untimed) replays for ~0.6 s before and ~0.3 s
        # after the timed region so the 100 ms nvidia-smi sampler sees it loaded
        lat0 = sg.time(engine.SLOT_PARALLEL, warmup=1, iters=5, flush_l2=False).median_ms
        roll = min(20000, max(1, int(600.0 / max(lat0, 0.01))))   # ~0.6 s of replays
        if not args.profile_region:
            sg.time(engine.SLOT_PARALLEL, warmup=0, iters=roll, flush_l2=False)
        torch.cuda.synchronize()
        if args.profile_region:   # ncu --profile-from-start off: capture only the timed replays
            torch.cuda.cudart().cudaProfilerStart()
        t_par = sg.time(engine.SLOT_PARALLEL, warmup=args.warmup, iters=args.steps, flush_l2=True)
        torch.cuda.synchronize()
        if args.profile_region:
            torch.cuda.cudart().cudaProfilerStop()
        else:
            sg.time(engine.SLOT_PARALLEL, warmup=0, iters=max(1, roll // 2), flush_l2=False)
            torch.cuda.synchronize()
    t_seq = sg.time(engine.SLOT_SEQUENTIAL, warmup=args.warmup, iters=args.steps, flush_l2=True)
    t_warm = sg.time(engine.SLOT_PARALLEL, warmup=args.warmup, iters=args.steps, flush_l2=False)
    t_seq_warm = sg.time(engine.SLOT_SEQUENTIAL, warmup=args.warmup, iters=args.steps, flush_l2=False)
    step_total_s = sum(t_par.samples) / 1e3

    # launch-order sensitivity (the paper's Fig. 2 question): the same kernels and
    # Alg. 1 plan captured with the baseline orders, timed like the Opara graph
    orders = {}
    from paper_2312_10351_b200.order import make_order
    for slot, pol in ((10, "dfs"), (11, "wavefront")):
        sg.capture(slot, sg.plan, make_order(sg.graph, pol, sg.gpu_config))
        orders[pol] = round(sg.time(slot, warmup=args.warmup, iters=args.steps, flush_l2=True).median_ms, 4)

    # e2e through the public API: pinned host in -> H2D -> replay -> D2H logits
    e2e = sg.time_host_roundtrip(x, warmup=args.warmup, iters=args.steps)

    if world > 1:
        tt = torch.tensor([step_total_s, e2e["seconds"]], dtype=torch.float64, device=torch.device("cuda", local))
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_total_s, e2e_s = tt.tolist()
    else:
        e2e_s = e2e["seconds"]

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    peaks = _peaks()
    work = sg.work()
    cp_us = sg.critical_path_us()
    lat_ms = t_par.median_ms
    # Compute peaks per engine.  tcgen05 kind::tf32 runs at half the bf16 rate
    # (tensor throughput scales with operand bytes), and 3xTF32 issues three
    # MMAs per product: effective peak = measured bf16 / 2 / 3.  The SIMT
    # engine's peak is the nominal fp32 FFMA rate (no measured figure exists).
    tc_peak_tflops = peaks["bf16_tflops"] / 2 / 3
    fam = {}
    for k, (op, p) in enumerate(zip(sg.program.ops, sg.profile)):
        if op.kind == 0:
            continue
        if op.kind == 1:
            name = {0: "conv2d_f32_simt", 1: "conv2d_tc_tf32x3", 2: "conv2d_tc_bf16"}[sg.engines[k]]
        else:
            name = {2: "maxpool2d", 3: "avgpool2d", 4: "global_avgpool", 5: "linear_f32", 6: "add",
                    7: "layernorm", 9: "embedding", 10: "attention_tc", 11: "copy", 12: "fm", 13: "dwconv2d",
                    14: "relu", 16: "field_embedding", 17: "first_order", 18: "pack_input"}[op.kind]
        f = fam.setdefault(name, {"us": 0.0, "flops": 0, "bytes": 0, "launches": 0})
        f["us"] += p["isolated_us"]
        f["flops"] += op.flops
        f["bytes"] += op.bytes_min
        f["launches"] += 1
    peak_of = {"conv2d_tc_tf32x3": tc_peak_tflops, "conv2d_f32_simt": FP32_SIMT_NOMINAL_TFLOPS,
               "linear_f32": FP32_SIMT_NOMINAL_TFLOPS, "conv2d_tc_bf16": peaks["bf16_tflops"],
               "attention_tc": peaks["bf16_tflops"]}
    # DAG roofline: max(critical path, FLOPs at compute peak + bytes at HBM peak)
    flop_term_us = sum(f["flops"] / (peak_of.get(k, FP32_SIMT_NOMINAL_TFLOPS) * 1e12) * 1e6
                       for k, f in fam.items() if k in peak_of)
    byte_term_us = work["bytes"] / (peaks["hbm_gbs"] * 1e9) * 1e6
    roof_us = max(cp_us, flop_term_us + byte_term_us)

    dom = max(fam, key=lambda k: fam[k]["us"])
    d = fam[dom]
    total_us = sum(f["us"] for f in fam.values())
    if dom in peak_of:
        achieved = d["flops"] / (d["us"] * 1e-6) / 1e12
        peak, unit, bound = peak_of[dom], "TFLOP/s", "tensor"
    else:
        achieved = d["bytes"] / (d["us"] * 1e-6) / 1e9
        peak, unit, bound = peaks["hbm_gbs"], "GB/s", "hbm"
    traffic = None
    prof = ROOT / "profiles" / f"r01_{args.model}_{args.dtype}_full.md"
    if prof.exists() and dom in prof.read_text():
        vals = {}
        for ln in prof.read_text().splitlines():
            parts = [x.strip() for x in ln.split("|")]
            if len(parts) > 3 and parts[1].startswith("dram__bytes_"):
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(parts[2], 1)
                vals[parts[1]] = float(parts[3]) * mult
        if vals:
            traffic = int(sum(vals.values()))
    roofline = {
        "kernel": dom,
        "bound": bound,
        "achieved": round(achieved, 3), "peak": round(peak, 1),
        "unit": unit, "frac": round(achieved / peak, 4),
        "peak_source": ("measured bf16 (MEASURED_PEAKS.json) / 2 (tf32 rate) / 3 (3xTF32 passes)"
                        if dom == "conv2d_tc_tf32x3" else
                        "measured bf16 dense (MEASURED_PEAKS.json)" if dom in ("conv2d_tc_bf16", "attention_tc") else
                        "nominal fp32 FFMA (148 SM x 128 lanes x 2 x 1.965 GHz)" if unit == "TFLOP/s"
                        else "measured HBM copy (MEASURED_PEAKS.json)"),
        "traffic": traffic,
        "traffic_note": f"dram read+write bytes of one {dom} launch from the committed ncu --set full capture "
                        f"({prof.name}, cold cache under ncu)" if traffic else None,
        "share_of_step": round(d["us"] / total_us, 3),
        "launches_per_step": d["launches"],
        "flops_per_step": d["flops"],
        "timing": "CUDA events around a graph of back-to-back launches of each op (opara_exec_profile), "
                  "summed over the family's launches",
    }

    # CPU baseline: the reference's path on the same profiled DAG, 1 core
    gd = graph_to_dict(sg.graph)
    gcfg = {"num_sms": sg.gpu_config.num_sms, "threads_per_sm": sg.gpu_config.threads_per_sm,
            "shared_mem_per_sm": sg.gpu_config.shared_mem_per_sm,
            "registers_per_sm": sg.gpu_config.registers_per_sm,
            "max_blocks_per_sm": sg.gpu_config.max_blocks_per_sm,
            "same_class_slowdown": sg.gpu_config.same_class_slowdown}
    cpu = cpu_reference(gd, gcfg, args.cpu_seconds, 1)

    launches = sg.num_launches(engine.SLOT_PARALLEL)
    value = world * args.batch * args.steps / step_total_s
    line = {
        "metric": "batch-1 inference throughput (inferences/s); batch-1 latency ms and speed-up vs the "
                  "sequential single-stream CUDA Graph of the same kernels reported beside it",
        "value": round(value, 2),
        "unit": "inferences/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_total_s * 1e3 / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic input, random-init weights (seed 0), BN stats randomised",
        "config": {"workload": workload_name(args, x),
                   "parallelism": f"{world} independent replica(s), no collective",
                   "l2": "flushed (256 MiB memset) before every timed step, outside the event bracket",
                   "dag_nodes": len(sg.graph), "dag_edges": len(sg.graph.edges),
                   "streams": sg.plan.num_streams, "syncs": len(sg.plan.sync_events)},
        "latency_ms": round(lat_ms, 4),
        "latency_ms_mean": round(t_par.mean_ms, 4),
        "sequential_latency_ms": round(t_seq.median_ms, 4),
        "speedup_vs_sequential": round(t_seq.median_ms / lat_ms, 4),
        "grids": "bounded" if sg.bound_grids else "full",
        "splitk_reduction": sg.splitk,
        "bound_scale": sg.bound_scale if sg.bound_grids else None,
        "conv_engines": {name: sum(1 for e in sg.engines.values() if e == code)
                         for code, name in ((0, "simt_f32"), (1, "tc_tf32x3"), (2, "tc_bf16"))},
        "grid_autotune": getattr(sg, "autotune", None),
        "sequential_best_latency_ms": round(min([t_seq.median_ms] + [a["sequential_ms"] for a in (
            getattr(sg, "autotune", None) or [])]), 4),
        "latency_warm_l2_ms": round(t_warm.median_ms, 4),
        "sequential_latency_warm_l2_ms": round(t_seq_warm.median_ms, 4),
        "speedup_vs_sequential_warm_l2": round(t_seq_warm.median_ms / t_warm.median_ms, 4),
        "launch_order_latency_ms": {"opara": round(lat_ms, 4), **orders,
                                    "sequential": round(t_seq.median_ms, 4)},
        "speedup_vs_best_sequential": round(min([t_seq.median_ms] + [a["sequential_ms"] for a in (
            getattr(sg, "autotune", None) or [])]) / lat_ms, 4),
        "dag_roofline": {"critical_path_us": round(cp_us, 2), "flop_term_us": round(flop_term_us, 2),
                         "byte_term_us": round(byte_term_us, 2), "roofline_us": round(roof_us, 2),
                         "frac": round(roof_us / (lat_ms * 1e3), 4),
                         "flops": work["flops"], "bytes": work["bytes"],
                         "compute_peak_tflops": {k: round(v, 1) for k, v in peak_of.items()},
                         "hbm_peak_gbs": peaks["hbm_gbs"]},
        "roofline": roofline,
        "rel_err_vs_torch_fp32": rel,
        "rel_tolerance": 1e-4 if args.dtype == "f32" else 1e-2,
        "e2e": {"value": round(world * args.batch * args.steps / e2e_s, 2), "unit": "inferences/s",
                "h2d_bytes_per_step": e2e["h2d_bytes"], "d2h_bytes_per_step": e2e["d2h_bytes"],
                "path": "ScheduledGraph.run_host: pinned host input(s) -> H2D -> graph replay -> "
                        "D2H of the output, per step, CUDA events around all three"},
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
        "clocks": clk.summary(),
        "cpu_baseline": {"value": round(cpu["value"] * args.batch, 3), "unit": "inferences/s", "cores": 1,
                         "kind": "port",
                         "sample": f"{cpu['runs']} runs of oracle allocate_streams + order_opara + "
                                   f"simulate (the reference's 'run') on the profiled {args.model} DAG, "
                                   f"{args.cpu_seconds:.0f} s budget, 1 process"},
        "peaks": peaks,
    }
    if world > 1:
        dist.destroy_process_group()
    return line


def run_reference(args) -> dict | None:
    """--impl reference: the reference's CPU path on all host cores."""
    world, rank, _ = _dist()
    if rank != 0:
        return None
    from paper_2312_10351_b200 import frontend
    from paper_2312_10351_b200.dag import graph_to_dict
    import paper_2312_10351_b200.engine as engine
    model, _, x = build_workload(args)
    prog = frontend.lower(model, x, args.dtype)
    g = engine.static_dag(prog)  # same topology / classes; launch-config demands
    gd = graph_to_dict(g)
    cfg = {"num_sms": 148, "threads_per_sm": 2048, "shared_mem_per_sm": 233472,
           "registers_per_sm": 65536, "max_blocks_per_sm": 32, "same_class_slowdown": 1.4}
    cores = len(os.sched_getaffinity(0))
    per_step = max(1.0, args.cpu_seconds / max(1, args.steps))
    vals = []
    for _ in range(args.warmup):
        cpu_reference(gd, cfg, 0.2, 1)
    t0 = time.perf_counter()
    runs = 0
    for _ in range(args.steps):
        r = cpu_reference(gd, cfg, per_step, cores)
        vals.append(r["value"])
        runs += r["runs"]
    el = time.perf_counter() - t0
    v = statistics.median(vals) * args.batch   # one simulated DAG run serves `batch` requests
    return {
        "impl": "reference",
        "metric": "batch-1 inference throughput (inferences/s); batch-1 latency ms and speed-up vs the "
                  "sequential single-stream CUDA Graph of the same kernels reported beside it",
        "value": round(v, 3), "unit": "inferences/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 / v, 3) if v else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic DAG of the model (launch-config demands)",
        "config": {"workload": workload_name(args, x), "path": "reference CPU path (allocate_streams + "
                               "order_opara + simulate) on the model's DAG", "processes": cores},
        "cpu_baseline": {"value": round(v, 3), "unit": "inferences/s", "cores": cores, "kind": "port",
                         "sample": f"{runs} simulated runs in {el:.1f} s across {cores} processes"},
        "e2e": {"value": round(v, 3), "unit": "inferences/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--model", default="inception_v3",
                    choices=["inception_v3", "googlenet", "bert_base", "nasnet_large", "deepfm"])
    ap.add_argument("--batch", type=int, default=1, help="requests per inference (DeepFM batch sweep 1-32)")
    ap.add_argument("--profile-region", action="store_true",
                    help="bracket the timed Opara replays with cudaProfilerStart/Stop (for ncu)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--profile-reps", type=int, default=20,
                    help="launches per op when measuring its isolated in-graph time")
    ap.add_argument("--grids", default="auto", choices=["auto", "bounded", "full"],
                    help="bounded = size each conv for its DAG level's share of the SMs (Opara bounded "
                         "grids); full = whole GPU per conv; auto = build both, keep the faster Opara graph")
    args = ap.parse_args(argv)
    args.warmup = max(3, args.warmup)
    line = run_reference(args) if args.impl == "reference" else run_gpu(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
