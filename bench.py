"""Benchmark: batch-1 inference through the Opara multi-stream CUDA Graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model inception_v3|googlenet|...]
    python bench.py --impl reference ...     # the reference's CPU path on the same DAG

A "step" is one inference of `--batch` requests = one replay of the captured
graph.  Every rank (one per GPU, torchrun for N > 1) owns an independent
replica — the path does not shard and there is no collective
on the data path.  The only cross-rank traffic is control: a gloo (CPU)
process group broadcasts rank 0's tuning choice and reduces the timed
seconds with a max — no NCCL.

The JSON line carries: value (whole-job inferences/s, device-timed, L2
flushed before every step), latency and the speed-up over the sequential
single-stream CUDA Graph of the same kernels, the DAG and hardware roofline
fractions, the dominant kernel's roofline, e2e (pinned host input -> H2D ->
replay -> D2H of the output, through ScheduledGraph.run_host), clocks sampled
during the timed region, the schedule files of the timed graph, and
cpu_baseline (the reference's CPU path — its own ``opsched`` package from
baseline/_ref, else the oracle port — on the same profiled DAG).  The run
fails (exit 1) when the timed graph's output misses the north_star tolerance
or its schedule differs from the reference's.

``--impl reference`` never imports this repo's package: it loads the
profiled DAG committed under schedules/<workload>/ (written by an earlier GPU
run of this bench) and runs load_graph + allocate_streams + order_opara +
simulate through the reference package on every host core.
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

# read once by the CUDA driver at context creation: one hardware queue per plan stream
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
SCHEDULES = ROOT / "schedules"      # committed profiled DAGs + schedules, one dir per workload
REF_PKG = ROOT / "baseline" / "_ref"  # pip --target install of the reference (stdlib-only)

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


def _reference_api():
    """"reference" when the reference's own ``opsched`` (pip-installed into
    baseline/_ref, stdlib-only) imports, else "port" (the oracle restatement)."""
    if REF_PKG.is_dir() and str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))
    try:
        import opsched  # noqa: F401
        return "reference"
    except ImportError:
        return "port"


def _cpu_sim_worker(args):
    """One process: the reference's 'scheduled graph out, run' on the DAG file —
    load_graph + allocate_streams + order_opara + simulate — repeated until
    `budget_s` elapses.  Returns (runs, seconds, kind)."""
    graph_path, cfg_path, budget_s = args
    sys.path.insert(0, str(ROOT))
    kind = _reference_api()
    runs = 0
    t0 = time.perf_counter()
    if kind == "reference":
        import opsched
        cfg = opsched.load_gpu_config(cfg_path)
        while True:
            g = opsched.load_graph(graph_path)
            plan = opsched.allocate_streams(g)
            sched = opsched.order_opara(g, cfg)
            opsched.simulate(g, plan, sched, cfg)
            runs += 1
            el = time.perf_counter() - t0
            if el >= budget_s:
                return runs, el, kind
    from oracle import opsched_oracle as orc
    cfg = json.loads(Path(cfg_path).read_text())
    while True:
        d = json.loads(Path(graph_path).read_text())
        g = orc.Dag(d["nodes"], d["edges"])
        a, ns, sync = orc.allocate_streams(g)
        order = orc.order_opara(g, cfg)
        orc.simulate_makespan_ns(g, a, ns, sync, order, cfg)
        runs += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            return runs, el, kind


def cpu_reference(graph_path, cfg_path, budget_s: float, procs: int) -> dict:
    """The reference's CPU path on this host: `procs` processes in parallel."""
    if procs <= 1:
        runs, el, kind = _cpu_sim_worker((str(graph_path), str(cfg_path), budget_s))
        total = runs / el
    else:
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            res = pool.map(_cpu_sim_worker, [(str(graph_path), str(cfg_path), budget_s)] * procs)
        total = sum(r / e for r, e, _ in res)
        runs = sum(r for r, _, _ in res)
        kind = res[0][2]
    return {"value": total, "runs": runs, "kind": kind}


def reference_schedule(graph_path, cfg_path) -> dict:
    """The checker: the reference's (or the oracle's) Alg. 1 plan and Alg. 2
    order of the DAG file, as plain data."""
    kind = _reference_api()
    if kind == "reference":
        import opsched
        g = opsched.load_graph(graph_path)
        plan = opsched.allocate_streams(g)
        order = opsched.order_opara(g, opsched.load_gpu_config(cfg_path)).order
        return {"assignment": dict(plan.assignment), "num_streams": plan.num_streams,
                "sync": [tuple(e) for e in plan.sync_events], "order": list(order), "kind": kind}
    from oracle import opsched_oracle as orc
    d = json.loads(Path(graph_path).read_text())
    g = orc.Dag(d["nodes"], d["edges"])
    a, ns, sync = orc.allocate_streams(g)
    return {"assignment": a, "num_streams": ns, "sync": [tuple(e) for e in sync],
            "order": orc.order_opara(g, json.loads(Path(cfg_path).read_text())), "kind": kind}


def cpu_model_execution(model, x, budget_s: float) -> dict:
    """BASELINE.md §3's CPU model-execution analog: PyTorch eager fp32 forward on
    every host core, repeated for `budget_s`."""
    import torch
    cores = len(os.sched_getaffinity(0))
    prev = torch.get_num_threads()
    torch.set_num_threads(cores)
    model = model.cpu().eval()
    xs = tuple(t.cpu() for t in x) if isinstance(x, tuple) else (x.cpu(),)
    runs = 0
    with torch.no_grad():
        model(*xs)
        t0 = time.perf_counter()
        while True:
            model(*xs)
            runs += 1
            el = time.perf_counter() - t0
            if el >= budget_s:
                break
    torch.set_num_threads(prev)
    return {"runs": runs, "seconds": el, "cores": cores}


# ----------------------------------------------------------------- GPU arm


def build_workload(args):
    """(model, reference model, example input(s)) of the configured workload."""
    from paper_2312_10351_b200 import zoo
    if args.model == "bert_base":
        model, ref_model, x = zoo.build_bert()
        return model, ref_model, x
    if args.model == "deepfm":
        model, x = zoo.build_deepfm(args.batch)
        return model, model, x
    model, x = zoo.build(args.model, batch=args.batch)
    return model, model, x


def resolve_dtype(args) -> None:
    if args.model == "bert_base":
        args.dtype = "bf16"  # BASELINE config: BERT-base seq 128 bf16
    elif args.model == "deepfm":
        args.dtype = "f32"   # fp32 recommendation model (exact-fp32 engines)


def workload_key(args) -> str:
    return f"{args.model}_{args.dtype}_b{args.batch}"


def workload_name(args, x) -> str:
    shape = "+".join("x".join(map(str, t.shape)) for t in (x if isinstance(x, tuple) else (x,)))
    return f"{args.model} batch={args.batch} {args.dtype} ({shape})"


def bench_config(meta: dict, world: int) -> dict:
    """The `config` object both arms print (same workload, same DAG)."""
    return {"workload": meta["workload"], "parallelism": f"{world} independent replica(s), no collective",
            "l2": "flushed (256 MiB memset) before every timed step, outside the event bracket",
            "dag_nodes": meta["dag_nodes"], "dag_edges": meta["dag_edges"],
            "streams": meta["streams"], "syncs": meta["syncs"], "schedule": meta["schedule"]}


def broadcast_value(dist, rank: int, compute):
    """compute() on rank 0, its (picklable) result on every rank."""
    box = [compute() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def replica_compile(dist, rank: int, world: int, search, build_choice, cache_dir):
    """Replicas run identical graphs.  Rank 0 runs `search(cache_path)` (the
    sizing-variant search, which writes its tile choices into the tuning cache
    file), then broadcasts its variant and the cache CONTENTS; every other rank
    writes them into its own local cache file and calls
    `build_choice(variant, cache_path)`.  Control traffic only, over the
    (gloo) process group.  Returns (scheduled graph, variant)."""
    cache = os.path.join(cache_dir, f"opara_tune_rank{rank}.json")
    sg = search(cache) if rank == 0 else None
    variant, text = broadcast_value(dist, rank, lambda: (sg_variant(sg), Path(cache).read_text()
                                                         if os.path.exists(cache) else "{}"))
    if rank != 0:
        Path(cache).write_text(text)
        sg = build_choice(variant, cache)
    return sg, variant


def sg_variant(sg) -> tuple:
    return (bool(sg.bound_grids), sg.splitk, sg.bound_scale)


def time_max(dist, world: int, values: list[float]) -> list[float]:
    """Max over ranks of per-rank device-timed seconds (gloo, CPU tensors)."""
    if world <= 1:
        return values
    import torch
    t = torch.tensor(values, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def measure_tf32_tflops(dev) -> float:
    """Dense TF32 tensor throughput of this GPU (cuBLAS 8192^3 GEMM, TF32 on):
    the measured denominator of the 3xTF32 engine's roofline (÷3 passes)."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    e0.record()
    for _ in range(it):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    torch.backends.cuda.matmul.allow_tf32 = old
    ms = e0.elapsed_time(e1) / it
    del a, b
    return 2 * n ** 3 / (ms * 1e-3) / 1e12


def save_schedule(sg, args, meta: dict, root: Path) -> Path:
    """The timed graph's profiled DAG, plan, order and GpuConfig (reference file
    formats) plus the workload meta, so the numbers tie to a re-checkable schedule."""
    from paper_2312_10351_b200.device import gpu_config_to_dict
    d = root / workload_key(args)
    sg.save(d)
    (d / "gpu_config.json").write_text(json.dumps(gpu_config_to_dict(sg.gpu_config), indent=2, sort_keys=True) + "\n")
    (d / "meta.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    return d


def run_gpu(args) -> tuple[dict | None, int]:
    import torch
    import torch.distributed as dist

    world, rank, local = _dist()
    if world > 1:
        # control plane only (tuning choice broadcast, max-over-ranks timing): gloo on the host
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False

    from paper_2312_10351_b200 import engine

    model, ref_model, x = build_workload(args)
    bound = {"auto": "auto", "bounded": True, "full": False}[args.grids]

    def compile_auto(cache_path=None):
        if cache_path:
            os.environ["OPARA_TUNE_CACHE"] = cache_path
        return engine.compile(model, x, device=local, bound_grids=bound, profile_reps=args.profile_reps,
                              dtype=args.dtype)

    def compile_choice(variant, cache_path):
        os.environ["OPARA_TUNE_CACHE"] = cache_path
        bounded, splitk, scale = variant
        return engine.ScheduledGraph(engine.lower(model, x, args.dtype), local, profile_reps=args.profile_reps,
                                     bound_grids=bounded, splitk=splitk, bound_scale=scale)

    if world > 1:
        import tempfile
        sg, _ = replica_compile(dist, rank, world, compile_auto, compile_choice, tempfile.gettempdir())
    else:
        sg = compile_auto()
    xd = tuple(t.cuda(local) for t in x) if isinstance(x, tuple) else x.cuda(local)
    # correctness gate on every rank, on the graph that is timed: a fast wrong answer is not a result
    y = sg.run(xd)
    y = y[0] if isinstance(y, tuple) else y
    with torch.no_grad():
        ref = ref_model.cuda(local)(*xd) if isinstance(xd, tuple) else ref_model.cuda(local)(xd)
    ref = ref[0] if isinstance(ref, tuple) else ref
    y = y.float().reshape(ref.shape)
    rel = (torch.linalg.vector_norm(y.double() - ref.double()) / torch.linalg.vector_norm(ref.double())).item()
    tol = 1e-4 if args.dtype == "f32" else 1e-2
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
    # diagnostic (not a reference policy): longest-remaining-path-first list order
    # over the profiled kernel times, the order the B200 sub-DAG search favours
    from paper_2312_10351_b200.order import LaunchSchedule
    from paper_2312_10351_b200.search import critical_path_first_order
    cpf = critical_path_first_order(sg.graph, {v: sg.profile[v - 1]["isolated_us"] for v in sg.graph.node_ids})
    sg.capture(12, sg.plan, LaunchSchedule(cpf, "critical_path_first"))
    orders["critical_path_first"] = round(sg.time(12, warmup=args.warmup, iters=args.steps,
                                                  flush_l2=True).median_ms, 4)

    # e2e through the public API: pinned host in -> H2D -> replay -> D2H output
    e2e = sg.time_host_roundtrip(x, warmup=args.warmup, iters=args.steps)

    step_total_s, e2e_s = time_max(dist, world, [step_total_s, e2e["seconds"]])
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None, 0 if rel <= tol else 1

    peaks = _peaks()
    tf32_tflops = measure_tf32_tflops(sg.dev)
    work = sg.work()
    cp_us = sg.critical_path_us()
    lat_ms = t_par.median_ms
    # compute peaks per engine: 3xTF32 = measured TF32 / 3 passes; bf16 = measured
    # (MEASURED_PEAKS.json); the SIMT engine's peak is the nominal fp32 FFMA rate
    tc_peak_tflops = tf32_tflops / 3
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
        peak, unit, bound_kind = peak_of[dom], "TFLOP/s", "tensor"
    else:
        achieved = d["bytes"] / (d["us"] * 1e-6) / 1e9
        peak, unit, bound_kind = peaks["hbm_gbs"], "GB/s", "hbm"
    traffic, traffic_note = _ncu_traffic(args, dom)
    roofline = {
        "kernel": dom,
        "bound": bound_kind,
        "achieved": round(achieved, 3), "peak": round(peak, 1),
        "unit": unit, "frac": round(achieved / peak, 4),
        "peak_source": ("measured TF32 (cuBLAS 8192^3 GEMM, TF32 on, this run) / 3 (3xTF32 passes)"
                        if dom == "conv2d_tc_tf32x3" else
                        "measured bf16 dense (MEASURED_PEAKS.json)" if dom in ("conv2d_tc_bf16", "attention_tc") else
                        "nominal fp32 FFMA (148 SM x 128 lanes x 2 x 1.965 GHz)" if unit == "TFLOP/s"
                        else "measured HBM copy (MEASURED_PEAKS.json)"),
        "traffic": traffic,
        "traffic_note": traffic_note,
        "share_of_step": round(d["us"] / total_us, 3),
        "launches_per_step": d["launches"],
        "flops_per_step": d["flops"],
        "bytes_per_step": d["bytes"],
        "avg_launch_us": round(d["us"] / d["launches"], 3),
        "timing": "CUDA events around a graph of back-to-back launches of each op (opara_exec_profile), "
                  "summed over the family's launches",
    }

    # the timed graph's schedule, saved in the reference's file formats and
    # re-checked against the reference's own Alg. 1 / Alg. 2 on the same DAG file
    meta = {"workload": workload_name(args, x), "dag_nodes": len(sg.graph), "dag_edges": len(sg.graph.edges),
            "streams": sg.plan.num_streams, "syncs": len(sg.plan.sync_events),
            "schedule": f"schedules/{workload_key(args)}"}
    out_root = Path(args.save_schedule) if args.save_schedule else ROOT / "gpurun_out" / "schedules"
    sdir = save_schedule(sg, args, meta, out_root)
    chk = reference_schedule(sdir / "graph.json", sdir / "gpu_config.json")
    sched_ok = (chk["assignment"] == dict(sg.plan.assignment) and chk["num_streams"] == sg.plan.num_streams
                and chk["sync"] == [tuple(e) for e in sg.plan.sync_events]
                and chk["order"] == list(sg.schedule.order))

    cpu = cpu_reference(sdir / "graph.json", sdir / "gpu_config.json", args.cpu_seconds, 1)
    cpu_exec = cpu_model_execution(ref_model, x, args.cpu_model_seconds) if args.cpu_model_seconds > 0 else None

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
        "config": bench_config(meta, world),
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
                         "hw_frac": round((flop_term_us + byte_term_us) / (lat_ms * 1e3), 4),
                         "note": "frac = north_star DAG roofline (critical path of this build's own isolated "
                                 "kernel times); hw_frac = hardware term only (FLOPs at peak + bytes at HBM)",
                         "flops": work["flops"], "bytes": work["bytes"],
                         "compute_peak_tflops": {k: round(v, 1) for k, v in peak_of.items()},
                         "tf32_tflops_measured": round(tf32_tflops, 1),
                         "hbm_peak_gbs": peaks["hbm_gbs"]},
        "roofline": roofline,
        "rel_err_vs_torch_fp32": rel,
        "rel_tolerance": tol,
        "parity_ok": rel <= tol,
        "schedule_parity": {"ok": sched_ok, "checker": chk["kind"],
                            "files": [f"{meta['schedule']}/{n}" for n in
                                      ("graph.json", "plan.json", "order.json", "gpu_config.json")],
                            "written_to": str(sdir.relative_to(ROOT)) if sdir.is_relative_to(ROOT) else str(sdir)},
        "e2e": {"value": round(world * args.batch * args.steps / e2e_s, 2), "unit": "inferences/s",
                "h2d_bytes_per_step": e2e["h2d_bytes"], "d2h_bytes_per_step": e2e["d2h_bytes"],
                "path": "ScheduledGraph.run_host: pinned host input(s) -> H2D -> graph replay -> "
                        "D2H of the output, per step, CUDA events around all three"},
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
        "clocks": clk.summary(),
        "cpu_baseline": {"value": round(cpu["value"] * args.batch, 3), "unit": "inferences/s", "cores": 1,
                         "kind": cpu["kind"],
                         "sample": f"{cpu['runs']} runs of load_graph + allocate_streams + order_opara + "
                                   f"simulate (the reference's 'scheduled graph out, run') on this run's "
                                   f"profiled {args.model} DAG file, {args.cpu_seconds:.0f} s budget, 1 process"},
        "cpu_model_execution": None if cpu_exec is None else {
            "value": round(cpu_exec["runs"] * args.batch / cpu_exec["seconds"], 3), "unit": "inferences/s",
            "cores": cpu_exec["cores"],
            "sample": f"PyTorch eager fp32 forward of the same model on the host, torch.set_num_threads("
                      f"{cpu_exec['cores']}), {cpu_exec['runs']} runs in {cpu_exec['seconds']:.1f} s"},
        "peaks": peaks,
        "version": _version(),
    }
    if world > 1:
        dist.destroy_process_group()
    return line, 0 if (rel <= tol and sched_ok) else 1


def _version() -> str:
    from paper_2312_10351_b200 import _lib
    return _lib.version()


def _ncu_traffic(args, dom: str):
    """DRAM bytes of one launch of the dominant kernel from the committed
    `ncu --set full` summary of this workload (newest round first)."""
    for rnd in ("r02", "r01"):
        prof = ROOT / "profiles" / f"{rnd}_{args.model}_{args.dtype}_full.md"
        if not prof.exists() or dom not in prof.read_text():
            continue
        vals, shape = {}, None
        for ln in prof.read_text().splitlines():
            parts = [x.strip() for x in ln.split("|")]
            if len(parts) > 3 and parts[1] == f"family dram bytes per launch: {dom}":
                # mean over every launch of the family in one timed step (launch list pass)
                return int(float(parts[3])), (f"dram read+write bytes per {dom} launch, averaged over every "
                                              f"launch of one timed step (ncu launch-list pass, {prof.name})")
            if len(parts) > 3 and parts[1].startswith("dram__bytes_"):
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(parts[2], 1)
                vals[parts[1]] = float(parts[3]) * mult
            if len(parts) > 3 and parts[1] == "conv shape":
                shape = parts[3]
        if vals:
            note = (f"dram read+write bytes of one {dom} launch from the committed ncu --set full capture "
                    f"({prof.name}, cold cache under ncu)" + (f"; launch shape {shape}" if shape else ""))
            return int(sum(vals.values())), note
    return None, None


def run_reference(args) -> dict | None:
    """--impl reference: the reference's CPU path on all host cores, on the
    profiled DAG the GPU arm scheduled (committed under schedules/).  Imports
    nothing from this repo's package."""
    world, rank, _ = _dist()
    if rank != 0:
        return None
    sdir = SCHEDULES / workload_key(args)
    if not (sdir / "graph.json").exists():
        return {"impl": "reference", "unavailable": f"no committed profiled DAG at {sdir.relative_to(ROOT)}"}
    meta = json.loads((sdir / "meta.json").read_text())
    graph, cfgp = sdir / "graph.json", sdir / "gpu_config.json"
    cores = len(os.sched_getaffinity(0))
    per_step = max(1.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(args.warmup):
        cpu_reference(graph, cfgp, 0.2, 1)
    vals, runs, kind = [], 0, None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = cpu_reference(graph, cfgp, per_step, cores)
        vals.append(r["value"])
        runs += r["runs"]
        kind = r["kind"]
    el = time.perf_counter() - t0
    v = statistics.median(vals) * args.batch   # one scheduled + simulated DAG run serves `batch` requests
    return {
        "impl": "reference",
        "metric": "batch-1 inference throughput (inferences/s); batch-1 latency ms and speed-up vs the "
                  "sequential single-stream CUDA Graph of the same kernels reported beside it",
        "value": round(v, 3), "unit": "inferences/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 / v, 3) if v else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "the GPU arm's profiled DAG of the synthetic model (committed schedule files)",
        "config": bench_config(meta, world),
        "path": ("the reference package itself (baseline/_ref/opsched): load_graph + allocate_streams + "
                 "order_opara + simulate" if kind == "reference" else
                 "oracle port of load_graph + allocate_streams + order_opara + simulate"),
        "cpu_baseline": {"value": round(v, 3), "unit": "inferences/s", "cores": cores, "kind": kind,
                         "sample": f"{runs} scheduled+simulated runs of {sdir.relative_to(ROOT)}/graph.json "
                                   f"in {el:.1f} s across {cores} processes"},
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
    ap.add_argument("--cpu-model-seconds", type=float, default=3.0,
                    help="budget of the PyTorch-eager CPU forward baseline (0 = skip)")
    ap.add_argument("--save-schedule", default=None,
                    help="directory for the timed graph's schedule files (default gpurun_out/schedules)")
    args = ap.parse_args(argv)
    args.warmup = max(3, args.warmup)
    resolve_dtype(args)
    if args.impl == "reference":
        line, rc = run_reference(args), 0
    else:
        line, rc = run_gpu(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    if rc:
        print("bench: the timed graph failed its parity gate (output tolerance or schedule)", file=sys.stderr)
    return rc


if __name__ == "__main__":
    sys.exit(main())
