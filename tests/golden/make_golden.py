"""Generate the scheduler golden vectors FROM THE REFERENCE ITSELF.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports the reference ``opsched`` package (pure Python, stdlib only) from
/root/reference/pkg/src, builds the graphs its own tests use (generators,
seeded ``random_dag`` corpora with the seeds of test_allocator.py:20,
test_orderer.py:27, test_simulator.py:208, test_acceptance.py:77) and records
what the reference computes: topological order, Alg. 1 plan, Alg. 2 order,
the baseline orders and simulated makespans.  The output
``sched_golden.json`` is committed; tests never read /root/reference.

Graph encoding (compact): node = [id, class(0=compute,1=memory), blocks,
threads_per_block, shared_mem_bytes, registers_per_thread, block_duration_us].
"""

from __future__ import annotations

import json
import os
import sys
import warnings
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).with_name("sched_golden.json")


def main() -> None:
    sys.path.insert(0, str(REF))
    import opsched
    from opsched import (ComputationGraph, GpuConfig, OpClass, OperatorNode, ResourceDemand,
                         allocate_streams, make_order, simulate, single_stream_plan, GPU_PRESETS)
    from opsched import generators as gen

    warnings.simplefilter("ignore")

    def mk(nid, name="conv", dur=10.0, blocks=1, threads=256, smem=0, regs=32, cls=None):
        if cls is None:
            cls = OpClass.COMPUTE if name in ("conv", "matmul", "gemm") else OpClass.MEMORY
        return OperatorNode(nid, name, cls, ResourceDemand(threads, smem, regs, blocks), dur)

    def antichain(n, **kw):
        return ComputationGraph([mk(i, **kw) for i in range(1, n + 1)], [])

    def hog_and_chains():
        nodes = [mk(1, "conv", dur=200, blocks=2, threads=900)]
        edges, nid = [], 1
        for _ in range(4):
            nid += 1
            root = nid
            nodes.append(mk(root, "conv", dur=25, threads=224))
            prev = root
            for _ in range(20):
                nid += 1
                nodes.append(mk(nid, "conv", dur=10, threads=32))
                edges.append((prev, nid))
                prev = nid
        return ComputationGraph(nodes, edges)

    configs = {
        "orderer_cfg": GpuConfig(1, 1000, 65536, 65536, 16),
        "2080s-like": GPU_PRESETS["2080s-like"],
        "a100-like": GPU_PRESETS["a100-like"],
        "b200-like": GpuConfig(148, 2048, 233472, 65536, 32),
        "crit5": GpuConfig(2, 1024, 65536, 65536, 16, 1.0),
        "crit6": GpuConfig(1, 1024, 65536, 65536, 16, 1.4),
    }

    graphs: list[tuple[str, object]] = []
    graphs += [(f"antichain{n}", antichain(n)) for n in (1, 2, 5)]
    graphs += [(f"chain{n}", gen.chain(n)) for n in (1, 2, 3, 5, 12)]
    graphs += [(f"fork{k}", gen.fork(k)) for k in (1, 2, 3, 5)]
    graphs += [("diamond", gen.diamond()), ("cases13", gen.placement_cases()),
               ("inception3x2", gen.inception_block(3, 2)), ("inception4x3", gen.inception_block(4, 3))]
    graphs.append(("orderer_four", ComputationGraph(
        [mk(1, "relu", threads=100), mk(2, "conv", threads=50),
         mk(3, "relu", threads=30), mk(4, "conv", threads=200)], [])))
    graphs.append(("orderer_fork", ComputationGraph(
        [mk(1, "conv", threads=100), mk(2, "relu", threads=20), mk(3, "conv", threads=10)],
        [(1, 2), (1, 3)])))
    graphs.append(("orderer_uniform", ComputationGraph(
        [mk(i, "conv", threads=64) for i in range(1, 8)],
        [(1, 3), (1, 4), (2, 5), (3, 6), (4, 6), (5, 7)])))
    graphs.append(("crit6", ComputationGraph(
        [mk(i, "relu", dur=100, threads=512) for i in range(1, 5)]
        + [mk(i, "conv", dur=100, threads=512) for i in range(5, 9)], [])))
    graphs.append(("hog_and_chains", hog_and_chains()))
    graphs.append(("dfs_two_chains", ComputationGraph(
        [mk(i) for i in range(1, 7)], [(1, 3), (3, 5), (2, 4), (4, 6)])))
    graphs += [(f"alloc_corpus_{i}", gen.random_dag(3 + i % 12, max_width=4, seed=200 + i)) for i in range(30)]
    graphs += [(f"order_corpus_{i}", gen.random_dag(3 + i % 12, max_width=4, seed=300 + i)) for i in range(30)]
    graphs += [(f"sim_corpus_{i}", gen.random_dag(4 + i % 20, max_width=5, seed=500 + i)) for i in range(30)]
    graphs += [(f"crit3_{i}", gen.random_dag(5 + (i % 26), max_width=6, seed=1000 + i)) for i in range(0, 200, 4)]
    graphs += [(f"wide_{s}", gen.random_dag(300, max_width=20, seed=s)) for s in (1, 2, 3)]
    graphs.append(("big_4242", gen.random_dag(2000, max_width=20, seed=4242)))

    cases = []
    for name, g in graphs:
        nodes = [[n.id, 0 if n.op_class is OpClass.COMPUTE else 1, n.demand.num_blocks,
                  n.demand.threads_per_block, n.demand.shared_mem_per_block,
                  n.demand.registers_per_thread, n.block_duration_us] for n in g.nodes]
        plan = allocate_streams(g)
        rec = {
            "name": name,
            "nodes": nodes,
            "edges": [list(e) for e in g.edges],
            "topo": g.topo_sort(),
            "assignment": [[v, plan.assignment[v]] for v in sorted(plan.assignment)],
            "num_streams": plan.num_streams,
            "sync": [list(e) for e in plan.sync_events],
            "orders": {},
            "makespan_ns": {},
        }
        small = len(g) <= 400
        for cname, cfg in configs.items():
            rec["orders"][cname] = {
                "opara": list(make_order(g, "opara", cfg).order),
            }
            if cname == "b200-like":
                for pol in ("sequential", "dfs", "wavefront"):
                    rec["orders"][cname][pol] = list(make_order(g, pol, cfg).order)
            feasible = all(
                n.demand.threads_per_block <= cfg.threads_per_sm
                and n.demand.shared_mem_per_block <= cfg.shared_mem_per_sm
                and n.demand.registers_per_block <= cfg.registers_per_sm for n in g.nodes)
            if small and feasible and cname in ("2080s-like", "b200-like", "crit5", "crit6"):
                rec["makespan_ns"][cname] = {
                    "opara": simulate(g, plan, make_order(g, "opara", cfg), cfg).makespan_ns,
                    "sequential": simulate(g, single_stream_plan(g), g.topo_sort(), cfg).makespan_ns,
                }
        cases.append(rec)

    out = {
        "generator": "tests/golden/make_golden.py",
        "reference": f"opsched {opsched.__version__} @ /root/reference/pkg/src",
        "configs": {k: {"num_sms": c.num_sms, "threads_per_sm": c.threads_per_sm,
                        "shared_mem_per_sm": c.shared_mem_per_sm,
                        "registers_per_sm": c.registers_per_sm,
                        "max_blocks_per_sm": c.max_blocks_per_sm,
                        "same_class_slowdown": c.same_class_slowdown}
                    for k, c in configs.items()},
        "cases": cases,
    }
    OUT.write_text(json.dumps(out, separators=(",", ":")) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(cases)} cases)")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def model_dags() -> None:
    """Model DAG fixtures: the DAGs our frontend extracts for every
    BASELINE config (GoogLeNet, Inception-v3, NASNet-A Large, BERT-base,
    DeepFM at batch 1 and 32; static launch-config demands), scheduled by the
    REFERENCE (its own load_graph / allocate_streams / make_order)."""
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
    from opsched import GpuConfig, allocate_streams, make_order
    from opsched.graph import load_graph
    from paper_2312_10351_b200 import engine, frontend, zoo
    from paper_2312_10351_b200.dag import graph_to_dict
    import tempfile

    cfg = GpuConfig(148, 2048, 233472, 65536, 32)
    out = {}
    workloads = {
        "googlenet": lambda: zoo.build("googlenet") + ("f32",),
        "inception_v3": lambda: zoo.build("inception_v3") + ("f32",),
        "nasnet_large": lambda: zoo.build("nasnet_large") + ("f32",),
        "bert_base": lambda: (zoo.build_bert()[0], zoo.build_bert()[2], "bf16"),
        "deepfm": lambda: zoo.build_deepfm(1) + ("f32",),
        "deepfm_b32": lambda: zoo.build_deepfm(32) + ("f32",),
    }
    for name, make in workloads.items():
        model, x, dtype = make()
        g = engine.static_dag(frontend.lower(model, x, dtype))
        d = graph_to_dict(g)
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            json.dump(d, f)
        rg = load_graph(f.name)  # the reference parses our DAG file
        plan = allocate_streams(rg)
        out[name] = {
            "graph": d,
            "assignment": [[v, plan.assignment[v]] for v in sorted(plan.assignment)],
            "num_streams": plan.num_streams,
            "sync": [list(e) for e in plan.sync_events],
            "opara": list(make_order(rg, "opara", cfg).order),
            "sequential": list(make_order(rg, "sequential", cfg).order),
        }
    path = OUT.with_name("model_dags_golden.json")
    path.write_text(json.dumps(out, separators=(",", ":")) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "models":
    model_dags()


def cli_fixtures() -> None:
    """CLI golden outputs: the REFERENCE CLI (python -m opsched) run on two
    graph files — the 13-node placement cases and the GoogLeNet DAG — with a
    B200 GpuConfig file; tests/test_cli.py replays our CLI byte for byte."""
    import shutil
    import subprocess
    import tempfile
    out = OUT.parent / "cli"
    out.mkdir(exist_ok=True)
    (out / "b200.json").write_text(json.dumps({"num_sms": 148, "threads_per_sm": 2048,
                                               "shared_mem_per_sm": 233472, "registers_per_sm": 65536,
                                               "max_blocks_per_sm": 32, "same_class_slowdown": 1.4},
                                              indent=2, sort_keys=True) + "\n")
    env = dict(os.environ, PYTHONPATH=str(REF))
    gold = json.loads(OUT.with_name("model_dags_golden.json").read_text())
    (out / "googlenet.json").write_text(json.dumps(gold["googlenet"]["graph"], indent=2, sort_keys=True) + "\n")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([sys.executable, "-m", "opsched", "gen", "cases", "--out", "cases.json"], cwd=td, env=env,
                       check=True, capture_output=True)
        shutil.copy(Path(td) / "cases.json", out / "cases.json")
    for name in ("cases", "googlenet"):
        with tempfile.TemporaryDirectory() as td:
            shutil.copy(out / f"{name}.json", Path(td) / "g.json")
            shutil.copy(out / "b200.json", Path(td) / "b200.json")
            run = lambda *a: subprocess.run([sys.executable, "-m", "opsched", *a], cwd=td, env=env, check=True,
                                            capture_output=True, text=True).stdout
            stdout = run("schedule", "g.json", "--gpu-config", "b200.json")
            run("simulate", "g.json", "g.plan.json", "g.order.json", "--trace", "g.tsv", "--out", "g.sim.json",
                "--gpu-config", "b200.json")
            table = run("compare", "g.json", "--policies", "sequential,opara,dfs,wavefront,random", "--out",
                        "g.compare.json", "--gpu-config", "b200.json")
            for suffix in ("plan.json", "order.json", "tsv", "sim.json", "compare.json"):
                shutil.copy(Path(td) / f"g.{suffix}", out / f"{name}.{suffix}")
            (out / f"{name}.stdout").write_text(stdout + table)
    print(f"wrote {out}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "cli":
    cli_fixtures()
