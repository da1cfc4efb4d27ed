"""Bit-exact parity of the C++ scheduler (through the C ABI) with the
reference: golden vectors produced by the reference itself, plus a seeded fuzz
corpus checked against the oracle restatement."""

from __future__ import annotations

import random

import pytest

import paper_2312_10351_b200 as op
from conftest import golden_nodes, golden_sched
from oracle import opsched_oracle as orc

GOLD = golden_sched()
CASES = GOLD["cases"]


def to_graph(nodes, edges):
    return op.ComputationGraph(
        [op.OperatorNode(n["id"], n["name"], op.OpClass(n["class"]),
                         op.ResourceDemand(n["threads_per_block"], n["shared_mem_bytes"],
                                           n["registers_per_thread"], n["blocks"]),
                         n["block_duration_us"]) for n in nodes], edges)


def cfg_of(d):
    return op.GpuConfig(d["num_sms"], d["threads_per_sm"], d["shared_mem_per_sm"],
                        d["registers_per_sm"], d["max_blocks_per_sm"], d["same_class_slowdown"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_native_matches_reference_golden(case):
    g = to_graph(golden_nodes(case), case["edges"])
    assert g.topo_sort() == case["topo"]
    assert [list(e) for e in g.edges] == sorted(case["edges"])
    plan = op.allocate_streams(g)
    assert sorted(plan.assignment.items()) == [tuple(x) for x in case["assignment"]]
    assert plan.num_streams == case["num_streams"]
    assert [list(e) for e in plan.sync_events] == case["sync"]
    assert op.validate_plan(g, plan) == []
    for cname, orders in case["orders"].items():
        cfg = cfg_of(GOLD["configs"][cname])
        assert list(op.order_opara(g, cfg).order) == orders["opara"], cname
        for pol in ("sequential", "dfs", "wavefront"):
            if pol in orders:
                assert list(op.make_order(g, pol, cfg).order) == orders[pol], pol


def _random_nodes(rng, n, ids):
    out = []
    for v in ids:
        out.append({"id": v, "name": "op", "class": rng.choice(["compute", "memory"]),
                    "blocks": rng.choice([1, 2, 7, 148, 296, 1000, 2 ** 20]),
                    "threads_per_block": rng.choice([0, 32, 64, 96, 128, 256, 384, 512, 1024]),
                    "shared_mem_bytes": rng.choice([0, 1, 4096, 49152, 100000, 232448]),
                    "registers_per_thread": rng.choice([0, 16, 32, 40, 64, 96, 168, 255]),
                    "block_duration_us": rng.choice([0.5, 1.0, 3.25, 10.0])})
    return out


def _random_dag(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 60)
    ids = rng.sample(range(-50, 10_000), n)  # arbitrary, non-contiguous, negative ids
    order = ids[:]
    rng.shuffle(order)
    edges = set()
    for j in range(1, n):
        for _ in range(rng.randint(0, 3)):
            i = rng.randrange(j)
            edges.add((order[i], order[j]))
    e = list(edges)
    rng.shuffle(e)
    return _random_nodes(rng, n, ids), e


CFGS = [op.GPU_PRESETS["b200"], op.GPU_PRESETS["2080s-like"],
        op.GpuConfig(3, 1000, 7000, 12345, 4), op.GpuConfig(1, 1, 1, 1, 1)]


@pytest.mark.parametrize("seed", range(300))
def test_native_matches_oracle_fuzz(seed):
    nodes, edges = _random_dag(seed)
    g = to_graph(nodes, edges)
    o = orc.Dag(nodes, edges)
    assert g.topo_sort() == o.topo
    plan = op.allocate_streams(g)
    a, ns, sync = orc.allocate_streams(o)
    assert dict(plan.assignment) == a and plan.num_streams == ns
    assert list(plan.sync_events) == sync
    for cfg in CFGS:
        cd = {"threads_per_sm": cfg.threads_per_sm, "shared_mem_per_sm": cfg.shared_mem_per_sm,
              "registers_per_sm": cfg.registers_per_sm}
        assert list(op.order_opara(g, cfg).order) == orc.order_opara(o, cd)
        for n in nodes:
            d = op.ResourceDemand(n["threads_per_block"], n["shared_mem_bytes"],
                                  n["registers_per_thread"], n["blocks"])
            assert op.dominant_share(d, cfg) == orc.dominant_share(n, cd)  # bit-exact double
    assert list(op.order_baseline(g, "dfs").order) == orc.order_dfs(o)
    assert list(op.order_baseline(g, "wavefront").order) == orc.order_wavefront(o)


@pytest.mark.parametrize("seed", range(40))
def test_validate_plan_messages_match_oracle(seed):
    rng = random.Random(1000 + seed)
    nodes, edges = _random_dag(seed)
    g = to_graph(nodes, edges)
    o = orc.Dag(nodes, edges)
    plan = op.allocate_streams(g)
    assign = dict(plan.assignment)
    sync = list(plan.sync_events)
    # corrupt the plan in several ways
    if assign and rng.random() < 0.5:
        del assign[rng.choice(list(assign))]
    if rng.random() < 0.3:
        assign[99_999] = 0
    if rng.random() < 0.3 and assign:
        k = rng.choice(list(assign))
        assign[k] = assign[k] + rng.choice([1, 5])
    if sync and rng.random() < 0.5:
        sync.pop(rng.randrange(len(sync)))
    if rng.random() < 0.3:
        sync.append((nodes[0]["id"], 123_456))
    if edges and rng.random() < 0.3:
        sync.append(tuple(edges[0]))
    ns = plan.num_streams + rng.choice([0, 0, 1, -1])
    bad = op.StreamPlan(assign, ns, tuple(sync))
    assert op.validate_plan(g, bad) == orc.validate_plan(o, assign, ns, sync)


@pytest.mark.parametrize("nodes,edges,msg", [
    ([1, 1], [], "duplicate node id 1"),
    ([2, 1, 2], [], "duplicate node id 2"),
    ([1], [(1, 9)], "edge (1, 9) references an unknown node"),
    ([1], [(1, 1)], "self-edge (1, 1)"),
    ([1, 2], [(1, 2), (1, 2)], "duplicate edge (1, 2)"),
    ([1, 2], [(1, 2), (2, 1)], "cycle involving nodes [1, 2]"),
    ([1, 2, 3, 4], [(1, 2), (2, 3), (3, 2), (3, 4)], "cycle involving nodes [2, 3, 4]"),
])
def test_validation_messages_verbatim(nodes, edges, msg):
    mk = lambda i: op.OperatorNode(i, "conv", op.OpClass.COMPUTE, op.ResourceDemand(32, 0, 32, 1), 1.0)
    with pytest.raises(op.GraphValidationError) as e:
        op.ComputationGraph([mk(i) for i in nodes], edges)
    assert str(e.value) == msg


def test_unknown_id_is_key_error():
    g = op.ComputationGraph([op.OperatorNode(1, "conv", op.OpClass.COMPUTE,
                                             op.ResourceDemand(32, 0, 32, 1), 1.0)], [])
    with pytest.raises(KeyError, match="unknown node id 7"):
        g.predecessors(7)
    with pytest.raises(KeyError, match="unknown node id 7"):
        g.node(7)


def test_empty_graph():
    g = op.ComputationGraph([], [])
    plan = op.allocate_streams(g)
    assert plan.num_streams == 0 and plan.sync_events == () and dict(plan.assignment) == {}
    assert op.single_stream_plan(g).num_streams == 0
    assert op.order_opara(g, op.GPU_PRESETS["b200"]).order == ()
    assert op.validate_plan(g, plan) == []
