"""Pin the oracle: it must reproduce every golden vector the reference produced
(tests/golden/make_golden.py) and the reference tests' hand-traced KATs."""

from __future__ import annotations

import pytest

from conftest import golden_nodes, golden_sched
from oracle import opsched_oracle as orc

CASES = golden_sched()["cases"]
CFGS = golden_sched()["configs"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_vectors(case):
    g = orc.Dag(golden_nodes(case), case["edges"])
    assert g.topo == case["topo"]
    assign, ns, sync = orc.allocate_streams(g)
    assert sorted(assign.items()) == [tuple(x) for x in case["assignment"]]
    assert ns == case["num_streams"]
    assert [list(e) for e in sync] == case["sync"]
    assert orc.validate_plan(g, assign, ns, sync) == []
    for cname, orders in case["orders"].items():
        cfg = CFGS[cname]
        assert orc.order_opara(g, cfg) == orders["opara"], cname
        if "dfs" in orders:
            assert orc.order_sequential(g) == orders["sequential"]
            assert orc.order_dfs(g) == orders["dfs"]
            assert orc.order_wavefront(g) == orders["wavefront"]
    for cname, spans in case["makespan_ns"].items():
        cfg = CFGS[cname]
        got = orc.simulate_makespan_ns(g, assign, ns, sync, orc.order_opara(g, cfg), cfg)
        assert got == spans["opara"], cname
        a1, n1, s1 = orc.single_stream_plan(g)
        assert orc.simulate_makespan_ns(g, a1, n1, s1, orc.order_sequential(g), cfg) == spans["sequential"]


def _n(i, cls="compute", blocks=1, threads=256, smem=0, regs=32, dur=10.0):
    return {"id": i, "name": "op", "class": cls, "blocks": blocks, "threads_per_block": threads,
            "shared_mem_bytes": smem, "registers_per_thread": regs, "block_duration_us": dur}


def test_kat_acceptance_criterion_1():
    """test_acceptance.py:58-82 hand-traced placements."""
    g = orc.Dag([_n(1), _n(2)], [])
    assert orc.allocate_streams(g)[0] == {1: 0, 2: 1}
    g = orc.Dag([_n(i) for i in range(1, 5)], [(1, 2), (1, 3), (1, 4)])
    assert orc.allocate_streams(g)[0] == {1: 0, 2: 0, 3: 1, 4: 2}
    g = orc.Dag([_n(i) for i in range(1, 5)], [(1, 2), (1, 3), (2, 4), (3, 4)])
    assert orc.allocate_streams(g)[0] == {1: 0, 2: 0, 3: 1, 4: 0}


def test_kat_dominant_share_and_orders():
    """test_orderer.py:30-33, :51-62, :65-76; test_acceptance.py:190."""
    cfg = {"threads_per_sm": 1000, "shared_mem_per_sm": 65536, "registers_per_sm": 65536}
    assert orc.dominant_share(_n(1, threads=500, smem=32768, regs=16, blocks=2), cfg) == pytest.approx(1.0)
    g = orc.Dag([_n(1, "memory", threads=100), _n(2, threads=50), _n(3, "memory", threads=30),
                 _n(4, threads=200)], [])
    assert orc.order_opara(g, cfg) == [3, 2, 1, 4]
    g = orc.Dag([_n(1, threads=100), _n(2, "memory", threads=20), _n(3, threads=10)], [(1, 2), (1, 3)])
    assert orc.order_opara(g, cfg) == [1, 2, 3]
    g = orc.Dag([_n(i, "memory", dur=100, threads=512) for i in range(1, 5)]
                + [_n(i, dur=100, threads=512) for i in range(5, 9)], [])
    c6 = {"num_sms": 1, "threads_per_sm": 1024, "shared_mem_per_sm": 65536,
          "registers_per_sm": 65536, "max_blocks_per_sm": 16, "same_class_slowdown": 1.4}
    assert orc.order_opara(g, c6) == [1, 5, 2, 6, 3, 7, 4, 8]
    a, ns, s = orc.allocate_streams(g)
    assert orc.simulate_makespan_ns(g, a, ns, s, [1, 5, 2, 6, 3, 7, 4, 8], c6) == 400000
    assert orc.simulate_makespan_ns(g, a, ns, s, list(range(1, 9)), c6) == 560000


@pytest.mark.parametrize("nodes,edges,msg", [
    ([1, 1], [], "duplicate node id 1"),
    ([1], [(1, 9)], "edge (1, 9) references an unknown node"),
    ([1], [(1, 1)], "self-edge (1, 1)"),
    ([1, 2], [(1, 2), (1, 2)], "duplicate edge (1, 2)"),
    ([1, 2], [(1, 2), (2, 1)], "cycle involving nodes [1, 2]"),
])
def test_kat_validation_messages(nodes, edges, msg):
    """graph.py:115-152 message text, test_graph.py:83-105."""
    with pytest.raises(orc.OracleGraphError) as e:
        orc.Dag([_n(i) for i in nodes], edges)
    assert str(e.value) == msg
