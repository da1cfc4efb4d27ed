"""Exhaustive order search: the C++ linear-extension
enumerator and best_order against the oracle restatement of oracle.py:52-122
(the reference's own test_oracle.py also runs against search.py through the
shim in test_reference_suite.py)."""

from __future__ import annotations

import math
import random

import pytest

import paper_2312_10351_b200 as op
from oracle import opsched_oracle as orc
from paper_2312_10351_b200 import search
from paper_2312_10351_b200.dag import graph_from_dict


def _tiny(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 8)
    ids = rng.sample(range(-20, 200), n)   # arbitrary ids: enumeration is by id, not position
    nodes = [{"id": v, "name": "op", "class": rng.choice(["compute", "memory"]), "blocks": rng.randint(1, 40),
              "threads_per_block": rng.choice([64, 128, 256]), "shared_mem_bytes": rng.choice([0, 4096, 65536]),
              "registers_per_thread": rng.choice([16, 32, 64]),
              "block_duration_us": round(rng.uniform(0.5, 20.0), 3)} for v in ids]
    topo = ids[:]
    rng.shuffle(topo)
    edges = sorted({(topo[i], topo[j]) for j in range(1, n) for i in rng.sample(range(j), min(j, rng.randint(0, 2)))})
    return nodes, edges


CFG = dict(num_sms=4, threads_per_sm=2048, shared_mem_per_sm=233472, registers_per_sm=65536,
           max_blocks_per_sm=8, same_class_slowdown=1.4)


@pytest.mark.parametrize("seed", range(80))
def test_linear_extensions_match_oracle(seed):
    nodes, edges = _tiny(seed)
    g = graph_from_dict({"nodes": nodes, "edges": [list(e) for e in edges]})
    o = orc.Dag(nodes, edges)
    got = list(search.linear_extensions(g))
    assert got == list(orc.linear_extensions(o))
    assert got == sorted(got) and len(set(got)) == len(got)
    assert all(g.is_linear_extension(e) for e in got)


@pytest.mark.parametrize("seed", range(25))
def test_best_order_matches_oracle(seed):
    nodes, edges = _tiny(seed)
    g = graph_from_dict({"nodes": nodes, "edges": [list(e) for e in edges]})
    o = orc.Dag(nodes, edges)
    cfg = op.GpuConfig(**CFG)
    plan = op.allocate_streams(g)
    a, ns, s = orc.allocate_streams(o)
    for limit in (None, 3):
        res = search.best_order(g, plan, cfg, limit=limit)
        want = orc.best_order(o, a, ns, s, CFG, limit=limit)
        assert (res.best_makespan_ns, res.best_order, res.orders_examined,
                res.search_space_exhausted) == want


def test_enumeration_spans_chunks():
    """An antichain of 8 has 8! = 40320 extensions: more than one native chunk."""
    nodes = [{"id": i, "name": "op", "class": "compute", "blocks": 1, "threads_per_block": 32,
              "shared_mem_bytes": 0, "registers_per_thread": 16, "block_duration_us": 1.0} for i in range(1, 9)]
    g = graph_from_dict({"nodes": nodes, "edges": []})
    exts = list(search.linear_extensions(g))
    assert len(exts) == math.factorial(8)
    assert exts[0] == tuple(range(1, 9)) and exts[-1] == tuple(range(8, 0, -1))
    assert exts == sorted(exts)
    assert search.count_linear_extensions(g, cap=100) == (100, False)


def test_empty_graph_has_one_empty_extension():
    g = graph_from_dict({"nodes": [], "edges": []})
    assert list(search.linear_extensions(g)) == [()]
