"""Parity on exactly what bench.py times, and dependency safety of the replay.

bench.py compiles every workload with ``bound_grids="auto"``: the fastest of
{full, bounded} grids x {push, pull, auto} split-K reductions (plus SM-share
scales for the bounded winner).  These tests build that same graph per
BASELINE config through bench.py's own workload builder and assert the
north_star tolerance (1e-4 fp32, 1e-2 bf16) against the PyTorch fp32 eager
forward, that the Opara graph equals the sequential graph of the same kernels
bit for bit, and that the replayed timeline respects every DAG edge — the
analog of the reference's dependency check on a simulated trace
(`/root/reference/pkg/tests/helpers.py:120-124`: every consumer starts after
its producer ends).  Kernel start stamps are taken after griddepcontrol.wait
(PDL), end stamps after the last store of the last CTA.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return (torch.linalg.vector_norm(a.double() - b.double()) / torch.linalg.vector_norm(b.double())).item()


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False


def edge_violations(sg, slot) -> list[tuple[int, int, int, int]]:
    """(producer, consumer, producer_end_ns, consumer_start_ns) for every DAG
    edge whose consumer kernel started before its producer finished.  NOP
    joins launch nothing: they pass their predecessors' finish time through."""
    from paper_2312_10351_b200 import engine
    tr = {nid: (s, e) for nid, s, e in sg.trace(slot)}
    nop = {k + 1 for k, op in enumerate(sg.program.ops) if op.kind == engine.NOP}
    ready = {}   # node -> (latest producer end, producer id) over its (transitive through NOPs) inputs
    done = {}
    bad = []
    for v in sg.graph.topo_sort():
        r = max(((done[p], p) for p in sg.graph.predecessors(v)), default=(None, None))
        if v in nop:
            done[v] = r[0] if r[0] is not None else tr[v][0]
            continue
        if r[0] is not None and tr[v][0] < r[0]:
            bad.append((r[1], v, r[0], tr[v][0]))
        done[v] = tr[v][1]
    return bad


def _bench_workload(model, dtype, batch):
    import bench
    args = argparse.Namespace(model=model, dtype=dtype, batch=batch)
    bench.resolve_dtype(args)
    m, ref, x = bench.build_workload(args)
    return args.dtype, m, ref, x


def _check(sg, ref_model, x, tol):
    from paper_2312_10351_b200 import engine
    xd = tuple(t.cuda() for t in x) if isinstance(x, tuple) else x.cuda()
    y = sg.run(xd)
    y_seq = sg.run(xd, slot=engine.SLOT_SEQUENTIAL)
    ys = y if isinstance(y, tuple) else (y,)
    yss = y_seq if isinstance(y_seq, tuple) else (y_seq,)
    assert all(torch.equal(a, b) for a, b in zip(ys, yss)), "Opara and sequential graphs disagree"
    with torch.no_grad():
        ref = ref_model.cuda()(*xd) if isinstance(xd, tuple) else ref_model.cuda()(xd)
    refs = ref if isinstance(ref, tuple) else (ref,)
    rels = [_rel(a.float().reshape(b.shape), b) for a, b in zip(ys, refs)]
    assert max(rels) <= tol, rels
    for slot in (engine.SLOT_PARALLEL, engine.SLOT_SEQUENTIAL):
        bad = edge_violations(sg, slot)
        assert not bad, f"slot {slot}: {len(bad)} edges violated, first {bad[:3]}"
    return rels


BENCH_CONFIGS = [("googlenet", "f32", 1), ("googlenet", "bf16", 1), ("inception_v3", "f32", 1),
                 ("inception_v3", "bf16", 1), ("bert_base", "bf16", 1), ("nasnet_large", "f32", 1),
                 ("nasnet_large", "bf16", 1), ("deepfm", "f32", 1), ("deepfm", "f32", 32)]


@pytest.mark.parametrize("model,dtype,batch", BENCH_CONFIGS)
def test_bench_graph_parity(model, dtype, batch):
    """The graph bench.py times for this config: compile(bound_grids="auto")."""
    from paper_2312_10351_b200 import engine
    dtype, m, ref, x = _bench_workload(model, dtype, batch)
    sg = engine.compile(m, x, device=0, bound_grids="auto", profile_reps=3, dtype=dtype)
    try:
        _check(sg, ref, x, 1e-4 if dtype == "f32" else 1e-2)
    finally:
        sg.close()


@pytest.mark.parametrize("bounded,splitk,scale", [(False, "push", 1.0), (False, "pull", 1.0), (False, "l2", 1.0),
                                                  (False, "auto", 1.0), (True, "push", 1.0), (True, "pull", 1.0),
                                                  (True, "l2", 1.0), (True, "auto", 1.0),
                                                  (True, "pull", 0.75), (True, "pull", 1.5), (True, "pull", 2.0)])
@pytest.mark.parametrize("model,dtype", [("inception_v3", "f32"), ("googlenet", "bf16")])
def test_every_autotune_variant(model, dtype, bounded, splitk, scale):
    """Every candidate compile(bound_grids="auto") may pick is correct, so the
    timing-dependent choice cannot select a wrong graph."""
    from paper_2312_10351_b200 import engine
    dtype, m, ref, x = _bench_workload(model, dtype, 1)
    sg = engine.ScheduledGraph(engine.lower(m, x, dtype), 0, profile_reps=2, bound_grids=bounded,
                               splitk=splitk, bound_scale=scale)
    try:
        _check(sg, ref, x, 1e-4 if dtype == "f32" else 1e-2)
    finally:
        sg.close()


def test_trace_order_follows_capture_order():
    """Kernels that share a plan stream start in the order the schedule
    launched them (the instantiated graph keeps the capture order per stream),
    and the same holds for the single-stream sequential graph."""
    from paper_2312_10351_b200 import engine, zoo
    model, x = zoo.build("inception_v3")
    sg = engine.compile(model, x, device=0, profile_reps=2)
    try:
        tr = {nid: s for nid, s, _ in sg.trace(engine.SLOT_PARALLEL)}
        nop = {k + 1 for k, op in enumerate(sg.program.ops) if op.kind == engine.NOP}
        per_stream = {}
        for v in sg.schedule.order:
            if v not in nop:
                per_stream.setdefault(sg.plan.assignment[v], []).append(tr[v])
        for sid, starts in per_stream.items():
            assert starts == sorted(starts), f"stream {sid} started out of launch order"
        seq = {nid: s for nid, s, _ in sg.trace(engine.SLOT_SEQUENTIAL)}
        starts = [seq[v] for v in sg.graph.topo_sort() if v not in nop]
        assert starts == sorted(starts)
    finally:
        sg.close()
