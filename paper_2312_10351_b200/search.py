"""Exhaustive launch-order search on tiny DAGs: simulated and measured on the B200.

Drop-in for the reference's ``opsched.oracle`` (oracle.py:1-204): the same
``linear_extensions`` enumeration order (lexicographic by node id, computed by
``opara_linear_extensions`` in libopara), ``best_order`` / ``best_plan`` over
the bit-exact execution model (``simulate``) with the same tie-breaks (first
minimum wins) and result types.

The B200 addition: ``measure_orders`` captures the same
kernels and Alg. 1 plan once per launch order into a scratch graph slot of a
compiled ``ScheduledGraph`` and times each replay on the device, so Alg. 2's
order can be ranked against every order of a sub-DAG on real hardware.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from . import _lib
from .dag import ComputationGraph
from .order import LaunchSchedule, make_order
from .plan import DEFAULT_SYNC_OVERHEAD_US, StreamPlan, single_stream_plan
from .simulator import simulate

_CHUNK = 4096


@dataclass(frozen=True)
class OracleResult:
    """Best launch order found for a fixed plan (oracle.py:21-32)."""

    best_makespan_ns: int
    best_order: tuple[int, ...]
    orders_examined: int
    search_space_exhausted: bool

    @property
    def best_makespan_us(self) -> float:
        return self.best_makespan_ns / 1000


@dataclass(frozen=True)
class PlanSearchResult:
    """Best (plan, order) pair under the sync-overhead-inclusive objective (oracle.py:35-49)."""

    best_total_ns: int
    best_makespan_ns: int
    best_plan: StreamPlan
    best_order: tuple[int, ...]
    plans_examined: int
    orders_examined: int
    search_space_exhausted: bool

    @property
    def best_total_us(self) -> float:
        return self.best_total_ns / 1000


def linear_extensions(g: ComputationGraph) -> Iterator[tuple[int, ...]]:
    """Every linear extension in lexicographic order by node id (oracle.py:52-84)."""
    n = len(g)
    if n == 0:
        yield ()
        return
    L = _lib.lib()
    buf = np.zeros(_CHUNK * n, dtype=np.int64)
    skip = 0
    while True:
        written = C.c_int64(0)
        done = C.c_int32(0)
        _lib.check(L.opara_linear_extensions(g.handle, skip, _CHUNK, _lib.ptr(buf), C.byref(written),
                                             C.byref(done)))
        rows = buf[: written.value * n].reshape(-1, n).tolist()
        yield from (tuple(r) for r in rows)
        if done.value:
            return
        skip += written.value


def count_linear_extensions(g: ComputationGraph, cap: int | None = None) -> tuple[int, bool]:
    """(number of extensions up to `cap`, whether that is all of them)."""
    k = 0
    for _ in linear_extensions(g):
        if cap is not None and k >= cap:
            return k, False
        k += 1
    return k, True


def best_order(g: ComputationGraph, plan: StreamPlan, cfg, limit: int | None = None) -> OracleResult:
    """Simulate every linear extension under a fixed plan and keep the minimum
    (oracle.py:87-122); the first-found minimum wins ties."""
    best_ns: int | None = None
    best: tuple[int, ...] = ()
    examined = 0
    exhausted = True
    for order in linear_extensions(g):
        if limit is not None and examined >= limit:
            exhausted = False
            break
        examined += 1
        ns = simulate(g, plan, order, cfg, blocks=False).makespan_ns
        if best_ns is None or ns < best_ns:
            best_ns, best = ns, order
    return OracleResult(best_makespan_ns=0 if best_ns is None else best_ns, best_order=best,
                        orders_examined=examined, search_space_exhausted=exhausted)


def _partitions(ids: list[int], max_streams: int) -> Iterator[dict[int, int]]:
    """Canonical stream assignments in first-seen numbering (oracle.py:125-141)."""
    assignment: dict[int, int] = {}

    def walk(i: int, used: int) -> Iterator[dict[int, int]]:
        if i == len(ids):
            yield dict(assignment)
            return
        v = ids[i]
        for s in range(min(used + 1, max_streams)):
            assignment[v] = s
            yield from walk(i + 1, max(used, s + 1))
        del assignment[v]

    yield from walk(0, 0)


def best_plan(g: ComputationGraph, cfg, max_streams: int | None = None, limit: int | None = None,
              sync_overhead_us: float = DEFAULT_SYNC_OVERHEAD_US) -> PlanSearchResult:
    """Joint search over stream assignments and launch orders; objective =
    makespan + syncs x overhead; `limit` caps simulated pairs (oracle.py:144-204)."""
    ids = g.topo_sort()
    cap = len(ids) if max_streams is None else max_streams
    overhead_ns = round(sync_overhead_us * 1000)
    best_total = None
    best_span = 0
    best_pl = None
    best_ord: tuple[int, ...] = ()
    plans = orders = 0
    exhausted = True
    budget_left = limit
    for assignment in _partitions(ids, cap):
        if budget_left is not None and budget_left <= 0:
            exhausted = False
            break
        num_streams = max(assignment.values()) + 1 if assignment else 0
        sync = tuple(sorted((u, v) for (u, v) in g.edges if assignment[u] != assignment[v]))
        plan = StreamPlan(assignment=assignment, num_streams=num_streams, sync_events=sync)
        sub = best_order(g, plan, cfg, limit=budget_left)
        plans += 1
        orders += sub.orders_examined
        if budget_left is not None:
            budget_left -= sub.orders_examined
        if not sub.search_space_exhausted:
            exhausted = False
        if sub.orders_examined == 0:
            continue
        total = sub.best_makespan_ns + len(sync) * overhead_ns
        if best_total is None or total < best_total:
            best_total, best_span, best_pl, best_ord = total, sub.best_makespan_ns, plan, sub.best_order
    if best_pl is None:
        best_pl = single_stream_plan(g)
        best_total = 0
    return PlanSearchResult(best_total_ns=best_total, best_makespan_ns=best_span, best_plan=best_pl,
                            best_order=best_ord, plans_examined=plans, orders_examined=orders,
                            search_space_exhausted=exhausted)


# ----------------------------------------------------------- on the B200

SCRATCH_SLOT = 20


def measure_orders(sg, orders, iters: int = 200, warmup: int = 20, flush_l2: bool = False,
                   plan: StreamPlan | None = None) -> list[float]:
    """Median device latency (ms) of each launch order: the compiled graph's
    kernels and Alg. 1 plan (or `plan`) re-captured per order into a scratch
    slot and replayed `iters` times under CUDA events."""
    plan = plan or sg.plan
    out = []
    for order in orders:
        sg.capture(SCRATCH_SLOT, plan, LaunchSchedule(tuple(order), "search"))
        out.append(sg.time(SCRATCH_SLOT, warmup=warmup, iters=iters, flush_l2=flush_l2).median_ms)
    return out


def critical_path_first_order(g: ComputationGraph, cost: dict[int, float]) -> tuple[int, ...]:
    """Diagnostic baseline (not a reference policy): list scheduling that
    always launches the ready op with the longest remaining path (its own
    cost plus the longest cost path to a sink), ties by ascending id."""
    import heapq
    tail: dict[int, float] = {}
    for v in reversed(g.topo_sort()):
        tail[v] = cost[v] + max((tail[w] for w in g.successors(v)), default=0.0)
    missing = {v: len(g.predecessors(v)) for v in g.node_ids}
    ready = [(-tail[v], v) for v in g.node_ids if missing[v] == 0]
    heapq.heapify(ready)
    out = []
    while ready:
        _, v = heapq.heappop(ready)
        out.append(v)
        for w in g.successors(v):
            missing[w] -= 1
            if missing[w] == 0:
                heapq.heappush(ready, (-tail[w], w))
    return tuple(out)


def search_measured(sg, limit: int = 5000, iters: int = 200, recheck: int = 8, rounds: int = 3) -> dict:
    """Rank Alg. 2's order among every linear extension of `sg`'s DAG (up to
    `limit`) by measured latency.  Every order is timed in `rounds` interleaved
    passes (median of the per-pass medians, so clock and thermal drift spread
    over all orders); the `recheck` fastest plus the named policies are then
    re-timed together for the final ranking."""
    g = sg.graph
    orders = []
    exhausted = True
    for o in linear_extensions(g):
        if len(orders) >= limit:
            exhausted = False
            break
        orders.append(o)
    passes = [measure_orders(sg, orders, iters=iters) for _ in range(rounds)]
    lat = np.median(np.asarray(passes), axis=0)
    named = {pol: tuple(make_order(g, pol, sg.gpu_config).order) for pol in ("opara", "dfs", "wavefront",
                                                                              "sequential")}
    named["critical_path_first"] = critical_path_first_order(
        g, {v: sg.profile[v - 1]["isolated_us"] for v in g.node_ids})
    top = [orders[i] for i in np.argsort(lat)[:recheck]]
    final_set = list(dict.fromkeys(top + list(named.values())))
    fin = np.median(np.asarray([measure_orders(sg, final_set, iters=iters * 2) for _ in range(rounds)]), axis=0)
    fin_of = dict(zip(final_set, fin.tolist()))
    index = {o: i for i, o in enumerate(orders)}
    sorted_lat = np.sort(lat)

    def rank(o):   # 1-based rank of o's first-pass latency among all orders
        i = index.get(o)
        return None if i is None else int(np.searchsorted(sorted_lat, lat[i], side="left")) + 1

    return {
        "nodes": len(g), "edges": len(g.edges), "streams": sg.plan.num_streams,
        "orders_examined": len(orders), "search_space_exhausted": exhausted,
        "latency_ms": {"min": float(sorted_lat[0]), "median": float(np.median(lat)),
                       "max": float(sorted_lat[-1])},
        "best_order": list(min(fin_of, key=fin_of.get)), "best_ms": float(min(fin_of.values())),
        "policies": {pol: {"ms": fin_of[o], "rank": rank(o), "percentile": (rank(o) or 0) / len(orders),
                           "order": list(o)} for pol, o in named.items()},
        "isolated_us": {v: sg.profile[v - 1]["isolated_us"] for v in g.node_ids},
        "classes": {v: g.node(v).op_class.value for v in g.node_ids},
        "iters": iters, "rounds": rounds,
    }
