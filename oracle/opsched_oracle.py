"""CPU restatement of the reference scheduler — TEST INFRASTRUCTURE ONLY.

This module is the parity oracle for the stream allocator (Alg. 1), the
resource-aware launch orderer (Alg. 2), the deterministic topological order
they both walk, plan validation, and the reference's execution model (the
discrete-event "run" the B200 CUDA Graph replaces).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it, and only as the checker or the timed CPU
baseline.  The product path (``paper_2312_10351_b200``) never imports it.

Parity pinning: every function here is checked against the reference's own
known-answer tests (``/root/reference/pkg/tests``) and against golden vectors
produced by the reference itself (``tests/golden/make_golden.py`` imports the
reference package in the build container; the vectors are committed).

Everything is a plain restatement over plain data — nodes are dicts with the
graph-file schema keys of ``graph.py:264-268`` plus ``class``; edges are
``(u, v)`` integer pairs — written for clarity, not speed.  Citations are
``file:line`` into ``/root/reference/pkg/src/opsched``.
"""

from __future__ import annotations

import heapq

COMPUTE = "compute"
MEMORY = "memory"


class OracleGraphError(Exception):
    """Structural problem; message text equals GraphValidationError's."""


class OracleCoverageError(Exception):
    """Launch order problem; message text equals CoverageError's."""


class OracleInfeasibleError(Exception):
    """Block larger than an SM; message text equals InfeasibleBlockError's."""


# --------------------------------------------------------------------- graph


class Dag:
    """Validated DAG with id-sorted adjacency (graph.py:110-136)."""

    def __init__(self, nodes, edges):
        # graph.py:111-116 — sort by id, the first repeated id (in sorted order) wins
        ordered = sorted(nodes, key=lambda n: int(n["id"]))
        self.node = {}
        for n in ordered:
            nid = int(n["id"])
            if nid in self.node:
                raise OracleGraphError(f"duplicate node id {nid}")
            self.node[nid] = n
        self.ids = [int(n["id"]) for n in ordered]
        # graph.py:117-130 — per edge: unknown endpoint, self-edge, duplicate
        self.pred = {i: [] for i in self.ids}
        self.succ = {i: [] for i in self.ids}
        seen = set()
        for raw in edges:
            u, v = int(raw[0]), int(raw[1])
            if u not in self.node or v not in self.node:
                raise OracleGraphError(f"edge ({u}, {v}) references an unknown node")
            if u == v:
                raise OracleGraphError(f"self-edge ({u}, {v})")
            if (u, v) in seen:
                raise OracleGraphError(f"duplicate edge ({u}, {v})")
            seen.add((u, v))
            self.succ[u].append(v)
            self.pred[v].append(u)
        for i in self.ids:  # graph.py:133-134 — ascending id adjacency
            self.pred[i].sort()
            self.succ[i].sort()
        self.edges = sorted(seen)  # graph.py:135
        self.topo = self._lexicographic_topo()

    def _lexicographic_topo(self):
        """Kahn with a min-heap of ids (graph.py:138-153)."""
        missing = {i: len(self.pred[i]) for i in self.ids}
        heap = [i for i in self.ids if missing[i] == 0]
        heapq.heapify(heap)
        out = []
        while heap:
            v = heapq.heappop(heap)
            out.append(v)
            for s in self.succ[v]:
                missing[s] -= 1
                if missing[s] == 0:
                    heapq.heappush(heap, s)
        if len(out) != len(self.ids):
            stuck = sorted(i for i in self.ids if missing[i] > 0)
            raise OracleGraphError(f"cycle involving nodes {stuck}")
        return out

    def is_linear_extension(self, order):
        """graph.py:197-202."""
        if sorted(order) != sorted(self.ids):
            return False
        at = {v: k for k, v in enumerate(order)}
        return all(at[u] < at[v] for (u, v) in self.edges)


# ------------------------------------------------------------ Alg. 1 / plans


def allocate_streams(g: Dag):
    """Donate-once stream inheritance over the topo order (allocator.py:43-67).

    Returns (assignment dict id->stream, num_streams, sorted sync pairs).
    """
    spent = set()
    stream = {}
    opened = 0
    for v in g.topo:
        donor = next((p for p in g.pred[v] if p not in spent), None)
        if donor is None:
            stream[v] = opened
            opened += 1
        else:
            stream[v] = stream[donor]
            spent.add(donor)
    sync = sorted(e for e in g.edges if stream[e[0]] != stream[e[1]])
    return stream, opened, sync


def single_stream_plan(g: Dag):
    """allocator.py:70-77."""
    return {v: 0 for v in g.ids}, (1 if g.ids else 0), []


def validate_plan(g: Dag, assignment, num_streams, sync):
    """Violation strings in the reference's order (allocator.py:80-109)."""
    out = []
    ids = set(g.ids)
    out += [f"node {v} unassigned" for v in sorted(ids) if v not in assignment]
    out += [f"assigned node {v} not in graph" for v in sorted(assignment) if v not in ids]
    used = sorted(set(assignment.values()))
    if used and used != list(range(num_streams)):
        out.append(f"stream ids must be dense 0..{num_streams - 1}, got {used}")
    if not assignment and num_streams != 0:
        out.append("num_streams must be 0 for an empty assignment")
    sync_set = {(int(u), int(v)) for (u, v) in sync}
    edge_set = set(g.edges)
    out += [f"sync event ({u}, {v}) is not a graph edge" for (u, v) in sorted(sync_set - edge_set)]
    for (u, v) in g.edges:
        if u not in assignment or v not in assignment:
            continue
        cross = assignment[u] != assignment[v]
        if cross and (u, v) not in sync_set:
            out.append(f"missing sync for cross-stream edge ({u}, {v})")
        if not cross and (u, v) in sync_set:
            out.append(f"sync event ({u}, {v}) joins same-stream nodes")
    return out


# -------------------------------------------------------------- Alg. 2 / orders


def dominant_share(node, cfg):
    """orderer.py:45-53: max of three per-SM fractions, times the block count."""
    threads = int(node["threads_per_block"])
    fractions = (
        threads / int(cfg["threads_per_sm"]),
        int(node["shared_mem_bytes"]) / int(cfg["shared_mem_per_sm"]),
        (int(node["registers_per_thread"]) * threads) / int(cfg["registers_per_sm"]),
    )
    return max(fractions) * int(node["blocks"])


def order_opara(g: Dag, cfg):
    """Two class heaps keyed (share, id), memory first, flip to the class not
    just launched (orderer.py:60-88)."""
    key = {v: (dominant_share(g.node[v], cfg), v) for v in g.ids}
    cls = {v: g.node[v]["class"] for v in g.ids}
    missing = {v: len(g.pred[v]) for v in g.ids}
    heaps = {MEMORY: [], COMPUTE: []}
    for v in g.ids:
        if missing[v] == 0:
            heapq.heappush(heaps[cls[v]], key[v])
    flip = {MEMORY: COMPUTE, COMPUTE: MEMORY}
    want = MEMORY
    out = []
    while heaps[MEMORY] or heaps[COMPUTE]:
        took = want if heaps[want] else flip[want]
        _, v = heapq.heappop(heaps[took])
        out.append(v)
        for s in g.succ[v]:
            missing[s] -= 1
            if missing[s] == 0:
                heapq.heappush(heaps[cls[s]], key[s])
        want = flip[took]
    return out


def order_sequential(g: Dag):
    """orderer.py:151-152: the topological order."""
    return list(g.topo)


def order_dfs(g: Dag):
    """Emit a node the moment its last predecessor is emitted, walking depth
    first from the roots in id order (orderer.py:91-110)."""
    missing = {v: len(g.pred[v]) for v in g.ids}
    out = []
    for root in [v for v in g.ids if missing[v] == 0]:
        out.append(root)
        stack = [[root, 0]]
        while stack:
            frame = stack[-1]
            v, k = frame
            succs = g.succ[v]
            pushed = False
            while k < len(succs):
                s = succs[k]
                k += 1
                missing[s] -= 1
                if missing[s] == 0:
                    out.append(s)
                    frame[1] = k
                    stack.append([s, 0])
                    pushed = True
                    break
            if not pushed:
                stack.pop()
    return out


def order_wavefront(g: Dag):
    """Level order, ids ascending within a level (orderer.py:113-118)."""
    level = {}
    for v in g.topo:
        level[v] = 1 + max((level[p] for p in g.pred[v]), default=-1)
    return sorted(g.ids, key=lambda v: (level[v], v))


# ------------------------------------------------------- execution model (run)


def py_round(x):
    """Python's round-half-even on a float, as used by graph.py:99 / simulator.py:331."""
    return round(x)


def simulate_makespan_ns(g: Dag, assignment, num_streams, sync, order, cfg):
    """Discrete-event run of (plan, order): FIFO streams, per-edge record/wait,
    head-of-line block dispatch to the lowest-index SM that fits, same-class
    co-residency slowdown decided per dispatch round (simulator.py:212-415).

    Returns the makespan in integer nanoseconds.
    """
    ids = set(g.ids)
    if set(order) != ids or len(order) != len(ids):
        missing = sorted(ids - set(order))
        extra = sorted(set(order) - ids)
        raise OracleCoverageError(
            f"launch order must cover the graph exactly (missing {missing}, extra {extra})")
    if not g.is_linear_extension(order):
        raise OracleCoverageError("launch order is not a linear extension of the graph")
    nsm = int(cfg["num_sms"])
    cap = (int(cfg["threads_per_sm"]), int(cfg["shared_mem_per_sm"]),
           int(cfg["registers_per_sm"]), int(cfg["max_blocks_per_sm"]))
    need = {}
    for v in g.ids:
        n = g.node[v]
        t = int(n["threads_per_block"])
        need[v] = (t, int(n["shared_mem_bytes"]), int(n["registers_per_thread"]) * t, 1)
        if need[v][0] > cap[0] or need[v][1] > cap[1] or need[v][2] > cap[2]:
            raise OracleInfeasibleError(
                f"operator {v} ({n['name']}): one block exceeds a single SM's capacity")
    if not order:
        return 0
    slowdown = float(cfg.get("same_class_slowdown", 1.4))
    dur = {v: py_round(float(g.node[v]["block_duration_us"]) * 1000) for v in g.ids}
    cls = {v: g.node[v]["class"] for v in g.ids}

    fifo = {s: [] for s in range(num_streams)}
    for v in order:
        fifo[assignment[v]].append(v)
    head = {s: 0 for s in fifo}
    waits = {v: 0 for v in order}
    listeners = {v: [] for v in order}
    for (u, v) in sync:
        waits[v] += 1
        listeners[u].append(v)

    todo = {v: int(g.node[v]["blocks"]) for v in order}
    live_count = {v: 0 for v in order}
    free = [list(cap) for _ in range(nsm)]
    resident = [dict() for _ in range(nsm)]  # token -> op
    at_head = set()
    went_eligible = set()
    done_at = {}
    queue = []  # (eligibility seq, op)
    seq = 0
    token = 0
    finish = []  # (end, token, op, sm)

    def enqueue(v):
        nonlocal seq
        went_eligible.add(v)
        heapq.heappush(queue, (seq, v))
        seq += 1

    def fit(v):
        d = need[v]
        for i in range(nsm):
            f = free[i]
            if f[0] >= d[0] and f[1] >= d[1] and f[2] >= d[2] and f[3] >= 1:
                return i
        return None

    def dispatch(t):
        nonlocal token
        placed = []
        while queue:
            v = queue[0][1]
            blocked = False
            while todo[v] > 0:
                sm = fit(v)
                if sm is None:
                    blocked = True
                    break
                for k in range(4):
                    free[sm][k] -= need[v][k]
                resident[sm][token] = v
                placed.append((token, v, sm))
                token += 1
                todo[v] -= 1
                live_count[v] += 1
            if blocked:
                break
            heapq.heappop(queue)
        for tok, v, sm in placed:
            hit = any(o != v and cls[o] == cls[v] for tk, o in resident[sm].items() if tk != tok)
            end = t + (py_round(dur[v] * slowdown) if hit else dur[v])
            heapq.heappush(finish, (end, tok, v, sm))

    for s, members in fifo.items():
        if members:
            at_head.add(members[0])
    for v in order:
        if v in at_head and waits[v] == 0:
            enqueue(v)
    dispatch(0)

    while finish:
        t = finish[0][0]
        ended = []
        while finish and finish[0][0] == t:
            _, tok, v, sm = heapq.heappop(finish)
            for k in range(4):
                free[sm][k] += need[v][k]
            del resident[sm][tok]
            live_count[v] -= 1
            if live_count[v] == 0 and todo[v] == 0 and v not in done_at:
                done_at[v] = t
                ended.append(v)
        fresh = []
        for v in ended:
            s = assignment[v]
            head[s] += 1
            if head[s] < len(fifo[s]):
                w = fifo[s][head[s]]
                at_head.add(w)
                if waits[w] == 0:
                    fresh.append(w)
            for c in listeners[v]:
                waits[c] -= 1
                if waits[c] == 0 and c in at_head and c not in went_eligible:
                    fresh.append(c)
        for v in sorted(fresh, key=lambda x: assignment[x]):
            enqueue(v)
        dispatch(t)

    if len(done_at) != len(order):
        raise RuntimeError("simulation ended with unfinished operators")
    return max(done_at.values())


# ------------------------------------------------------ exhaustive search


def linear_extensions(g: Dag):
    """Every linear extension, lexicographic by id (oracle.py:52-84)."""
    indeg = {v: len(g.pred[v]) for v in g.ids}
    prefix = []

    def walk():
        if len(prefix) == len(g.ids):
            yield tuple(prefix)
            return
        for v in [u for u in g.ids if indeg[u] == 0 and u not in placed]:
            placed.add(v)
            prefix.append(v)
            for s in g.succ[v]:
                indeg[s] -= 1
            yield from walk()
            for s in g.succ[v]:
                indeg[s] += 1
            prefix.pop()
            placed.discard(v)

    placed = set()
    yield from walk()


def best_order(g: Dag, assignment, num_streams, sync, cfg, limit=None):
    """(best makespan ns, best order, examined, exhausted) — first minimum wins
    (oracle.py:87-122)."""
    best_ns, best, examined, exhausted = None, (), 0, True
    for order in linear_extensions(g):
        if limit is not None and examined >= limit:
            exhausted = False
            break
        examined += 1
        ns = simulate_makespan_ns(g, assignment, num_streams, sync, list(order), cfg)
        if best_ns is None or ns < best_ns:
            best_ns, best = ns, order
    return (0 if best_ns is None else best_ns), best, examined, exhausted


# ------------------------------------------------------------------ helpers


def critical_path(g: Dag, weight):
    """Longest path under per-node weights (tests/helpers.py:90-96 pattern)."""
    dist = {}
    for v in g.topo:
        dist[v] = max((dist[p] for p in g.pred[v]), default=0) + weight[v]
    return max(dist.values()) if dist else 0
