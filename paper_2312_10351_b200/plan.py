"""Stream plans: Alg. 1 allocation, validation and plan files.

Drop-in for the reference allocator API (allocator.py:21-206).  The
allocation and the validation run in C++ (``opara_allocate_streams``,
``opara_validate_plan``); plan files use the reference JSON schema.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Mapping

import numpy as np

from . import _lib
from .dag import ComputationGraph, _read_json
from .errors import FormatError, PlanViolationError

DEFAULT_SYNC_OVERHEAD_US = 5.0


@dataclass(frozen=True)
class StreamPlan:
    """Operator -> stream assignment plus the cross-stream sync edges."""

    assignment: Mapping[int, int]
    num_streams: int
    sync_events: tuple[tuple[int, int], ...]

    def stream_of(self, node_id: int) -> int:
        return self.assignment[node_id]

    def streams(self) -> dict[int, list[int]]:
        """Stream id -> member ids ascending."""
        out: dict[int, list[int]] = {s: [] for s in range(self.num_streams)}
        for v in sorted(self.assignment):
            out[self.assignment[v]].append(v)
        return out


class _NativePlan(StreamPlan):
    """A StreamPlan whose ``assignment`` / ``sync_events`` are materialised from
    the C++ result arrays on first access.  Building V + E Python objects
    eagerly would dominate (and de-linearise) allocate_streams on large DAGs;
    equality with any StreamPlan is field-wise, as for the dataclass."""

    def __init__(self, ids, stream_of: np.ndarray, num_streams: int, sync_flat: np.ndarray):
        object.__setattr__(self, "_ids", ids)
        object.__setattr__(self, "_stream_of", stream_of)
        object.__setattr__(self, "_sync_flat", sync_flat)
        object.__setattr__(self, "num_streams", num_streams)

    @property
    def assignment(self) -> Mapping[int, int]:
        cached = self.__dict__.get("_assignment")
        if cached is None:
            cached = dict(zip(self._ids, self._stream_of.tolist()))
            object.__setattr__(self, "_assignment", cached)
        return cached

    @property
    def sync_events(self) -> tuple[tuple[int, int], ...]:
        cached = self.__dict__.get("_sync")
        if cached is None:
            f = self._sync_flat
            cached = tuple(zip(f[0::2].tolist(), f[1::2].tolist()))
            object.__setattr__(self, "_sync", cached)
        return cached

    def __eq__(self, other):
        if not isinstance(other, StreamPlan):
            return NotImplemented
        return (self.assignment, self.num_streams, self.sync_events) == \
               (other.assignment, other.num_streams, other.sync_events)

    __hash__ = None

    def __reduce__(self):
        return (StreamPlan, (self.assignment, self.num_streams, self.sync_events))


def allocate_streams(g: ComputationGraph) -> StreamPlan:
    """Alg. 1: walk the topo order; a node joins the stream
    of its first (ascending id) predecessor that has not yet donated, else it
    opens stream ``num_streams``.  Computed by ``opara_allocate_streams``."""
    L = _lib.lib()
    n = len(g)
    stream_of = np.empty(n, dtype=np.int32)
    sync = np.empty(2 * max(1, len(g.edges)), dtype=np.int64)
    ns = C.c_int32(0)
    nsync = C.c_int64(0)
    _lib.check(L.opara_allocate_streams(g.handle, _lib.ptr(stream_of), C.byref(ns),
                                        _lib.ptr(sync), C.byref(nsync)))
    return _NativePlan(g.node_ids, stream_of, int(ns.value), sync[: 2 * nsync.value].copy())


def single_stream_plan(g: ComputationGraph) -> StreamPlan:
    """Everything on stream 0 — the sequential-CUDA-Graph baseline plan."""
    L = _lib.lib()
    stream_of = np.empty(len(g), dtype=np.int32)
    ns = C.c_int32(0)
    _lib.check(L.opara_single_stream_plan(g.handle, _lib.ptr(stream_of), C.byref(ns)))
    return StreamPlan(assignment=dict(zip(g.node_ids, stream_of.tolist())),
                      num_streams=int(ns.value), sync_events=())


def validate_plan(g: ComputationGraph, plan: StreamPlan) -> list[str]:
    """Human-readable violations (empty = valid), computed in C++."""
    L = _lib.lib()
    items = list(plan.assignment.items())
    ids = np.asarray([int(k) for k, _ in items], dtype=np.int64)
    streams = np.asarray([int(s) for _, s in items], dtype=np.int64)
    sync = np.asarray([(int(u), int(v)) for (u, v) in plan.sync_events], dtype=np.int64).reshape(-1)
    count = C.c_int64(0)
    cap = 256 + 96 * (len(items) + len(g) + len(g.edges) + len(plan.sync_events)) + 32 * len(items)
    buf = C.create_string_buffer(cap)
    _lib.check(L.opara_validate_plan(g.handle, _lib.ptr(ids), _lib.ptr(streams), len(items),
                                     int(plan.num_streams), _lib.ptr(sync), len(plan.sync_events),
                                     buf, cap, C.byref(count)))
    if count.value == 0:
        return []
    return buf.value.decode().split("\n")


def plan_to_dict(plan: StreamPlan, g: ComputationGraph) -> dict:
    """Plan file dict; each stream lists its members in topological order."""
    rank = {v: k for k, v in enumerate(g.topo_sort())}
    return {
        "streams": {str(s): sorted(m, key=rank.__getitem__) for s, m in plan.streams().items()},
        "sync": [list(e) for e in plan.sync_events],
        "num_streams": plan.num_streams,
    }


def save_plan(plan: StreamPlan, g: ComputationGraph, path) -> None:
    Path(path).write_text(json.dumps(plan_to_dict(plan, g), indent=2, sort_keys=True) + "\n")


def load_plan(path) -> StreamPlan:
    data = _read_json(path)
    for key in ("streams", "sync", "num_streams"):
        if key not in data:
            raise FormatError(f"{path}: missing {key!r}")
    if not isinstance(data["streams"], dict):
        raise FormatError(f"{path}: 'streams' must be an object")
    assignment: dict[int, int] = {}
    for sid_raw, members in data["streams"].items():
        try:
            sid = int(sid_raw)
        except ValueError:
            raise FormatError(f"{path}: stream id {sid_raw!r} is not an integer") from None
        if not isinstance(members, list):
            raise FormatError(f"{path}: stream {sid_raw} members must be a list")
        for v in members:
            v = int(v)
            if v in assignment:
                raise FormatError(f"{path}: node {v} appears in more than one stream")
            assignment[v] = sid
    sync = []
    for raw in data["sync"]:
        if not isinstance(raw, (list, tuple)) or len(raw) != 2:
            raise FormatError(f"{path}: sync entries must be [u, v] pairs")
        sync.append((int(raw[0]), int(raw[1])))
    return StreamPlan(assignment=assignment, num_streams=int(data["num_streams"]),
                      sync_events=tuple(sorted(sync)))


@dataclass(frozen=True)
class PlanCost:
    """Eq. (1) decomposition of one (plan, order): total = parallel + syncs x
    t_overhead; parallel_ratio above 1 is flagged, never clamped."""

    sequential_us: float
    parallel_us: float
    parallel_ratio: float
    sync_count: int
    sync_overhead_us: float
    total_us: float
    exceeds_sequential: bool


def plan_cost(sequential_us: float, parallel_us: float, sync_count: int,
              sync_overhead_us: float = DEFAULT_SYNC_OVERHEAD_US) -> PlanCost:
    """Assemble a PlanCost from two makespans (simulated or measured)."""
    return PlanCost(
        sequential_us=sequential_us, parallel_us=parallel_us,
        parallel_ratio=parallel_us / sequential_us if sequential_us else 0.0,
        sync_count=sync_count, sync_overhead_us=sync_overhead_us,
        total_us=parallel_us + sync_count * sync_overhead_us,
        exceeds_sequential=parallel_us > sequential_us)


def evaluate_plan(g: ComputationGraph, plan: StreamPlan, order, cfg,
                  sync_overhead_us: float = DEFAULT_SYNC_OVERHEAD_US) -> PlanCost:
    """Eq. (1)-(3) cost of (plan, order) on the execution model (allocator.py:180-206):
    the plan is validated first (PlanViolationError on any violation), then the
    sequential and parallel makespans come from the C++ port of ``simulate``.
    ``parallel_ratio`` above 1 is flagged by ``exceeds_sequential``, not clamped."""
    from .simulator import sequential_makespan_ns, simulate   # simulator imports this module
    require_valid(g, plan)
    seq_ns = sequential_makespan_ns(g, cfg)
    para_ns = simulate(g, plan, order, cfg).makespan_ns
    count = len(plan.sync_events)
    return PlanCost(sequential_us=seq_ns / 1000, parallel_us=para_ns / 1000,
                    parallel_ratio=para_ns / seq_ns if seq_ns else 0.0,
                    sync_count=count, sync_overhead_us=sync_overhead_us,
                    total_us=para_ns / 1000 + count * sync_overhead_us,
                    exceeds_sequential=para_ns > seq_ns)


def require_valid(g: ComputationGraph, plan: StreamPlan) -> None:
    problems = validate_plan(g, plan)
    if problems:
        raise PlanViolationError("; ".join(problems))
