"""The reference's execution model, on the C++ port (`opara_simulate`).

Drop-in for ``opsched.simulator`` (simulator.py:148-475): the same
``SimResult`` / ``OpRecord`` / ``BlockRecord`` records, ``simulate``,
``sequential_makespan[_ns]``, ``trace`` / ``trace_tsv`` / ``write_trace`` and
``result_to_dict``.  Input checks (coverage, linear extension, plan validity,
infeasible blocks) run here with the reference's wording (_check_inputs,
simulator.py:187-209); the discrete-event loop — where the reference spends
50-340 ms per model DAG — runs in csrc/simulate.cpp and is bit-exact with
it (integer nanoseconds, Python-round slowdowns, identical tie-breaks).

On the B200 the real multi-stream CUDA Graph (engine.ScheduledGraph) is the
"run"; this model predicts a schedule's makespan without a device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .dag import ComputationGraph, OpClass
from .device import DEFAULT_GPU, GPU_PRESETS, GpuConfig, gpu_config_to_dict, load_gpu_config  # noqa: F401
from .errors import CoverageError, InfeasibleBlockError, PlanViolationError
from .plan import StreamPlan, single_stream_plan, validate_plan


@dataclass(frozen=True)
class BlockRecord:
    """One placed thread block (simulator.py:127-135)."""

    op_id: int
    index: int
    sm: int
    start_ns: int
    end_ns: int


@dataclass(frozen=True)
class OpRecord:
    """Per-operator execution summary (simulator.py:138-147)."""

    op_id: int
    name: str
    op_class: OpClass
    stream: int
    start_ns: int
    end_ns: int
    sms: tuple[int, ...]


@dataclass(frozen=True)
class SimResult:
    """Outcome of one simulation run (simulator.py:148-179)."""

    makespan_ns: int
    ops: tuple[OpRecord, ...]
    blocks: tuple[BlockRecord, ...]
    sm_busy_ns: tuple[int, ...]
    sm_efficiency: float
    blocked_ns: int
    sync_wait_ns: int

    @property
    def makespan_us(self) -> float:
        return self.makespan_ns / 1000

    def op_start_ns(self, op_id: int) -> int:
        return self._op(op_id).start_ns

    def op_end_ns(self, op_id: int) -> int:
        return self._op(op_id).end_ns

    def _op(self, op_id: int) -> OpRecord:
        for rec in self.ops:
            if rec.op_id == op_id:
                return rec
        raise KeyError(f"unknown op id {op_id}")


def _order_of(schedule) -> list[int]:
    return list(getattr(schedule, "order", schedule))


def _check_inputs(g: ComputationGraph, plan: StreamPlan, order: list[int], cfg: GpuConfig) -> None:
    """simulator.py:187-209, same checks in the same order and wording."""
    ids = set(g.node_ids)
    if set(order) != ids or len(order) != len(ids):
        missing = sorted(ids - set(order))
        extra = sorted(set(order) - ids)
        raise CoverageError(f"launch order must cover the graph exactly (missing {missing}, extra {extra})")
    if not g.is_linear_extension(order):
        raise CoverageError("launch order is not a linear extension of the graph")
    problems = validate_plan(g, plan)
    if problems:
        raise PlanViolationError("; ".join(problems))
    for n in g.nodes:
        d = n.demand
        if (d.threads_per_block > cfg.threads_per_sm or d.shared_mem_per_block > cfg.shared_mem_per_sm
                or d.registers_per_block > cfg.registers_per_sm):
            raise InfeasibleBlockError(f"operator {n.id} ({n.name}): one block exceeds a single SM's capacity")


def simulate(g: ComputationGraph, plan: StreamPlan, schedule, cfg: GpuConfig, *,
             blocks: bool = True) -> SimResult:
    """Run the execution model for one (plan, launch order) pair.

    ``blocks=False`` skips materialising the per-block log: the makespan, SM
    busy times and every per-op timing field are unaffected, but ``OpRecord.sms``
    (rebuilt from the block log) is empty and ``blocks`` is ``()``."""
    order = _order_of(schedule)
    _check_inputs(g, plan, order, cfg)
    if not order:
        return SimResult(0, (), (), (0,) * cfg.num_sms, 0.0, 0, 0)
    ids = g.node_ids
    n = len(ids)
    dur = np.asarray([nd.block_duration_ns for nd in g.nodes], dtype=np.int64)
    stream_of = np.asarray([plan.assignment[v] for v in ids], dtype=np.int32)
    order_a = np.asarray(order, dtype=np.int64)
    sync = np.asarray([(u, v) for (u, v) in plan.sync_events], dtype=np.int64).reshape(-1)
    start = np.zeros(n, dtype=np.int64)
    end = np.zeros(n, dtype=np.int64)
    busy = np.zeros(cfg.num_sms, dtype=np.int64)
    total_blocks = sum(nd.demand.num_blocks for nd in g.nodes)
    log = np.zeros((total_blocks if blocks else 0, 5), dtype=np.int64)
    res = _lib.OparaSimResult()
    nb = C.c_int64(0)
    L = _lib.lib()
    _lib.check(L.opara_simulate(g.handle, _lib.ptr(dur), _lib.ptr(stream_of), int(plan.num_streams),
                                _lib.ptr(order_a), _lib.ptr(sync), len(plan.sync_events),
                                C.byref(_lib.gpu_config_struct(cfg)), C.byref(res), _lib.ptr(start),
                                _lib.ptr(end), _lib.ptr(busy), _lib.ptr(log) if blocks else None,
                                log.shape[0], C.byref(nb)))
    sms: dict[int, set] = {v: set() for v in ids}
    block_recs: tuple = ()
    if blocks:
        rows = sorted(map(tuple, log[: nb.value].tolist()))
        block_recs = tuple(BlockRecord(*r) for r in rows)
        for r in rows:
            sms[r[0]].add(r[2])
    ops = tuple(OpRecord(op_id=v, name=nd.name, op_class=nd.op_class, stream=plan.assignment[v],
                         start_ns=int(start[k]), end_ns=int(end[k]), sms=tuple(sorted(sms[v])))
                for k, (v, nd) in enumerate(zip(ids, g.nodes)))
    return SimResult(makespan_ns=int(res.makespan_ns), ops=ops, blocks=block_recs,
                     sm_busy_ns=tuple(int(x) for x in busy), sm_efficiency=float(res.sm_efficiency),
                     blocked_ns=int(res.blocked_ns), sync_wait_ns=int(res.sync_wait_ns))


def sequential_makespan_ns(g: ComputationGraph, cfg: GpuConfig) -> int:
    """Makespan of the single-stream topological schedule (simulator.py:418-426)."""
    return simulate(g, single_stream_plan(g), g.topo_sort(), cfg, blocks=False).makespan_ns


def sequential_makespan(g: ComputationGraph, cfg: GpuConfig) -> float:
    return sequential_makespan_ns(g, cfg) / 1000


def trace(result: SimResult) -> list[OpRecord]:
    """Per-operator timeline rows sorted by start time (ties by op id)."""
    return sorted(result.ops, key=lambda r: (r.start_ns, r.op_id))


TRACE_HEADER = "op_id\tname\tclass\tstream\tstart_ns\tend_ns"


def trace_tsv(result: SimResult) -> str:
    lines = [TRACE_HEADER]
    for r in trace(result):
        lines.append(f"{r.op_id}\t{r.name}\t{r.op_class.value}\t{r.stream}\t{r.start_ns}\t{r.end_ns}")
    return "\n".join(lines) + "\n"


def write_trace(result: SimResult, path) -> None:
    Path(path).write_text(trace_tsv(result))


def result_to_dict(result: SimResult) -> dict:
    """SimResult as a JSON-serialisable dict (simulator.py:455-475)."""
    return {
        "makespan_ns": result.makespan_ns,
        "makespan_us": result.makespan_ns / 1000,
        "sm_busy_ns": list(result.sm_busy_ns),
        "sm_efficiency": result.sm_efficiency,
        "blocked_ns": result.blocked_ns,
        "sync_wait_ns": result.sync_wait_ns,
        "ops": {
            str(r.op_id): {"name": r.name, "class": r.op_class.value, "stream": r.stream,
                           "start_ns": r.start_ns, "end_ns": r.end_ns, "sms": list(r.sms)}
            for r in result.ops
        },
    }
