"""Launch orders: Alg. 2 and the baseline policies.

Drop-in for the reference orderer API (orderer.py:25-180).  ``opara``,
``sequential``, ``dfs`` and ``wavefront`` are computed in C++ by
``opara_order``; ``random`` stays host-side because its definition *is*
CPython's Mersenne Twister (``random.Random(seed).randrange``).
"""

from __future__ import annotations

import bisect
import ctypes as C
import json
import random
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .dag import ComputationGraph, ResourceDemand, _read_json
from .errors import FormatError

POLICIES = ("opara", "dfs", "wavefront", "random", "sequential")
_POLICY_CODE = {"opara": 0, "sequential": 1, "dfs": 2, "wavefront": 3}


@dataclass(frozen=True)
class LaunchSchedule:
    """A launch order and the policy (and seed) that produced it."""

    order: tuple[int, ...]
    policy: str
    seed: int | None = None


@dataclass(frozen=True, order=True)
class ResourceScore:
    """Alg. 2 sort key: dominant share, then node id."""

    dominant_share: float
    node_id: int


def dominant_share(demand: ResourceDemand, cfg) -> float:
    """max(threads/threads_per_sm, smem/smem_per_sm, regs/regs_per_sm) x blocks,
    in IEEE double exactly as orderer.py:48-53 (computed by libopara)."""
    node = _lib.OparaNode(0, 0, 0, int(demand.num_blocks), int(demand.threads_per_block),
                          int(demand.shared_mem_per_block), int(demand.registers_per_thread))
    out = C.c_double(0.0)
    cfg_s = _lib.gpu_config_struct(cfg)
    _lib.check(_lib.lib().opara_dominant_share(C.byref(node), C.byref(cfg_s), C.byref(out)))
    return out.value


def resource_score(g: ComputationGraph, node_id: int, cfg) -> ResourceScore:
    return ResourceScore(dominant_share(g.node(node_id).demand, cfg), node_id)


def _native_order(g: ComputationGraph, code: int, cfg) -> tuple[int, ...]:
    out = np.empty(len(g), dtype=np.int64)
    cfg_s = _lib.gpu_config_struct(cfg) if cfg is not None else None
    _lib.check(_lib.lib().opara_order(g.handle, code, C.byref(cfg_s) if cfg_s is not None else None,
                                      _lib.ptr(out)))
    return tuple(out.tolist())


def order_opara(g: ComputationGraph, cfg) -> LaunchSchedule:
    """Alg. 2: memory and compute ready lists, cheapest
    (dominant share, id) first, alternating to the class not just launched,
    starting with memory."""
    return LaunchSchedule(order=_native_order(g, 0, cfg), policy="opara")


def _order_random(g: ComputationGraph, seed: int) -> tuple[int, ...]:
    rng = random.Random(seed)
    indeg = {v: len(g.predecessors(v)) for v in g.node_ids}
    ready = sorted(v for v in g.node_ids if indeg[v] == 0)
    out = []
    while ready:
        v = ready.pop(rng.randrange(len(ready)))
        out.append(v)
        for s in g.successors(v):
            indeg[s] -= 1
            if indeg[s] == 0:
                bisect.insort(ready, s)
    return tuple(out)


def order_baseline(g: ComputationGraph, policy: str, seed: int | None = None) -> LaunchSchedule:
    """dfs / wavefront / sequential (C++) and random (seeded, host-side)."""
    if policy in ("dfs", "wavefront", "sequential"):
        return LaunchSchedule(order=_native_order(g, _POLICY_CODE[policy], None), policy=policy)
    if policy == "random":
        actual = 0 if seed is None else seed
        return LaunchSchedule(order=_order_random(g, actual), policy="random", seed=actual)
    raise ValueError(f"unknown baseline policy {policy!r}")


def make_order(g: ComputationGraph, policy: str, cfg, seed: int | None = None) -> LaunchSchedule:
    if policy == "opara":
        return order_opara(g, cfg)
    return order_baseline(g, policy, seed)


def schedule_to_dict(sched: LaunchSchedule) -> dict:
    return {"policy": sched.policy, "seed": sched.seed, "order": list(sched.order)}


def save_schedule(sched: LaunchSchedule, path) -> None:
    Path(path).write_text(json.dumps(schedule_to_dict(sched), indent=2, sort_keys=True) + "\n")


def load_schedule(path) -> LaunchSchedule:
    data = _read_json(path)
    if "order" not in data or not isinstance(data["order"], list):
        raise FormatError(f"{path}: missing 'order' list")
    seed = data.get("seed")
    return LaunchSchedule(order=tuple(int(v) for v in data["order"]),
                          policy=str(data.get("policy", "unknown")),
                          seed=None if seed is None else int(seed))
