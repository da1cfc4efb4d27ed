"""Shared pytest setup: markers, repo root on sys.path, golden-vector loaders."""

from __future__ import annotations

import json
import os
import sys
import tempfile
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: longer CPU-only cases")
    # One tile-tuning cache per test session: the GPU suite compiles the same
    # models many times (per split-K mode, grid policy and bench variant), and
    # every (shape, budget, reduction) key is tuned once instead of per compile.
    # Any cached choice is a measured-valid tile; tests that need a private
    # cache set their own (monkeypatch).
    if "OPARA_TUNE_CACHE" not in os.environ:
        os.environ["OPARA_TUNE_CACHE"] = os.path.join(tempfile.mkdtemp(prefix="opara_tune_"), "tune.json")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@lru_cache(maxsize=None)
def golden_sched():
    return json.loads((GOLDEN / "sched_golden.json").read_text())


def golden_nodes(case):
    """Golden compact nodes -> graph-file node dicts (oracle schema)."""
    out = []
    for nid, cls, blocks, thr, smem, regs, dur in case["nodes"]:
        out.append({"id": nid, "name": "op", "class": "compute" if cls == 0 else "memory",
                    "blocks": blocks, "threads_per_block": thr, "shared_mem_bytes": smem,
                    "registers_per_thread": regs, "block_duration_us": dur})
    return out
