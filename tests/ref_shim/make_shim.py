"""Assemble a throw-away ``opsched`` package whose hot path is OURS.

The reference test suite (/root/reference/pkg/tests, 158 tests) imports
``opsched``.  This shim answers those imports with:

* errors / graph / allocator / orderer / simulator  ->  paper_2312_10351_b200
  (C++ via the C ABI: scheduler, and the bit-exact port of the execution model)
* oracle  ->  paper_2312_10351_b200.search (exhaustive order / plan search)
* generators / cli / __init__ / __main__  ->  the reference modules
  themselves (symlinked into a temp dir, never copied into the repo); they are
  out of the hot path and are the consumers of our outputs.

Used only by tests/test_reference_suite.py in the build container (where
/root/reference exists).
"""

from __future__ import annotations

import os
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src/opsched")

ERRORS = "from paper_2312_10351_b200.errors import *  # noqa\n" \
         "from paper_2312_10351_b200.errors import (SchedulerError, FormatError, GraphValidationError,\n" \
         "    PlanViolationError, CoverageError, InfeasibleBlockError)\n"
GRAPH = "from paper_2312_10351_b200.dag import (OpClass, classify, ResourceDemand, OperatorNode,\n" \
        "    ComputationGraph, load_graph, save_graph, graph_to_dict, apply_profile, _read_json)\n"
ALLOCATOR = "from paper_2312_10351_b200.plan import (DEFAULT_SYNC_OVERHEAD_US, PlanCost, StreamPlan,\n" \
            "    allocate_streams, evaluate_plan, load_plan, plan_to_dict, save_plan, single_stream_plan,\n" \
            "    validate_plan)\n"
SIMULATOR = "from paper_2312_10351_b200.simulator import *  # noqa\n" \
            "from paper_2312_10351_b200.simulator import (BlockRecord, OpRecord, SimResult, TRACE_HEADER,\n" \
            "    DEFAULT_GPU, GPU_PRESETS, GpuConfig, gpu_config_to_dict, load_gpu_config, result_to_dict,\n" \
            "    sequential_makespan, sequential_makespan_ns, simulate, trace, trace_tsv, write_trace,\n" \
            "    _check_inputs, _order_of)\n"
ORACLE = "from paper_2312_10351_b200.search import (OracleResult, PlanSearchResult, linear_extensions,\n" \
         "    best_order, best_plan, _partitions)\n"
ORDERER = "from paper_2312_10351_b200.order import (POLICIES, LaunchSchedule, ResourceScore,\n" \
          "    dominant_share, resource_score, order_opara, order_baseline, make_order,\n" \
          "    schedule_to_dict, save_schedule, load_schedule)\n" \
          "from .simulator import GpuConfig  # noqa: F401\n"


def make_shim(root: Path) -> Path:
    pkg = root / "opsched"
    pkg.mkdir(parents=True, exist_ok=True)
    (pkg / "errors.py").write_text(ERRORS)
    (pkg / "graph.py").write_text(GRAPH)
    (pkg / "allocator.py").write_text(ALLOCATOR)
    (pkg / "orderer.py").write_text(ORDERER)
    (pkg / "simulator.py").write_text(SIMULATOR)
    (pkg / "oracle.py").write_text(ORACLE)
    for name in ("__init__.py", "__main__.py", "generators.py", "cli.py"):
        link = pkg / name
        if not link.exists():
            os.symlink(REF_SRC / name, link)
    return root
