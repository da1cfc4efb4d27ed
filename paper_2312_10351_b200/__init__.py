"""paper_2312_10351_b200 — Opara's operator-parallel DAG executor, B200-native.

Drop-in for the reference ``opsched`` package's hot path: the same public
names for the graph model, the stream allocator (Alg. 1) and the launch
orderer (Alg. 2), computed by the C++ scheduler in libopara.so; and, in place
of the reference's simulated "run", a real multi-stream CUDA Graph executor
with hand-written sm_100a kernels (``compile`` / ``ScheduledGraph.run``); the
simulated run itself is kept as a bit-exact C++ port (``simulate``).
"""

__version__ = "0.1.0"  # the reference opsched version this package is a drop-in for (cli metadata)

import os as _os

# The driver reads CUDA_DEVICE_MAX_CONNECTIONS once, when the CUDA context is
# created: set it before any CUDA call so every plan stream can map onto its
# own hardware queue (bench.py sets it before importing torch as well).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .dag import (ComputationGraph, OpClass, OperatorNode, ResourceDemand, apply_profile,
                  classify, graph_from_dict, graph_to_dict, load_graph, save_graph)
from .device import (DEFAULT_GPU, GPU_PRESETS, GpuConfig, device_gpu_config, gpu_config_to_dict,
                     load_gpu_config)
from .errors import (CoverageError, CudaError, FormatError, GraphValidationError,
                     InfeasibleBlockError, PlanViolationError, SchedulerError)
from .order import (POLICIES, LaunchSchedule, ResourceScore, dominant_share, load_schedule,
                    make_order, order_baseline, order_opara, resource_score, save_schedule,
                    schedule_to_dict)
from .plan import (DEFAULT_SYNC_OVERHEAD_US, PlanCost, StreamPlan, allocate_streams, evaluate_plan,
                   load_plan, plan_to_dict, save_plan, single_stream_plan, validate_plan)
from .simulator import (BlockRecord, OpRecord, SimResult, result_to_dict, sequential_makespan,
                        sequential_makespan_ns, simulate, trace, trace_tsv, write_trace)

__all__ = [
    "__version__", "ComputationGraph", "CoverageError", "CudaError", "DEFAULT_GPU",
    "DEFAULT_SYNC_OVERHEAD_US", "FormatError", "GPU_PRESETS", "GpuConfig", "GraphValidationError",
    "InfeasibleBlockError", "LaunchSchedule", "OpClass", "OperatorNode", "POLICIES", "PlanCost",
    "PlanViolationError", "ResourceDemand", "ResourceScore", "SchedulerError", "StreamPlan",
    "allocate_streams", "apply_profile", "evaluate_plan", "classify", "device_gpu_config", "dominant_share",
    "gpu_config_to_dict", "graph_from_dict", "graph_to_dict", "load_gpu_config", "load_graph",
    "load_plan", "load_schedule", "make_order", "order_baseline", "order_opara", "plan_to_dict",
    "resource_score", "save_graph", "save_plan", "save_schedule", "schedule_to_dict",
    "single_stream_plan", "validate_plan", "BlockRecord", "OpRecord", "SimResult", "result_to_dict",
    "sequential_makespan", "sequential_makespan_ns", "simulate", "trace", "trace_tsv", "write_trace",
]
