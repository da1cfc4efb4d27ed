"""GPU capacity model (GpuConfig) and the B200 preset.

Same fields, presets and file schema as the reference (simulator.py:42-121),
plus a ``b200`` preset and ``device_gpu_config`` which reads the live
capacities from cudaGetDeviceProperties through libopara.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

from . import _lib
from .dag import _read_json
from .errors import FormatError


@dataclass(frozen=True)
class GpuConfig:
    """Per-SM capacities (plus SM count and the same-class slowdown knob)."""

    num_sms: int
    threads_per_sm: int
    shared_mem_per_sm: int
    registers_per_sm: int
    max_blocks_per_sm: int
    same_class_slowdown: float = 1.4

    def __post_init__(self) -> None:
        for name in ("num_sms", "threads_per_sm", "shared_mem_per_sm", "registers_per_sm",
                     "max_blocks_per_sm"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.same_class_slowdown < 1.0:
            raise ValueError("same_class_slowdown must be >= 1.0")


GPU_PRESETS: dict[str, GpuConfig] = {
    "a100-like": GpuConfig(108, 2048, 167936, 65536, 32),
    "2080s-like": GpuConfig(48, 1024, 65536, 65536, 16),
    # cudaGetDeviceProperties on a B200 (sm_100): 148 SMs, 2048 threads,
    # 228 KiB smem, 64 Ki registers, 32 resident blocks per SM.
    "b200": GpuConfig(148, 2048, 233472, 65536, 32),
    # same capacities, same-class slowdown fitted to measured B200 graph
    # latencies of the seven block-bound BASELINE configs (scripts/calibrate.py,
    # profiles/r02_calibration.md: mean |log error| 0.065 vs 0.102 at 1.4)
    "b200-calibrated": GpuConfig(148, 2048, 233472, 65536, 32, 1.9),
}

DEFAULT_GPU = "2080s-like"


def load_gpu_config(spec) -> GpuConfig:
    """Preset name or GpuConfig JSON file."""
    if isinstance(spec, str) and spec in GPU_PRESETS:
        return GPU_PRESETS[spec]
    path = Path(spec)
    if not path.exists():
        raise FormatError(f"gpu config {spec!r} is neither a preset "
                          f"({', '.join(sorted(GPU_PRESETS))}) nor an existing file")
    data = _read_json(path)
    keys = ("num_sms", "threads_per_sm", "shared_mem_per_sm", "registers_per_sm",
            "max_blocks_per_sm")
    for key in keys:
        if key not in data:
            raise FormatError(f"{path}: missing {key!r}")
    try:
        return GpuConfig(*(int(data[k]) for k in keys),
                         same_class_slowdown=float(data.get("same_class_slowdown", 1.4)))
    except ValueError as exc:
        raise FormatError(f"{path}: {exc}") from None


def gpu_config_to_dict(cfg: GpuConfig) -> dict:
    return {"num_sms": cfg.num_sms, "threads_per_sm": cfg.threads_per_sm,
            "shared_mem_per_sm": cfg.shared_mem_per_sm, "registers_per_sm": cfg.registers_per_sm,
            "max_blocks_per_sm": cfg.max_blocks_per_sm,
            "same_class_slowdown": cfg.same_class_slowdown}


def device_gpu_config(device: int = 0) -> GpuConfig:
    """Live capacities of a CUDA device (requires a GPU)."""
    out = _lib.OparaGpuConfig()
    _lib.check(_lib.lib().opara_device_gpu_config(int(device), C.byref(out)))
    return GpuConfig(out.num_sms, out.threads_per_sm, out.shared_mem_per_sm, out.registers_per_sm,
                     out.max_blocks_per_sm, out.same_class_slowdown)
