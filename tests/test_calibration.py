"""The b200-calibrated preset (§8f rank 1) against the committed measured run:
its fitted same-class slowdown predicts the measured multi-stream graph
latencies of the block-bound configs better than the reference default 1.4."""

from __future__ import annotations

import sys
from pathlib import Path

import paper_2312_10351_b200 as op

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "scripts"))


def test_calibrated_preset_beats_default_on_committed_run():
    import calibrate
    rows = [r for r in calibrate.load(ROOT / "profiles" / "r02_run_a") if not r["name"].startswith("deepfm")]
    assert len(rows) >= 5
    s = op.GPU_PRESETS["b200-calibrated"].same_class_slowdown
    fitted = calibrate.err(rows, [calibrate.predict(r, s) for r in rows])
    default = calibrate.err(rows, [calibrate.predict(r, 1.4) for r in rows])
    assert fitted < default and fitted < 0.1, (fitted, default)
