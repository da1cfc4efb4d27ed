"""Run the reference's OWN test suite (158 tests) against our C++ scheduler
and our C++ port of its execution model.

The shim (tests/ref_shim/make_shim.py) routes the reference's graph /
allocator / orderer / simulator imports to paper_2312_10351_b200.  Needs /root/reference,
so it runs in the build container and skips elsewhere (e.g. the GPU box).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = Path("/root/reference/pkg/tests")


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference tree not present")
def test_reference_suite_passes_against_native_scheduler(tmp_path):
    sys.path.insert(0, str(ROOT / "tests" / "ref_shim"))
    from make_shim import make_shim
    shim = make_shim(tmp_path / "shim")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(shim), str(ROOT), str(REF_TESTS)])
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x",
         "--rootdir", str(tmp_path), str(REF_TESTS)],
        capture_output=True, text=True, env=env, cwd=tmp_path, timeout=900)
    tail = res.stdout[-3000:] + res.stderr[-2000:]
    assert res.returncode == 0, tail
    # every reference test ran against the shim and passed
    assert " passed" in res.stdout and "failed" not in res.stdout, tail
    # prove the hot path really was ours
    probe = subprocess.run(
        [sys.executable, "-c", "import opsched, opsched.allocator as a; print(a.allocate_streams.__module__)"],
        capture_output=True, text=True, env=env, cwd=tmp_path)
    assert probe.stdout.strip() == "paper_2312_10351_b200.plan", probe.stderr
    probe = subprocess.run(
        [sys.executable, "-c", "import opsched.simulator as s; print(s.simulate.__module__)"],
        capture_output=True, text=True, env=env, cwd=tmp_path)
    assert probe.stdout.strip() == "paper_2312_10351_b200.simulator", probe.stderr
    probe = subprocess.run(
        [sys.executable, "-c", "import opsched.oracle as o; print(o.best_order.__module__, o.linear_extensions.__module__)"],
        capture_output=True, text=True, env=env, cwd=tmp_path)
    assert probe.stdout.split() == ["paper_2312_10351_b200.search"] * 2, probe.stderr
