"""Our CLI against the reference CLI's own outputs (tests/golden/cli, made by
`python -m opsched` in the build container): schedule / simulate / compare
write byte-identical plan, order, trace, result and report files, print the
same lines, and keep the exit-code contract (0 / 2)."""

from __future__ import annotations

import shutil
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT

CLI = GOLDEN / "cli"


def _run(td, *args):
    return subprocess.run([sys.executable, "-m", "paper_2312_10351_b200", *args], cwd=td, capture_output=True,
                          text=True, env={"PYTHONPATH": str(ROOT), "PATH": "/usr/bin:/bin"})


@pytest.mark.parametrize("name", ["cases", "googlenet"])
def test_cli_matches_reference_outputs(tmp_path, name):
    shutil.copy(CLI / f"{name}.json", tmp_path / "g.json")
    shutil.copy(CLI / "b200.json", tmp_path / "b200.json")
    r1 = _run(tmp_path, "schedule", "g.json", "--gpu-config", "b200.json")
    assert r1.returncode == 0, r1.stderr
    r2 = _run(tmp_path, "simulate", "g.json", "g.plan.json", "g.order.json", "--trace", "g.tsv", "--out",
              "g.sim.json", "--gpu-config", "b200.json")
    assert r2.returncode == 0, r2.stderr
    r3 = _run(tmp_path, "compare", "g.json", "--policies", "sequential,opara,dfs,wavefront,random", "--out",
              "g.compare.json", "--gpu-config", "b200.json")
    assert r3.returncode == 0, r3.stderr
    for suffix in ("plan.json", "order.json", "tsv", "sim.json", "compare.json"):
        assert (tmp_path / f"g.{suffix}").read_bytes() == (CLI / f"{name}.{suffix}").read_bytes(), suffix
    assert r1.stdout + r3.stdout == (CLI / f"{name}.stdout").read_text()


def test_cli_exit_codes(tmp_path):
    assert _run(tmp_path, "schedule", "missing.json").returncode == 2
    shutil.copy(CLI / "cases.json", tmp_path / "g.json")
    r = _run(tmp_path, "compare", "g.json", "--policies", "opara")
    assert r.returncode == 2 and "at least two policies" in r.stderr
    r = _run(tmp_path, "compare", "g.json", "--policies", "opara,nope")
    assert r.returncode == 2 and "unknown policy" in r.stderr
