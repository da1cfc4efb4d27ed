"""Exhaustive launch-order search on a sub-DAG block, on the B200 (§8f rank 4):
every linear extension of Inception-v3's InceptionB block captured with the
Alg. 1 plan gives the bit-identical output, and the measured search ranks the
Opara order among all of them."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_every_order_of_a_block_gives_identical_output():
    from paper_2312_10351_b200 import engine, search, zoo
    from paper_2312_10351_b200.order import LaunchSchedule
    model, x = zoo.build("inception_v3_b")
    sg = engine.compile(model, x, device=0, profile_reps=2)
    try:
        want = sg.run(x.cuda()).clone()
        orders = list(search.linear_extensions(sg.graph))
        assert len(orders) == 20
        for o in orders:
            sg.capture(search.SCRATCH_SLOT, sg.plan, LaunchSchedule(o, "search"))
            assert torch.equal(sg.run(x.cuda(), slot=search.SCRATCH_SLOT), want), o
        res = search.search_measured(sg, iters=20, rounds=1, recheck=3)
        assert res["orders_examined"] == 20 and res["search_space_exhausted"]
        assert 1 <= res["policies"]["opara"]["rank"] <= 20
        assert res["best_ms"] <= res["policies"]["opara"]["ms"] * 1.0001
    finally:
        sg.close()
