"""Sweep tile width (variant) and split-K of the bf16 tcgen05 GEMM on BERT's
linear shapes (Q/K/V/O 768->768, FFN1 768->3072, FFN2 3072->768, 128 tokens):
isolated in-graph time per launch (back-to-back launches, PDL)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2312_10351_b200 import _lib, engine, zoo


def profile(recs, idx, reps=50):
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.opara_exec_create(0, C.cast(recs, C.c_void_p), len(recs), C.byref(h)))
    out = (_lib.OparaOpProfile * len(recs))()
    _lib.check(L.opara_exec_profile(h, reps, C.cast(out, C.c_void_p)))
    L.opara_exec_destroy(h)
    return [out[i] for i in idx]


model, _, ids = zoo.build_bert()
sg = engine.compile(model, ids, device=0, dtype="bf16", profile_reps=5)
ops = sg.program.ops
pick = {}
for i, o in enumerate(ops):
    if o.kind == 1:
        pick.setdefault((o.ints["Cin"], o.ints["Cout"]), i)
idx = list(pick.values())
for (k, n), i in pick.items():
    print(f"K={k} N={n} op {i}: auto {sg.profile[i]['isolated_us']:.2f} us blocks {sg.profile[i]['num_blocks']}")
for var in range(4):
    for splits in (1, 2, 3, 4, 6, 8):
        recs = (_lib.OparaOp * len(sg._recs))()
        C.memmove(recs, sg._recs, C.sizeof(sg._recs))
        for i in idx:
            recs[i].variant = var
            recs[i].i[19] = splits
        try:
            ps = profile(recs, idx)
            print(f"bn{[32, 64, 128, 256][var]:3d} split {splits}: " +
                  "  ".join(f"{k}x{n} {p.isolated_us:6.2f}us/{p.num_blocks}" for (k, n), p in zip(pick, ps)))
        except Exception as e:  # noqa: BLE001
            print("fail", var, splits, e)
