"""Compile a stem->conv->pool model for one conv shape and replay it (ncu target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch
from test_gpu_kernels import Wrap
from paper_2312_10351_b200 import engine

cin, cout, k, s, p, hw = (int(v) for v in sys.argv[1:7])
eng = sys.argv[7] if len(sys.argv) > 7 else "tc"
torch.manual_seed(0)
m = Wrap(cin, cout, k, s, p, hw).eval()
x = torch.randn(1, 3, hw, hw)
sg = engine.compile(m, x, device=0, profile_reps=1, conv_engine=eng)
for _ in range(3):
    sg.run(x.cuda())
torch.cuda.synchronize()
for o, pr in zip(sg.program.ops, sg.profile):
    print(o.kind, o.ints, pr)
if sg.debug_ts:
    torch.cuda.synchronize()
    for k, buf in sg.debug_ts.items():
        allb = buf.cpu()
        t = allb[:64].view(8, 8)
        t0s = int(allb[0])
        iss = [int(v) - t0s for v in allb[768:832].tolist() if v > 0]
        cvt = [int(v) - t0s for v in allb[256:320].tolist() if v > 0]
        mma = [int(v) - t0s for v in allb[512:576].tolist() if v > 0]
        print("  issue", iss[:16]); print("  cvt  ", cvt[:16]); print("  mma  ", mma[:16])
        ct = allb[64:256].view(-1, 2)
        ct = ct[ct[:, 0] > 0]
        cs = ct[:, 0] - ct[:, 0].min()
        ce = ct[:, 1] - ct[:, 0].min()
        print("  ctas", ct.shape[0], "start spread ns", int(cs.max()), "lifetimes ns min/med/max",
              int((ce - cs).min()), int((ce - cs).median()), int((ce - cs).max()), "window", int(ce.max()))
        t0 = int(t[t > 0].min()) if (t > 0).any() else 0
        print("op", k, "phase ns (rows = warps 0..4; cols = start, alloc, mma_done, epi_enter, accum_ready, epi_done, end)")
        for w in range(5):
            print("  w", w, [int(v) - t0 if v > 0 else -1 for v in t[w][:7].tolist()])
tr = sg.trace(engine.SLOT_SEQUENTIAL)
print("trace (seq):", [(i, s, e, e - s) for i, s, e in tr])
t = sg.time(engine.SLOT_SEQUENTIAL, warmup=5, iters=20, flush_l2=False)
print("seq replay median ms", t.median_ms)
