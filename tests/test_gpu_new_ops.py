"""Numerics of the NASNet / DeepFM operator families on the B200 through the
executor (C ABI) against the plain PyTorch fp32 forward of the same module
(TF32 off): depthwise conv with fused input ReLU, n-ary ADD, fused input ReLU
on the three conv engines, subsample-folded 1x1 convs, global pooling of a
ReLU, and the DeepFM gather / first-order / FM kernels."""

from __future__ import annotations

import pytest
import torch
import torch.nn as nn

from paper_2312_10351_b200 import zoo

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return (torch.linalg.vector_norm(a.double() - b.double()) / torch.linalg.vector_norm(b.double())).item()


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False


def _bn(c):
    bn = nn.BatchNorm2d(c, eps=1e-3)
    with torch.no_grad():
        bn.running_mean.normal_(0, 0.1)
        bn.running_var.uniform_(0.5, 1.5)
        bn.weight.uniform_(0.5, 1.5)
        bn.bias.normal_(0, 0.1)
    return bn


class SepBlock(nn.Module):
    """stem conv -> ReLU -> depthwise k x k / s -> 1x1 + BN -> ReLU -> depthwise -> 1x1 + BN, added to a pool."""

    def __init__(self, c, k, s):
        super().__init__()
        self.stem = nn.Conv2d(3, c, 1, bias=False)
        self.sbn = _bn(c)
        self.dw1 = nn.Conv2d(c, c, k, s, k // 2, groups=c, bias=False)
        self.pw1 = nn.Conv2d(c, c, 1, bias=False)
        self.bn1 = _bn(c)
        self.dw2 = nn.Conv2d(c, c, k, 1, k // 2, groups=c, bias=False)
        self.pw2 = nn.Conv2d(c, c, 1, bias=False)
        self.bn2 = _bn(c)
        self.pool = nn.AvgPool2d(3, s, 1, count_include_pad=False)

    def forward(self, x):
        x = self.sbn(self.stem(x))
        y = self.bn1(self.pw1(self.dw1(torch.relu(x))))
        y = self.bn2(self.pw2(self.dw2(torch.relu(y))))
        return y + self.pool(x)


@pytest.mark.parametrize("c,k,s,hw,dtype,tol", [(32, 3, 1, 21, "f32", 1e-4), (48, 5, 2, 42, "f32", 1e-4),
                                                (64, 7, 2, 83, "f32", 1e-4), (40, 3, 1, 11, "f32", 1e-4),
                                                (64, 5, 2, 42, "bf16", 1e-2), (96, 7, 1, 21, "bf16", 1e-2),
                                                (42, 5, 2, 83, "bf16", 1e-2), (84, 7, 2, 42, "bf16", 1e-2),
                                                (42, 3, 1, 21, "f32", 1e-4), (36, 5, 1, 11, "bf16", 1e-2)])
def test_separable_block(c, k, s, hw, dtype, tol):
    from paper_2312_10351_b200 import engine
    torch.manual_seed(0)
    m = SepBlock(c, k, s).eval()
    x = torch.randn(1, 3, hw, hw)
    sg = engine.compile(m, x, device=0, profile_reps=2, dtype=dtype)
    kinds = {op.kind for op in sg.program.ops}
    assert 13 in kinds and 6 in kinds  # DWCONV2D and ADD launched, ReLUs fused
    assert 14 not in kinds
    y = sg.run(x.cuda()).float()
    with torch.no_grad():
        ref = m.cuda()(x.cuda()).permute(0, 2, 3, 1)
    assert _rel(y.reshape(ref.shape), ref) <= tol


class ReluConvHead(nn.Module):
    """relu -> 1x1 conv (fused input ReLU on the engine) and factorized
    reduction (subsample offsets 0/1 folded into stride-2 1x1 convs), then
    global average pool of a ReLU -> linear."""

    def __init__(self, c, cout):
        super().__init__()
        self.stem = nn.Conv2d(3, c, 3, 1, 1, bias=False)
        self.sbn = _bn(c)
        self.conv = nn.Conv2d(c, cout, 1, bias=False)
        self.bn = _bn(cout)
        self.p1 = nn.Conv2d(c, cout // 2, 1, bias=False)
        self.b1 = _bn(cout // 2)
        self.p2 = nn.Conv2d(c, cout // 2, 1, bias=False)
        self.b2 = _bn(cout // 2)
        self.fc = nn.Linear(3 * cout + c, 10)

    def forward(self, x):
        x = self.sbn(self.stem(x))
        r = torch.relu(x)            # x is also read raw below, so the ReLU fuses into the consumers
        a = self.bn(self.conv(r))
        b = torch.cat([self.b1(self.p1(zoo.subsample2d(r, 0))), self.b2(self.p2(zoo.subsample2d(r, 1)))], 1)
        gap = nn.functional.adaptive_avg_pool2d
        feats = [gap(torch.relu(a), 1), gap(a, 1), gap(torch.relu(b), 1), gap(x, 1)]
        return self.fc(torch.flatten(torch.cat(feats, 1), 1))


@pytest.mark.parametrize("c,cout,hw,dtype,tol", [(64, 128, 21, "f32", 1e-4), (96, 64, 42, "f32", 1e-4),
                                                 (64, 128, 21, "bf16", 1e-2), (128, 256, 11, "bf16", 1e-2)])
def test_relu_in_and_subsample(c, cout, hw, dtype, tol):
    from paper_2312_10351_b200 import engine
    torch.manual_seed(1)
    m = ReluConvHead(c, cout).eval()
    x = torch.randn(1, 3, hw, hw)
    sg = engine.compile(m, x, device=0, profile_reps=2, dtype=dtype)
    assert any(op.ints.get("relu_in") for op in sg.program.ops if op.kind == 1)
    assert any(op.ints.get("ph", 0) < 0 for op in sg.program.ops if op.kind == 1)
    y = sg.run(x.cuda())
    with torch.no_grad():
        ref = m.cuda()(x.cuda())
    assert _rel(y, ref) <= tol


@pytest.mark.parametrize("batch", [1, 2, 4, 8, 16, 32])
def test_deepfm_parity(batch):
    """The BASELINE DeepFM batch sweep 1-32 at the bench's 100k-row vocab per field."""
    from paper_2312_10351_b200 import engine, zoo
    model, (dense, ids) = zoo.build_deepfm(batch)
    sg = engine.compile(model, (dense, ids), device=0, profile_reps=2)
    y = sg.run((dense.cuda(), ids.cuda()))
    y_seq = sg.run((dense.cuda(), ids.cuda()), slot=engine.SLOT_SEQUENTIAL)
    assert torch.equal(y, y_seq)
    with torch.no_grad():
        ref = model.cuda()(dense.cuda(), ids.cuda())
    assert _rel(y, ref) <= 1e-5
    assert sg.plan.num_streams > 20  # the per-field gathers run as parallel branches


@pytest.mark.parametrize("cin,cout,k,s,hw", [(32, 32, 3, 1, 37), (64, 48, 1, 1, 29), (16, 64, 3, 2, 41),
                                           (192, 32, 5, 1, 17)])
def test_pixel_major_tf32x3_tile(cin, cout, k, s, hw):
    """The pixel-major 3xTF32 tile (pixels on UMMA M, <= 64 channels on N,
    variant 4/5 with its own weight packing) against the fp32 reference."""
    import ctypes as C

    import numpy as np

    from paper_2312_10351_b200 import _lib, engine
    torch.manual_seed(2)
    conv = nn.Conv2d(cin, cout, k, s, k // 2, bias=False)
    bn = _bn(cout)
    stem = nn.Conv2d(3, cin, 1, bias=False)
    m = nn.Sequential(stem, nn.ReLU(), conv, bn, nn.ReLU()).eval()
    x = torch.randn(1, 3, hw, hw)
    sg = engine.ScheduledGraph(engine.lower(m, x, "f32"), 0, profile_reps=1, tune=False)
    k_conv = max(i for i, op in enumerate(sg.program.ops) if op.kind == 1)
    op = sg.program.ops[k_conv]
    var, nw = (4, 32) if cout <= 32 else (5, 64)
    wpx = torch.from_numpy(engine.pack_conv_weights_tf32x3(op.weight, rows=nw)).cuda()
    recs = (_lib.OparaOp * len(sg._recs))()
    C.memmove(recs, sg._recs, C.sizeof(sg._recs))
    recs[k_conv].variant, recs[k_conv].p[1], recs[k_conv].i[19], recs[k_conv].i[22] = var, wpx.data_ptr(), 0, 1
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.opara_exec_create(0, C.cast(recs, C.c_void_p), len(recs), C.byref(h)))
    try:
        sg.input_buffer.copy_(x.cuda())
        order = np.asarray(range(len(recs)), dtype=np.int64)
        _lib.check(L.opara_exec_run_eager(h, _lib.ptr(order), len(order),
                                          C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        y = sg.output_buffer.clone()
    finally:
        L.opara_exec_destroy(h)
    with torch.no_grad():   # float64 on the CPU: cuDNN may pick Winograd / FFT for 5x5 (~1e-4 error)
        ref = m.double()(x.double()).permute(0, 2, 3, 1)
    assert _rel(y.cpu().reshape(ref.shape), ref) <= 1e-5
