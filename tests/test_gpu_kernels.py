"""Kernel-level numerics on the B200: each op family through the executor
(C ABI) against a plain PyTorch fp32 reference of the same op (TF32 off)."""

from __future__ import annotations

import pytest
import torch
import torch.nn as nn
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return (torch.linalg.vector_norm(a.double() - b.double()) / torch.linalg.vector_norm(b.double())).item()


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False


class ConvBnRelu(nn.Module):
    def __init__(self, cin, cout, k, s, p, relu=True):
        super().__init__()
        self.conv = nn.Conv2d(cin, cout, k, s, p, bias=False)
        self.bn = nn.BatchNorm2d(cout, eps=1e-3)
        self.relu = relu
        with torch.no_grad():
            self.bn.running_mean.normal_(0, 0.1)
            self.bn.running_var.uniform_(0.5, 1.5)
            self.bn.weight.uniform_(0.5, 1.5)
            self.bn.bias.normal_(0, 0.1)

    def forward(self, x):
        y = self.bn(self.conv(x))
        return F.relu(y) if self.relu else y


class Wrap(nn.Module):
    """Stem conv (NCHW input) -> the conv under test (NHWC view) -> maxpool."""

    def __init__(self, cin, cout, k, s, p, hw_in):
        super().__init__()
        self.stem = ConvBnRelu(3, cin, 1, 1, 0)
        self.body = ConvBnRelu(cin, cout, k, s, p)
        self.pool = nn.MaxPool2d(3, 2, ceil_mode=True)

    def forward(self, x):
        return self.pool(self.body(self.stem(x)))


CONV_CASES = [
    # cin, cout, kernel, stride, pad, hw
    (64, 64, 1, 1, 0, 56),
    (192, 96, 3, 1, 1, 28),
    (480, 192, 1, 1, 0, 14),
    (832, 384, 1, 1, 0, 7),
    (160, 192, (1, 7), 1, (0, 3), 17),
    (160, 192, (7, 1), 1, (3, 0), 17),
    (288, 384, 3, 2, 0, 35),
    (2048, 320, 1, 1, 0, 8),
    (48, 64, 5, 1, 2, 35),
    (7, 13, 3, 1, 1, 9),      # odd channels -> scalar gather
]


@pytest.mark.parametrize("engine_name", ["tc", "tc-pull", "tc-l2", "simt"])
@pytest.mark.parametrize("case", CONV_CASES, ids=[str(c) for c in CONV_CASES])
def test_conv_matches_torch(case, engine_name):
    """Oracle: the same module in float64 on the CPU (cuDNN fp32 may pick
    Winograd/FFT algorithms whose own error is ~1e-4 on 5x5 kernels)."""
    from paper_2312_10351_b200 import engine
    cin, cout, k, s, p, hw = case
    torch.manual_seed(0)
    m = Wrap(cin, cout, k, s, p, hw).eval()
    x = torch.randn(1, 3, hw, hw)
    sg = engine.compile(m, x, device=0, profile_reps=2, conv_engine=engine_name.split("-")[0],
                        splitk=engine_name.split("-")[1] if "-" in engine_name else None)
    y = sg.run(x.cuda())
    with torch.no_grad():
        ref = m.double()(x.double())
    y_nchw = y.permute(0, 3, 1, 2).cpu()
    assert y_nchw.shape == ref.shape
    # 3xTF32 drops the lo*lo term: ~1e-6 over K ~ 2.6k; exact-fp32 SIMT ~3e-7
    assert _rel(y_nchw, ref) < (1e-5 if engine_name.startswith("tc") else 2e-6)
    # replaying twice is idempotent (split-K counters reset themselves)
    y2 = sg.run(x.cuda())
    assert torch.equal(y, y2)


BF16_CASES = [
    (64, 64, 1, 1, 0, 56),
    (192, 96, 3, 1, 1, 28),
    (160, 192, (1, 7), 1, (0, 3), 17),
    (288, 384, 3, 2, 0, 35),
    (2048, 320, 1, 1, 0, 8),
    (12, 20, 3, 1, 1, 9),     # Cin % 8 != 0 -> register gather path
]


@pytest.mark.parametrize("splitk", ["push", "pull", "l2"])
@pytest.mark.parametrize("case", BF16_CASES, ids=[str(c) for c in BF16_CASES])
def test_conv_bf16_matches_torch(case, splitk):
    """bf16 tcgen05 engine (kind::f16, fp32 accumulation) vs the fp64 module;
    bf16 storage of inputs/weights/outputs bounds the error near 1e-2.  Both
    split-K reductions: push (receive buffers behind the ring) and pull (one
    cluster barrier, blocks bulk-copied into the owners' rings)."""
    from paper_2312_10351_b200 import engine
    cin, cout, k, s, p, hw = case
    torch.manual_seed(0)
    m = Wrap(cin, cout, k, s, p, hw).eval()
    x = torch.randn(1, 3, hw, hw)
    sg = engine.compile(m, x, device=0, profile_reps=2, dtype="bf16", splitk=splitk)
    assert all(engine.conv_engine_for(o, 1) == 2 for o in sg.program.ops if o.kind == 1)
    y = sg.run(x.cuda())
    with torch.no_grad():
        ref = m.double()(x.double())
    y_nchw = y.permute(0, 3, 1, 2).float().cpu()
    assert _rel(y_nchw, ref) < 1.5e-2
    assert torch.equal(sg.run(x.cuda()), y)


def test_attention_and_layernorm_rows():
    """One BERT layer in isolation (embedding, Q/K/V GEMMs, tcgen05 attention,
    residual LayerNorm) vs the torch restatement in fp64."""
    import torch.nn.functional as F
    from paper_2312_10351_b200 import engine, zoo
    from transformers import BertConfig, BertModel

    class OneLayer(torch.nn.Module):
        def __init__(self, hf):
            super().__init__()
            self.hf = hf

        def forward(self, ids):
            e = self.hf.embeddings
            x = zoo.bert_embeddings(ids, e.word_embeddings.weight, e.position_embeddings.weight,
                                    e.token_type_embeddings.weight, e.LayerNorm.weight, e.LayerNorm.bias, 1e-12)
            at = self.hf.encoder.layer[0].attention
            q = F.linear(x, at.self.query.weight, at.self.query.bias)
            k = F.linear(x, at.self.key.weight, at.self.key.bias)
            v = F.linear(x, at.self.value.weight, at.self.value.bias)
            ctx = zoo.self_attention(q, k, v, 12)
            return zoo.add_layer_norm(ctx, x, at.output.LayerNorm.weight, at.output.LayerNorm.bias, 1e-12)

    torch.manual_seed(0)
    cfg = BertConfig(num_hidden_layers=1)
    hf = BertModel(cfg).eval()
    m = OneLayer(hf).eval()
    ids = torch.randint(0, cfg.vocab_size, (1, 128))
    sg = engine.compile(m, ids, device=0, profile_reps=2, dtype="bf16")
    y = sg.run(ids.cuda())
    with torch.no_grad():
        ref = m.double()(ids)
    assert _rel(y.float().reshape(ref.shape).cpu(), ref) < 1e-2


class PoolNet(nn.Module):
    """Stem conv -> the pool under test, with a second conv on a channel
    view so the pool also reads at a channel offset."""

    def __init__(self, c, pool):
        super().__init__()
        self.stem = ConvBnRelu(3, c, 3, 1, 1)
        self.pool = pool

    def forward(self, x):
        return self.pool(self.stem(x))


POOL_CASES = [
    ("max3s2ceil", lambda: nn.MaxPool2d(3, 2, ceil_mode=True)),
    ("max3s2", lambda: nn.MaxPool2d(3, 2)),
    ("max3s1p1", lambda: nn.MaxPool2d(3, 1, padding=1)),
    ("max2s2", lambda: nn.MaxPool2d(2, 2)),
    ("avg3s1p1", lambda: nn.AvgPool2d(3, 1, padding=1)),
    ("avg3s1p1_nopad", lambda: nn.AvgPool2d(3, 1, padding=1, count_include_pad=False)),
    ("avg3s2ceil", lambda: nn.AvgPool2d(3, 2, padding=1, ceil_mode=True, count_include_pad=False)),
    ("avg5s3", lambda: nn.AvgPool2d(5, 3)),
]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("c", [64, 36, 30])
@pytest.mark.parametrize("name,make", POOL_CASES, ids=[c[0] for c in POOL_CASES])
def test_pool_matches_torch(name, make, c, dtype):
    """Every pooling path (3x3 all-taps-in-flight and generic windows; 16-,
    8-byte and scalar channel vectors) against torch on the same stem output."""
    from paper_2312_10351_b200 import engine
    torch.manual_seed(1)
    m = PoolNet(c, make()).eval()
    x = torch.randn(1, 3, 23, 23)
    sg = engine.compile(m, x, device=0, profile_reps=2, dtype=dtype)
    y = sg.run(x.cuda()).float().permute(0, 3, 1, 2).cpu()   # executor activations are NHWC
    with torch.no_grad():
        ref = m.double()(x.double()).float()
    assert y.shape == ref.shape
    assert _rel(y, ref) < (1e-2 if dtype == "bf16" else 1e-5), name


TMA_CASES = [
    # cin, cout, kernel, stride, pad, hw, batch
    (64, 64, 1, 1, 0, 56, 1),
    (192, 96, 3, 1, 1, 28, 2),          # image wrap inside a pixel tile
    (160, 192, (1, 7), 1, (0, 3), 17, 1),
    (160, 192, (7, 1), 1, (3, 0), 17, 3),
    (288, 384, 3, 2, 0, 35, 1),
    (48, 64, 5, 1, 2, 35, 2),
    (2048, 320, 1, 1, 0, 8, 1),
]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("case", TMA_CASES, ids=[str(c) for c in TMA_CASES])
def test_tma_im2col_equals_gather(case, dtype, monkeypatch, tmp_path):
    """The TMA im2col activation loads deliver exactly the bytes the cp.async
    gathers do (same smem tiles, same MMA order), so the two builds of the same
    graph agree bit for bit, on every autotuned tile; batch > 1 covers the
    image wrap inside a pixel tile."""
    from paper_2312_10351_b200 import engine
    cin, cout, k, s, p, hw, n = case
    torch.manual_seed(0)
    m = Wrap(cin, cout, k, s, p, hw).eval()
    x = torch.randn(n, 3, hw, hw)
    outs = []
    monkeypatch.setenv("OPARA_TUNE_CACHE", str(tmp_path / "tune.json"))   # same tiles in both builds
    for flag in ("1", "0"):
        monkeypatch.setenv("OPARA_TMA", flag)
        sg = engine.compile(m, x, device=0, profile_reps=2, dtype=dtype)
        outs.append(sg.run(x.cuda()).clone())
    assert torch.equal(outs[0], outs[1])
    with torch.no_grad():
        ref = m.double()(x.double())
    rel = _rel(outs[0].permute(0, 3, 1, 2).float().cpu(), ref)
    assert rel < (1e-5 if dtype == "f32" else 1.5e-2)


class _StemReduce(nn.Module):
    """Stem conv -> NASNet's factorized reduction (ReLU, stride-2 1x1 paths at
    pixel offsets 0 and 1 of the zero-extended map, concatenated)."""

    def __init__(self, cin, cout):
        super().__init__()
        from paper_2312_10351_b200 import zoo
        self.stem = ConvBnRelu(3, cin, 1, 1, 0)
        self.red = zoo._FactorizedReduction(cin, cout)

    def forward(self, x):
        return self.red(self.stem(x))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("hw", [21, 22, 83])
def test_tma_im2col_subsample_paths(hw, dtype, monkeypatch, tmp_path):
    """Offset-1 subsample convs have padding -1: their TMA box runs one pixel
    past the edge (zeros, like the zero-extended map); odd and even sizes."""
    from paper_2312_10351_b200 import engine
    torch.manual_seed(0)
    m = _StemReduce(64, 128).eval()
    x = torch.randn(1, 3, hw, hw)
    outs = []
    monkeypatch.setenv("OPARA_TUNE_CACHE", str(tmp_path / "tune.json"))
    for flag in ("1", "0"):
        monkeypatch.setenv("OPARA_TMA", flag)
        sg = engine.compile(m, x, device=0, profile_reps=2, dtype=dtype)
        outs.append(sg.run(x.cuda()).clone())
    assert torch.equal(outs[0], outs[1])
    with torch.no_grad():
        ref = m.double()(x.double())
    rel = _rel(outs[0].permute(0, 3, 1, 2).float().cpu(), ref)
    assert rel < (1e-5 if dtype == "f32" else 1.5e-2)
