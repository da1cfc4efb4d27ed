"""Benchmark models of BASELINE.json's configs, random-init and seeded.

Synthetic inputs and random weights only (there is no network for
checkpoints).  BatchNorm running statistics and affine parameters are
randomised (mean ~ N(0, 0.1), var ~ U(0.5, 1.5), gamma ~ U(0.5, 1.5),
beta ~ N(0, 0.1)) so that BN folding is exercised, not trivial
(SURVEY.md §8d).
"""

from __future__ import annotations

import torch
import torch.nn as nn


def _randomise_bn(model: nn.Module, gen: torch.Generator) -> None:
    for m in model.modules():
        if isinstance(m, nn.BatchNorm2d):
            c = m.num_features
            with torch.no_grad():
                m.running_mean.copy_(torch.randn(c, generator=gen) * 0.1)
                m.running_var.copy_(torch.rand(c, generator=gen) + 0.5)
                m.weight.copy_(torch.rand(c, generator=gen) + 0.5)
                m.bias.copy_(torch.randn(c, generator=gen) * 0.1)


def googlenet(seed: int = 0) -> nn.Module:
    import torchvision
    torch.manual_seed(seed)
    m = torchvision.models.googlenet(weights=None, aux_logits=False, init_weights=True)
    _randomise_bn(m, torch.Generator().manual_seed(seed + 1))
    return m.eval()


def inception_v3(seed: int = 0) -> nn.Module:
    import torchvision
    torch.manual_seed(seed)
    m = torchvision.models.inception_v3(weights=None, aux_logits=False, init_weights=True)
    _randomise_bn(m, torch.Generator().manual_seed(seed + 1))
    return m.eval()


MODELS = {
    "googlenet": (googlenet, (1, 3, 224, 224)),
    "inception_v3": (inception_v3, (1, 3, 299, 299)),
}


def _block(make):
    def fn(seed: int = 0) -> nn.Module:
        torch.manual_seed(seed)
        m = make()
        for mod in m.modules():
            if isinstance(mod, nn.Conv2d):
                nn.init.kaiming_normal_(mod.weight, nonlinearity="relu")
        _randomise_bn(m, torch.Generator().manual_seed(seed + 1))
        return m.eval()
    return fn


def _googlenet_3a():
    from torchvision.models.googlenet import Inception
    return Inception(192, 64, 96, 128, 16, 32, 32)


def _inception_a():
    from torchvision.models.inception import InceptionA
    return InceptionA(192, pool_features=32)


def _inception_b():
    from torchvision.models.inception import InceptionB
    return InceptionB(288)


def _inception_e():
    from torchvision.models.inception import InceptionE
    return InceptionE(1280)


# Tiny sub-DAGs (one multi-branch block each) for the exhaustive launch-order
# search measured on the GPU: the block's input is the
# NCHW activation the full network feeds it.
BLOCKS = {
    "googlenet_3a": (_block(_googlenet_3a), (1, 192, 28, 28)),
    "inception_v3_a": (_block(_inception_a), (1, 192, 35, 35)),
    "inception_v3_b": (_block(_inception_b), (1, 288, 35, 35)),
    "inception_v3_e": (_block(_inception_e), (1, 1280, 8, 8)),
}


def build(name: str, batch: int = 1, seed: int = 0):
    """(model, example input) for a named config (or a sub-DAG block of BLOCKS)."""
    fn, shape = MODELS[name] if name in MODELS else BLOCKS[name]
    model = fn(seed)
    g = torch.Generator().manual_seed(seed + 2)
    x = torch.randn((batch,) + tuple(shape[1:]), generator=g)
    return model, x


# ---------------------------------------------------------------- BERT-base
#
# The benchmark model is HF `BertModel(BertConfig())` (random init, seeded).
# torch.fx cannot trace it directly, so `OparaBert` restates its forward over
# the SAME parameter tensors with a few fx-visible primitives (wrapped leaf
# functions the frontend lowers to fused kernels).  Eagerly, each primitive
# runs the exact torch computation, so OparaBert(x) == BertModel(x).


@torch.fx.wrap
def bert_embeddings(ids, word, pos, typ, gamma, beta, eps: float):
    """HF BertEmbeddings: (word[ids] + type[0]) + pos[:T], then LayerNorm."""
    t = ids.shape[-1]
    x = torch.nn.functional.embedding(ids[0], word) + typ[0] + pos[:t]
    return torch.nn.functional.layer_norm(x, (x.shape[-1],), gamma, beta, eps)


@torch.fx.wrap
def self_attention(q, k, v, heads: int):
    """Unmasked multi-head softmax(QK^T / sqrt(d)) V over [T, C] rows."""
    t, c = q.shape
    d = c // heads
    qh = q.view(t, heads, d).transpose(0, 1)
    kh = k.view(t, heads, d).transpose(0, 1)
    vh = v.view(t, heads, d).transpose(0, 1)
    p = torch.softmax(qh @ kh.transpose(1, 2) * (d ** -0.5), dim=-1)
    return (p @ vh).transpose(0, 1).reshape(t, c)


@torch.fx.wrap
def add_layer_norm(x, res, gamma, beta, eps: float):
    return torch.nn.functional.layer_norm(x + res, (x.shape[-1],), gamma, beta, eps)


@torch.fx.wrap
def first_token(x):
    return x[:1]


class OparaBert(nn.Module):
    """BERT encoder + pooler over a BertModel's parameters (batch 1)."""

    def __init__(self, hf):
        super().__init__()
        self.hf = hf
        cfg = hf.config
        self.heads = cfg.num_attention_heads
        self.eps = cfg.layer_norm_eps
        self.nlayers = cfg.num_hidden_layers

    def forward(self, input_ids):
        e = self.hf.embeddings
        x = bert_embeddings(input_ids, e.word_embeddings.weight, e.position_embeddings.weight,
                            e.token_type_embeddings.weight, e.LayerNorm.weight, e.LayerNorm.bias, self.eps)
        F = torch.nn.functional
        for layer in self.hf.encoder.layer:
            at = layer.attention
            q = F.linear(x, at.self.query.weight, at.self.query.bias)
            k = F.linear(x, at.self.key.weight, at.self.key.bias)
            v = F.linear(x, at.self.value.weight, at.self.value.bias)
            ctx = self_attention(q, k, v, self.heads)
            o = F.linear(ctx, at.output.dense.weight, at.output.dense.bias)
            x = add_layer_norm(o, x, at.output.LayerNorm.weight, at.output.LayerNorm.bias, self.eps)
            h = F.gelu(F.linear(x, layer.intermediate.dense.weight, layer.intermediate.dense.bias))
            o2 = F.linear(h, layer.output.dense.weight, layer.output.dense.bias)
            x = add_layer_norm(o2, x, layer.output.LayerNorm.weight, layer.output.LayerNorm.bias, self.eps)
        pooled = torch.tanh(F.linear(first_token(x), self.hf.pooler.dense.weight, self.hf.pooler.dense.bias))
        return x, pooled


class HFBertReference(nn.Module):
    """The reference forward: BertModel(input_ids) -> (last_hidden_state[0], pooler_output)."""

    def __init__(self, hf):
        super().__init__()
        self.hf = hf

    def forward(self, input_ids):
        out = self.hf(input_ids=input_ids)
        return out.last_hidden_state[0], out.pooler_output


def bert_base(seed: int = 0):
    from transformers import BertConfig, BertModel
    torch.manual_seed(seed)
    cfg = BertConfig()
    cfg._attn_implementation = "eager"
    hf = BertModel(cfg).eval()
    g = torch.Generator().manual_seed(seed + 1)
    with torch.no_grad():  # non-trivial LayerNorm affine parameters
        for m in hf.modules():
            if isinstance(m, nn.LayerNorm):
                m.weight.copy_(torch.rand(m.weight.shape, generator=g) + 0.5)
                m.bias.copy_(torch.randn(m.bias.shape, generator=g) * 0.1)
    return OparaBert(hf).eval(), HFBertReference(hf).eval()


def build_bert(seq: int = 128, seed: int = 0):
    """(OparaBert, HF reference, input_ids [1, seq])."""
    model, ref = bert_base(seed)
    g = torch.Generator().manual_seed(seed + 2)
    ids = torch.randint(0, model.hf.config.vocab_size, (1, seq), generator=g)
    return model, ref, ids


# ------------------------------------------------------------------ DeepFM
#
# DeepFM (Guo et al. 2017) in the Criteo layout the SURVEY proposes (§8d):
# 13 dense + 26 sparse fields, 100k ids per field, embedding dim 16, MLP
# 400-400-400.  The per-field lookups are independent branches feeding both
# the FM interaction and the MLP — the wide, shallow DAG Opara exploits.
# Primitives are fx-visible leaf functions the frontend lowers to kernels;
# eagerly they run the plain torch computation.


@torch.fx.wrap
def field_embedding(ids, field: int, table):
    """Rows table[ids[:, field]] -> [B, dim]."""
    return torch.nn.functional.embedding(ids[:, field], table)


@torch.fx.wrap
def first_order(ids, w1, dense, wd, bias):
    """DeepFM linear part: sum_f w1[f, ids[:, f]] + dense . wd + bias -> [B, 1]."""
    f = torch.arange(ids.shape[1], device=ids.device)
    return w1[f, ids].sum(1, keepdim=True) + dense @ wd.reshape(-1, 1) + bias


@torch.fx.wrap
def fm_interaction(v, fields: int):
    """0.5 * sum_d ((sum_f v_fd)^2 - sum_f v_fd^2) over [B, fields * dim] -> [B, 1]."""
    v = v.reshape(v.shape[0], fields, -1)
    s = v.sum(1)
    return 0.5 * (s * s - (v * v).sum(1)).sum(1, keepdim=True)


class DeepFM(nn.Module):
    def __init__(self, n_dense: int = 13, n_sparse: int = 26, vocab: int = 100_000, dim: int = 16,
                 hidden=(400, 400, 400)):
        super().__init__()
        self.n_sparse = n_sparse
        self.tables = nn.ParameterList(nn.Parameter(torch.randn(vocab, dim) * 0.05) for _ in range(n_sparse))
        self.w1 = nn.Parameter(torch.randn(n_sparse, vocab) * 0.05)
        self.wd = nn.Parameter(torch.randn(n_dense) * 0.05)
        self.b = nn.Parameter(torch.zeros(1))
        layers, width = [], n_dense + n_sparse * dim
        for h in hidden:
            layers += [nn.Linear(width, h), nn.ReLU()]
            width = h
        layers.append(nn.Linear(width, 1))
        self.mlp = nn.Sequential(*layers)

    def forward(self, dense, ids):
        embs = [field_embedding(ids, f, self.tables[f]) for f in range(self.n_sparse)]
        emb = torch.cat(embs, 1)
        deep = self.mlp(torch.cat([dense, emb], 1))
        fm = fm_interaction(emb, self.n_sparse)
        lin = first_order(ids, self.w1, dense, self.wd, self.b)
        return torch.sigmoid(lin + fm + deep)


def build_deepfm(batch: int = 1, seed: int = 0, vocab: int = 100_000):
    """(DeepFM, (dense [B, 13], ids [B, 26])) with seeded random weights and inputs."""
    torch.manual_seed(seed)
    model = DeepFM(vocab=vocab).eval()
    g = torch.Generator().manual_seed(seed + 2)
    dense = torch.rand(batch, 13, generator=g)
    ids = torch.randint(0, vocab, (batch, 26), generator=g)
    return model, (dense, ids)


# ----------------------------------------------------------- NASNet-A Large
#
# NASNet-A Large (Zoph et al. 2018; 331x331, penultimate 4032 filters, 18
# normal cells + 2 stem cells + 2 reduction cells), written here from the
# architecture description because the image has no timm.  Padding is
# PyTorch-symmetric (k//2) everywhere, which gives the canonical spatial sizes
# 165 -> 83 -> 42 -> 21 -> 11; the factorized-reduction paths are
# subsample(x, 0) and subsample(x, 1) (= TF's pad-and-shift) each followed by
# its own BatchNorm (identical to one BN over their concatenation).


@torch.fx.wrap
def subsample2d(x, offset: int):
    """x[:, :, off::2, off::2] of x zero-extended by one row/column (offset 0 or 1)."""
    if offset:
        x = torch.nn.functional.pad(x, (0, offset, 0, offset))[:, :, offset:, offset:]
    return x[:, :, ::2, ::2]


def _bn(c):
    return nn.BatchNorm2d(c, eps=1e-3)


class _SepConv(nn.Module):
    """ReLU -> depthwise k x k (stride s) -> 1x1 -> BN -> ReLU -> depthwise k x k -> 1x1 -> BN."""

    def __init__(self, cin, cout, k, stride, mid=None):
        super().__init__()
        mid = cin if mid is None else mid
        self.relu = nn.ReLU()
        self.dw1 = nn.Conv2d(cin, cin, k, stride, k // 2, groups=cin, bias=False)
        self.pw1 = nn.Conv2d(cin, mid, 1, bias=False)
        self.bn1 = _bn(mid)
        self.relu1 = nn.ReLU()
        self.dw2 = nn.Conv2d(mid, mid, k, 1, k // 2, groups=mid, bias=False)
        self.pw2 = nn.Conv2d(mid, cout, 1, bias=False)
        self.bn2 = _bn(cout)

    def forward(self, x):
        x = self.bn1(self.pw1(self.dw1(self.relu(x))))
        return self.bn2(self.pw2(self.dw2(self.relu1(x))))


class _ReluConvBn(nn.Module):
    def __init__(self, cin, cout):
        super().__init__()
        self.relu = nn.ReLU()
        self.conv = nn.Conv2d(cin, cout, 1, bias=False)
        self.bn = _bn(cout)

    def forward(self, x):
        return self.bn(self.conv(self.relu(x)))


class _FactorizedReduction(nn.Module):
    """ReLU, then two stride-2 1x1 paths offset by one pixel, concatenated."""

    def __init__(self, cin, cout):
        super().__init__()
        self.relu = nn.ReLU()
        self.conv1 = nn.Conv2d(cin, cout // 2, 1, bias=False)
        self.bn1 = _bn(cout // 2)
        self.conv2 = nn.Conv2d(cin, cout - cout // 2, 1, bias=False)
        self.bn2 = _bn(cout - cout // 2)

    def forward(self, x):
        x = self.relu(x)
        return torch.cat([self.bn1(self.conv1(subsample2d(x, 0))), self.bn2(self.conv2(subsample2d(x, 1)))], 1)


def _avg3(stride=1):
    return nn.AvgPool2d(3, stride, 1, count_include_pad=False)


class _StemCell0(nn.Module):
    def __init__(self, cin, c):
        super().__init__()
        self.conv_1x1 = _ReluConvBn(cin, c)
        self.b0l = _SepConv(c, c, 5, 2)
        self.b0r = _SepConv(cin, c, 7, 2, mid=c)
        self.b1l = nn.MaxPool2d(3, 2, 1)
        self.b1r = _SepConv(cin, c, 7, 2, mid=c)
        self.b2l = _avg3(2)
        self.b2r = _SepConv(cin, c, 5, 2, mid=c)
        self.b3r = _avg3()
        self.b4l = _SepConv(c, c, 3, 1)
        self.b4r = nn.MaxPool2d(3, 2, 1)

    def forward(self, x):
        x1 = self.conv_1x1(x)
        c0 = self.b0l(x1) + self.b0r(x)
        c1 = self.b1l(x1) + self.b1r(x)
        c2 = self.b2l(x1) + self.b2r(x)
        c3 = self.b3r(c0) + c1
        c4 = self.b4l(c0) + self.b4r(x1)
        return torch.cat([c1, c2, c3, c4], 1)


class _ReductionCell(nn.Module):
    """Stem cell 1 and the two reduction cells: left = 1x1(prev) or factorized
    reduction, right = 1x1(x); five stride-2 combinations."""

    def __init__(self, c_left_in, c_right_in, c, left_factorized=False):
        super().__init__()
        self.left = _FactorizedReduction(c_left_in, c) if left_factorized else _ReluConvBn(c_left_in, c)
        self.right = _ReluConvBn(c_right_in, c)
        self.b0l = _SepConv(c, c, 5, 2)
        self.b0r = _SepConv(c, c, 7, 2)
        self.b1l = nn.MaxPool2d(3, 2, 1)
        self.b1r = _SepConv(c, c, 7, 2)
        self.b2l = _avg3(2)
        self.b2r = _SepConv(c, c, 5, 2)
        self.b3r = _avg3()
        self.b4l = _SepConv(c, c, 3, 1)
        self.b4r = nn.MaxPool2d(3, 2, 1)

    def forward(self, x, x_prev):
        xl = self.left(x_prev)
        xr = self.right(x)
        c0 = self.b0l(xr) + self.b0r(xl)
        c1 = self.b1l(xr) + self.b1r(xl)
        c2 = self.b2l(xr) + self.b2r(xl)
        c3 = self.b3r(c0) + c1
        c4 = self.b4l(c0) + self.b4r(xr)
        return torch.cat([c1, c2, c3, c4], 1)


class _NormalCell(nn.Module):
    """NASNet-A normal cell (the first cell after a reduction takes its left
    input through a factorized reduction)."""

    def __init__(self, c_left_in, c_right_in, c, left_factorized=False):
        super().__init__()
        self.left = _FactorizedReduction(c_left_in, c) if left_factorized else _ReluConvBn(c_left_in, c)
        self.right = _ReluConvBn(c_right_in, c)
        self.b0l = _SepConv(c, c, 5, 1)
        self.b0r = _SepConv(c, c, 3, 1)
        self.b1l = _SepConv(c, c, 5, 1)
        self.b1r = _SepConv(c, c, 3, 1)
        self.b2l = _avg3()
        self.b3l = _avg3()
        self.b3r = _avg3()
        self.b4l = _SepConv(c, c, 3, 1)

    def forward(self, x, x_prev):
        xl = self.left(x_prev)
        xr = self.right(x)
        c0 = self.b0l(xr) + self.b0r(xl)
        c1 = self.b1l(xl) + self.b1r(xl)
        c2 = self.b2l(xr) + xl
        c3 = self.b3l(xl) + self.b3r(xl)
        c4 = self.b4l(xr) + xr
        return torch.cat([xl, c0, c1, c2, c3, c4], 1)


class NASNetALarge(nn.Module):
    def __init__(self, num_classes: int = 1001, stem: int = 96, penultimate: int = 4032, cells_per_stage: int = 6):
        super().__init__()
        f = penultimate // 24                     # 168
        self.conv0 = nn.Conv2d(3, stem, 3, 2, 0, bias=False)
        self.bn0 = _bn(stem)
        self.stem0 = _StemCell0(stem, f // 4)                                  # 4 * 42 = 168 ch @ 83
        self.stem1 = _ReductionCell(stem, 4 * (f // 4), f // 2, left_factorized=True)  # 4 * 84 = 336 @ 42
        cells = []
        prev, cur = 4 * (f // 4), 4 * (f // 2)   # channels of (x_prev, x) entering the next cell
        for stage, width in enumerate((f, 2 * f, 4 * f)):
            if stage > 0:   # reduction cell: 4 * width channels at half resolution
                cells.append(_ReductionCell(prev, cur, width))
                prev, cur = cur, 4 * width
            for k in range(cells_per_stage):
                cells.append(_NormalCell(prev, cur, width, left_factorized=k == 0))
                prev, cur = cur, 6 * width
        self.cells = nn.ModuleList(cells)
        self.relu = nn.ReLU()
        self.avg_pool = nn.AvgPool2d(11, 1, 0)
        self.dropout = nn.Dropout(0.5)
        self.last_linear = nn.Linear(cur, num_classes)

    def forward(self, x):
        x0 = self.bn0(self.conv0(x))
        s0 = self.stem0(x0)
        x_prev, x = s0, self.stem1(s0, x0)
        for cell in self.cells:
            x_prev, x = x, cell(x, x_prev)
        x = self.avg_pool(self.relu(x))
        return self.last_linear(self.dropout(torch.flatten(x, 1)))


def nasnet_large(seed: int = 0) -> nn.Module:
    """Random-init NASNet-A Large whose BatchNorm running statistics are
    calibrated on one seeded random image (a train-mode pass with cumulative
    averaging), so activations keep a trained network's scale through the 22
    cells instead of compounding; BN affine parameters are then randomised."""
    torch.manual_seed(seed)
    m = NASNetALarge()
    for mod in m.modules():
        if isinstance(mod, nn.BatchNorm2d):
            mod.momentum = None
    g = torch.Generator().manual_seed(seed + 3)
    m.train()
    with torch.no_grad():
        m(torch.randn(1, 3, 331, 331, generator=g))
    gen = torch.Generator().manual_seed(seed + 1)
    for mod in m.modules():
        if isinstance(mod, nn.BatchNorm2d):
            c = mod.num_features
            with torch.no_grad():
                mod.weight.copy_(torch.rand(c, generator=gen) + 0.5)
                mod.bias.copy_(torch.randn(c, generator=gen) * 0.1)
    return m.eval()


MODELS["nasnet_large"] = (nasnet_large, (1, 3, 331, 331))
