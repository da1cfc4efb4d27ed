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


def build(name: str, batch: int = 1, seed: int = 0):
    """(model, example input) for a named config."""
    fn, shape = MODELS[name]
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
