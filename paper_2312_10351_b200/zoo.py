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
