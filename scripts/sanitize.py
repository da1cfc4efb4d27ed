"""One small scheduled graph per kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck) on the B200:

    compute-sanitizer --tool racecheck python scripts/sanitize.py conv_f32_pull

Cases: conv_f32_{push,pull,l2} (3xTF32 tcgen05 conv with TMA im2col loads,
cluster split-K with bulk-copy push / DSMEM pull / L2 partials),
conv_bf16_{push,pull,l2} (kind::f16 conv), bert_layer (embedding + LN, Q/K/V
GEMMs, tcgen05 attention, residual LayerNorm), bert_fold (a full encoder layer
with its first LayerNorm folded into the GEMMs).  Tuning
is off (no candidate sweep) so the sanitized launches are the graph's own:
the profiling launches, one eager pass and two graph replays (Opara and
sequential), each output checked against PyTorch."""
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2312_10351_b200 import engine, zoo  # noqa: E402


def conv_case(dtype, splitk):
    from test_gpu_kernels import Wrap
    torch.manual_seed(0)
    cin, cout, k, s, p, hw = (480, 192, 1, 1, 0, 14) if dtype == "f32" else (288, 384, 3, 2, 0, 35)
    m = Wrap(cin, cout, k, s, p, hw).eval()
    return m, torch.randn(1, 3, hw, hw), dtype, splitk


def bert_case():
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
    m = OneLayer(BertModel(cfg).eval()).eval()
    return m, torch.randint(0, cfg.vocab_size, (1, 128)), "bf16", "push"


def bert_fold_case():
    """One full encoder layer: its first add_layer_norm folds into the O-projection
    (residual + stats epilogue) and FFN1 (LayerNorm on load, writes the rows FFN2
    adds back); the output LayerNorm stays a kernel."""
    from transformers import BertConfig, BertModel

    class Layer(torch.nn.Module):
        def __init__(self, hf):
            super().__init__()
            self.hf = hf

        def forward(self, ids):
            e = self.hf.embeddings
            x = zoo.bert_embeddings(ids, e.word_embeddings.weight, e.position_embeddings.weight,
                                    e.token_type_embeddings.weight, e.LayerNorm.weight, e.LayerNorm.bias, 1e-12)
            layer = self.hf.encoder.layer[0]
            at = layer.attention
            q = F.linear(x, at.self.query.weight, at.self.query.bias)
            k = F.linear(x, at.self.key.weight, at.self.key.bias)
            v = F.linear(x, at.self.value.weight, at.self.value.bias)
            o = F.linear(zoo.self_attention(q, k, v, 12), at.output.dense.weight, at.output.dense.bias)
            x = zoo.add_layer_norm(o, x, at.output.LayerNorm.weight, at.output.LayerNorm.bias, 1e-12)
            h = F.gelu(F.linear(x, layer.intermediate.dense.weight, layer.intermediate.dense.bias))
            o2 = F.linear(h, layer.output.dense.weight, layer.output.dense.bias)
            return zoo.add_layer_norm(o2, x, layer.output.LayerNorm.weight, layer.output.LayerNorm.bias, 1e-12)

    torch.manual_seed(0)
    cfg = BertConfig(num_hidden_layers=1)
    m = Layer(BertModel(cfg).eval()).eval()
    return m, torch.randint(0, cfg.vocab_size, (1, 128)), "bf16", "auto"


CASES = {"conv_f32_push": lambda: conv_case("f32", "push"), "conv_f32_pull": lambda: conv_case("f32", "pull"),
         "conv_f32_l2": lambda: conv_case("f32", "l2"),
         "conv_bf16_push": lambda: conv_case("bf16", "push"), "conv_bf16_pull": lambda: conv_case("bf16", "pull"),
         "conv_bf16_l2": lambda: conv_case("bf16", "l2"),
         "bert_layer": bert_case, "bert_fold": bert_fold_case}

if __name__ == "__main__":
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    name = sys.argv[1]
    m, x, dtype, splitk = CASES[name]()
    fold = not (len(sys.argv) > 2 and sys.argv[2] == "nofold")
    sg = engine.ScheduledGraph(engine.lower(m, x, dtype, fold_ln=fold), 0, profile_reps=1, tune=False, splitk=splitk)
    y_eager = sg.run_eager(x.cuda()).clone()
    y = sg.run(x.cuda())
    y_seq = sg.run(x.cuda(), slot=engine.SLOT_SEQUENTIAL)
    torch.cuda.synchronize()
    with torch.no_grad():
        ref = m.double()(x.double() if x.is_floating_point() else x)
    ref = ref.permute(0, 2, 3, 1) if ref.dim() == 4 else ref
    rel = (torch.linalg.vector_norm(y.double().cpu().reshape(ref.shape) - ref)
           / torch.linalg.vector_norm(ref)).item()
    tol = 1e-5 if dtype == "f32" else 1.5e-2
    ok = torch.equal(y, y_seq) and torch.equal(y, y_eager) and rel < tol
    print(f"{name}: launches={sg.num_launches()} rel={rel:.2e} ok={ok}")
    sys.exit(0 if ok else 1)
