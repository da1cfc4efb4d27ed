"""CPU-side checks of the model path: fx lowering, concat elimination, the
static DAG, and bit-exact scheduling of the model DAGs against what the
reference computed on the same DAG JSON (tests/golden/model_dags_golden.json)."""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

import paper_2312_10351_b200 as op
from conftest import GOLDEN
from oracle import opsched_oracle as orc
from paper_2312_10351_b200 import engine, frontend, zoo
from paper_2312_10351_b200.dag import graph_from_dict, graph_to_dict

MODELS = json.loads((GOLDEN / "model_dags_golden.json").read_text())
B200 = op.GPU_PRESETS["b200"]


@pytest.mark.parametrize("name", sorted(MODELS))
def test_model_dag_schedule_matches_reference(name):
    gold = MODELS[name]
    g = graph_from_dict(gold["graph"])
    plan = op.allocate_streams(g)
    assert sorted(plan.assignment.items()) == [tuple(x) for x in gold["assignment"]]
    assert plan.num_streams == gold["num_streams"]
    assert [list(e) for e in plan.sync_events] == gold["sync"]
    assert list(op.order_opara(g, B200).order) == gold["opara"]
    assert list(op.make_order(g, "sequential", B200).order) == gold["sequential"]


@pytest.mark.parametrize("name,v,e,streams", [("googlenet", 82, 108, 28), ("inception_v3", 125, 159, 36)])
def test_lowering_matches_fixture_and_paper_anchor(name, v, e, streams):
    """Our frontend reproduces the committed DAG exactly; GoogLeNet's 28
    streams equal the paper's count.  The DAGs carry one node
    more than the torch graph: the PACK_INPUT op in front of the stem conv,
    which chains onto the stem's stream (the stream count is unchanged)."""
    model, x = zoo.build(name)
    prog = frontend.lower(model, x)
    g = engine.static_dag(prog)
    d = graph_to_dict(g)
    gold = MODELS[name]["graph"]
    assert d["edges"] == gold["edges"]
    assert [(n["id"], n["name"], n["class"]) for n in d["nodes"]] == \
           [(n["id"], n["name"], n["class"]) for n in gold["nodes"]]
    assert (len(g), len(g.edges), op.allocate_streams(g).num_streams) == (v, e, streams)


def test_concat_slices_are_disjoint_and_cover():
    model, x = zoo.build("googlenet")
    prog = frontend.lower(model, x)
    for k, o in enumerate(prog.ops):
        if o.kind != frontend.NOP:
            continue
        root, base = o.output.root()
        spans = sorted((t.root()[1], t.root()[1] + t.shape[3]) for t in o.inputs)
        assert spans[0][0] == base and spans[-1][1] == base + o.output.shape[3]
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_bn_folding_is_exact_in_float64():
    torch.manual_seed(0)
    conv = torch.nn.Conv2d(8, 16, 3, padding=1, bias=False)
    bn = torch.nn.BatchNorm2d(16, eps=1e-3)
    with torch.no_grad():
        bn.running_mean.normal_(0, 0.1)
        bn.running_var.uniform_(0.5, 1.5)
        bn.weight.uniform_(0.5, 1.5)
        bn.bias.normal_(0, 0.1)
    bn.eval()
    wk, b = frontend._fold_bn(conv, bn)
    x = torch.randn(1, 8, 5, 5)
    ref = bn(conv(x)).detach()
    w = torch.from_numpy(wk).reshape(3, 3, 8, 16).permute(3, 2, 0, 1)
    y = torch.nn.functional.conv2d(x, w, torch.from_numpy(b), padding=1)
    assert torch.allclose(y, ref, atol=1e-5)


def test_static_dag_schedules_equal_oracle():
    model, x = zoo.build("inception_v3")
    g = engine.static_dag(frontend.lower(model, x))
    d = graph_to_dict(g)
    o = orc.Dag(d["nodes"], d["edges"])
    a, ns, sync = orc.allocate_streams(o)
    plan = op.allocate_streams(g)
    assert dict(plan.assignment) == a and plan.num_streams == ns
    cfg = {"threads_per_sm": B200.threads_per_sm, "shared_mem_per_sm": B200.shared_mem_per_sm,
           "registers_per_sm": B200.registers_per_sm}
    assert list(op.order_opara(g, B200).order) == orc.order_opara(o, cfg)


def test_pack_conv_weights_layout():
    """The tcgen05 W image: 64-byte swizzle, hi + lo == w (tf32 split)."""
    rng = np.random.default_rng(0)
    wk = rng.standard_normal((40, 130)).astype(np.float32)  # K=40, Cout=130
    p = engine.pack_conv_weights_tf32x3(wk)
    mt, kb = 2, 3
    img = p.reshape(mt, kb, 2, 16, 8, 4, 4)
    for co in (0, 7, 77, 129):
        for k in (0, 5, 17, 39):
            m, row = divmod(co, 128)
            atom, r = divmod(row, 8)
            b, kk = divmod(k, 16)
            pos = (kk // 4) ^ ((r >> 1) & 3)
            hi = img[m, b, 0, atom, r, pos, kk % 4]
            lo = img[m, b, 1, atom, r, pos, kk % 4]
            assert hi + lo == pytest.approx(float(wk[k, co]), rel=1e-6)
            assert (np.float32(hi).view(np.uint32) & 0x1FFF) == 0


def test_concurrency_targets_share_levels():
    model, x = zoo.build("googlenet")
    prog = frontend.lower(model, x)
    t = engine.concurrency_targets(prog)
    assert t and all(8 <= v <= 148 for v in t.values())


def test_serial_ops_keep_full_grids():
    """BERT: Q/K/V projections run beside each other and get SM shares; the
    output projection and the FFN are alone in the DAG and keep full grids."""
    m, _, ids = zoo.build_bert()
    prog = frontend.lower(m, ids, "bf16")
    serial, t = engine.serial_ops(prog), engine.concurrency_targets(prog)
    convs = [v for v, o in enumerate(prog.ops) if o.kind == frontend.CONV2D]
    assert len(t) == 36 and all(v not in serial for v in t)
    assert sum(1 for v in convs if v in serial) == 37
    assert all(t[v] == round(148 / 3) for v in t)
    model, x = zoo.build("googlenet")
    g = frontend.lower(model, x)
    assert 0 in engine.serial_ops(g) and 1 in engine.serial_ops(g)   # PACK_INPUT -> stem conv


def _workload(name):
    if name == "bert_base":
        m, _, ids = zoo.build_bert()
        return m, ids, "bf16"
    if name.startswith("deepfm"):
        m, x = zoo.build_deepfm(32 if name.endswith("b32") else 1)
        return m, x, "f32"
    m, x = zoo.build(name)
    return m, x, "f32"


@pytest.mark.parametrize("name,v,e,streams", [("nasnet_large", 697, 912, 159), ("bert_base", 87, 168, 25),
                                              ("deepfm", 36, 36, 29), ("deepfm_b32", 36, 36, 29)])
def test_new_config_dags_match_fixture(name, v, e, streams):
    """NASNet-A Large, BERT-base and DeepFM lower to exactly the DAG the
    reference scheduled for the golden fixture."""
    model, x, dtype = _workload(name)
    g = engine.static_dag(frontend.lower(model, x, dtype))
    d = graph_to_dict(g)
    gold = MODELS[name]["graph"]
    assert d["edges"] == gold["edges"]
    assert [(n["id"], n["name"], n["class"]) for n in d["nodes"]] == \
           [(n["id"], n["name"], n["class"]) for n in gold["nodes"]]
    assert (len(g), len(g.edges), op.allocate_streams(g).num_streams) == (v, e, streams)


def test_nasnet_relus_are_fused():
    """Every NASNet ReLU folds into a producer epilogue or a consumer's input
    (no standalone RELU launches); subsampled factorized-reduction paths fold
    into stride-2 1x1 convs with padding -offset."""
    model, x = zoo.build("nasnet_large")
    prog = frontend.lower(model, x)
    kinds = [o.kind for o in prog.ops]
    assert frontend.RELU not in kinds
    assert sum(1 for o in prog.ops if o.kind == frontend.DWCONV2D and o.ints["relu_in"]) > 50
    fr = [o for o in prog.ops if o.kind == frontend.CONV2D and o.ints["sh"] == 2 and o.ints["R"] == 1]
    assert {o.ints["ph"] for o in fr} == {0, -1} and all(o.ints["relu_in"] for o in fr)


def test_deepfm_lowering_shape():
    """26 parallel field gathers write straight into the MLP-input concat; the
    dense features are copied in; the three heads fold into one sigmoid ADD."""
    model, x = zoo.build_deepfm(8)
    prog = frontend.lower(model, x)
    fields = [o for o in prog.ops if o.kind == frontend.FIELD_EMBEDDING]
    assert len(fields) == 26
    offs = sorted(t.root()[1] for o in fields for t in [o.output])
    assert offs == [13 + 16 * f for f in range(26)]
    last = prog.ops[-1]
    assert last.kind == frontend.ADD and last.ints["n"] == 3 and last.ints["act"] == frontend.ACT_SIGMOID
    assert len(prog.inputs) == 2 and prog.inputs[1].dtype == "i64"


def test_bert_layernorm_folding_lowering():
    """bf16 BERT: 23 of 24 add_layer_norms fold into the GEMMs around them
    (frontend.PendingLN); the output LayerNorm stays a kernel.  Producers get
    the residual as a second input and the stats tensor as an extra output;
    every consumer reads (o, stats, residual); exactly one consumer per folded
    LayerNorm writes the normalised rows, before any GEMM reads them as a
    residual; fold_ln=False keeps every LayerNorm kernel."""
    m, _, ids = zoo.build_bert()
    prog = frontend.lower(m, ids, "bf16")
    ops = prog.ops
    assert sum(1 for o in ops if o.kind == frontend.LAYERNORM) == 1
    prods = [k for k, o in enumerate(ops) if o.ints.get("res_stats")]
    cons = [k for k, o in enumerate(ops) if o.ints.get("ln_in")]
    writers = [k for k in cons if ops[k].ints.get("ln_write")]
    assert (len(prods), len(writers), len(cons)) == (23, 23, 23 + 11 * 2)
    edges = set(prog.edges)
    for k in prods:
        o = ops[k]
        assert len(o.inputs) == 2 and len(o.extra_outputs) == 1 and o.ints.get("act", 0) == 0
        assert o.extra_outputs[0].producers == {k} and o.extra_outputs[0].shape == (128, 12)
    for k in cons:
        o = ops[k]
        assert len(o.inputs) == 3 and o.ints["ln_tiles"] == 6 and o.arrays["gb"].shape == (2, 768)
        producer = min(o.inputs[1].producers)
        assert ops[producer].ints.get("res_stats") and (producer, k) in edges
    for k in writers:   # the normalised rows exist before any GEMM reads them as its residual
        out = ops[k].extra_outputs[0]
        readers = [j for j, o in enumerate(ops) if any(t is out for t in o.inputs)]
        assert readers and all(j > k and (k, j) in edges for j in readers)
    unfolded = frontend.lower(m, ids, "bf16", fold_ln=False)
    assert sum(1 for o in unfolded.ops if o.kind == frontend.LAYERNORM) == 24
    assert not any(o.ints.get("ln_in") or o.ints.get("res_stats") for o in unfolded.ops)
