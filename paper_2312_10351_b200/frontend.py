"""Model -> operator DAG lowering (torch.fx).

PyTorch is used here only to define the model and to trace it.  The traced
graph is lowered to the executor's operator records:

* Conv2d -> BatchNorm2d -> ReLU chains fold into one CONV2D op (BN folded in
  float64 on the host; the kernel applies bias + ReLU in its epilogue).
* ``torch.cat`` disappears: every concat input is produced straight into its
  channel slice of the concatenated buffer (nested concats flatten).
* Views (flatten, eval-mode dropout) alias their producer.

The resulting DAG has one node per kernel launch, ids 1..V in trace order,
edges from every producer of an op's input buffer region.  This is the DAG
the scheduler (Alg. 1 / Alg. 2) sees, and the JSON the reference consumes.
"""

from __future__ import annotations

import operator
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.fx as fx
import torch.nn as nn
import torch.nn.functional as F

from .dag import OpClass

# opara_op_kind values (include/opara.h)
NOP, CONV2D, MAXPOOL2D, AVGPOOL2D, GLOBAL_AVGPOOL, LINEAR, ADD = 0, 1, 2, 3, 4, 5, 6
LAYERNORM, EMBEDDING, ATTENTION, COPY, FM, DWCONV2D, RELU = 7, 9, 10, 11, 12, 13, 14
FIELD_EMBEDDING, FIRST_ORDER, PACK_INPUT = 16, 17, 18

# linear + residual + LayerNorm fusion (opt-in): deepest reduction (K) one CTA streams whole.
# Measured on BERT-base: the fused O-proj + LN (48 unsplit CTAs streaming 196 KB of weights
# each) takes 10.7 us against 5.3 + 1.7 us unfused, so compile() leaves it off by default.

# fused activations (csrc kernels): 0 none, 1 ReLU, 2 GELU (erf), 3 tanh, 4 sigmoid
ACT_NONE, ACT_RELU, ACT_GELU, ACT_TANH, ACT_SIGMOID = 0, 1, 2, 3, 4


@dataclass
class Tensor:
    """A value of the lowered program.  4-D values are NHWC channel views of a
    root buffer; 2-D values are dense row-major [rows, features]."""

    tid: int
    shape: tuple            # (N, H, W, C) or (M, K)
    producers: set = field(default_factory=set)   # op indices writing this region
    alias: "Tensor | None" = None                  # concat parent
    coff_in_alias: int = 0
    nchw_input: bool = False                       # the graph input (dense NCHW)
    is_graph_input: bool = False
    dtype: str = "f32"                             # "f32" | "bf16" element type of the buffer

    def root(self) -> tuple["Tensor", int]:
        t, off = self, 0
        while t.alias is not None:
            off += t.coff_in_alias
            t = t.alias
        return t, off


@dataclass
class LoweredOp:
    kind: int
    name: str                 # label used in the DAG (classify-table names)
    op_class: OpClass
    ints: dict                # named integer parameters
    inputs: list              # [Tensor]
    output: Tensor
    weight: np.ndarray | None = None    # host float32, executor layout
    bias: np.ndarray | None = None
    flops: int = 0            # algorithmic FLOPs (2*MAC for conv/linear)
    bytes_min: int = 0        # algorithmic bytes: inputs read once + weights + output written
    label: str = ""           # fx node name, for reports
    arrays: dict = field(default_factory=dict)  # extra host arrays (tables, LN affine)
    floats: tuple = ()        # float parameters (eps, scale)
    extra_outputs: list = field(default_factory=list)   # further tensors this op writes


@dataclass
class PendingLN:
    """add_layer_norm(o, res) folded into the GEMMs around it (bf16 rows path):
    the GEMM producing `o` also stores, per (token, 128-channel tile), the sum
    and sum of squares of o + res into `stats`; every consuming GEMM loads the
    o and res tiles and normalises o + res on load from those sums and gamma /
    beta (the unfolded kernel's roundings), and the first one also stores the
    normalised rows into `out`, which later add_layer_norms read as their
    residual.  No LayerNorm kernel is launched."""

    o: Tensor
    res: Tensor
    stats: Tensor
    gb: np.ndarray            # [2][C] fp32: gamma, beta
    eps: float
    out: Tensor
    writer: int | None = None


class LoweringError(RuntimeError):
    pass


_PENDING_ADD = object()   # an add folded into the n-ary ADD of its single add consumer


@dataclass
class Lazy:
    """A value whose producing transform is folded into its consumers instead
    of being launched: ReLU (consumers with a fused input ReLU: convs,
    depthwise convs, global pooling) and/or a stride-2 subsample at offset
    `sub` (folded into a consuming 1x1 conv as stride 2 and padding -sub)."""

    tensor: Tensor
    relu: bool = False
    sub: int | None = None


@dataclass
class Program:
    ops: list
    tensors: list
    input: Tensor             # first graph input
    output: Tensor            # first graph output
    edges: list               # (u, v) op indices
    outputs: list = field(default_factory=list)
    inputs: list = field(default_factory=list)


def _pool_out(size, k, s, p, ceil_mode):
    """torch's pooling output size (pooling_output_shape)."""
    num = size + 2 * p - (k - 1) - 1 + ((s - 1) if ceil_mode else 0)
    out = num // s + 1
    if ceil_mode and (out - 1) * s >= size + p:
        out -= 1
    return out


def _pair(v):
    return tuple(v) if isinstance(v, (tuple, list)) else (v, v)


def _fold_bn(conv: nn.Conv2d, bn: nn.BatchNorm2d | None):
    w = conv.weight.detach().double().cpu()
    b = conv.bias.detach().double().cpu() if conv.bias is not None else torch.zeros(w.shape[0], dtype=torch.float64)
    if bn is not None:
        scale = bn.weight.detach().double().cpu() / torch.sqrt(bn.running_var.detach().double().cpu() + bn.eps)
        w = w * scale[:, None, None, None]
        b = (b - bn.running_mean.detach().double().cpu()) * scale + bn.bias.detach().double().cpu()
    # [Cout, Cin, R, S] -> [R, S, Cin, Cout] -> [K, Cout]
    cout, cin, r, s = w.shape
    wk = w.permute(2, 3, 1, 0).reshape(r * s * cin, cout).contiguous()
    return wk.float().numpy(), b.float().numpy()


class _Lowerer:
    def __init__(self, gm: fx.GraphModule, dtype: str = "f32", fold_ln: bool = True):
        self.gm = gm
        self.act_dtype = dtype          # element type of conv / pool activations
        self.fold_ln = fold_ln          # fold add_layer_norm into the GEMMs around it (bf16)
        self.esize = 2 if dtype == "bf16" else 4
        self.ops: list[LoweredOp] = []
        self.tensors: list[Tensor] = []
        self.env: dict = {}
        self.consumed: set[fx.Node] = set()
        self._materialized: dict[int, Tensor] = {}
        self._packed = None

    def new_tensor(self, shape, producers=(), dtype=None):
        t = Tensor(len(self.tensors), tuple(int(x) for x in shape), set(producers),
                   dtype=dtype or self.act_dtype)
        self.tensors.append(t)
        return t

    def emit(self, op: LoweredOp) -> None:
        idx = len(self.ops)
        self.ops.append(op)
        op.output.producers = {idx}
        for t in op.extra_outputs:
            t.producers = {idx}

    @staticmethod
    def _esz(t: Tensor) -> int:
        return {"bf16": 2, "f32": 4, "i64": 8}[t.dtype]

    # ------------------------------------------------ lazy values (fusion)

    def value(self, arg) -> Tensor:
        """The materialised tensor of an fx argument: a pending ReLU is
        launched once as a RELU op (the unfused fallback) and cached; a folded
        LayerNorm is its normalised rows (written by its first consuming GEMM)."""
        v = self.env[arg]
        if isinstance(v, PendingLN):
            if v.writer is None:
                raise LoweringError(f"{arg}: folded LayerNorm read before a consuming GEMM wrote it")
            return v.out
        if not isinstance(v, Lazy):
            return v
        if v.sub is not None:
            raise LoweringError(f"{arg}: a subsample must feed a 1x1 convolution")
        key = id(v)
        if key not in self._materialized:
            t = v.tensor
            out = self.new_tensor(t.shape, dtype=t.dtype)
            p, c = self._pixels(t)
            self.emit(LoweredOp(RELU, "relu", OpClass.MEMORY, dict(P=p, C=c, n=1, act=ACT_RELU), [t], out,
                                flops=p * c, bytes_min=2 * self._esz(t) * p * c, label=str(arg)))
            self._materialized[key] = out
        return self._materialized[key]

    def lazy(self, arg) -> Lazy:
        v = self.env[arg]
        return v if isinstance(v, Lazy) else Lazy(v)

    @staticmethod
    def _pixels(t: Tensor):
        if len(t.shape) == 4:
            n, h, w, c = t.shape
            return n * h * w, c
        return int(np.prod(t.shape[:-1])), t.shape[-1]

    # ----------------------------------------------------------- patterns

    def _single_user(self, node, pred):
        users = list(node.users)
        if len(users) == 1 and pred(users[0]):
            return users[0]
        return None

    def _is_bn(self, n):
        return n.op == "call_module" and isinstance(self.gm.get_submodule(n.target), nn.BatchNorm2d)

    def _is_relu(self, n):
        if n.op == "call_function" and n.target in (F.relu, torch.relu):
            return True
        if n.op == "call_method" and n.target in ("relu", "relu_"):
            return True
        return n.op == "call_module" and isinstance(self.gm.get_submodule(n.target), nn.ReLU)

    def _is_sigmoid(self, n):
        if n.op == "call_function" and n.target in (torch.sigmoid, F.sigmoid):
            return True
        return n.op == "call_module" and isinstance(self.gm.get_submodule(n.target), nn.Sigmoid)

    def _is_add(self, n):
        return n.op == "call_function" and n.target in (operator.add, torch.add) and not n.kwargs

    def _bn_relu_tail(self, node):
        """conv -> [BatchNorm2d] -> [ReLU] chain starting at `node` (single users only)."""
        bn_node = self._single_user(node, self._is_bn)
        tail, bn = node, None
        if bn_node is not None:
            bn = self.gm.get_submodule(bn_node.target)
            self.consumed.add(bn_node)
            tail = bn_node
        relu_node = self._single_user(tail, self._is_relu)
        if relu_node is not None:
            self.consumed.add(relu_node)
            tail = relu_node
        return tail, bn, relu_node is not None

    def lower_conv(self, node, conv: nn.Conv2d):
        if _pair(conv.dilation) != (1, 1):
            raise LoweringError(f"{node.name}: dilated conv not supported")
        if conv.padding_mode != "zeros" or isinstance(conv.padding, str):
            raise LoweringError(f"{node.name}: only explicit zero padding is supported")
        if conv.groups != 1:
            if conv.groups == conv.in_channels == conv.out_channels:
                return self.lower_dwconv(node, conv)
            raise LoweringError(f"{node.name}: grouped conv (other than depthwise) not supported")
        lz = self.lazy(node.args[0])
        x = lz.tensor
        tail, bn, relu = self._bn_relu_tail(node)
        n, h, w, cin = x.shape
        cin_model = cin
        if x.nchw_input and cin % (8 if self.act_dtype == "bf16" else 4) and not lz.relu and lz.sub is None:
            # stem over the fp32 NCHW image: read a zero-padded NHWC copy in the
            # activation dtype instead (one 16-byte gather per tap), weights padded to match
            x = self._packed_input(x)
            cin = x.shape[3]
        r, s = conv.kernel_size
        sh, sw = _pair(conv.stride)
        ph, pw = _pair(conv.padding)
        if lz.sub is not None:
            # subsample(x, off) -> 1x1 conv  ==  1x1 conv with stride 2 reading pixel 2*o + off
            if (r, s, sh, sw, ph, pw) != (1, 1, 1, 1, 0, 0):
                raise LoweringError(f"{node.name}: a subsample folds only into a 1x1/s1/p0 conv")
            sh = sw = 2
            ph = pw = -lz.sub
            oh, ow = (h + 1) // 2, (w + 1) // 2   # samples off, off + 2, ... of the zero-extended map
        else:
            oh = (h + 2 * ph - r) // sh + 1
            ow = (w + 2 * pw - s) // sw + 1
        cout = conv.out_channels
        out = self.new_tensor((n, oh, ow, cout))
        wk, b = _fold_bn(conv, bn)
        if cin != cin_model:   # zero rows for the padded input channels: k = (r*S + s)*Cin + c
            wk = np.pad(wk.reshape(r * s, cin_model, cout), ((0, 0), (0, cin - cin_model), (0, 0))
                        ).reshape(r * s * cin, cout)
        macs = n * oh * ow * cout * r * s * cin_model
        op = LoweredOp(CONV2D, "conv", OpClass.COMPUTE,
                       dict(N=n, H=h, W=w, Cin=cin, OH=oh, OW=ow, Cout=cout, R=r, S=s, sh=sh,
                            sw=sw, ph=ph, pw=pw, relu=int(relu), relu_in=int(lz.relu)),
                       [x], out, wk, b, flops=2 * macs,
                       bytes_min=self._esz(x) * n * h * w * cin + self.esize * wk.size
                       + 4 * b.size + self.esize * n * oh * ow * cout,
                       label=node.name)
        self.emit(op)
        self.env[tail] = out

    def _packed_input(self, x: Tensor) -> Tensor:
        """The NHWC copy of the NCHW graph image in the activation dtype, channels padded to a 16-byte vector (one PACK_INPUT op)."""
        if getattr(self, "_packed", None) is None:
            n, h, w, c = x.shape
            v = 8 if self.act_dtype == "bf16" else 4
            cp = (c + v - 1) // v * v
            out = self.new_tensor((n, h, w, cp))
            self.emit(LoweredOp(PACK_INPUT, "copy", OpClass.MEMORY, dict(N=n, H=h, W=w, C=c, Cp=cp), [x], out,
                                bytes_min=4 * n * h * w * c + self.esize * n * h * w * cp, label="pack_input"))
            self._packed = out
        return self._packed

    def lower_dwconv(self, node, conv: nn.Conv2d):
        lz = self.lazy(node.args[0])
        if lz.sub is not None:
            raise LoweringError(f"{node.name}: subsample before a depthwise conv")
        x = lz.tensor
        tail, bn, relu = self._bn_relu_tail(node)
        n, h, w, c = x.shape
        r, s = conv.kernel_size
        sh, sw = _pair(conv.stride)
        ph, pw = _pair(conv.padding)
        oh = (h + 2 * ph - r) // sh + 1
        ow = (w + 2 * pw - s) // sw + 1
        wt = conv.weight.detach().double().cpu()[:, 0]          # [C, r, s]
        b = conv.bias.detach().double().cpu() if conv.bias is not None else torch.zeros(c, dtype=torch.float64)
        if bn is not None:
            scale = bn.weight.detach().double().cpu() / torch.sqrt(bn.running_var.detach().double().cpu() + bn.eps)
            wt = wt * scale[:, None, None]
            b = (b - bn.running_mean.detach().double().cpu()) * scale + bn.bias.detach().double().cpu()
        wk = wt.permute(1, 2, 0).reshape(r * s, c).float().numpy()   # [r*s][C]
        has_bias = conv.bias is not None or bn is not None
        out = self.new_tensor((n, oh, ow, c))
        op = LoweredOp(DWCONV2D, "dwconv", OpClass.MEMORY,
                       dict(N=n, H=h, W=w, C=c, OH=oh, OW=ow, kh=r, kw=s, sh=sh, sw=sw, ph=ph, pw=pw,
                            relu_in=int(lz.relu), act=int(relu)),
                       [x], out, np.ascontiguousarray(wk), b.float().numpy() if has_bias else None,
                       flops=2 * n * oh * ow * c * r * s,
                       bytes_min=self._esz(x) * n * h * w * c + 4 * wk.size + self.esize * n * oh * ow * c,
                       label=node.name)
        self.emit(op)
        self.env[tail] = out

    def lower_pool(self, node, is_max, k, s, p, ceil_mode, include_pad=True, dilation=1):
        if _pair(dilation) != (1, 1):
            raise LoweringError(f"{node.name}: dilated pooling not supported")
        kh, kw = _pair(k)
        sh, sw = _pair(s if s not in (None, ()) else k)
        ph, pw = _pair(p)
        lz = self.lazy(node.args[0])
        n, h, w, c = lz.tensor.shape
        if not is_max and (kh, kw) == (h, w) and (ph, pw) == (0, 0) and lz.sub is None:
            return self.lower_gap(node)          # window == whole map: global average pool
        x = self.value(node.args[0])
        oh = _pool_out(h, kh, sh, ph, ceil_mode)
        ow = _pool_out(w, kw, sw, pw, ceil_mode)
        out = self.new_tensor((n, oh, ow, c))
        op = LoweredOp(MAXPOOL2D if is_max else AVGPOOL2D, "pool", OpClass.MEMORY,
                       dict(N=n, H=h, W=w, C=c, OH=oh, OW=ow, kh=kh, kw=kw, sh=sh, sw=sw, ph=ph,
                            pw=pw, include_pad=int(include_pad)),
                       [x], out, flops=n * oh * ow * c * kh * kw,
                       bytes_min=self.esize * (n * h * w * c + n * oh * ow * c), label=node.name)
        self.emit(op)
        self.env[node] = out

    def lower_gap(self, node):
        lz = self.lazy(node.args[0])
        if lz.sub is not None:
            raise LoweringError(f"{node.name}: subsample before global pooling")
        x = lz.tensor
        n, h, w, c = x.shape
        out = self.new_tensor((n, c), dtype="f32")  # feeds the fp32 classifier head
        op = LoweredOp(GLOBAL_AVGPOOL, "pool", OpClass.MEMORY, dict(N=n, H=h, W=w, C=c, relu_in=int(lz.relu)),
                       [x], out, flops=n * h * w * c, bytes_min=self.esize * n * h * w * c + 4 * n * c,
                       label=node.name)
        self.emit(op)
        self.env[node] = out

    def lower_linear(self, node, lin: nn.Linear):
        x = self.value(node.args[0])
        if len(x.shape) != 2:
            raise LoweringError(f"{node.name}: linear expects a [rows, features] input")
        m, k = x.shape
        nout = lin.out_features
        act = 0
        tail = node
        relu_node = self._single_user(node, self._is_relu)
        if relu_node is not None:
            act = 1
            self.consumed.add(relu_node)
            tail = relu_node
        if x.dtype != "f32":
            raise LoweringError(f"{node.name}: the SIMT linear head expects fp32 rows")
        out = self.new_tensor((m, nout), dtype="f32")
        if m > 1 and k % 4 == 0:
            # a real GEMM (several rows, e.g. a DeepFM request batch): a 1x1 conv over
            # [rows, 1, 1, features], so it runs on the fp32 tensor-core engine (3xTF32
            # tcgen05) or the exact-FFMA SIMT conv, whichever the per-shape tuner measures
            # faster.  Single-row GEMVs stay on the bandwidth-bound SIMT linear kernel.
            wk = lin.weight.detach().double().cpu().numpy().T.astype(np.float32).copy()
            bias = (lin.bias.detach().float().cpu().numpy() if lin.bias is not None
                    else np.zeros(nout, dtype=np.float32))
            self.emit(LoweredOp(CONV2D, "gemm", OpClass.COMPUTE,
                                dict(N=m, H=1, W=1, Cin=k, OH=1, OW=1, Cout=nout, R=1, S=1, sh=1, sw=1, ph=0,
                                     pw=0, relu=act, relu_in=0),
                                [x], out, wk, bias, flops=2 * m * k * nout,
                                bytes_min=4 * (m * k + wk.size + bias.size + m * nout), label=node.name))
            self.env[tail] = out
            return
        wt = lin.weight.detach().float().cpu().contiguous().numpy()
        b = lin.bias.detach().float().cpu().numpy() if lin.bias is not None else None
        op = LoweredOp(LINEAR, "gemm", OpClass.COMPUTE, dict(M=m, K=k, N=nout, act=act), [x], out,
                       wt, b, flops=2 * m * k * nout,
                       bytes_min=4 * (m * k + wt.size + (0 if b is None else b.size) + m * nout),
                       label=node.name)
        self.emit(op)
        self.env[tail] = out

    def _copy_into(self, t: Tensor, label: str) -> Tensor:
        """A fresh buffer holding `t` (COPY op) — for graph inputs or values
        already placed in another concat, which cannot alias a concat slice."""
        out = self.new_tensor(t.shape, dtype=t.dtype)
        p, c = self._pixels(t)
        self.emit(LoweredOp(COPY, "copy", OpClass.MEMORY, dict(P=p, C=c, n=1, act=ACT_NONE), [t], out,
                            bytes_min=2 * self._esz(t) * p * c, label=label))
        return out

    def lower_cat(self, node):
        parts = node.args[0]
        dim = node.args[1] if len(node.args) > 1 else node.kwargs.get("dim", 0)
        ins = [self.value(p) for p in parts]
        rank = len(ins[0].shape)
        if any(len(t.shape) != rank for t in ins) or rank not in (2, 4):
            raise LoweringError(f"{node.name}: concat of 2-D rows or 4-D NCHW maps only")
        if (rank == 4 and dim not in (1, -3)) or (rank == 2 and dim not in (1, -1)):
            raise LoweringError(f"{node.name}: only channel / feature concat is supported")
        lead = ins[0].shape[:-1]
        if any(t.shape[:-1] != lead for t in ins):
            raise LoweringError(f"{node.name}: concat inputs disagree outside the channel dim")
        if any(t.dtype != ins[0].dtype for t in ins):
            # COPY kernels move one element type; a converting copy does not exist
            raise LoweringError(f"{node.name}: concat of mixed dtypes {sorted({t.dtype for t in ins})}")
        ctot = sum(t.shape[-1] for t in ins)
        out = self.new_tensor(tuple(lead) + (ctot,), dtype=ins[0].dtype)
        off = 0
        placed = []
        for p, t in zip(parts, ins):
            if t.alias is not None or t.nchw_input or t.is_graph_input:
                t = self._copy_into(t, f"{node.name}.copy")
            t.alias = out
            t.coff_in_alias = off
            off += t.shape[-1]
            placed.append(t)
        # The concat stays a DAG node (the paper's operator graph has it) but
        # launches nothing: its producers already wrote their slices, so it is
        # a pure join — capture applies its waits and records only.
        self.emit(LoweredOp(NOP, "concat", OpClass.MEMORY, {}, placed, out, label=node.name))
        self.env[node] = out

    def lower_add(self, node):
        """A tree of single-use binary adds (+ an optional sigmoid/ReLU user)
        becomes one n-ary ADD op (csrc/elementwise.cu)."""
        leaves = []

        def collect(n):
            for a in n.args[:2]:
                if isinstance(a, fx.Node) and self.env.get(a) is _PENDING_ADD:
                    collect(a)
                else:
                    leaves.append(a)
        collect(node)
        if len(leaves) > 4:
            raise LoweringError(f"{node.name}: more than 4 addends")
        ins = [self.value(a) for a in leaves]
        shape = ins[0].shape
        if any(t.shape != shape for t in ins):
            raise LoweringError(f"{node.name}: broadcasting adds are not supported")
        tail, act = node, ACT_NONE
        for pred, code in ((self._is_sigmoid, ACT_SIGMOID), (self._is_relu, ACT_RELU)):
            u = self._single_user(node, pred)
            if u is not None:
                tail, act = u, code
                self.consumed.add(u)
                break
        out = self.new_tensor(shape, dtype=ins[0].dtype)
        p, c = self._pixels(out)
        self.emit(LoweredOp(ADD, "add", OpClass.MEMORY, dict(P=p, C=c, n=len(ins), act=act), ins, out,
                            flops=(len(ins) - 1) * p * c,
                            bytes_min=(len(ins) + 1) * self._esz(out) * p * c, label=node.name))
        self.env[tail] = out

    def lower_relu(self, node):
        lz = self.lazy(node.args[0])
        self.env[node] = Lazy(lz.tensor, True, lz.sub)

    def lower_subsample(self, node):
        lz = self.lazy(node.args[0])
        if lz.sub is not None:
            raise LoweringError(f"{node.name}: nested subsample")
        self.env[node] = Lazy(lz.tensor, lz.relu, int(node.args[1]))

    # ------------------------------------------------- transformer rows path
    # Token activations are [T, C] row blocks stored as (1, 1, T, C) channel
    # views, so a linear layer is a 1x1 conv over T "pixels".

    def _param(self, node):
        if not (isinstance(node, fx.Node) and node.op == "get_attr"):
            raise LoweringError(f"{node}: expected a parameter (get_attr)")
        obj = self.gm
        for part in node.target.split("."):
            obj = getattr(obj, part)
        return obj.detach().float().cpu()

    def lower_linear_rows(self, node):
        pend = self.env[node.args[0]]
        pend = pend if isinstance(pend, PendingLN) else None
        x = pend.o if pend is not None else self.value(node.args[0])
        w = self._param(node.args[1])
        b = self._param(node.args[2]) if len(node.args) > 2 and node.args[2] is not None else None
        n, h, t, k = x.shape
        nout = w.shape[0]
        tail, act = node, 0
        for pred_fn, code in ((lambda u: u.op == "call_function" and u.target is F.gelu, 2),
                              (lambda u: u.op == "call_function" and u.target is torch.tanh, 3),
                              (self._is_relu, 1)):
            nxt = self._single_user(node, pred_fn)
            if nxt is not None:
                if code == 2 and nxt.kwargs.get("approximate", "none") != "none":
                    continue
                tail, act = nxt, code
                self.consumed.add(nxt)
                break
        bias = (b if b is not None else torch.zeros(nout)).numpy()
        ints = dict(N=1, H=1, W=t, Cin=k, OH=1, OW=t, Cout=nout, R=1, S=1, sh=1, sw=1, ph=0, pw=0,
                    relu=int(act == 1), act=act)
        out = self.new_tensor((1, 1, t, nout))
        op = LoweredOp(CONV2D, "gemm", OpClass.COMPUTE, ints, [x], out, w.t().contiguous().numpy(), bias,
                       flops=2 * t * k * nout, bytes_min=self.esize * (t * k + k * nout + t * nout) + 4 * nout,
                       label=node.name)
        if pend is not None:
            # LayerNorm of the activation rows on load (stats from the producing GEMM)
            ints.update(ln_in=1, ln_tiles=k // 128)
            op.inputs += [pend.stats, pend.res]
            op.arrays = {"gb": pend.gb}
            op.floats = (pend.eps,)
            op.flops += 4 * t * k
            op.bytes_min += 4 * pend.stats.shape[0] * pend.stats.shape[1] + 8 * k + self.esize * t * k
            if pend.writer is None:   # the first consumer materialises the normalised rows
                ints["ln_write"] = 1
                op.extra_outputs.append(pend.out)
                op.bytes_min += self.esize * t * k
                pend.writer = len(self.ops)
        self.emit(op)
        self.env[tail] = out

    def lower_embeddings(self, node):
        ids = self.value(node.args[0])
        word, pos, typ, gamma, beta = (self._param(a) for a in node.args[1:6])
        eps = float(node.args[6])
        t, c = ids.shape[-1], word.shape[1]
        out = self.new_tensor((1, 1, t, c))
        op = LoweredOp(EMBEDDING, "embedding", OpClass.MEMORY, dict(rows=t, C=c), [ids], out,
                       flops=8 * t * c, bytes_min=8 * t + 3 * 4 * t * c + self.esize * t * c, label=node.name,
                       arrays={"gamma": gamma.numpy(), "beta": beta.numpy(), "word": word.numpy(),
                               "pos": pos.numpy(), "type": typ.numpy()}, floats=(eps,))
        self.emit(op)
        self.env[node] = out

    def lower_attention(self, node):
        q, k, v = (self.value(a) for a in node.args[:3])
        heads = int(node.args[3])
        t, c = q.shape[2], q.shape[3]
        out = self.new_tensor((1, 1, t, c))
        op = LoweredOp(ATTENTION, "attention", OpClass.COMPUTE, dict(T=t, C=c, heads=heads), [q, k, v], out,
                       flops=4 * t * t * c, bytes_min=self.esize * 4 * t * c, label=node.name,
                       floats=((c // heads) ** -0.5,))
        self.emit(op)
        self.env[node] = out

    def _ln_foldable(self, node) -> bool:
        """add_layer_norm(o, res) folds into GEMMs when o comes from a bf16 row
        GEMM without activation used only here, every user is a linear layer
        reading it (at least one, lowered before any residual user) or a later
        add_layer_norm reading it as its residual, and C is whole 128-channel
        tiles.  The model's output LayerNorm (read by first_token / returned)
        stays a kernel."""
        if self.act_dtype != "bf16" or not self.fold_ln:
            return False
        o = node.args[0]
        ot = self.env.get(o)
        if not isinstance(ot, Tensor) or len(o.users) != 1 or not ot.producers or ot.alias is not None:
            return False
        prod = self.ops[min(ot.producers)]
        if (prod.kind != CONV2D or prod.name != "gemm" or prod.ints.get("act", 0) != 0 or prod.ints.get("ln_in")
                or ot.shape[-1] % 128 or ot.dtype != "bf16"):
            return False
        order = {n: i for i, n in enumerate(self.gm.graph.nodes)}
        lin = [u for u in node.users if u.op == "call_function" and u.target is F.linear and u.args[0] is node]
        res = [u for u in node.users if u.op == "call_function" and getattr(u.target, "__name__", "") ==
               "add_layer_norm" and u.args[1] is node and u.args[0] is not node]
        if not lin or len(lin) + len(res) != len(node.users):
            return False
        first = min(order[u] for u in lin)
        return all(order[u] > first for u in res)

    def lower_add_layernorm(self, node):
        if self._ln_foldable(node):
            o = self.env[node.args[0]]
            pidx = min(o.producers)
            prod = self.ops[pidx]
            r = self.value(node.args[1])
            t, c = o.shape[2], o.shape[3]
            stats = self.new_tensor((t, (c // 128) * 2), dtype="f32")
            stats.producers = {pidx}
            prod.inputs.append(r)
            prod.extra_outputs.append(stats)
            prod.ints["res_stats"] = 1
            prod.flops += 3 * t * c
            prod.bytes_min += self.esize * t * c + 4 * t * (c // 128) * 2   # residual read, stats written
            gb = np.stack([self._param(node.args[2]).numpy(), self._param(node.args[3]).numpy()]).astype(np.float32)
            self.env[node] = PendingLN(o, r, stats, gb, float(node.args[4]), self.new_tensor((1, 1, t, c)))
            return
        x, r = self.value(node.args[0]), self.value(node.args[1])
        gamma, beta = self._param(node.args[2]), self._param(node.args[3])
        eps = float(node.args[4])
        t, c = x.shape[2], x.shape[3]
        out = self.new_tensor((1, 1, t, c))
        op = LoweredOp(LAYERNORM, "layernorm", OpClass.MEMORY, dict(rows=t, C=c), [x, r], out,
                       flops=8 * t * c, bytes_min=self.esize * 3 * t * c, label=node.name,
                       arrays={"gamma": gamma.numpy(), "beta": beta.numpy()}, floats=(eps,))
        self.emit(op)
        self.env[node] = out

    def lower_first_token(self, node):
        x = self.value(node.args[0])
        view = self.new_tensor((1, 1, 1, x.shape[3]), dtype=x.dtype)
        view.alias, view.coff_in_alias = x, 0   # pixel 0 of x's buffer: a shorter view
        view.producers = set(x.producers)
        self.env[node] = view

    # -------------------------------------------------------- DeepFM path

    def lower_field_embedding(self, node):
        ids = self.value(node.args[0])
        field_idx = int(node.args[1])
        table = self._param(node.args[2])
        b = ids.shape[0]
        vocab, dim = table.shape
        out = self.new_tensor((b, dim), dtype="f32")
        self.emit(LoweredOp(FIELD_EMBEDDING, "embedding", OpClass.MEMORY,
                            dict(B=b, dim=dim, field=field_idx, vocab=vocab), [ids], out,
                            bytes_min=8 * b + 2 * 4 * b * dim, label=node.name,
                            arrays={"table": table.numpy()}))
        self.env[node] = out

    def lower_first_order(self, node):
        ids, w1, dense, wd, bias = node.args[:5]
        ids_t, dense_t = self.value(ids), self.value(dense)
        w1a, wda, ba = self._param(w1), self._param(wd), self._param(bias)
        b = ids_t.shape[0]
        fields, vocab = w1a.shape
        out = self.new_tensor((b, 1), dtype="f32")
        self.emit(LoweredOp(FIRST_ORDER, "gather", OpClass.MEMORY,
                            dict(B=b, fields=fields, vocab=vocab, n_dense=dense_t.shape[-1]), [ids_t, dense_t], out,
                            flops=2 * b * (fields + dense_t.shape[-1]),
                            bytes_min=8 * b * fields + 4 * b * fields + 4 * b * dense_t.shape[-1] + 4 * b,
                            label=node.name, arrays={"w1": w1a.numpy(), "wd": wda.reshape(-1).numpy()},
                            floats=(float(ba.reshape(-1)[0]),)))
        self.env[node] = out

    def lower_fm(self, node):
        x = self.value(node.args[0])
        fields = int(node.args[1])
        b, c = x.shape
        out = self.new_tensor((b, 1), dtype="f32")
        self.emit(LoweredOp(FM, "fm", OpClass.MEMORY, dict(B=b, fields=fields, dim=c // fields), [x], out,
                            flops=3 * b * c, bytes_min=4 * b * c + 4 * b, label=node.name))
        self.env[node] = out

    # ------------------------------------------------------------- driver

    def _graph_input(self, example: torch.Tensor) -> Tensor:
        if example.dim() == 4 and example.is_floating_point():
            n, c, h, w = example.shape
            t = self.new_tensor((n, h, w, c), dtype="f32")
            t.nchw_input = True
        elif not example.is_floating_point():
            t = self.new_tensor(tuple(example.shape), dtype="i64")
        elif example.dim() == 2:
            t = self.new_tensor(tuple(example.shape), dtype="f32")
        else:
            raise LoweringError("graph inputs: 4-D NCHW images, 2-D fp32 feature rows or integer ids")
        t.is_graph_input = True
        return t

    FUNCTIONS = {
        "bert_embeddings": "lower_embeddings", "self_attention": "lower_attention",
        "add_layer_norm": "lower_add_layernorm", "first_token": "lower_first_token",
        "field_embedding": "lower_field_embedding", "first_order": "lower_first_order",
        "fm_interaction": "lower_fm", "subsample2d": "lower_subsample",
    }

    def run(self, examples) -> Program:
        examples = list(examples) if isinstance(examples, (tuple, list)) else [examples]
        inputs = []
        for node in self.gm.graph.nodes:
            if node in self.consumed:
                continue
            if node.op == "placeholder":
                if len(inputs) >= len(examples):
                    raise LoweringError("more graph inputs than example tensors")
                t = self._graph_input(examples[len(inputs)])
                inputs.append(t)
                self.env[node] = t
            elif node.op == "get_attr":
                self.env[node] = None  # parameters are read where they are consumed
            elif node.op == "output":
                res = node.args[0]
                outs = list(res) if isinstance(res, (tuple, list)) else [res]
                self.env["__outs__"] = [self.value(r) for r in outs]
            elif node.op == "call_module":
                mod = self.gm.get_submodule(node.target)
                if isinstance(mod, nn.Conv2d):
                    self.lower_conv(node, mod)
                elif isinstance(mod, nn.MaxPool2d):
                    self.lower_pool(node, True, mod.kernel_size, mod.stride, mod.padding,
                                    mod.ceil_mode, dilation=mod.dilation)
                elif isinstance(mod, nn.AvgPool2d):
                    if mod.divisor_override is not None:
                        raise LoweringError(f"{node.name}: divisor_override unsupported")
                    self.lower_pool(node, False, mod.kernel_size, mod.stride, mod.padding,
                                    mod.ceil_mode, mod.count_include_pad)
                elif isinstance(mod, nn.AdaptiveAvgPool2d):
                    if _pair(mod.output_size) != (1, 1):
                        raise LoweringError(f"{node.name}: only global adaptive pooling")
                    self.lower_gap(node)
                elif isinstance(mod, (nn.Dropout, nn.Identity)):
                    self.env[node] = self.env[node.args[0]]
                elif isinstance(mod, nn.Linear):
                    self.lower_linear(node, mod)
                elif isinstance(mod, nn.ReLU):
                    self.lower_relu(node)
                else:
                    raise LoweringError(f"{node.name}: unsupported module {type(mod).__name__}")
            elif node.op == "call_method" and node.target in ("relu", "relu_"):
                self.lower_relu(node)
            elif node.op == "call_function":
                tgt = node.target
                name = getattr(tgt, "__name__", "")
                if tgt is torch.cat:
                    self.lower_cat(node)
                elif tgt is F.linear:
                    self.lower_linear_rows(node)
                elif name in self.FUNCTIONS:
                    getattr(self, self.FUNCTIONS[name])(node)
                elif self._is_relu(node):
                    self.lower_relu(node)
                elif self._is_add(node):
                    users = list(node.users)
                    if len(users) == 1 and self._is_add(users[0]):
                        self.env[node] = _PENDING_ADD   # folded into its consumer's n-ary ADD
                    else:
                        self.lower_add(node)
                elif tgt is torch.flatten:
                    x = self.value(node.args[0])
                    if len(x.shape) == 2:
                        self.env[node] = x
                    elif len(x.shape) == 4 and x.shape[1] == 1 and x.shape[2] == 1:
                        raise LoweringError(f"{node.name}: flatten of an unpooled 1x1 map")
                    else:
                        raise LoweringError(f"{node.name}: flatten of a spatial map unsupported")
                elif tgt is F.avg_pool2d:
                    a = node.args
                    kw = node.kwargs
                    k = a[1] if len(a) > 1 else kw["kernel_size"]
                    s = a[2] if len(a) > 2 else kw.get("stride", None)
                    p = a[3] if len(a) > 3 else kw.get("padding", 0)
                    cm = a[4] if len(a) > 4 else kw.get("ceil_mode", False)
                    cip = a[5] if len(a) > 5 else kw.get("count_include_pad", True)
                    self.lower_pool(node, False, k, s, p, cm, cip)
                elif tgt is F.max_pool2d:
                    a = node.args
                    kw = node.kwargs
                    k = a[1] if len(a) > 1 else kw["kernel_size"]
                    s = a[2] if len(a) > 2 else kw.get("stride", None)
                    p = a[3] if len(a) > 3 else kw.get("padding", 0)
                    d = a[4] if len(a) > 4 else kw.get("dilation", 1)
                    cm = a[5] if len(a) > 5 else kw.get("ceil_mode", False)
                    self.lower_pool(node, True, k, s, p, cm, dilation=d)
                elif tgt is F.adaptive_avg_pool2d:
                    size = node.args[1] if len(node.args) > 1 else node.kwargs["output_size"]
                    if _pair(size) != (1, 1):
                        raise LoweringError(f"{node.name}: only global adaptive pooling")
                    self.lower_gap(node)
                elif tgt in (F.dropout,):
                    self.env[node] = self.env[node.args[0]]
                else:
                    raise LoweringError(f"{node.name}: unsupported function {tgt}")
            else:
                raise LoweringError(f"{node.name}: unsupported fx op {node.op}")
        if len(inputs) != len(examples):
            raise LoweringError(f"model takes {len(inputs)} inputs, {len(examples)} example tensors given")
        outs = self.env["__outs__"]
        for t in outs:  # graph outputs leave the GEMM engine in fp32
            if t.producers and self.ops[min(t.producers)].kind == CONV2D and t.alias is None:
                t.dtype = "f32"
        edges = set()
        for v, op in enumerate(self.ops):
            for t in op.inputs:
                for u in t.producers:
                    edges.add((u, v))
        return Program(self.ops, self.tensors, inputs[0], outs[0], sorted(edges), outs, inputs)


def lower(model: nn.Module, example, dtype: str = "f32", fold_ln: bool = True) -> Program:
    """Trace `model` with torch.fx and lower it to executor operators.

    `example` is one input tensor or a tuple of them (one per forward
    argument).  dtype "f32": fp32 activations end to end (3xTF32 tensor-core
    convs).  dtype "bf16": bf16 activations and weights with fp32
    accumulation; the graph input stays fp32 NCHW and the classifier head
    stays fp32.  fold_ln: bf16 add_layer_norm(o, res) whose users are GEMMs
    launches no kernel (PendingLN)."""
    if dtype not in ("f32", "bf16"):
        raise ValueError(f"unknown dtype {dtype!r}")
    model = model.eval()
    gm = fx.symbolic_trace(model)
    return _Lowerer(gm, dtype, fold_ln).run(example)
