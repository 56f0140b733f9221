"""Synthetic workloads named by BASELINE.json: inference graphs of the
paper's models (ResNet-50, BERT-base, NasNet-A, NasRNN), a random DAG
generator, and the paper's backend set (cuDNN / cuBLAS / TensorRT / TVM)
as simulated backends with cost profiles.

Graphs are built op by op with real shapes (batch 1); weights and other
parameters are graph inputs.  Cost tables are synthetic stand-ins for the
paper's measured ones (the reference ships none): per (backend, op) a
per-element coefficient and a launch overhead, with TVM fusing cheaply via
rules and TensorRT acting as the graph inference library whose contiguous
regions are discounted.
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field

from .cost import OpCost, SimMeasurer, SimProfile
from .graph import ComputationGraph, GraphInput, InputRef, OperatorNode
from .registry import BackendDescriptor, BackendKind, PatternRegistry
from .rules import FusionTransition, OpClass, OpValidity, PatternRule


class GraphBuilder:
    def __init__(self):
        self.inputs: list[GraphInput] = []
        self.nodes: list[OperatorNode] = []
        self.shapes: dict[int, tuple[int, ...]] = {}

    def input(self, name: str, shape) -> InputRef:
        self.inputs.append(GraphInput(name, tuple(shape)))
        return InputRef(name)

    def op(self, kind: str, inputs, shape, **attrs) -> int:
        nid = len(self.nodes)
        self.nodes.append(OperatorNode(nid, kind, dict(sorted(attrs.items())), tuple(inputs),
                                       tuple(int(d) for d in shape)))
        self.shapes[nid] = tuple(shape)
        return nid

    def param(self, shape) -> InputRef:
        return self.input(f"p{len(self.inputs)}", shape)

    def build(self, outputs) -> ComputationGraph:
        return ComputationGraph(self.inputs, self.nodes, outputs)


# -- ResNet-50 ---------------------------------------------------------------------------

def _conv(b: GraphBuilder, x, cin, cout, k, s, hw):
    ho = (hw + s - 1) // s
    w = b.param((cout, cin, k, k))
    return b.op("conv2d", (x, w), (1, cout, ho, ho), channels=cout, kernel_size=[k, k],
                strides=[s, s], data_layout="NCHW", groups=1), ho


def _bn(b: GraphBuilder, x, c, hw):
    return b.op("batch_norm", (x, b.param((c,)), b.param((c,))), (1, c, hw, hw), axis=1)


def resnet50(batch: int = 1) -> ComputationGraph:
    b = GraphBuilder()
    x = b.input("data", (batch, 3, 224, 224))
    y, hw = _conv(b, x, 3, 64, 7, 2, 224)
    y = _bn(b, y, 64, hw)
    y = b.op("relu", (y,), (1, 64, hw, hw))
    hw = hw // 2
    y = b.op("max_pool2d", (y,), (1, 64, hw, hw), pool_size=[3, 3], strides=[2, 2])
    cin = 64
    for stage, (blocks, width) in enumerate(((3, 64), (4, 128), (6, 256), (3, 512))):
        for i in range(blocks):
            stride = 2 if (i == 0 and stage > 0) else 1
            cout = width * 4
            t, hw2 = _conv(b, y, cin, width, 1, 1, hw)
            t = b.op("relu", (_bn(b, t, width, hw2),), (1, width, hw2, hw2))
            t, hw2 = _conv(b, t, width, width, 3, stride, hw)
            t = b.op("relu", (_bn(b, t, width, hw2),), (1, width, hw2, hw2))
            t, _ = _conv(b, t, width, cout, 1, 1, hw2)
            t = _bn(b, t, cout, hw2)
            if i == 0:
                sc, _ = _conv(b, y, cin, cout, 1, stride, hw)
                sc = _bn(b, sc, cout, hw2)
            else:
                sc = y
            y = b.op("add", (t, sc), (1, cout, hw2, hw2))
            y = b.op("relu", (y,), (1, cout, hw2, hw2))
            cin, hw = cout, hw2
    y = b.op("global_avg_pool2d", (y,), (1, cin, 1, 1))
    y = b.op("batch_flatten", (y,), (1, cin))
    y = b.op("dense", (y, b.param((1000, cin))), (1, 1000), units=1000)
    y = b.op("bias_add", (y, b.param((1000,))), (1, 1000), axis=1)
    y = b.op("softmax", (y,), (1, 1000), axis=-1)
    return b.build([y])


# -- BERT-base -----------------------------------------------------------------------------

def bert_base(seq: int = 128, layers: int = 12, hidden: int = 768, heads: int = 12,
              ffn: int = 3072) -> ComputationGraph:
    b = GraphBuilder()
    ids = b.input("input_ids", (1, seq))
    seg = b.input("segment_ids", (1, seq))
    mask = b.input("attention_mask", (1, 1, 1, seq))
    hd = hidden // heads
    x = b.op("take", (b.param((30522, hidden)), ids), (1, seq, hidden), axis=0)
    x = b.op("add", (x, b.op("take", (b.param((2, hidden)), seg), (1, seq, hidden), axis=0)),
             (1, seq, hidden))
    x = b.op("add", (x, b.param((1, seq, hidden))), (1, seq, hidden))
    x = b.op("layer_norm", (x, b.param((hidden,)), b.param((hidden,))), (1, seq, hidden),
             axis=-1)

    def proj(inp, units, rows=seq):
        d = b.op("dense", (inp, b.param((units, hidden))), (1, rows, units), units=units)
        return b.op("bias_add", (d, b.param((units,))), (1, rows, units), axis=-1)

    for _ in range(layers):
        heads_out = []
        for _name in ("q", "k", "v"):
            t = proj(x, hidden)
            t = b.op("reshape", (t,), (1, seq, heads, hd), newshape=[1, seq, heads, hd])
            t = b.op("transpose", (t,), (1, heads, seq, hd), axes=[0, 2, 1, 3])
            heads_out.append(t)
        q, k, v = heads_out
        s = b.op("batch_matmul", (q, k), (1, heads, seq, seq), transpose_b=1)
        s = b.op("divide", (s, b.param((1,))), (1, heads, seq, seq))
        s = b.op("add", (s, mask), (1, heads, seq, seq))
        s = b.op("softmax", (s,), (1, heads, seq, seq), axis=-1)
        o = b.op("batch_matmul", (s, v), (1, heads, seq, hd), transpose_b=0)
        o = b.op("transpose", (o,), (1, seq, heads, hd), axes=[0, 2, 1, 3])
        o = b.op("reshape", (o,), (1, seq, hidden), newshape=[1, seq, hidden])
        o = proj(o, hidden)
        o = b.op("add", (o, x), (1, seq, hidden))
        x = b.op("layer_norm", (o, b.param((hidden,)), b.param((hidden,))), (1, seq, hidden),
                 axis=-1)
        f = b.op("dense", (x, b.param((ffn, hidden))), (1, seq, ffn), units=ffn)
        f = b.op("bias_add", (f, b.param((ffn,))), (1, seq, ffn), axis=-1)
        f = b.op("gelu", (f,), (1, seq, ffn))
        f = b.op("dense", (f, b.param((hidden, ffn))), (1, seq, hidden), units=hidden)
        f = b.op("bias_add", (f, b.param((hidden,))), (1, seq, hidden), axis=-1)
        f = b.op("add", (f, x), (1, seq, hidden))
        x = b.op("layer_norm", (f, b.param((hidden,)), b.param((hidden,))), (1, seq, hidden),
                 axis=-1)
    cls = b.op("strided_slice", (x,), (1, 1, hidden), begin=[0, 0, 0], end=[1, 1, hidden])
    cls = b.op("reshape", (cls,), (1, hidden), newshape=[1, hidden])
    p = b.op("dense", (cls, b.param((hidden, hidden))), (1, hidden), units=hidden)
    p = b.op("bias_add", (p, b.param((hidden,))), (1, hidden), axis=-1)
    p = b.op("tanh", (p,), (1, hidden))
    return b.build([x, p])


# -- NasNet-A ------------------------------------------------------------------------------

def _sep_conv(b: GraphBuilder, x, c, k, hw, stride=1):
    y = x
    for rep in range(2):
        s = stride if rep == 0 else 1
        h2 = (hw + s - 1) // s
        y = b.op("relu", (y,), (1, c, hw, hw))
        y = b.op("conv2d", (y, b.param((c, 1, k, k))), (1, c, h2, h2), channels=c,
                 kernel_size=[k, k], strides=[s, s], groups=c, data_layout="NCHW")
        y = b.op("conv2d", (y, b.param((c, c, 1, 1))), (1, c, h2, h2), channels=c,
                 kernel_size=[1, 1], strides=[1, 1], groups=1, data_layout="NCHW")
        y = _bn(b, y, c, h2)
        hw = h2
    return y


def _squeeze(b: GraphBuilder, x, cin, c, hw):
    y = b.op("relu", (x,), (1, cin, hw, hw))
    y = b.op("conv2d", (y, b.param((c, cin, 1, 1))), (1, c, hw, hw), channels=c,
             kernel_size=[1, 1], strides=[1, 1], groups=1, data_layout="NCHW")
    return _bn(b, y, c, hw)


_NORMAL = (("sep5", 1, "sep3", 0), ("sep5", 0, "sep3", 0), ("avg3", 1, "id", 0),
           ("avg3", 0, "avg3", 0), ("sep3", 0, "id", 0))
_REDUCE = (("sep5", 1, "sep7", 0), ("max3", 1, "sep7", 0), ("avg3", 1, "sep5", 0),
           ("id", 2, "max3", 1), ("avg3", 2, "sep3", 1))


def _branch(b: GraphBuilder, kind, x, c, hw, stride):
    h2 = (hw + stride - 1) // stride
    if kind.startswith("sep"):
        return _sep_conv(b, x, c, int(kind[3]), hw, stride)
    if kind == "avg3":
        return b.op("avg_pool2d", (x,), (1, c, h2, h2), pool_size=[3, 3], strides=[stride, stride])
    if kind == "max3":
        return b.op("max_pool2d", (x,), (1, c, h2, h2), pool_size=[3, 3], strides=[stride, stride])
    if stride == 1:
        return x
    return b.op("avg_pool2d", (x,), (1, c, h2, h2), pool_size=[1, 1], strides=[stride, stride])


def nasnet_a(cells_per_stack: int = 4, stem_channels: int = 32, filters: int = 44) -> ComputationGraph:
    """NASNet-A (mobile-style): conv stem, two reduction cells, then three
    stacks of `cells_per_stack` normal cells separated by reduction cells.
    Every cell squeezes its two inputs (relu, 1x1 conv, bn) and combines
    them through five blocks of two branch ops joined by add; unused block
    outputs are concatenated."""
    b = GraphBuilder()
    x = b.input("data", (1, 3, 224, 224))
    hw = 112
    stem = b.op("conv2d", (x, b.param((stem_channels, 3, 3, 3))), (1, stem_channels, hw, hw),
                channels=stem_channels, kernel_size=[3, 3], strides=[2, 2], groups=1,
                data_layout="NCHW")
    stem = _bn(b, stem, stem_channels, hw)
    prev, cur, cprev, ccur = stem, stem, stem_channels, stem_channels
    c = filters // 4
    plan = ["reduce", "reduce"]
    for stack in range(3):
        if stack:
            plan.append("reduce")
        plan.extend(["normal"] * cells_per_stack)
    for cell in plan:
        reduce = cell == "reduce"
        if reduce:
            c *= 2
        stride = 2 if reduce else 1
        out_hw = (hw + stride - 1) // stride
        states = [_squeeze(b, cur, ccur, c, hw), _squeeze(b, prev, cprev, c, hw)]
        used = set()
        for left, li, right, ri in (_REDUCE if reduce else _NORMAL):
            branches = []
            for kind, idx in ((left, li), (right, ri)):
                in_stride, in_hw = (stride, hw) if idx < 2 else (1, out_hw)
                branches.append(_branch(b, kind, states[idx], c, in_hw, in_stride))
                used.add(idx)
            states.append(b.op("add", tuple(branches), (1, c, out_hw, out_hw)))
        outs = tuple(states[i] for i in range(2, len(states)) if i not in used)
        nxt = b.op("concatenate", outs, (1, c * len(outs), out_hw, out_hw), axis=1)
        if reduce:
            prev, cprev = b.op("avg_pool2d", (cur,), (1, ccur, out_hw, out_hw), pool_size=[1, 1],
                               strides=[2, 2]), ccur
        else:
            prev, cprev = cur, ccur
        cur, ccur, hw = nxt, c * len(outs), out_hw
    y = b.op("relu", (cur,), (1, ccur, hw, hw))
    y = b.op("global_avg_pool2d", (y,), (1, ccur, 1, 1))
    y = b.op("batch_flatten", (y,), (1, ccur))
    y = b.op("dense", (y, b.param((1000, ccur))), (1, 1000), units=1000)
    y = b.op("bias_add", (y, b.param((1000,))), (1, 1000), axis=1)
    y = b.op("softmax", (y,), (1, 1000), axis=-1)
    return _prune(b, [y])


def _prune(b: GraphBuilder, outputs) -> ComputationGraph:
    """Drop nodes that reach no output and renumber densely."""
    consumers: dict[int, list[int]] = {n.id: [] for n in b.nodes}
    for n in b.nodes:
        for r in n.input_ids:
            if isinstance(r, int):
                consumers[r].append(n.id)
    live = set(outputs)
    for n in reversed(b.nodes):
        if n.id in live:
            for r in n.input_ids:
                if isinstance(r, int):
                    live.add(r)
    remap = {}
    nodes = []
    for n in b.nodes:
        if n.id in live:
            remap[n.id] = len(remap)
    used_inputs = set()
    for n in b.nodes:
        if n.id not in live:
            continue
        refs = tuple(remap[r] if isinstance(r, int) else r for r in n.input_ids)
        used_inputs.update(r.name for r in refs if isinstance(r, InputRef))
        nodes.append(OperatorNode(remap[n.id], n.op_kind, n.attrs, refs, n.output_shape))
    inputs = [gi for gi in b.inputs if gi.name in used_inputs]
    return ComputationGraph(inputs, nodes, [remap[o] for o in outputs])


# -- NasRNN ----------------------------------------------------------------------------------

def nasrnn(steps: int = 10, hidden: int = 512, batch: int = 1) -> ComputationGraph:
    """The NAS recurrent cell (Zoph & Le, 2017) unrolled over `steps`:
    eight gated linear leaves of (x_t, h_{t-1}) combined by a fixed tree of
    add / mul with tanh / sigmoid / relu / identity activations."""
    b = GraphBuilder()
    shape = (batch, hidden)
    h = b.input("h0", shape)
    cstate = b.input("c0", shape)
    leaf_acts = ("sigmoid", "relu", "sigmoid", "identity", "tanh", "sigmoid", "tanh", "relu")
    pair_ops = (("add", "tanh"), ("mul", "sigmoid"), ("mul", "tanh"), ("mul", "tanh"))
    for t in range(steps):
        x = b.input(f"x{t}", shape)
        leaves = []
        for i in range(8):
            wx = b.op("dense", (x, b.param((hidden, hidden))), shape, units=hidden)
            wh = b.op("dense", (h, b.param((hidden, hidden))), shape, units=hidden)
            s = b.op("add", (wx, wh), shape)
            act = leaf_acts[i]
            leaves.append(s if act == "identity" else b.op(act, (s,), shape))
        level = []
        for i, (comb, act) in enumerate(pair_ops):
            y = b.op(comb, (leaves[2 * i], leaves[2 * i + 1]), shape)
            level.append(b.op(act, (y,), shape))
        # cell-state injection
        inj = b.op("add", (level[0], cstate), shape)
        level[0] = b.op("tanh", (inj,), shape)
        a = b.op("tanh", (b.op("mul", (level[0], level[1]), shape),), shape)
        c2 = b.op("relu", (b.op("add", (level[2], level[3]), shape),), shape)
        cstate = c2
        h = b.op("tanh", (b.op("mul", (a, c2), shape),), shape)
    return b.build([h, cstate])


# -- random DAG -------------------------------------------------------------------------------

RANDOM_OPS = ("conv2d", "add", "relu", "mul", "tanh", "dense", "sigmoid", "batch_norm")
RANDOM_SHAPES = ((1, 4, 4, 4), (1, 8, 8, 8), (1, 16, 4, 4), (1, 32, 8, 8))


def random_dag(n: int, seed: int = 0, ops=RANDOM_OPS[:4], p_node_input: float = 0.75,
               window: int | None = None) -> ComputationGraph:
    """Random DAG, ids in topological order; each node has 1-2 inputs drawn
    from earlier nodes (within `window` if given) or the graph input, and the
    outputs are exactly the sinks."""
    rng = random.Random(seed)
    nodes = []
    consumed = set()
    for i in range(n):
        refs = []
        for _ in range(rng.choice((1, 1, 2))):
            if i > 0 and rng.random() < p_node_input:
                lo = 0 if window is None else max(0, i - window)
                j = rng.randrange(lo, i)
                refs.append(j)
                consumed.add(j)
            else:
                refs.append(InputRef("x"))
        nodes.append(OperatorNode(i, rng.choice(ops), {"variant": rng.randrange(3)},
                                  tuple(refs), rng.choice(RANDOM_SHAPES)))
    outputs = [i for i in range(n) if i not in consumed]
    return ComputationGraph([GraphInput("x", RANDOM_SHAPES[0])], nodes, outputs)


# -- backends ------------------------------------------------------------------------------------

ELEMWISE = ("relu", "add", "mul", "tanh", "sigmoid", "gelu", "bias_add", "divide", "copy",
            "identity")
INJECTIVE = ("reshape", "transpose", "batch_flatten", "strided_slice", "take", "concatenate")
REDUCE = ("softmax", "layer_norm", "batch_norm", "global_avg_pool2d", "avg_pool2d", "max_pool2d")
HEAVY = ("conv2d", "dense", "batch_matmul")


@dataclass
class BackendSet:
    registry: PatternRegistry
    measurer: SimMeasurer
    graph_backend: str
    rules: dict[str, PatternRule] = field(default_factory=dict)


def _profile(bid: str, table: dict[str, tuple[float, float]], **kw) -> SimProfile:
    return SimProfile(bid, {op: OpCost(c, o) for op, (c, o) in table.items()}, **kw)


def paper_backends(g: ComputationGraph, with_rules: bool = True, verify: bool = True) -> BackendSet:
    """cuDNN, cuBLAS and TVM (op kernel libraries) and TensorRT (graph
    inference library) with simulated cost tables; TVM's fused patterns are
    generated from its fusion rule against `g`."""
    present = sorted({n.op_kind for n in g.nodes.values()})
    reg = PatternRegistry()
    profiles = {}

    def cost_table(scale_heavy, scale_light, over_heavy, over_light, ops):
        t = {}
        for op in ops:
            if op in HEAVY:
                t[op] = (scale_heavy, over_heavy)
            elif op in REDUCE:
                t[op] = (scale_light * 1.5, over_light * 1.2)
            else:
                t[op] = (scale_light, over_light)
        return t

    # cuDNN: convolutions, pooling, activations, softmax
    cudnn_ops = [op for op in present if op in ("conv2d", "relu", "tanh", "sigmoid", "add",
                                                "max_pool2d", "avg_pool2d", "global_avg_pool2d",
                                                "softmax", "batch_norm")]
    reg.add_backend(BackendDescriptor("cudnn", BackendKind.OP_KERNEL_LIBRARY))
    for op in cudnn_ops:
        reg.add_pattern("cudnn", f"{op}()")
    if "conv2d" in present:
        for text in ("relu(conv2d(*, *))", "relu(batch_norm(conv2d(*, *), *, *))",
                     "batch_norm(conv2d(*, *), *, *)", "relu(add(batch_norm(conv2d(*, *), *, *), *))"):
            reg.add_pattern("cudnn", text)
    profiles["cudnn"] = _profile("cudnn", cost_table(2.0e-9, 1.0e-9, 0.012, 0.006, cudnn_ops),
                                 fusion_discount=0.85)
    # cuBLAS: GEMMs
    blas_ops = [op for op in present if op in ("dense", "batch_matmul", "bias_add")]
    if blas_ops:
        reg.add_backend(BackendDescriptor("cublas", BackendKind.OP_KERNEL_LIBRARY))
        for op in blas_ops:
            reg.add_pattern("cublas", f"{op}()")
        if "dense" in present and "bias_add" in present:
            reg.add_pattern("cublas", "bias_add(dense(*, *), *)")
        profiles["cublas"] = _profile("cublas", cost_table(1.2e-9, 1.0e-9, 0.010, 0.006, blas_ops),
                                      fusion_discount=0.9)
    # TVM: every op, fusion rule (kFusable anchor + elementwise/injective tail)
    reg.add_backend(BackendDescriptor("tvm", BackendKind.OP_KERNEL_LIBRARY))
    for op in present:
        reg.add_pattern("tvm", f"{op}()")
    rules = {}
    if with_rules:
        validity = []
        for op in present:
            if op in HEAVY:
                cls = OpClass.FUSABLE
            elif op in ELEMWISE:
                cls = OpClass.ELEMWISE
            elif op in INJECTIVE:
                cls = OpClass.INJECTIVE
            else:
                cls = OpClass.OPAQUE
            validity.append(OpValidity(op, (), cls))
        rule = PatternRule("tvm", tuple(validity), (
            FusionTransition(OpClass.FUSABLE, OpClass.ELEMWISE, OpClass.FUSABLE),
            FusionTransition(OpClass.ELEMWISE, OpClass.ELEMWISE, OpClass.ELEMWISE),
            FusionTransition(OpClass.INJECTIVE, OpClass.INJECTIVE, OpClass.INJECTIVE),
            FusionTransition(OpClass.INJECTIVE, OpClass.ELEMWISE, OpClass.INJECTIVE),
        ), max_fusion_size=8)
        rules["tvm"] = rule
        reg.add_pattern_rule("tvm", rule, g, verify=verify)
    profiles["tvm"] = _profile("tvm", cost_table(3.0e-9, 0.8e-9, 0.015, 0.005, present),
                               fusion_discount=0.75)
    # TensorRT: graph inference library
    trt_ops = [op for op in present if op not in ("take", "strided_slice")]
    reg.add_backend(BackendDescriptor("tensorrt", BackendKind.GRAPH_INFERENCE_LIBRARY))
    for op in trt_ops:
        reg.add_pattern("tensorrt", f"{op}()")
    if "conv2d" in present:
        reg.add_pattern("tensorrt", "relu(batch_norm(conv2d(*, *), *, *))")
    if "dense" in present and "bias_add" in present:
        reg.add_pattern("tensorrt", "bias_add(dense(*, *), *)")
    profiles["tensorrt"] = _profile("tensorrt", cost_table(1.8e-9, 1.1e-9, 0.014, 0.008, trt_ops),
                                    fusion_discount=0.8, region_alpha=0.05, region_floor=0.7)
    return BackendSet(reg, SimMeasurer(profiles), "tensorrt", rules)


def random_backends(g: ComputationGraph, n_backends: int = 8, n_graph: int = 1, seed: int = 0,
                    fused_per_backend: int = 6) -> BackendSet:
    """`n_backends` simulated backends over the graph's op kinds: backend 0
    carries every singleton, the others random singleton subsets and
    depth-2 fused patterns copied from the graph; the last `n_graph` are
    graph inference libraries."""
    rng = random.Random(seed)
    present = sorted({n.op_kind for n in g.nodes.values()})
    reg = PatternRegistry()
    profiles = {}
    with_preds = [n for n in g.nodes.values() if any(isinstance(r, int) for r in n.input_ids)]
    for b in range(n_backends):
        is_graph = b >= n_backends - n_graph
        bid = f"{'g' if is_graph else 'b'}{b}"
        reg.add_backend(BackendDescriptor(bid, BackendKind.GRAPH_INFERENCE_LIBRARY if is_graph
                                          else BackendKind.OP_KERNEL_LIBRARY))
        ops = present if b == 0 or is_graph else [op for op in present if rng.random() < 0.7]
        for op in ops:
            reg.add_pattern(bid, f"{op}()")
        for _ in range(fused_per_backend if b else 0):
            if not with_preds:
                break
            node = rng.choice(with_preds)
            args = []
            for r in node.input_ids:
                if isinstance(r, int) and rng.random() < 0.8:
                    args.append(f"{g.nodes[r].op_kind}()")
                else:
                    args.append("*")
            reg.add_pattern(bid, f"{node.op_kind}({', '.join(args)})")
        profiles[bid] = SimProfile(
            bid, {op: OpCost(rng.choice((0.0, 1e-6, 2e-6)), round(rng.uniform(0.05, 1.0), 3))
                  for op in present},
            fusion_discount=rng.choice((1.0, 0.95, 0.9, 0.8)),
            region_alpha=rng.choice((0.02, 0.05)), region_floor=rng.choice((0.7, 0.9)))
    graph_ids = reg.graph_backend_ids()
    return BackendSet(reg, SimMeasurer(profiles), graph_ids[-1] if graph_ids else "")


CONFIGS = {
    "resnet50": lambda: resnet50(),
    "bert_base": lambda: bert_base(),
    "nasnet_a": lambda: nasnet_a(),
    "nasrnn": lambda: nasrnn(),
    "random100k": lambda: random_dag(100_000, seed=0, ops=RANDOM_OPS, window=64),
}
