"""Python image of the reference operator API for the decode hot path.

Names, argument meaning and error behaviour follow the reference's header-only C++ library
(`infersim`): gemm.hpp (SBI-GeMM schedule, packed layout, exec), fusion.hpp (Deep-Fusion
partition), model.hpp (accounting) and costmodel.hpp (roofline / collectives).  Every call goes
through the C ABI of libdsinf.so (include/dsinf.h); nothing here computes on its own.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Set

import numpy as np

from . import _capi as capi
from ._capi import ConfigError, InfeasibleError  # noqa: F401  (re-exported, errors.hpp:24-34)

# ---------------------------------------------------------------- gemm.hpp

kOutputTileWidth = int(capi.lib.dsinf_output_tile_width())  # gemm.hpp:45


class TilingMode(enum.IntEnum):  # gemm.hpp:42
    oneD = capi.TILING_1D
    twoD = capi.TILING_2D


@dataclass
class GemmShape:  # gemm.hpp:28-40
    out_dim: int = 0
    in_dim: int = 0
    batch: int = 1
    dtype_bytes: int = 2

    def _c(self) -> capi.GemmShape:
        return capi.GemmShape(self.out_dim, self.in_dim, self.batch, self.dtype_bytes)

    def validate(self) -> None:
        if self.out_dim < 1 or self.in_dim < 1 or self.batch < 1:
            raise ConfigError("gemm shape dims must be positive")
        if self.dtype_bytes not in (1, 2, 4):
            raise ConfigError("dtype_bytes must be one of {1, 2, 4}")


@dataclass
class GemmSchedule:  # gemm.hpp:47-54
    mode: TilingMode = TilingMode.oneD
    output_tiles: int = 1
    input_tiles: int = 1
    warps_per_block: int = 1
    kernel_count: int = 1
    pack_M: int = 1

    def _c(self) -> capi.GemmSchedule:
        return capi.GemmSchedule(int(self.mode), self.output_tiles, self.input_tiles, self.warps_per_block,
                                 self.kernel_count, self.pack_M)


@dataclass
class DeviceSpec:  # hardware.hpp:36-69 (peak map as three slots)
    mem_bytes: int = 0
    mem_bw: float = 0.0
    sm_count: int = 0
    kernel_launch_overhead: float = 5e-6
    peak_flops_by_dtype: Dict[int, float] = field(default_factory=dict)

    def _c(self) -> capi.DeviceSpec:
        p = self.peak_flops_by_dtype
        return capi.DeviceSpec(self.mem_bytes, self.mem_bw, self.sm_count, self.kernel_launch_overhead,
                               p.get(4, 0.0), p.get(2, 0.0), p.get(1, 0.0))


def b200_device() -> DeviceSpec:
    d = capi.DeviceSpec()
    capi.lib.dsinf_b200_device_spec(C.byref(d))
    return DeviceSpec(d.mem_bytes, d.mem_bw, d.sm_count, d.kernel_launch_overhead,
                      {4: d.peak_flops_fp32, 2: d.peak_flops_fp16, 1: d.peak_flops_int8})


def cache_line_pack(dtype_bytes: int) -> int:  # gemm.hpp:57-60
    return int(capi.lib.dsinf_cache_line_pack(dtype_bytes))


def derive_schedule(shape: GemmShape, device: DeviceSpec) -> GemmSchedule:  # gemm.hpp:65-96
    out = capi.GemmSchedule()
    capi.check(capi.lib.dsinf_derive_schedule(C.byref(shape._c()), C.byref(device._c()), C.byref(out)))
    return GemmSchedule(TilingMode(out.mode), out.output_tiles, out.input_tiles, out.warps_per_block,
                        out.kernel_count, out.pack_M)


def packed_index(n: int, k: int, out_dim: int, pack_M: int) -> int:  # gemm.hpp:108-111
    return int(capi.lib.dsinf_packed_index(n, k, out_dim, pack_M))


@dataclass
class PackedWeights:  # gemm.hpp:101-106
    data: np.ndarray
    shape: GemmShape
    pack_M: int
    padded_in_dim: int


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel())


def _ptr(a: np.ndarray, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def pack_weights(matrix, shape: GemmShape, pack_M: int) -> PackedWeights:  # gemm.hpp:113-130
    m = _f64(matrix)
    kp = C.c_int64()
    capi.check(capi.lib.dsinf_pack_weights_f64(_ptr(m), m.size, C.byref(shape._c()), pack_M, None, 0, C.byref(kp)))
    out = np.zeros(shape.out_dim * kp.value, dtype=np.float64)
    capi.check(capi.lib.dsinf_pack_weights_f64(_ptr(m), m.size, C.byref(shape._c()), pack_M, _ptr(out), out.size,
                                               C.byref(kp)))
    return PackedWeights(out, GemmShape(**shape.__dict__), pack_M, kp.value)


def unpack_weights(packed: PackedWeights) -> np.ndarray:  # gemm.hpp:132-139
    out = np.zeros(packed.shape.out_dim * packed.shape.in_dim, dtype=np.float64)
    data = _f64(packed.data)
    capi.check(capi.lib.dsinf_unpack_weights_f64(_ptr(data), data.size, C.byref(packed.shape._c()), packed.pack_M,
                                                 _ptr(out), out.size))
    return out


def exec_device(packed: PackedWeights, x, batch: int, schedule: GemmSchedule,
                compute_dtype: int = capi.DT_F16) -> np.ndarray:
    """exec_reference (gemm.hpp:147-202) run by the sm_100a SBI-GeMM kernel.

    Same inputs and output layout as the reference (row-major B x N); the device computes in
    fp16 with fp32 accumulation (or W8A8 int8 with int32 accumulation)."""
    xv = _f64(x)
    data = _f64(packed.data)
    out = np.zeros(batch * packed.shape.out_dim, dtype=np.float64)
    shape = GemmShape(packed.shape.out_dim, packed.shape.in_dim, batch, packed.shape.dtype_bytes)
    capi.check(capi.lib.dsinf_exec_device(_ptr(data), data.size, packed.pack_M, C.byref(shape._c()), C.byref(schedule._c()),
                                          _ptr(xv), xv.size, batch, compute_dtype, _ptr(out), out.size))
    return out


# ---------------------------------------------------------------- model.hpp

@dataclass
class ModelConfig:  # model.hpp:42-64 (dense)
    name: str = ""
    hidden_dim: int = 0
    num_layers: int = 0
    num_heads: int = 1
    vocab_size: int = 50257
    max_seq: int = 2048
    dtype_bytes: int = 2

    def _c(self) -> capi.ModelConfig:
        return capi.ModelConfig(self.hidden_dim, self.num_layers, self.num_heads, self.vocab_size, self.max_seq,
                                self.dtype_bytes)


@dataclass
class SeqWorkload:  # model.hpp:68-80
    batch: int = 1
    prompt_len: int = 0
    gen_tokens: int = 0


class Phase(enum.IntEnum):  # model.hpp:82
    prompt = capi.PHASE_PROMPT
    generation = capi.PHASE_GENERATION


def param_count(cfg: ModelConfig) -> int:  # model.hpp:93-101
    out = C.c_int64()
    capi.check(capi.lib.dsinf_param_count(C.byref(cfg._c()), C.byref(out)))
    return out.value


def param_bytes(cfg: ModelConfig) -> int:  # model.hpp:103-105
    out = C.c_int64()
    capi.check(capi.lib.dsinf_param_bytes(C.byref(cfg._c()), C.byref(out)))
    return out.value


def layer_flops(cfg: ModelConfig, w: SeqWorkload, phase: Phase) -> float:  # model.hpp:121-132
    out = C.c_double()
    capi.check(capi.lib.dsinf_layer_flops(C.byref(cfg._c()), w.batch, w.prompt_len, w.gen_tokens, int(phase),
                                          C.byref(out)))
    return out.value


def kv_cache_bytes(cfg: ModelConfig, w: SeqWorkload) -> int:  # model.hpp:135-140
    out = C.c_int64()
    capi.check(capi.lib.dsinf_kv_cache_bytes(C.byref(cfg._c()), w.batch, w.prompt_len, w.gen_tokens, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- costmodel.hpp

@dataclass
class KernelCost:  # costmodel.hpp:31-38
    compute_time: float
    memory_time: float
    launch_overhead: float
    total: float

    def memory_bound(self) -> bool:
        return self.memory_time >= self.compute_time


def kernel_time(flops: float, bytes_moved: float, device: DeviceSpec, dtype_bytes: int, fused_launches: int = 1,
                cuda_graph: bool = False) -> KernelCost:  # costmodel.hpp:42-56
    out = capi.KernelCost()
    capi.check(capi.lib.dsinf_kernel_time(flops, bytes_moved, C.byref(device._c()), dtype_bytes, fused_launches,
                                          int(cuda_graph), C.byref(out)))
    return KernelCost(out.compute_time, out.memory_time, out.launch_overhead, out.total)


class CollectiveKind(enum.IntEnum):  # costmodel.hpp:40
    allreduce = capi.COLL_ALLREDUCE
    allgather = capi.COLL_ALLGATHER
    alltoall = capi.COLL_ALLTOALL
    broadcast = capi.COLL_BROADCAST
    p2p = capi.COLL_P2P


@dataclass
class LinkSpec:  # hardware.hpp:30-34
    bandwidth: float = 0.0
    latency: float = 0.0


@dataclass
class Topology:  # the fields of hardware.hpp:80-123 that the cost model reads
    num_nodes: int = 1
    gpus_per_node: int = 1
    device: DeviceSpec = field(default_factory=DeviceSpec)
    intra: LinkSpec = field(default_factory=LinkSpec)
    inter: LinkSpec = field(default_factory=LinkSpec)

    def _c(self) -> capi.Topology:
        return capi.Topology(self.num_nodes, self.gpus_per_node, capi.LinkSpec(self.intra.bandwidth, self.intra.latency),
                             capi.LinkSpec(self.inter.bandwidth, self.inter.latency), self.device._c())


def collective_time(kind: CollectiveKind, bytes_per_rank: float, group: Sequence[int], topo: Topology) -> float:
    g = (C.c_int32 * max(1, len(group)))(*group)
    out = C.c_double()
    capi.check(capi.lib.dsinf_collective_time(int(kind), bytes_per_rank, g, len(group), C.byref(topo._c()),
                                              C.byref(out)))
    return out.value


@dataclass
class ParallelismPlan:  # costmodel.hpp:106-109
    tp: int = 1
    pp: int = 1


def min_latency_bound(cfg: ModelConfig, plan: ParallelismPlan, topo: Topology) -> float:  # costmodel.hpp:113-125
    out = C.c_double()
    capi.check(capi.lib.dsinf_min_latency_bound(C.byref(cfg._c()), plan.tp, plan.pp, C.byref(topo._c()),
                                                C.byref(out)))
    return out.value


# ---------------------------------------------------------------- fusion.hpp

class OpKind(enum.IntEnum):  # fusion.hpp:29
    elementwise = capi.OP_ELEMENTWISE
    reduction = capi.OP_REDUCTION
    transpose = capi.OP_TRANSPOSE
    gemm = capi.OP_GEMM
    quantize = capi.OP_QUANTIZE


class BatchRegime(enum.IntEnum):  # fusion.hpp:135
    small_batch = capi.REGIME_SMALL_BATCH
    large_batch = capi.REGIME_LARGE_BATCH


@dataclass
class OpNode:  # fusion.hpp:39-65 (dims are names only; legality uses tile structure)
    name: str
    kind: OpKind = OpKind.elementwise
    out_elems: int = 0
    tile_count: int = 1


@dataclass
class GraphEdge:  # fusion.hpp:68-72
    from_: int
    to: int
    tile_dep: Dict[int, Set[int]] = field(default_factory=dict)


@dataclass
class OpGraph:  # fusion.hpp:74-116
    nodes: List[OpNode] = field(default_factory=list)
    edges: List[GraphEdge] = field(default_factory=list)
    dtype_bytes: int = 2

    def edge_bytes(self, e: GraphEdge) -> int:
        return self.nodes[e.from_].out_elems * self.dtype_bytes


@dataclass
class FusionRegion:  # fusion.hpp:118-121
    node_ids: List[int]
    launch_count: int = 1


@dataclass
class FusionSavings:  # fusion.hpp:175-178
    launches_saved: int = 0
    bytes_saved: int = 0


class _FlatGraph:
    """Keeps the ctypes arrays of a flattened OpGraph alive for one call."""

    def __init__(self, g: OpGraph):
        n, e = len(g.nodes), len(g.edges)
        arr = lambda t, v: (t * max(1, len(v)))(*v)  # noqa: E731
        self.kind = arr(C.c_int32, [int(x.kind) for x in g.nodes])
        self.tiles = arr(C.c_int32, [x.tile_count for x in g.nodes])
        self.elems = arr(C.c_int64, [x.out_elems for x in g.nodes])
        self.efrom = arr(C.c_int32, [x.from_ for x in g.edges])
        self.eto = arr(C.c_int32, [x.to for x in g.edges])
        dep_off, cons, prod_off, prod = [0], [], [0], []
        for x in g.edges:
            for c in sorted(x.tile_dep):
                cons.append(c)
                prod.extend(sorted(x.tile_dep[c]))
                prod_off.append(len(prod))
            dep_off.append(len(cons))
        self.dep_off = arr(C.c_int32, dep_off)
        self.cons = arr(C.c_int32, cons)
        self.prod_off = arr(C.c_int32, prod_off)
        self.prod = arr(C.c_int32, prod)
        self.c = capi.OpGraph(n, self.kind, self.tiles, self.elems, e, self.efrom, self.eto, self.dep_off, self.cons,
                              self.prod_off, self.prod, g.dtype_bytes)


def fusable(graph: OpGraph, edge: GraphEdge) -> bool:  # fusion.hpp:126-133
    g = OpGraph(graph.nodes, [edge], graph.dtype_bytes)
    fg = _FlatGraph(g)
    out = C.c_int32()
    capi.check(capi.lib.dsinf_fusable(C.byref(fg.c), 0, C.byref(out)))
    return bool(out.value)


def partition_layer(graph: OpGraph, regime: BatchRegime) -> List[FusionRegion]:  # fusion.hpp:140-173
    fg = _FlatGraph(graph)
    region_of = (C.c_int32 * max(1, len(graph.nodes)))()
    nreg = C.c_int32()
    capi.check(capi.lib.dsinf_partition_layer(C.byref(fg.c), int(regime), region_of, C.byref(nreg)))
    regions = [FusionRegion([]) for _ in range(nreg.value)]
    for i in range(len(graph.nodes)):
        regions[region_of[i]].node_ids.append(i)
    return regions


def fusion_savings(regions: List[FusionRegion], graph: OpGraph) -> FusionSavings:  # fusion.hpp:183-215
    region_of = [-1] * len(graph.nodes)
    covered = 0
    for r, reg in enumerate(regions):
        for i in reg.node_ids:
            if i < 0 or i >= len(graph.nodes) or region_of[i] != -1:
                raise ConfigError("regions must partition the graph")
            region_of[i] = r
            covered += 1
    if covered != len(graph.nodes):
        raise ConfigError("regions must cover every node")
    fg = _FlatGraph(graph)
    ro = (C.c_int32 * max(1, len(region_of)))(*region_of)
    l, b = C.c_int64(), C.c_int64()
    capi.check(capi.lib.dsinf_fusion_savings(C.byref(fg.c), ro, len(regions), C.byref(l), C.byref(b)))
    return FusionSavings(l.value, b.value)


CANONICAL_NODE_NAMES = ("input_layernorm", "qkv_gemm", "attn_transpose", "attention", "post_attn_layernorm",
                        "intermediate_gemm", "bias_add", "residual_add")  # fusion.hpp:266-288


def canonical_layer_graph(hidden: int, batch: int, dtype_bytes: int = 2) -> OpGraph:  # fusion.hpp:242-357
    """The canonical decode-layer graph built by the library (dsinf_canonical_layer_graph)."""
    gb = capi.GraphBuffers()
    capi.check(capi.lib.dsinf_canonical_layer_graph(hidden, batch, dtype_bytes, C.byref(gb)))
    n, e, nd, npr = gb.num_nodes, gb.num_edges, gb.num_deps, gb.num_prods
    bufs = {"node_kind": (C.c_int32 * n)(), "node_tile_count": (C.c_int32 * n)(), "node_out_elems": (C.c_int64 * n)(),
            "edge_from": (C.c_int32 * e)(), "edge_to": (C.c_int32 * e)(), "dep_off": (C.c_int32 * (e + 1))(),
            "dep_consumer": (C.c_int32 * max(1, nd))(), "prod_off": (C.c_int32 * (nd + 1))(),
            "dep_prod": (C.c_int32 * max(1, npr))()}
    for k, v in bufs.items():
        setattr(gb, k, C.cast(v, type(getattr(gb, k))))
    capi.check(capi.lib.dsinf_canonical_layer_graph(hidden, batch, dtype_bytes, C.byref(gb)))
    g = OpGraph(dtype_bytes=gb.dtype_bytes)
    for i in range(n):
        g.nodes.append(OpNode(CANONICAL_NODE_NAMES[i], OpKind(bufs["node_kind"][i]), bufs["node_out_elems"][i],
                              bufs["node_tile_count"][i]))
    for j in range(e):
        dep = {}
        for c in range(bufs["dep_off"][j], bufs["dep_off"][j + 1]):
            dep[bufs["dep_consumer"][c]] = set(bufs["dep_prod"][bufs["prod_off"][c]:bufs["prod_off"][c + 1]])
        g.edges.append(GraphEdge(bufs["edge_from"][j], bufs["edge_to"][j], dep))
    return g


def canonical_layer_partition(hidden: int, batch: int, regime: BatchRegime, dtype_bytes: int = 2):
    """canonical_layer_graph (fusion.hpp:242-357) -> partition_layer -> fusion_savings, in one call.

    Returns (regions as lists of node names, FusionSavings)."""
    region_of = (C.c_int32 * 8)()
    nreg = C.c_int32()
    l, b = C.c_int64(), C.c_int64()
    capi.check(capi.lib.dsinf_canonical_layer_partition(hidden, batch, dtype_bytes, int(regime), region_of,
                                                        C.byref(nreg), C.byref(l), C.byref(b)))
    regions = [[] for _ in range(nreg.value)]
    for i in range(8):
        regions[region_of[i]].append(CANONICAL_NODE_NAMES[i])
    return regions, FusionSavings(l.value, b.value)
