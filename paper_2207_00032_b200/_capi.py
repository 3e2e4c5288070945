"""ctypes binding of include/dsinf.h (the C ABI of libdsinf.so).

The library is built in-tree (``make lib`` / ``__graft_entry__.build()``) and loaded from this
package directory.  There is no fallback: if the shared object is missing the import fails.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdsinf.so")

OK = 0
ERR_CONFIG = 2
ERR_INFEASIBLE = 3
ERR_CUDA = 4
ERR_NCCL = 5
ERR_INTERNAL = 6

DT_F16 = 1
DT_F32 = 2
DT_I8 = 3
DT_F64 = 4
DT_BF16 = 5

INT8_W8A8 = 0
INT8_W8A16 = 1
INT8_AUTO = 2
EPI_NONE = 0
EPI_GELU = 1
EPI_RESID = 2

TP_NONE = 0
TP_NCCL = 1
TP_LOCAL = 2
TP_SLICE = 3
TP_IPC = 4

TILING_1D = 0
TILING_2D = 1

(T_QKV, T_QKV_BIAS, T_O, T_O_BIAS, T_UP, T_UP_BIAS, T_DOWN, T_DOWN_BIAS, T_LN1_G, T_LN1_B, T_LN2_G,
 T_LN2_B, T_WTE, T_LNF_G, T_LNF_B) = range(1, 16)

COLL_ALLREDUCE, COLL_ALLGATHER, COLL_ALLTOALL, COLL_BROADCAST, COLL_P2P = range(5)
OP_ELEMENTWISE, OP_REDUCTION, OP_TRANSPOSE, OP_GEMM, OP_QUANTIZE = range(5)
REGIME_SMALL_BATCH, REGIME_LARGE_BATCH = 0, 1
PHASE_PROMPT, PHASE_GENERATION = 0, 1


class DsinfError(RuntimeError):
    code = ERR_INTERNAL


class ConfigError(DsinfError):
    """infersim::ConfigError (errors.hpp:24-27)."""
    code = ERR_CONFIG


class InfeasibleError(DsinfError):
    """infersim::InfeasibleError (errors.hpp:30-34)."""
    code = ERR_INFEASIBLE


class CudaError(DsinfError):
    code = ERR_CUDA


class NcclError(DsinfError):
    code = ERR_NCCL


_ERRORS = {ERR_CONFIG: ConfigError, ERR_INFEASIBLE: InfeasibleError, ERR_CUDA: CudaError, ERR_NCCL: NcclError}


class GemmShape(C.Structure):
    _fields_ = [("out_dim", C.c_int64), ("in_dim", C.c_int64), ("batch", C.c_int64), ("dtype_bytes", C.c_int32)]


class GemmSchedule(C.Structure):
    _fields_ = [("mode", C.c_int32), ("output_tiles", C.c_int64), ("input_tiles", C.c_int64),
                ("warps_per_block", C.c_int32), ("kernel_count", C.c_int32), ("pack_M", C.c_int32)]


class DeviceSpec(C.Structure):
    _fields_ = [("mem_bytes", C.c_int64), ("mem_bw", C.c_double), ("sm_count", C.c_int32),
                ("kernel_launch_overhead", C.c_double), ("peak_flops_fp32", C.c_double),
                ("peak_flops_fp16", C.c_double), ("peak_flops_int8", C.c_double)]


class GemmArgs(C.Structure):
    _fields_ = [("w_packed", C.c_void_p), ("w_dtype", C.c_int32), ("w_scales", C.c_void_p),
                ("N", C.c_int64), ("K", C.c_int64), ("B", C.c_int64), ("x", C.c_void_p),
                ("x_dtype", C.c_int32), ("x_scales", C.c_void_p), ("bias", C.c_void_p), ("out", C.c_void_p),
                ("out_dtype", C.c_int32), ("epilogue", C.c_int32), ("ksplit", C.c_int32), ("int8_act", C.c_int32),
                ("w_group_scales", C.c_void_p), ("group_size", C.c_int32)]


class LbArgs(C.Structure):
    _fields_ = [("w", C.c_void_p), ("w_dtype", C.c_int32), ("w_scales", C.c_void_p), ("N", C.c_int64),
                ("K", C.c_int64), ("M", C.c_int64), ("x", C.c_void_p), ("x_scales", C.c_void_p),
                ("bias", C.c_void_p), ("out", C.c_void_p), ("out_dtype", C.c_int32), ("epilogue", C.c_int32)]


class LaunchPlan(C.Structure):
    _fields_ = [("col_tile", C.c_int32), ("ksplit", C.c_int32), ("rows_per_split", C.c_int32),
                ("ctas", C.c_int32), ("stages", C.c_int32)]


class ModelConfig(C.Structure):
    _fields_ = [("hidden_dim", C.c_int64), ("num_layers", C.c_int64), ("num_heads", C.c_int64),
                ("vocab_size", C.c_int64), ("max_seq", C.c_int64), ("dtype_bytes", C.c_int32)]


class RuntimeConfig(C.Structure):
    _fields_ = [("batch", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32), ("tp_mode", C.c_int32),
                ("use_cuda_graph", C.c_int32), ("use_pdl", C.c_int32), ("max_ctx", C.c_int64),
                ("seed", C.c_uint64), ("ln_eps", C.c_float), ("rope_base", C.c_float), ("device", C.c_int32),
                ("use_step_kernel", C.c_int32), ("int8_act", C.c_int32), ("int8_group", C.c_int32)]


class ModelInfo(C.Structure):
    _fields_ = [("weight_bytes", C.c_int64), ("bytes_per_token", C.c_int64), ("kernels_per_step", C.c_int64),
                ("vocab_local", C.c_int64), ("heads_local", C.c_int64), ("kv_bytes", C.c_int64),
                ("shards", C.c_int32), ("graph_ready", C.c_int32), ("fused_allreduce", C.c_int32),
                ("plan_flags", C.c_int32)]


class KernelCost(C.Structure):
    _fields_ = [("compute_time", C.c_double), ("memory_time", C.c_double), ("launch_overhead", C.c_double),
                ("total", C.c_double), ("memory_bound", C.c_int32)]


class LinkSpec(C.Structure):
    _fields_ = [("bandwidth", C.c_double), ("latency", C.c_double)]


class Topology(C.Structure):
    _fields_ = [("num_nodes", C.c_int32), ("gpus_per_node", C.c_int32), ("intra", LinkSpec), ("inter", LinkSpec),
                ("device", DeviceSpec)]


class OpGraph(C.Structure):
    _fields_ = [("num_nodes", C.c_int32), ("node_kind", C.POINTER(C.c_int32)),
                ("node_tile_count", C.POINTER(C.c_int32)), ("node_out_elems", C.POINTER(C.c_int64)),
                ("num_edges", C.c_int32), ("edge_from", C.POINTER(C.c_int32)), ("edge_to", C.POINTER(C.c_int32)),
                ("dep_off", C.POINTER(C.c_int32)), ("dep_consumer", C.POINTER(C.c_int32)),
                ("prod_off", C.POINTER(C.c_int32)), ("dep_prod", C.POINTER(C.c_int32)), ("dtype_bytes", C.c_int32)]


class GraphBuffers(C.Structure):
    _fields_ = [("num_nodes", C.c_int32), ("num_edges", C.c_int32), ("num_deps", C.c_int32),
                ("num_prods", C.c_int32), ("dtype_bytes", C.c_int32),
                ("node_kind", C.POINTER(C.c_int32)), ("node_tile_count", C.POINTER(C.c_int32)),
                ("node_out_elems", C.POINTER(C.c_int64)), ("edge_from", C.POINTER(C.c_int32)),
                ("edge_to", C.POINTER(C.c_int32)), ("dep_off", C.POINTER(C.c_int32)),
                ("dep_consumer", C.POINTER(C.c_int32)), ("prod_off", C.POINTER(C.c_int32)),
                ("dep_prod", C.POINTER(C.c_int32))]


P = C.POINTER
vp = C.c_void_p
i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); every symbol declared in include/dsinf.h
SIGNATURES = {
    "dsinf_last_error": (C.c_char_p, []),
    "dsinf_version": (C.c_char_p, []),
    "dsinf_b200_device_spec": (None, [P(DeviceSpec)]),
    "dsinf_output_tile_width": (i64, []),
    "dsinf_cache_line_pack": (i32, [i32]),
    "dsinf_derive_schedule": (C.c_int, [P(GemmShape), P(DeviceSpec), P(GemmSchedule)]),
    "dsinf_packed_index": (i64, [i64, i64, i64, i32]),
    "dsinf_pack_weights_f64": (C.c_int, [P(f64), i64, P(GemmShape), i32, P(f64), i64, P(i64)]),
    "dsinf_unpack_weights_f64": (C.c_int, [P(f64), i64, P(GemmShape), i32, P(f64), i64]),
    "dsinf_exec_device": (C.c_int, [P(f64), i64, i32, P(GemmShape), P(GemmSchedule), P(f64), i64, i64, i32, P(f64), i64]),
    "dsinf_pack_weights_device": (C.c_int, [vp, i32, i64, i64, i32, vp, vp]),
    "dsinf_quantize_weights_int8": (C.c_int, [vp, i64, i64, vp, vp, vp]),
    "dsinf_quantize_weights_int8_groups": (C.c_int, [vp, i64, i64, C.c_int32, vp, vp, vp]),
    "dsinf_quantize_activations_int8": (C.c_int, [vp, i64, i64, vp, vp, vp]),
    "dsinf_gemm": (C.c_int, [P(GemmArgs), vp]),
    "dsinf_gemm_large_batch": (C.c_int, [P(LbArgs), vp]),
    "dsinf_gemm_launch_plan": (C.c_int, [i64, i64, i64, i32, P(LaunchPlan)]),
    "dsinf_attention_decode": (C.c_int, [vp, vp, vp, vp, i64, i64, i64, i64, vp, vp]),
    "dsinf_model_create": (C.c_int, [P(ModelConfig), P(RuntimeConfig), vp, P(vp)]),
    "dsinf_model_destroy": (C.c_int, [vp]),
    "dsinf_model_ipc_handle": (C.c_int, [vp, vp, C.c_int64, C.POINTER(C.c_int64)]),
    "dsinf_model_ipc_attach": (C.c_int, [vp, vp, C.c_int64]),
    "dsinf_nccl_window_check": (C.c_int, [vp, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_float)]),
    "dsinf_model_set_prompt": (C.c_int, [vp, P(i32), i64, vp]),
    "dsinf_model_set_prompt_device": (C.c_int, [vp, vp, i64, vp]),
    "dsinf_decode_step": (C.c_int, [vp, vp]),
    "dsinf_model_prefill": (C.c_int, [vp, vp]),
    "dsinf_decode_steps": (C.c_int, [vp, i64, vp]),
    "dsinf_decode_step_host": (C.c_int, [vp, P(i32), P(i32), vp]),
    "dsinf_model_outputs": (C.c_int, [vp, P(vp), P(i64), P(vp), P(vp), P(vp)]),
    "dsinf_model_read_logits": (C.c_int, [vp, P(C.c_float), i64, vp]),
    "dsinf_model_read_tokens": (C.c_int, [vp, P(i32), P(i32), i64, vp]),
    "dsinf_model_get_info": (C.c_int, [vp, P(ModelInfo)]),
    "dsinf_model_bytes_per_step": (i64, [vp, i64]),
    "dsinf_model_step_trace": (C.c_int, [vp, P(u64), i64, P(i64), P(i32), P(i32)]),
    "dsinf_model_launch_trace": (C.c_int, [vp, P(u64), i64, P(i64)]),
    "dsinf_model_launch_phases": (C.c_int, [vp, P(u64), i64]),
    "dsinf_model_cta_log": (C.c_int, [vp, P(u64), i64]),
    "dsinf_model_set_launch_trace": (C.c_int, [vp, i32]),
    "dsinf_synthetic_tensor": (C.c_int, [u64, i32, i32, i64, i64, P(C.c_float)]),
    "dsinf_shard_tensor": (C.c_int, [P(ModelConfig), i32, i32, i32, i32, u64, P(C.c_float), i64, P(i64), P(i64)]),
    "dsinf_nccl_get_unique_id": (C.c_int, [P(C.c_uint8)]),
    "dsinf_nccl_comm_create": (C.c_int, [P(C.c_uint8), i32, i32, i32, P(vp)]),
    "dsinf_nccl_comm_destroy": (C.c_int, [vp]),
    "dsinf_param_count": (C.c_int, [P(ModelConfig), P(i64)]),
    "dsinf_param_bytes": (C.c_int, [P(ModelConfig), P(i64)]),
    "dsinf_layer_flops": (C.c_int, [P(ModelConfig), i64, i64, i64, i32, P(f64)]),
    "dsinf_kv_cache_bytes": (C.c_int, [P(ModelConfig), i64, i64, i64, P(i64)]),
    "dsinf_kernel_time": (C.c_int, [f64, f64, P(DeviceSpec), i32, i64, i32, P(KernelCost)]),
    "dsinf_collective_time": (C.c_int, [i32, f64, P(i32), i32, P(Topology), P(f64)]),
    "dsinf_min_latency_bound": (C.c_int, [P(ModelConfig), i32, i32, P(Topology), P(f64)]),
    "dsinf_fusable": (C.c_int, [P(OpGraph), i32, P(i32)]),
    "dsinf_partition_layer": (C.c_int, [P(OpGraph), i32, P(i32), P(i32)]),
    "dsinf_fusion_savings": (C.c_int, [P(OpGraph), P(i32), i32, P(i64), P(i64)]),
    "dsinf_canonical_layer_partition": (C.c_int, [i64, i64, i32, i32, P(i32), P(i32), P(i64), P(i64)]),
    "dsinf_canonical_layer_graph": (C.c_int, [i64, i64, i32, P(GraphBuffers)]),
}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build())")

lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    return (lib.dsinf_last_error() or b"").decode()


def check(status: int) -> None:
    """Raise the Python image of the reference's exception for a non-zero status."""
    if status == OK:
        return
    exc = _ERRORS.get(status, DsinfError)
    raise exc(last_error())

# launch kinds of dsinf_model_launch_trace (DSINF_LK_*)
LK_NAMES = ["embed", "qkv", "attn", "attn_out", "mlp_up", "mlp_down", "lm_head", "argmax", "prep"]
