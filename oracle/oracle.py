"""ctypes wrappers for the CPU oracle (liboracle.so) and the reference shim (_ref/).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, as the checker.  Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libinfersim_ref.so")

P = C.POINTER
f64p = P(C.c_double)


class Schedule(C.Structure):
    _fields_ = [("two_d", C.c_int32), ("output_tiles", C.c_int64), ("input_tiles", C.c_int64),
                ("warps_per_block", C.c_int32), ("kernel_count", C.c_int32), ("pack_M", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("hidden", C.c_int64), ("layers", C.c_int64), ("heads", C.c_int64), ("vocab", C.c_int64),
                ("max_ctx", C.c_int64), ("dtype_bytes", C.c_int32), ("tp", C.c_int32), ("batch", C.c_int32),
                ("sm_count", C.c_int32), ("seed", C.c_uint64), ("ln_eps", C.c_float), ("rope_base", C.c_float),
                ("int8_act", C.c_int32), ("int8_group", C.c_int32)]


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


_or = _load(ORACLE_PATH)
_ref = _load(REF_PATH)


def oracle_lib():
    if _or is None:
        raise RuntimeError(f"{ORACLE_PATH} missing: run `make oracle`")
    return _or


def ref_lib() -> Optional[C.CDLL]:
    return _ref


if _or is not None:
    _or.or_cache_line_pack.restype = C.c_int32
    _or.or_derive_schedule.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, P(Schedule)]
    _or.or_packed_index.restype = C.c_int64
    _or.or_packed_index.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32]
    _or.or_pack.argtypes = [f64p, C.c_int64, C.c_int64, C.c_int32, f64p]
    _or.or_exec_sameorder.argtypes = [f64p, C.c_int64, C.c_int64, C.c_int32, P(Schedule), f64p, C.c_int64, f64p]
    _or.or_gemm_f64.argtypes = [P(C.c_float), C.c_int64, C.c_int64, P(Schedule), f64p, C.c_int64, f64p]
    _or.or_f32_to_f16.restype = C.c_uint16
    _or.or_f32_to_f16.argtypes = [C.c_float]
    _or.or_f16_to_f32.restype = C.c_float
    _or.or_f16_to_f32.argtypes = [C.c_uint16]
    _or.or_quant_rows.argtypes = [P(C.c_float), C.c_int64, C.c_int64, P(C.c_int8), P(C.c_float)]
    _or.or_quant_groups.argtypes = [P(C.c_float), C.c_int64, C.c_int64, C.c_int64, P(C.c_int8), P(C.c_uint16)]
    _or.or_gemm_i8.argtypes = [P(C.c_int8), P(C.c_float), P(C.c_int8), P(C.c_float), C.c_int64, C.c_int64,
                               C.c_int64, P(C.c_int32), P(C.c_float)]
    _or.or_synth_base.restype = C.c_uint64
    _or.or_synth_base.argtypes = [C.c_uint64, C.c_int32, C.c_int32]
    _or.or_synth_unit.restype = C.c_float
    _or.or_synth_unit.argtypes = [C.c_uint64, C.c_uint64]
    _or.or_model_create.restype = C.c_void_p
    _or.or_model_create.argtypes = [P(Config)]
    _or.or_model_destroy.argtypes = [C.c_void_p]
    _or.or_model_step.argtypes = [C.c_void_p, P(C.c_int32), C.c_int64, P(C.c_float), P(C.c_int32)]
    _or.or_model_final_hidden.argtypes = [C.c_void_p, P(C.c_float)]
    _or.or_synth_matrix.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                    P(C.c_float)]
    _or.or_synth_vector.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int64, P(C.c_float)]
    _or.or_model_set_int8_act.argtypes = [C.c_void_p, C.c_int32]
    _or.or_model_set_gemm_hook.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]

if _ref is not None:
    _ref.ref_packed_index.restype = C.c_int64
    _ref.ref_packed_index.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int]
    _ref.ref_derive_schedule.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, P(C.c_int64)]
    _ref.ref_pack_weights.argtypes = [f64p, C.c_int64, C.c_int64, C.c_int, C.c_int, f64p, C.c_int64]
    _ref.ref_unpack_weights.argtypes = [f64p, C.c_int64, C.c_int64, C.c_int, C.c_int, f64p]
    _ref.ref_exec_reference.argtypes = [f64p, C.c_int64, C.c_int64, C.c_int, P(C.c_int64), f64p, C.c_int64, f64p]
    _ref.ref_time_exec.restype = C.c_double
    _ref.ref_time_exec.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int,
                                   C.c_uint64, f64p]
    _ref.ref_step_create.restype = C.c_void_p
    _ref.ref_step_create.argtypes = [P(C.c_int64), P(C.c_int64), C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int,
                                     C.c_uint64]
    _ref.ref_step_run.restype = C.c_double
    _ref.ref_step_run.argtypes = [C.c_void_p, C.c_int]
    _ref.ref_step_destroy.argtypes = [C.c_void_p]
    _ref.ref_gemm_hook_clear.argtypes = []
    _ref.ref_param_count.argtypes = [C.c_int64] * 5 + [C.c_int, P(C.c_int64)]
    _ref.ref_layer_flops.argtypes = [C.c_int64] * 5 + [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int, f64p]
    _ref.ref_kv_cache_bytes.argtypes = [C.c_int64] * 5 + [C.c_int, C.c_int64, C.c_int64, C.c_int64, P(C.c_int64)]
    _ref.ref_kernel_time.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int64, C.c_int, f64p]
    _ref.ref_collective_time.argtypes = [C.c_int, C.c_double, P(C.c_int), C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.c_double, C.c_double, C.c_double, f64p]
    _ref.ref_min_latency_bound.argtypes = [C.c_int64] * 4 + [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int64, f64p]
    _ref.ref_canonical_partition.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, P(C.c_int32), P(C.c_int32),
                                             P(C.c_int64), P(C.c_int64)]
    _ref.ref_partition_graph.argtypes = [C.c_int, P(C.c_int32), P(C.c_int32), P(C.c_int64), C.c_int, P(C.c_int32),
                                         P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                         C.c_int, C.c_int, P(C.c_int32), P(C.c_int32), P(C.c_int64), P(C.c_int64)]


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(f64p)


# ---------------------------------------------------------------- oracle (restatement)

def derive_schedule(N, K, B, dtype_bytes, sm_count=148) -> Schedule:
    s = Schedule()
    rc = oracle_lib().or_derive_schedule(N, K, B, dtype_bytes, sm_count, C.byref(s))
    if rc:
        raise ValueError("invalid gemm shape")
    return s


def pack(W, M):
    N, K = W.shape
    kp = (K + M - 1) // M * M
    Wd, wp = _d(W)
    out = np.zeros(N * kp)
    oracle_lib().or_pack(wp, N, K, M, out.ctypes.data_as(f64p))
    return out


def exec_sameorder(packed, N, K, M, sched: Schedule, x, B):
    pd, pp = _d(packed)
    xd, xp = _d(x)
    out = np.zeros(B * N)
    oracle_lib().or_exec_sameorder(pp, N, K, M, C.byref(sched), xp, B, out.ctypes.data_as(f64p))
    return out.reshape(B, N)


def gemm_f64(W_f32, x, sched: Schedule):
    """exec_reference-order GEMM over row-major fp32 weights; returns [B][N] fp64."""
    W = np.ascontiguousarray(W_f32, dtype=np.float32)
    N, K = W.shape
    xd, xp = _d(x)
    B = xd.size // K
    out = np.zeros(B * N)
    oracle_lib().or_gemm_f64(W.ctypes.data_as(P(C.c_float)), N, K, C.byref(sched), xp, B, out.ctypes.data_as(f64p))
    return out.reshape(B, N)


def f32_to_f16_bits(v: float) -> int:
    return int(oracle_lib().or_f32_to_f16(v))


def quant_rows(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    R, K = x.shape
    q = np.zeros((R, K), dtype=np.int8)
    s = np.zeros(R, dtype=np.float32)
    oracle_lib().or_quant_rows(x.ctypes.data_as(P(C.c_float)), R, K, q.ctypes.data_as(P(C.c_int8)),
                               s.ctypes.data_as(P(C.c_float)))
    return q, s


def quant_groups(x, group=128):
    """or_quant_groups: (q int8 [R][K], fp16 scales [ceil(K/group)][R] as float16)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    R, K = x.shape
    q = np.zeros((R, K), dtype=np.int8)
    s = np.zeros(((K + group - 1) // group, R), dtype=np.uint16)
    oracle_lib().or_quant_groups(x.ctypes.data_as(P(C.c_float)), R, K, group, q.ctypes.data_as(P(C.c_int8)),
                                 s.ctypes.data_as(P(C.c_uint16)))
    return q, s.view(np.float16)


def dequant_groups(q, s16, group=128):
    """The K-group recipe's effective weights q * s (exact in fp64; the fp16 scale times an int8)."""
    R, K = q.shape
    sc = np.repeat(s16.astype(np.float64).T, group, axis=1)[:, :K]
    return q.astype(np.float64) * sc


def gemm_a16_groups(q, s16, x16, group=128):
    """y[B][N] = sum_g s_g * sum_{k in g} q x in fp64, rounded to fp32 (the GPU: each group's exact
    int8 x fp16 products summed in fp32, times its fp16 scale, groups summed in fp32)."""
    w = dequant_groups(q, s16, group)
    return (np.asarray(x16, dtype=np.float64) @ w.T).astype(np.float32)


def gemm_i8(wq, ws, xq, xs):
    wq = np.ascontiguousarray(wq, dtype=np.int8)
    xq = np.ascontiguousarray(xq, dtype=np.int8)
    ws = np.ascontiguousarray(ws, dtype=np.float32)
    xs = np.ascontiguousarray(xs, dtype=np.float32)
    N, K = wq.shape
    B = xq.shape[0]
    acc = np.zeros((B, N), dtype=np.int32)
    y = np.zeros((B, N), dtype=np.float32)
    oracle_lib().or_gemm_i8(wq.ctypes.data_as(P(C.c_int8)), ws.ctypes.data_as(P(C.c_float)),
                            xq.ctypes.data_as(P(C.c_int8)), xs.ctypes.data_as(P(C.c_float)), N, K, B,
                            acc.ctypes.data_as(P(C.c_int32)), y.ctypes.data_as(P(C.c_float)))
    return acc, y


def synth_unit(seed, layer, tensor, flat) -> float:
    base = oracle_lib().or_synth_base(seed, layer, tensor)
    return float(oracle_lib().or_synth_unit(base, flat))


class OracleModel:
    """CPU decoder with the GPU path's storage points (fp16 / fp32) and exec_reference GEMM order."""

    def __init__(self, hidden, layers, heads, vocab=50257, *, dtype_bytes=2, tp=1, batch=1, max_ctx=256,
                 seed=20220701, ln_eps=1e-5, rope_base=10000.0, sm_count=148, int8_act=0, int8_group=0):
        self.cfg = Config(hidden, layers, heads, vocab, max_ctx, dtype_bytes, tp, batch, sm_count, seed, ln_eps,
                          rope_base, int8_act, int8_group)
        self.batch, self.vocab, self.hidden = batch, vocab, hidden
        self._h = oracle_lib().or_model_create(C.byref(self.cfg))

    def step(self, tokens, pos):
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        logits = np.zeros((self.batch, self.vocab), dtype=np.float32)
        nxt = np.zeros(self.batch, dtype=np.int32)
        rc = oracle_lib().or_model_step(self._h, tok.ctypes.data_as(P(C.c_int32)), pos,
                                        logits.ctypes.data_as(P(C.c_float)), nxt.ctypes.data_as(P(C.c_int32)))
        if rc:
            raise ValueError("oracle step failed")
        return logits, nxt

    def set_int8_act(self, mode):
        oracle_lib().or_model_set_int8_act(self._h, mode)

    def use_reference_gemm(self, on=True):
        """Route every fp16-path GEMM through the reference's own exec_reference (oracle/_ref,
        compiled from the reference headers) instead of the same-order restatement."""
        ref = ref_lib()
        if on and ref is None:
            raise RuntimeError("oracle/_ref is not built")
        if on:
            self._sm = C.c_int(self.cfg.sm_count)
            fn = C.cast(ref.ref_gemm_hook, C.c_void_p)
            oracle_lib().or_model_set_gemm_hook(self._h, fn, C.cast(C.pointer(self._sm), C.c_void_p))
        else:
            oracle_lib().or_model_set_gemm_hook(self._h, None, None)

    def final_hidden(self):
        out = np.zeros((self.batch, self.hidden), dtype=np.float32)
        oracle_lib().or_model_final_hidden(self._h, out.ctypes.data_as(P(C.c_float)))
        return out

    def close(self):
        if self._h:
            if ref_lib() is not None:
                ref_lib().ref_gemm_hook_clear()
            oracle_lib().or_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- reference shim

def ref_derive_schedule(N, K, B, dtype, sm_count):
    out = (C.c_int64 * 6)()
    rc = ref_lib().ref_derive_schedule(N, K, B, dtype, sm_count, out)
    return rc, list(out)


def ref_exec_reference(W, dtype, sched6, x, B):
    W = np.ascontiguousarray(W, dtype=np.float64)
    N, K = W.shape
    xd, xp = _d(x)
    out = np.zeros(B * N)
    s = (C.c_int64 * 6)(*sched6)
    rc = ref_lib().ref_exec_reference(W.ctypes.data_as(f64p), N, K, dtype, s, xp, B, out.ctypes.data_as(f64p))
    if rc:
        raise ValueError(f"ref_exec_reference rc={rc}")
    return out.reshape(B, N)
