"""Host-side driver of the B200 decode path over the C ABI.

`DecoderModel` owns one dsinf_model handle (weights, KV cache, CUDA graph) and exposes the
per-token loop; the `gemm` / `attention_decode` / quantisation helpers call the device operators
on torch tensors (torch is only the device allocator and stream provider here).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _capi as capi

try:  # torch is plumbing (device memory, streams); the product is libdsinf.so
    import torch
except ImportError:  # pragma: no cover
    torch = None


from .presets import PRESETS, Preset  # noqa: E402,F401  (BASELINE.json configs)


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream if torch is not None and torch.cuda.is_available() else None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


class DecoderModel:
    """Greedy decode of a dense decoder (GPT-J-style block, pre-LN, rotary, tanh GeLU) on B200."""

    def __init__(self, hidden: int, layers: int, heads: int, vocab: int = 50257, max_seq: int = 2048, *,
                 dtype_bytes: int = 2, batch: int = 1, max_ctx: int = 256, tp_size: int = 1, tp_rank: int = 0,
                 tp_mode: int = capi.TP_NONE, nccl_comm: Optional[int] = None, use_cuda_graph: bool = True,
                 use_pdl: bool = True, use_step_kernel: bool = False, seed: int = 20220701, ln_eps: float = 1e-5, rope_base: float = 10000.0,
                 device: int = 0, int8_act: int = capi.INT8_W8A8, ipc_exchange=None, int8_group: int = 0):
        self.cfg = capi.ModelConfig(hidden, layers, heads, vocab, max_seq, dtype_bytes)
        self.rt = capi.RuntimeConfig(batch, tp_size, tp_rank, tp_mode, int(use_cuda_graph), int(use_pdl), max_ctx,
                                     seed, ln_eps, rope_base, device, int(use_step_kernel), int(int8_act),
                                     int(int8_group))
        self.batch, self.vocab, self.max_ctx = batch, vocab, max_ctx
        self.hidden, self.layers, self.heads = hidden, layers, heads
        self._h = C.c_void_p()
        capi.check(capi.lib.dsinf_model_create(C.byref(self.cfg), C.byref(self.rt), nccl_comm, C.byref(self._h)))
        self.info = self.get_info()
        if tp_mode == capi.TP_IPC and tp_size > 1:
            if ipc_exchange is None:
                raise capi.ConfigError("TP_IPC needs ipc_exchange(bytes) -> list of every rank's bytes")
            self.ipc_attach(ipc_exchange(self.ipc_handle()))

    # -- DSINF_TP_IPC: CUDA-IPC handles, exchanged by the caller over any host channel
    def ipc_handle(self) -> bytes:
        n = C.c_int64()
        capi.check(capi.lib.dsinf_model_ipc_handle(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        capi.check(capi.lib.dsinf_model_ipc_handle(self._h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def ipc_attach(self, blobs) -> None:
        allb = b"".join(blobs)
        buf = (C.c_uint8 * len(allb)).from_buffer_copy(allb)
        capi.check(capi.lib.dsinf_model_ipc_attach(self._h, buf, len(allb)))

    # -- lifecycle
    def close(self) -> None:
        if self._h:
            capi.check(capi.lib.dsinf_model_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def get_info(self) -> capi.ModelInfo:
        info = capi.ModelInfo()
        capi.check(capi.lib.dsinf_model_get_info(self._h, C.byref(info)))
        return info

    # -- prompt and steps
    def set_prompt(self, prompt: np.ndarray, stream=None) -> None:
        """prompt: int32 [B][P] host array; resets the position to 0."""
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        assert p.ndim == 2 and p.shape[0] == self.batch
        capi.check(capi.lib.dsinf_model_set_prompt(self._h, p.ctypes.data_as(C.POINTER(C.c_int32)), p.shape[1],
                                                   _stream_ptr(stream)))

    def set_prompt_device(self, prompt_dev, prompt_len: int, stream=None) -> None:
        capi.check(capi.lib.dsinf_model_set_prompt_device(self._h, _dptr(prompt_dev), prompt_len,
                                                          _stream_ptr(stream)))

    def step(self, n: int = 1, stream=None) -> None:
        capi.check(capi.lib.dsinf_decode_steps(self._h, n, _stream_ptr(stream)))

    def prefill(self, stream=None) -> None:
        """The whole prompt at once on the tensor cores (same resulting state as step(prompt_len))."""
        capi.check(capi.lib.dsinf_model_prefill(self._h, _stream_ptr(stream)))

    def outputs(self):
        logits, ld, nxt, hist, pos = C.c_void_p(), C.c_int64(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        capi.check(capi.lib.dsinf_model_outputs(self._h, C.byref(logits), C.byref(ld), C.byref(nxt), C.byref(hist),
                                                C.byref(pos)))
        return logits.value, ld.value, nxt.value, hist.value, pos.value

    def read_logits(self, stream=None) -> np.ndarray:
        """[shards, B, vocab_local_padded] fp32 (shards > 1 only for single-device TP)."""
        info = self.info
        out = np.zeros((info.shards, self.batch, info.vocab_local), dtype=np.float32)
        capi.check(capi.lib.dsinf_model_read_logits(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), out.size,
                                                    _stream_ptr(stream)))
        return out

    def full_logits(self, stream=None) -> np.ndarray:
        """Logits [B, vocab] assembled over the vocab shards resident on this device."""
        lg = self.read_logits(stream)
        return np.concatenate(list(lg), axis=1)[:, : self.vocab] if lg.shape[0] > 1 else lg[0, :, : self.vocab]

    def read_tokens(self, stream=None):
        nxt = np.zeros(self.batch, dtype=np.int32)
        hist = np.zeros((self.batch, self.max_ctx), dtype=np.int32)
        capi.check(capi.lib.dsinf_model_read_tokens(self._h, nxt.ctypes.data_as(C.POINTER(C.c_int32)),
                                                    hist.ctypes.data_as(C.POINTER(C.c_int32)), hist.size,
                                                    _stream_ptr(stream)))
        return nxt, hist

    def launch_trace(self, steps: int = 8, stream=None):
        """Per-launch device timeline of `steps` more decode steps: array [steps][launches][3] of
        (first CTA start ns, last CTA end ns, kind DSINF_LK_*) in the step's enqueue order, then for SBI-GeMM
        launches (first release, last prologue end, last main-loop end, longest CTA prologue, last release, 3 sub-phase probes) ns —
        [steps][launches][11]."""
        capi.check(capi.lib.dsinf_model_set_launch_trace(self._h, 1))
        out = []
        try:
            for _ in range(steps):
                self.step(1, stream=stream)
                n = C.c_int64()
                capi.check(capi.lib.dsinf_model_launch_trace(self._h, None, 0, C.byref(n)))
                buf = np.zeros(3 * n.value, dtype=np.uint64)
                capi.check(capi.lib.dsinf_model_launch_trace(self._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                             buf.size, None))
                ph = np.zeros(8 * n.value, dtype=np.uint64)
                capi.check(capi.lib.dsinf_model_launch_phases(self._h, ph.ctypes.data_as(C.POINTER(C.c_uint64)), ph.size))
                out.append(np.concatenate([buf.reshape(-1, 3), ph.reshape(-1, 8)], axis=1))
        finally:
            capi.check(capi.lib.dsinf_model_set_launch_trace(self._h, 0))
        return np.stack(out)

    def bytes_per_step(self, pos: int) -> int:
        return int(capi.lib.dsinf_model_bytes_per_step(self._h, pos))

    def generate(self, prompt: np.ndarray, gen_tokens: int, stream=None) -> np.ndarray:
        """Prefill the prompt token by token, then greedy-decode `gen_tokens`; returns [B, gen]."""
        P = prompt.shape[1]
        # the token sampled at step pos is stored at history[pos + 1]: the last one (pos = P + gen - 2)
        # needs P + gen - 1 < max_ctx, else the returned slice would come back one column short
        if P + gen_tokens > self.max_ctx:
            raise capi.InfeasibleError(f"prompt {P} + {gen_tokens} generated tokens exceed max_ctx {self.max_ctx}")
        self.set_prompt(prompt, stream)
        self.step(P + gen_tokens - 1, stream)
        _, hist = self.read_tokens(stream)
        return hist[:, P: P + gen_tokens]


# ---------------------------------------------------------------- device operators on torch tensors

def gemm(w_packed, x, N: int, K: int, *, w_scales=None, x_scales=None, bias=None, out=None, out_dtype=None,
         gelu: bool = False, ksplit: int = 0, a16: bool = False, w_group_scales=None, stream=None):
    """SBI-GeMM: out[B][N] = x[B][K] . W^T over the reference packed layout.

    w_packed: fp16 tensor [ceil(K/2)*2*N] (pack_M = 2) or int8 [ceil(K/4)*4*N] (pack_M = 4).
    w_group_scales: fp16 [ceil(K/128)][N] K-group scales (quantize_weights_int8_groups; W8A16)."""
    B = x.shape[0]
    i8w = w_packed.dtype == torch.int8
    if out is None:
        od = out_dtype or (torch.float16 if gelu else torch.float32)
        out = torch.empty((B, N), dtype=od, device=x.device)
    a = capi.GemmArgs()
    a.w_packed = _dptr(w_packed)
    a.w_dtype = capi.DT_I8 if i8w else capi.DT_F16
    a.w_scales = _dptr(w_scales)
    a.N, a.K, a.B = N, K, B
    a.x = _dptr(x)
    a.x_dtype = capi.DT_I8 if x.dtype == torch.int8 else capi.DT_F16
    a.x_scales = _dptr(x_scales)
    a.bias = _dptr(bias)
    a.out = _dptr(out)
    a.out_dtype = capi.DT_F32 if out.dtype == torch.float32 else capi.DT_F16
    a.epilogue = capi.EPI_GELU if gelu else capi.EPI_NONE
    a.ksplit = ksplit
    a.int8_act = capi.INT8_W8A16 if a16 or w_group_scales is not None else capi.INT8_W8A8
    if w_group_scales is not None:
        a.w_group_scales = _dptr(w_group_scales)
        a.group_size = 128
    capi.check(capi.lib.dsinf_gemm(C.byref(a), _stream_ptr(stream)))
    return out


def gemm_large_batch(w, x, *, w_scales=None, x_scales=None, bias=None, out=None, out_dtype=None, gelu=False,
                     resid=False, stream=None):
    """tcgen05 tensor-core GEMM of the large-batch regime: out[M][N] = x[M][K] . W[N][K]^T.

    w: row-major [N][K] fp16, or int8 with w_scales [N]; x: [M][K] of the same type (int8 with
    x_scales [M]).  gelu -> fp16 out; resid -> out (fp32) += result."""
    N, K = w.shape
    M = x.shape[0]
    i8 = w.dtype == torch.int8
    if out is None:
        od = out_dtype or (torch.float16 if gelu else torch.float32)
        out = torch.empty((M, N), dtype=od, device=x.device)
    a = capi.LbArgs()
    a.w = _dptr(w)
    a.w_dtype = capi.DT_I8 if i8 else (capi.DT_BF16 if w.dtype == torch.bfloat16 else capi.DT_F16)
    a.w_scales = _dptr(w_scales)
    a.N, a.K, a.M = N, K, M
    a.x = _dptr(x)
    a.x_scales = _dptr(x_scales)
    a.bias = _dptr(bias)
    a.out = _dptr(out)
    a.out_dtype = capi.DT_F32 if out.dtype == torch.float32 else capi.DT_F16
    a.epilogue = capi.EPI_GELU if gelu else (capi.EPI_RESID if resid else capi.EPI_NONE)
    capi.check(capi.lib.dsinf_gemm_large_batch(C.byref(a), _stream_ptr(stream)))
    return out


def pack_weights_device(w, pack_M: int = 2, stream=None):
    """Row-major [N][K] (fp16/fp32) -> packed fp16 [ceil(K/M)*M*N] (gemm.hpp:113-130 layout)."""
    N, K = w.shape
    kp = (K + pack_M - 1) // pack_M * pack_M
    out = torch.empty(N * kp, dtype=torch.float16, device=w.device)
    src = capi.DT_F32 if w.dtype == torch.float32 else capi.DT_F16
    capi.check(capi.lib.dsinf_pack_weights_device(_dptr(w.contiguous()), src, N, K, pack_M, _dptr(out),
                                                  _stream_ptr(stream)))
    return out


def quantize_weights_int8(w, stream=None):
    """Row-major fp16 [N][K] -> (packed int8 [ceil(K/4)*4*N], per-row fp32 scales [N])."""
    N, K = w.shape
    kp = (K + 3) // 4 * 4
    q = torch.empty(N * kp, dtype=torch.int8, device=w.device)
    s = torch.empty(N, dtype=torch.float32, device=w.device)
    capi.check(capi.lib.dsinf_quantize_weights_int8(_dptr(w.contiguous()), N, K, _dptr(q), _dptr(s),
                                                    _stream_ptr(stream)))
    return q, s


def quantize_weights_int8_groups(w, stream=None):
    """Row-major fp16 [N][K] -> (packed int8 [ceil(K/4)*4*N], fp16 K-group scales [ceil(K/128)][N])."""
    N, K = w.shape
    kp = (K + 3) // 4 * 4
    q = torch.zeros(N * kp, dtype=torch.int8, device=w.device)
    s = torch.empty(((K + 127) // 128, N), dtype=torch.float16, device=w.device)
    capi.check(capi.lib.dsinf_quantize_weights_int8_groups(_dptr(w.contiguous()), N, K, 128, _dptr(q), _dptr(s),
                                                           _stream_ptr(stream)))
    return q, s


def quantize_activations_int8(x, stream=None):
    B, K = x.shape
    q = torch.empty((B, K), dtype=torch.int8, device=x.device)
    s = torch.empty(B, dtype=torch.float32, device=x.device)
    capi.check(capi.lib.dsinf_quantize_activations_int8(_dptr(x.contiguous()), B, K, _dptr(q), _dptr(s),
                                                        _stream_ptr(stream)))
    return q, s


def attention_decode(q, kcache, vcache, pos_dev, out=None, stream=None):
    """q [B][H][d] fp16, caches [B][H][max_seq][d] fp16, pos_dev int32[1] -> out [B][H*d]."""
    B, H, d = q.shape
    max_seq = kcache.shape[2]
    if out is None:
        out = torch.empty((B, H * d), dtype=torch.float16, device=q.device)
    capi.check(capi.lib.dsinf_attention_decode(_dptr(q), _dptr(kcache), _dptr(vcache), _dptr(pos_dev), B, H, d,
                                               max_seq, _dptr(out), _stream_ptr(stream)))
    return out


def launch_plan(N: int, K: int, B: int, int8: bool = False) -> capi.LaunchPlan:
    p = capi.LaunchPlan()
    capi.check(capi.lib.dsinf_gemm_launch_plan(N, K, B, capi.DT_I8 if int8 else capi.DT_F16, C.byref(p)))
    return p


def shard_tensor(hidden: int, heads: int, vocab: int, tp: int, rank: int, layer: int, tensor: int,
                 seed: int) -> np.ndarray:
    """Rank `rank`'s tensor-parallel shard of a synthetic tensor (logical row-major), host-side."""
    cfg = capi.ModelConfig(hidden, 1, heads, vocab, 2048, 2)
    rows, cols = C.c_int64(), C.c_int64()
    capi.check(capi.lib.dsinf_shard_tensor(C.byref(cfg), tp, rank, layer, tensor, seed, None, 0, C.byref(rows),
                                           C.byref(cols)))
    out = np.zeros(rows.value * cols.value, dtype=np.float32)
    capi.check(capi.lib.dsinf_shard_tensor(C.byref(cfg), tp, rank, layer, tensor, seed,
                                           out.ctypes.data_as(C.POINTER(C.c_float)), out.size, None, None))
    return out.reshape(rows.value, cols.value)


def synthetic_tensor(seed: int, layer: int, tensor: int, rows: int, cols: int) -> np.ndarray:
    out = np.zeros(rows * cols, dtype=np.float32)
    capi.check(capi.lib.dsinf_synthetic_tensor(seed, layer, tensor, rows, cols,
                                               out.ctypes.data_as(C.POINTER(C.c_float))))
    return out.reshape(rows, cols)
