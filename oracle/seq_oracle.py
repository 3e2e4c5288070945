"""Teacher-forced sequence oracle: the CPU decoder of oracle.c (or_model_step) restated over whole
token sequences with numpy fp64 GEMMs, for parity at the BASELINE configs' full sizes.

TEST INFRASTRUCTURE ONLY -- imported by tests/ and tools/parity_baseline.py as the checker, never by
the product package.

Why a second restatement: or_model_step (oracle.c) runs one position at a time with the
exec_reference-order GEMM (gemm.hpp:147-202); a GPT-J-6B decode of a 128-token prompt plus 8 tokens
is ~10^12 MACs per sequence that way.  Here every position of every sequence goes through a layer at
once (causal attention), with the GEMMs as fp64 BLAS matrix products.  Given the tokens the GPU fed
itself (its prompt plus its own greedy tokens), the logits at each position depend only on the
tokens up to it, so one pass yields the logits the token-by-token decode would see at every step.

Numerics follow or_model_step line by line (oracle.c: LayerNorm in fp64 with the fp16 storage
point, the exec_reference fp64 GEMM -- here BLAS order, a difference at the 1e-16 relative level --,
the fp16-path epilogues in fp64, the int8-path epilogues in fp32 in the device's order, fp64
softmax attention, tanh GeLU, the TP partials summed in rank order in fp32, per-rank activation
quantisation for the row-parallel W8A8 GEMMs).  INT8 activation modes are per GEMM and per row
group: the prompt rows use `prefill_mode` (the tcgen05 prefill runs W8A8), the generated rows
`decode_mode` -- each 0 = W8A8, 1 = W8A16, or 0x100 | mask (bit g set = GEMM g W8A16; 0 QKV,
1 attn-out, 2 MLP-up, 3 MLP-down), as or_config.int8_act.

Pinned by tests/test_oracle_numerics.py::test_seq_oracle_matches_step_oracle against or_model_step.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import oracle as O

T_QKV, T_QKV_B, T_O, T_O_B, T_UP, T_UP_B, T_DOWN, T_DOWN_B = 1, 2, 3, 4, 5, 6, 7, 8
T_LN1_G, T_LN1_B, T_LN2_G, T_LN2_B, T_WTE, T_LNF_G, T_LNF_B = 9, 10, 11, 12, 13, 14, 15
FP = C.POINTER(C.c_float)


def f16r(x):
    """fp32 -> fp16 (round to nearest even) -> fp32: the GPU's fp16 storage point."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def _matrix(seed, layer, tensor, rows, cols, valid=None):
    out = np.empty((rows, cols), dtype=np.float32)
    O.oracle_lib().or_synth_matrix(seed, layer, tensor, rows, cols, rows if valid is None else valid,
                                   out.ctypes.data_as(FP))
    return out


def _vector(seed, layer, tensor, n):
    out = np.empty(n, dtype=np.float32)
    O.oracle_lib().or_synth_vector(seed, layer, tensor, n, out.ctypes.data_as(FP))
    return out


def _quant_rows(x):
    """or_quant_rows: per-row scale max|x| / 127 (fp32 divide; 1 for an all-zero row),
    q = clamp(rint(x / s), -127, 127) with an fp32 divide.  Large matrices (weights) go through
    the C function itself (OpenMP); activations through this numpy image of it."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.size > (1 << 22):
        return O.quant_rows(x)
    mx = np.abs(x).max(axis=1)
    s = np.where(mx > 0, mx / np.float32(127.0), np.float32(1.0)).astype(np.float32)
    q = np.clip(np.rint(x / s[:, None]), -127, 127).astype(np.int8)
    return q, s


def _layernorm(v, g, b, eps):
    """layernorm_row (oracle.c): fp64 statistics over fp32 rows, fp32 then fp16 output."""
    v64 = v.astype(np.float64)
    mean = v64.mean(axis=1, keepdims=True)
    var = ((v64 - mean) ** 2).mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + float(np.float32(eps)))
    return f16r(((v64 - mean) * rstd * g.astype(np.float64) + b.astype(np.float64)).astype(np.float32))


def _gelu(x):
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


class SeqOracle:
    """Teacher-forced decoder over whole sequences.  `forward` returns the logits (fp32) at the
    requested positions of every sequence; weights are regenerated per layer (nothing kept)."""

    def __init__(self, hidden, layers, heads, vocab=50257, *, dtype_bytes=2, tp=1, seed=20220701, ln_eps=1e-5,
                 rope_base=10000.0, acc="f64"):
        self.h, self.L, self.H, self.V = hidden, layers, heads, vocab
        self.d = hidden // heads
        self.t = tp
        self.Hl = heads // tp
        self.F = 4 * hidden
        self.Fl = self.F // tp
        self.i8 = dtype_bytes == 1
        self.seed = seed
        self.eps = ln_eps
        self.rope_base = rope_base
        # acc="f32": the same algorithm with fp32 GEMM and attention accumulation (the device's
        # accumulation width) -- a second correct implementation whose distance from the fp64 one
        # measures the intrinsic noise floor of the INT8 W8A8 activation quantisation (parity_baseline)
        assert acc in ("f64", "f32")
        self.ft = np.float64 if acc == "f64" else np.float32
        vq = 128 * tp
        self.Vpad = (vocab + vq - 1) // vq * vq

    # rotary table: the same expression as oracle.c / the device runtime's host-side table
    def _rope(self, n):
        d = self.d
        inv = np.array([math.pow(float(self.rope_base), -2.0 * k / d) for k in range(d // 2)])
        ang = np.arange(n, dtype=np.float64)[:, None] * inv[None, :]
        return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)

    # ---- GEMMs: out[M][N] for x[M][K] over the full (global) weight; K sliced per rank when row-parallel
    def _gemm16(self, x16, W):
        return (x16.astype(self.ft) @ W.astype(self.ft).T).astype(np.float64)

    def _gemm8(self, mode, x16, Wq, ws):
        """gemm8 (oracle.c): W8A16 y = fp32(sum q x) * s_w; W8A8 per-token int8 x, exact int32,
        y = fp32(fp32(acc) * s_x) * s_w."""
        if mode == 1:
            a = x16.astype(self.ft) @ Wq.astype(self.ft).T
            return a.astype(np.float32) * ws[None, :]
        xq, xs = _quant_rows(x16)
        acc = xq.astype(np.float64) @ Wq.astype(np.float64).T  # exact integers (< 2^53)
        t = acc.astype(np.int32).astype(np.float32) * xs[:, None]
        return t * ws[None, :]

    def _act(self, mode, g):
        return (mode >> g) & 1 if mode & 0x100 else mode

    def _col_gemm(self, x16, W, Wq, ws, modes, groups, g):
        """Column-parallel GEMM (QKV, MLP-up): no reduction, every rank sees the whole x."""
        if not self.i8:
            return self._gemm16(x16, W), None
        y = np.empty((x16.shape[0], Wq.shape[0]), dtype=np.float32)
        for rows, mode in zip(groups, modes):
            if rows.stop > rows.start:
                y[rows] = self._gemm8(self._act(mode, g), x16[rows], Wq, ws)
        return None, y

    def _row_gemm(self, x16, W, Wq, ws, modes, groups, g, kl):
        """Row-parallel GEMM (attn-out, MLP-down): per-rank K slice, fp32 partial per rank (fp16 path:
        fp32(fp64 sum)), partials added in rank order in fp32."""
        tot = None
        for rk in range(self.t):
            sl = slice(rk * kl, (rk + 1) * kl)
            if not self.i8:
                yf = self._gemm16(x16[:, sl], W[:, sl]).astype(np.float32)
            else:
                yf = np.empty((x16.shape[0], Wq.shape[0]), dtype=np.float32)
                for rows, mode in zip(groups, modes):
                    if rows.stop > rows.start:
                        yf[rows] = self._gemm8(self._act(mode, g), x16[rows, sl], Wq[:, sl], ws)
            tot = yf if tot is None else (tot + yf).astype(np.float32)
        return tot

    def forward(self, tokens, positions, *, prompt_len=None, prefill_mode=0, decode_mode=0, log=None):
        """tokens: int [S][T] (prompt + the tokens fed back); positions: list of positions p whose
        logits [S][len(positions)][V] are returned (p < T).  Rows t < prompt_len use `prefill_mode`,
        the others `decode_mode` (int8 only)."""
        tokens = np.asarray(tokens, dtype=np.int64)
        S, T = tokens.shape
        h, d, Hl, H = self.h, self.d, self.Hl, self.H
        P = T if prompt_len is None else min(prompt_len, T)
        M = S * T
        seed = self.seed
        # row groups of the flattened [S*T] rows by int8 activation mode
        tpos = np.tile(np.arange(T), S)
        order = np.argsort(tpos >= P, kind="stable")  # prompt rows first, then generated rows
        inv = np.empty_like(order)
        inv[order] = np.arange(M)
        n_prompt = int((tpos < P).sum())
        groups = (slice(0, n_prompt), slice(n_prompt, M))
        modes = (prefill_mode, decode_mode)
        tok = tokens.reshape(-1)[order]
        pos = tpos[order]
        seq = np.repeat(np.arange(S), T)[order]
        cos, sin = self._rope(T)
        c = cos[pos]  # [M][d/2]
        s = sin[pos]
        wte = _matrix(seed, -1, T_WTE, self.V, h)
        r = wte[tok].astype(np.float32)  # residual [M][h] fp32
        dsum = None
        for l in range(self.L):
            if log:
                log(f"layer {l}")
            bqkv = _vector(seed, l, T_QKV_B, 3 * h)
            bo = _vector(seed, l, T_O_B, h)
            bup = _vector(seed, l, T_UP_B, self.F)
            bdown_prev = _vector(seed, l - 1, T_DOWN_B, h) if l > 0 else None
            if l > 0:
                r = (r + (dsum + bdown_prev).astype(np.float32)).astype(np.float32)
            xln = _layernorm(r, _vector(seed, l, T_LN1_G, h), _vector(seed, l, T_LN1_B, h), self.eps)
            # ---- QKV + bias + RoPE (columns: [q | k | v], each h = H x d, global head order)
            Wqkv = _matrix(seed, l, T_QKV, 3 * h, h)
            Wq = ws = None
            if self.i8:
                Wq, ws = _quant_rows(Wqkv)
                Wqkv = None
            yd, yf = self._col_gemm(xln, Wqkv, Wq, ws, modes, groups, 0)
            del Wqkv, Wq
            if not self.i8:
                y = (yd + bqkv.astype(np.float64)[None, :]).reshape(M, 3, H, d // 2, 2)
                cc, ss = c.astype(np.float64)[:, None, None, :], s.astype(np.float64)[:, None, None, :]
                y0, y1 = y[:, :2, :, :, 0].copy(), y[:, :2, :, :, 1].copy()
                y[:, :2, :, :, 0] = y0 * cc - y1 * ss
                y[:, :2, :, :, 1] = y0 * ss + y1 * cc
                qkv = f16r(y.reshape(M, 3 * h).astype(np.float32))
            else:
                y = (yf + bqkv[None, :]).astype(np.float32).reshape(M, 3, H, d // 2, 2)
                cc, ss = c[:, None, None, :], s[:, None, None, :]
                y0, y1 = y[:, :2, :, :, 0].copy(), y[:, :2, :, :, 1].copy()
                p0, p1, p2, p3 = y0 * cc, y1 * ss, y0 * ss, y1 * cc
                y[:, :2, :, :, 0] = p0 - p1
                y[:, :2, :, :, 1] = p2 + p3
                qkv = f16r(y.reshape(M, 3 * h))
            del yd, yf, y
            # ---- causal attention per (sequence, head), fp64 softmax, fp16 output
            q = qkv[:, :h].reshape(M, H, d)
            k = qkv[:, h:2 * h].reshape(M, H, d)
            v = qkv[:, 2 * h:].reshape(M, H, d)
            a16 = np.empty((M, h), dtype=np.float32)
            scale = 1.0 / math.sqrt(d)
            for sq in range(S):
                rows = inv[sq * T:(sq + 1) * T]  # flattened rows of this sequence in position order
                qs = q[rows].astype(self.ft).transpose(1, 0, 2)  # [H][T][d]
                ks = k[rows].astype(self.ft).transpose(1, 0, 2)
                vs = v[rows].astype(self.ft).transpose(1, 0, 2)
                sc = (qs @ ks.transpose(0, 2, 1)) * scale  # [H][T][T]
                mask = np.triu(np.ones((T, T), dtype=bool), 1)
                sc[:, mask] = -np.inf
                sc -= sc.max(axis=2, keepdims=True)
                p = np.exp(sc)
                o = (p @ vs) / p.sum(axis=2, keepdims=True)  # [H][T][d]
                a16[rows] = f16r(o.transpose(1, 0, 2).reshape(T, h).astype(np.float32))
            del q, k, v, qkv
            # ---- attn-out (row parallel) + bias + residual
            Wo = _matrix(seed, l, T_O, h, h)
            Woq = wos = None
            if self.i8:
                Woq, wos = _quant_rows(Wo)
                Wo = None
            da = self._row_gemm(a16, Wo, Woq, wos, modes, groups, 1, Hl * d)
            del Wo, Woq
            r = (r + (da + bo).astype(np.float32)).astype(np.float32)
            xln = _layernorm(r, _vector(seed, l, T_LN2_G, h), _vector(seed, l, T_LN2_B, h), self.eps)
            # ---- MLP-up + bias + GeLU (column parallel)
            Wu = _matrix(seed, l, T_UP, self.F, h)
            Wuq = wus = None
            if self.i8:
                Wuq, wus = _quant_rows(Wu)
                Wu = None
            yd, yf = self._col_gemm(xln, Wu, Wuq, wus, modes, groups, 2)
            del Wu, Wuq
            if not self.i8:
                u16 = f16r(_gelu(yd + bup.astype(np.float64)[None, :]).astype(np.float32))
            else:
                u16 = f16r(_gelu((yf + bup[None, :]).astype(np.float32).astype(np.float64)).astype(np.float32))
            del yd, yf
            # ---- MLP-down (row parallel)
            Wd = _matrix(seed, l, T_DOWN, h, self.F)
            Wdq = wds = None
            if self.i8:
                Wdq, wds = _quant_rows(Wd)
                Wd = None
            dsum = self._row_gemm(u16, Wd, Wdq, wds, modes, groups, 3, self.Fl)
            del Wd, Wdq, u16
        # ---- final residual, LayerNorm, LM head (fp16 weights in both modes; vocab rows padded)
        sel = np.array([inv[sq * T + p] for sq in range(S) for p in positions], dtype=np.int64)
        rr = r[sel]
        if self.L > 0:
            rr = (rr + (dsum[sel] + _vector(seed, self.L - 1, T_DOWN_B, h)).astype(np.float32)).astype(np.float32)
        xf = _layernorm(rr, _vector(seed, -1, T_LNF_G, h), _vector(seed, -1, T_LNF_B, h), self.eps)
        logits = self._gemm16(xf, wte).astype(np.float32)
        return logits.reshape(S, len(positions), self.V)
