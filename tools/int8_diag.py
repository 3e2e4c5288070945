#!/usr/bin/env python3
"""INT8 parity diagnosis at full width: per-position max|dlogit| / tol of the GPU decode against the
step oracle (or_model_step) for W8A8 and W8A16, token-by-token and after the tcgen05 prefill.

  python tools/int8_diag.py [hidden heads layers prompt]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
L = int(sys.argv[3]) if len(sys.argv) > 3 else 1
P = int(sys.argv[4]) if len(sys.argv) > 4 else 8
V, GEN, SEED = 50257, 3, 20220701
prompt = np.random.default_rng(1).integers(0, V, (1, P)).astype(np.int32)


def run(mode, prefill, dtype_bytes=1):
    m = DecoderModel(h, L, H, V, dtype_bytes=dtype_bytes, batch=1, max_ctx=P + GEN + 4, seed=SEED, int8_act=mode)
    ora = O.OracleModel(h, L, H, V, dtype_bytes=dtype_bytes, batch=1, max_ctx=P + GEN + 4, seed=SEED,
                        int8_act=mode)
    m.set_prompt(prompt)
    rows = []
    if prefill:
        m.prefill()
        torch.cuda.synchronize()
        glog = [m.full_logits().copy()]
        for _ in range(GEN - 1):
            m.step(1)
            torch.cuda.synchronize()
            glog.append(m.full_logits().copy())
        _, hist = m.read_tokens()
        # the oracle steps through the prompt in the prefill's mode (W8A8 rows), then decodes in `mode`
        ora.set_int8_act(0)
        for pos in range(P - 1):
            ora.step(hist[:, pos], pos)
        for k in range(GEN):
            if k == 1:
                ora.set_int8_act(mode)
            ol, _ = ora.step(hist[:, P - 1 + k], P - 1 + k)
            tol = 0.06 * float(ol.std()) + 0.02
            rows.append((P - 1 + k, float(np.abs(glog[k] - ol).max()), tol))
    else:
        for pos in range(P + GEN - 1):
            m.step(1)
            torch.cuda.synchronize()
            lg = m.full_logits().copy()
            _, hist = m.read_tokens()
            ol, _ = ora.step(hist[:, pos], pos)
            tol = (0.06 if dtype_bytes == 1 else 0.03) * float(ol.std()) + (0.02 if dtype_bytes == 1 else 0.01)
            rows.append((pos, float(np.abs(lg - ol).max()), tol))
    m.close()
    ora.close()
    return rows


for name, mode, pre, dt in [("fp16 token", 0, False, 2), ("w8a8 token", capi.INT8_W8A8, False, 1),
                            ("w8a16 token", capi.INT8_W8A16, False, 1), ("w8a8 prefill", capi.INT8_W8A8, True, 1),
                            ("w8a16 prefill", capi.INT8_W8A16, True, 1)]:
    r = run(mode, pre, dt)
    print(f"h={h} L={L} {name:14s} " + " ".join(f"{p}:{e / t:.2f}" for p, e, t in r), flush=True)
