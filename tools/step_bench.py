#!/usr/bin/env python3
"""Decode ms/token of the persistent step kernel against the per-kernel graph path (CUDA events,
prompt 128, ctx 128 -> 128 + steps), and the step kernel's greedy tokens against the per-kernel path.

  python tools/step_bench.py [config] [dtypes] [batches] [steps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
dtypes = (sys.argv[2] if len(sys.argv) > 2 else "fp16,int8").split(",")
batches = [int(b) for b in (sys.argv[3] if len(sys.argv) > 3 else "1,8,16").split(",")]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 32
p = PRESETS[cfg]
P = 128


def run(dt, B, sk):
    m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B,
                     max_ctx=P + steps + 16, use_step_kernel=sk, int8_act=capi.INT8_W8A16 if dt == "int8" else 0)
    m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, P)).astype(np.int32))
    m.prefill()
    m.step(4)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    m.step(steps, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    _, hist = m.read_tokens()
    byts = m.bytes_per_step(P + 4 + steps // 2)
    m.close()
    return ms, hist[:, P:P + 4 + steps].copy(), byts


for dt in dtypes:
    for B in batches:
        base, htb, byts = run(dt, B, False)
        try:
            mine, hts, _ = run(dt, B, True)
        except Exception as ex:  # noqa: BLE001
            print(f"{cfg} {dt} B={B}: per-kernel {base:.3f} ms; step kernel failed: {ex}", flush=True)
            continue
        same = float(np.mean(htb == hts))
        print(f"{cfg} {dt} B={B}: per-kernel {base:.3f} ms ({byts / base / 1e6:.0f} GB/s), step kernel {mine:.3f} ms "
              f"({byts / mine / 1e6:.0f} GB/s), tokens equal {same:.3f}", flush=True)
