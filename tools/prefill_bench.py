"""Prefill latency of a preset (tcgen05 large-batch path) vs the token-by-token decode prefill.
python tools/prefill_bench.py [cfg] [fp16|int8] [B] [P]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200.engine import DecoderModel
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
dt = sys.argv[2] if len(sys.argv) > 2 else "fp16"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
P = int(sys.argv[4]) if len(sys.argv) > 4 else 128
p = PRESETS[cfg]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=P + 8)
prompt = np.random.default_rng(0).integers(0, p.vocab, (B, P)).astype(np.int32)


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        m.set_prompt(prompt)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


m.set_prompt(prompt)
m.prefill()  # builds the row-major weights and buffers
t_pf = timed(m.prefill)
t_dec = timed(lambda: m.step(P), reps=2)
h, L = p.hidden, p.layers
flops = 2.0 * B * P * 12 * h * h * L + 2.0 * B * P * P * h * L  # GEMMs + causal attention (QK, PV halves)
print(f"{cfg} {dt} B={B} P={P}: prefill {t_pf:.2f} ms ({B * P / t_pf * 1e3:.0f} tok/s, "
      f"{flops / (t_pf * 1e-3) / 1e12:.0f} TFLOP/s)  vs token-by-token {t_dec:.2f} ms  -> {t_dec / t_pf:.1f}x")
