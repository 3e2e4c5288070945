"""Tensor-parallel decode with every shard on ONE GPU (DSINF_TP_LOCAL): shards run one after the
other, so step_time / t is the per-rank compute time of a t-way TP step (no NVLink time).
python tools/tp_local_bench.py [cfg] [fp16|int8] [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
dt = sys.argv[2] if len(sys.argv) > 2 else "fp16"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = PRESETS[cfg]
for t in (1, 2, 4, 8):
    if p.heads % t:
        continue
    m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=200,
                     tp_size=t, tp_mode=capi.TP_LOCAL if t > 1 else capi.TP_NONE)
    m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32))
    m.step(130)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    m.step(32)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 32
    print(f"{cfg} {dt} B={B} TP={t} (all shards on one GPU): {ms:.3f} ms/step, per-rank compute {ms / t:.3f} ms")
    m.close()
