"""One prefill inside cudaProfilerStart/Stop (for ncu --profile-from-start off).
python tools/prof_prefill.py [cfg] [fp16|int8] [B] [P]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200.engine import DecoderModel
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
dt = sys.argv[2] if len(sys.argv) > 2 else "fp16"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 16
P = int(sys.argv[4]) if len(sys.argv) > 4 else 128
p = PRESETS[cfg]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=P + 8)
prompt = np.random.default_rng(0).integers(0, p.vocab, (B, P)).astype(np.int32)
m.set_prompt(prompt)
m.prefill()
m.set_prompt(prompt)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.prefill()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
