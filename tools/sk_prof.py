"""A few decode steps of GPT-J through the persistent step kernel (for ncu): python tools/sk_prof.py [fp16|int8] [B]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "int8"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m = DecoderModel(4096, 32, 32, 50257, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=160, use_step_kernel=True,
                 int8_act=capi.INT8_W8A16 if dt == "int8" else 0)
m.set_prompt(np.random.default_rng(0).integers(0, 50257, (B, 128)).astype(np.int32))
m.step(136)
torch.cuda.synchronize()
m.close()
