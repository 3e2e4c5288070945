"""Profile one decode step of a preset (for `ncu --profile-from-start off`).

python tools/prof_step.py [config] [fp16|int8] [batch] [graph 0/1]
Prefills a 128-token prompt, then wraps ONE decode step in cudaProfilerStart/Stop."""
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
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
graph = bool(int(sys.argv[4])) if len(sys.argv) > 4 else False
steps = int(os.environ.get("PROF_STEPS", "1"))
p = PRESETS[cfg]
# PROF_SLICE=1: rank 0's shard of the preset's TP config alone (DSINF_TP_SLICE); PROF_ACT: int8 mode
sl = dict(tp_size=p.tp, tp_rank=0, tp_mode=capi.TP_SLICE) if os.environ.get("PROF_SLICE") == "1" else {}
act = {"w8a8": capi.INT8_W8A8, "w8a16": capi.INT8_W8A16, "auto": capi.INT8_AUTO}[os.environ.get("PROF_ACT", "w8a8")]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=batch,
                 max_ctx=160, use_cuda_graph=graph, use_pdl=True, int8_act=act, **sl)
prompt = np.random.default_rng(0).integers(0, p.vocab, (batch, 128)).astype(np.int32)
m.set_prompt(prompt)
m.step(128)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.step(steps)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("kernels per step", m.get_info().kernels_per_step)
