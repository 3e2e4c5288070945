"""Profile one decode step of a preset (for `ncu --profile-from-start off`).

python tools/prof_step.py [config] [fp16|int8] [batch] [graph 0/1]
Prefills a 128-token prompt, then wraps ONE decode step in cudaProfilerStart/Stop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200.engine import PRESETS, DecoderModel  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
dt = sys.argv[2] if len(sys.argv) > 2 else "fp16"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
graph = bool(int(sys.argv[4])) if len(sys.argv) > 4 else False
steps = int(os.environ.get("PROF_STEPS", "1"))
p = PRESETS[cfg]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=batch,
                 max_ctx=160, use_cuda_graph=graph, use_pdl=True)
prompt = np.random.default_rng(0).integers(0, p.vocab, (batch, 128)).astype(np.int32)
m.set_prompt(prompt)
m.step(128)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.step(steps)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("kernels per step", m.get_info().kernels_per_step)
