"""In-situ timeline of the per-kernel decode step (CUDA graph as the bench runs it).

python tools/launch_trace.py [cfg] [fp16|int8] [B] [--pdl-off]

Every launch records its first-CTA start and last-CTA end (globaltimer); printed per launch kind:
mean duration, mean gap from the previous launch's end to this launch's first CTA, and the
step total.  Averaged over several decode steps (one step's trace is read after each)."""
import ctypes as C
import os
import sys

os.environ.setdefault("DSINF_LAUNCH_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import PRESETS, DecoderModel  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = args[0] if len(args) > 0 else "gptj-6b"
dt = args[1] if len(args) > 1 else "fp16"
B = int(args[2]) if len(args) > 2 else 1
p = PRESETS[cfg]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=192,
                 use_pdl="--pdl-off" not in sys.argv)
m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32))
m.step(128)
torch.cuda.synchronize()
L = p.layers
names = ["embed"] + [k for _ in range(L) for k in ("qkv", "attn", "o", "up", "down")] + ["lm", "argmax"]
durs, gaps, totals = {}, {}, []
for it in range(8):
    m.step(1)
    torch.cuda.synchronize()
    n = C.c_int64()
    capi.check(capi.lib.dsinf_model_launch_trace(m._h, None, 0, C.byref(n)))
    buf = np.zeros(2 * n.value, dtype=np.uint64)
    capi.check(capi.lib.dsinf_model_launch_trace(m._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size, None))
    t = buf.reshape(-1, 2).astype(np.float64) / 1e3
    assert len(t) == len(names), (len(t), len(names))
    totals.append(t[-1, 1] - t[0, 0])
    for i, k in enumerate(names):
        durs.setdefault(k, []).append(t[i, 1] - t[i, 0])
        if i > 0:
            gaps.setdefault(k, []).append(t[i, 0] - t[i - 1, 1])
print(f"{cfg} {dt} B={B}: step (first CTA -> last CTA) {np.median(totals):.1f} us")
tot_d = sum(np.sum(v) / 8 for v in durs.values())
for k in ["embed", "qkv", "attn", "o", "up", "down", "lm", "argmax"]:
    d = np.array(durs[k])
    g = np.array(gaps.get(k, [0.0]))
    cnt = len(d) // 8
    print(f"{k:7s} x{cnt:3d}  dur {d.mean():7.2f} us (min {d.min():6.2f})  gap-before {g.mean():6.2f} us  "
          f"share {100 * d.sum() / 8 / tot_d:5.1f}%")
g_all = sum(np.sum(v) / 8 for v in gaps.values())
print(f"sum of durations {tot_d:.1f} us, sum of gaps {g_all:.1f} us")
