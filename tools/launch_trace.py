"""In-situ timeline of the per-kernel decode step (CUDA graph as the bench runs it).

python tools/launch_trace.py [cfg] [fp16|int8] [B] [--pdl-off]

Every launch records its first-CTA start and last-CTA end (globaltimer); printed per launch kind:
mean duration, mean gap from the previous launch's end to this launch's first CTA, and the
step total.  Averaged over 8 decode steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = args[0] if len(args) > 0 else "gptj-6b"
dt = args[1] if len(args) > 1 else "fp16"
B = int(args[2]) if len(args) > 2 else 1
p = PRESETS[cfg]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=192,
                 use_pdl="--pdl-off" not in sys.argv)
m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32))
m.step(128)
tr = m.launch_trace(8).astype(np.float64)  # [steps][n][3]
kinds = tr[0, :, 2].astype(int)
dur = (tr[:, :, 1] - tr[:, :, 0]) / 1e3
gap = np.zeros_like(dur)
gap[:, 1:] = (tr[:, 1:, 0] - tr[:, :-1, 1]) / 1e3
span = np.median((tr[:, -1, 1] - tr[:, 0, 0]) / 1e3)
print(f"{cfg} {dt} B={B}: step (first CTA -> last CTA) {span:.1f} us, {len(kinds)} launches")
tot = dur.sum() / len(tr)
for k in sorted(set(kinds)):
    sel = kinds == k
    d, g = dur[:, sel], gap[:, sel]
    print(f"{capi.LK_NAMES[k]:9s} x{sel.sum():3d}  dur {d.mean():7.2f} us (min {d.min():6.2f})  gap-before {g.mean():6.2f} us"
          f"  share {100 * d.sum() / len(tr) / tot:5.1f}%")
print(f"sum of durations {tot:.1f} us, sum of gaps {gap.sum() / len(tr):.1f} us")
