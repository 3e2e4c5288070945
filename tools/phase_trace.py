"""Per-phase timeline of the SBI-GeMM launches inside the decode step (CUDA graph as the bench
runs it): for each launch kind, the mean of
  wait     previous launch's last CTA end -> this launch's dependency release
  pro      dependency release -> last CTA's prologue end
  loop     last prologue end -> last main-loop end
  epi      last main-loop end -> last CTA end
python tools/phase_trace.py [cfg] [fp16|int8|w8a16] [B] [--slice]"""
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
sl = dict(tp_size=p.tp, tp_rank=0, tp_mode=capi.TP_SLICE) if "--slice" in sys.argv else {}  # rank 0 of a TP config
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt in ("int8", "w8a16") else 2, batch=B, max_ctx=192,
                 int8_act=1 if dt == "w8a16" else 0, **sl)
m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32))
m.step(128)
tr = m.launch_trace(8).astype(np.float64)  # [steps][n][6]
kinds = tr[0, :, 2].astype(int)
span = np.median((tr[:, -1, 1] - tr[:, 0, 0]) / 1e3)
print(f"{cfg} {dt} B={B}: step {span:.1f} us, {len(kinds)} launches")
prev_end = np.zeros_like(tr[:, :, 1])
prev_end[:, 1:] = tr[:, :-1, 1]
for k in sorted(set(kinds)):
    sel = kinds == k
    t = tr[:, sel, :]
    st, en, rel, pro, loop, cpro, lrel, s1, s2, s3 = (t[..., i] for i in (0, 1, 3, 4, 5, 6, 7, 8, 9, 10))
    pe = prev_end[:, sel]
    if rel.max() > 1e19 or pro.min() == 0:  # not an SBI-GeMM launch
        d = (en - st) / 1e3
        g = (st - pe) / 1e3
        print(f"{capi.LK_NAMES[k]:9s} x{sel.sum():3d}  dur {d.mean():6.2f}  start-after-prev-end {g.mean():6.2f} us")
        continue
    f = lambda a: f"{a.mean():6.2f}"  # noqa: E731
    print(f"{capi.LK_NAMES[k]:9s} x{sel.sum():3d}  wait {f((rel - pe) / 1e3)}  pro {f((pro - rel) / 1e3)}  "
          f"loop {f((loop - pro) / 1e3)}  epi {f((en - loop) / 1e3)}  early-start {f((rel - st) / 1e3)} us"
          f"  | cta-pro-max {f(cpro / 1e3)}  release-spread {f((lrel - rel) / 1e3)}"
          f"  | sub(kcyc) {f(s1 / 1e3)} {f(s2 / 1e3)} {f(s3 / 1e3)}")
