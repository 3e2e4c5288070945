"""Per-CTA phase statistics of the persistent step kernel (DSINF_STEP_TRACE):
  python tools/step_trace2.py [cfg] [fp16|int8] [B]
Per phase kind, over layers 2..L-1 and CTAs: percentiles of the dependency wait (slot 1 - slot 0),
the consumer work after the dependency (slot 2 - slot 1), and per phase the span from the earliest
dependency release to the last tile publication; plus the gap between consecutive phases."""
import ctypes as C
import os
import sys

os.environ.setdefault("DSINF_STEP_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
dt = sys.argv[2] if len(sys.argv) > 2 else "int8"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = PRESETS[cfg]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=160,
                 use_step_kernel=True, int8_act=capi.INT8_W8A16 if dt == "int8" else 0)
m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32))
m.step(129)
torch.cuda.synchronize()
need, grid, ph = C.c_int64(), C.c_int32(), C.c_int32()
capi.check(capi.lib.dsinf_model_step_trace(m._h, None, 0, C.byref(need), C.byref(grid), C.byref(ph)))
m.step(1)  # the traced step: stamps are overwritten every step, read right after one
torch.cuda.synchronize()
buf = np.zeros(need.value, dtype=np.uint64)
capi.check(capi.lib.dsinf_model_step_trace(m._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size, None, None, None))
t = buf.reshape(grid.value, ph.value, 8).astype(np.float64)
step_start = np.min(t[:, 0, 7])  # every CTA stamps its start in (phase 0, slot 7)
valid = t >= step_start
t = np.where(valid, (t - step_start) / 1e3, np.nan)
names = ["embed"] + [n for _ in range(p.layers) for n in ("qkv", "attn", "o", "up", "down")] + ["lm"]
print(f"grid {grid.value} phases {ph.value}; step span {np.nanmax(t):.1f} us; {np.nanmax(t) / p.layers:.1f} us/layer")


def pct(a):
    a = a[~np.isnan(a)]
    if a.size == 0:
        return "   -      -      -"
    return f"{np.percentile(a, 50):6.2f} {np.percentile(a, 90):6.2f} {np.max(a):6.2f}"


print("kind   dep-wait p50/p90/max     work p50/p90/max      x-build p50/p90/max   release->published   prev-published->release")
for kind in ("qkv", "attn", "o", "up", "down", "lm"):
    idx = [i for i in range(1, ph.value) if names[i] == kind]
    if kind != "lm":
        idx = idx[2:-1] if len(idx) > 4 else idx
    w, k, xb, spans, gaps = [], [], [], [], []
    for i in idx:
        c = t[:, i, :]
        w.append(c[:, 1] - c[:, 0])
        k.append(c[:, 2] - c[:, 1])
        xb.append(c[:, 5] - c[:, 1])
        pub = np.nanmax(c[:, 6]) if kind != "attn" else np.nanmax(c[:, 2])
        spans.append(pub - np.nanmin(c[:, 1]))
        prev = t[:, i - 1, :]
        ppub = np.nanmax(prev[:, 6]) if names[i - 1] != "attn" else np.nanmax(prev[:, 2])
        gaps.append(np.nanmin(c[:, 1]) - ppub)
    print(f"{kind:5s} {pct(np.concatenate(w))}   {pct(np.concatenate(k))}   {pct(np.concatenate(xb))}   {np.nanmean(spans):8.2f}   {np.nanmean(gaps):8.2f}")
print("layer 3 timeline (us): phase  first-release  last-consumer-end  last-publish  producer-issued(max)")
for i in range(1 + 5 * 3, 1 + 5 * 4):
    c = t[:, i, :]
    print(f"  {names[i]:5s} {np.nanmin(c[:, 1]):9.2f} {np.nanmax(c[:, 2]):9.2f} {np.nanmax(c[:, 6]):9.2f} {np.nanmax(c[:, 3]):9.2f}")
m.close()
