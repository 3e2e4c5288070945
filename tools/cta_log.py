"""Per-CTA timeline of one SBI-GeMM launch inside the decode step.
DSINF_CTA_LOG=<n> python tools/cta_log.py [cfg] [fp16|int8] [B]   (n = index of the GEMM launch in the step)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
dt = sys.argv[2] if len(sys.argv) > 2 else "fp16"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = PRESETS[cfg]
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=192)
m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32))
m.step(130)
buf = np.zeros(6 * 4096, dtype=np.uint64)
capi.check(capi.lib.dsinf_model_cta_log(m._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size))
a = buf.reshape(-1, 6).astype(np.float64)
a = a[a[:, 1] > 0]
t0 = a[:, 2].min()
rel = (a[:, 2] - t0) / 1e3
st = (a[:, 1] - t0) / 1e3
pro = (a[:, 3] - a[:, 2]) / 1e3
loop = (a[:, 4] - a[:, 3]) / 1e3
epi = (a[:, 5] - a[:, 4]) / 1e3
end = (a[:, 5] - t0) / 1e3
print(f"launch {os.environ.get('DSINF_CTA_LOG')}: {len(a)} CTAs on {len(set(a[:, 0]))} SMs")
q = lambda v: " ".join(f"{x:6.2f}" for x in np.percentile(v, [0, 10, 50, 90, 100]))  # noqa: E731
print("percentiles       p0     p10    p50    p90   p100  (us)")
print("start-rel   ", q(st))
print("release     ", q(rel))
print("prologue    ", q(pro))
print("loop        ", q(loop))
print("epilogue    ", q(epi))
print("end         ", q(end))
smc = np.bincount(a[:, 0].astype(int))
print("CTAs per SM histogram:", np.bincount(smc[smc > 0]))
slow = pro > np.percentile(pro, 90)
print("slow-prologue CTAs: start-rel mean", st[slow].mean(), "vs others", st[~slow].mean())
