"""Phase timeline of the persistent step kernel: python tools/step_trace.py [cfg] [fp16|int8] [B]

Per phase (first layer in detail, then averages per phase kind): when the consumers first passed
the dependency wait, when the last consumer finished its units, when the last unit was ticketed
by a sync warp, when the last tile epilogue was published, and when the producers moved on."""
import ctypes as C
import os
import sys

os.environ.setdefault("DSINF_STEP_TRACE", "1")
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
m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B, max_ctx=160,
                 use_step_kernel=True, int8_act=capi.INT8_W8A16 if dt == "int8" else 0)
m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32))
m.step(130)
torch.cuda.synchronize()
need, grid, ph = C.c_int64(), C.c_int32(), C.c_int32()
capi.check(capi.lib.dsinf_model_step_trace(m._h, None, 0, C.byref(need), C.byref(grid), C.byref(ph)))
buf = np.zeros(need.value, dtype=np.uint64)
capi.check(capi.lib.dsinf_model_step_trace(m._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size, None, None, None))
t = buf.reshape(grid.value, ph.value, 8).astype(np.float64)
valid = t > 0
t0 = t[valid].min()
t = np.where(valid, (t - t0) / 1e3, np.nan)  # us


def mx(a):
    return np.nanmax(a) if np.any(~np.isnan(a)) else np.nan


def mn(a):
    return np.nanmin(a) if np.any(~np.isnan(a)) else np.nan


names = ["embed"] + [n for _ in range(p.layers) for n in ("qkv", "attn", "o", "up", "down")] + ["lm"]
print(f"grid {grid.value}  phases {ph.value}  step span {mx(t[:, :, :]):.1f} us")
print("phase          start  cons_end  sync_unit  tile_fin   done_pub  prod_moved")
for i in list(range(1, 7)) + [ph.value - 1]:
    c = t[:, i, :]
    print(f"{i:3d} {names[i]:6s} {mn(c[:, 1]):9.2f} {mx(c[:, 2]):9.2f} {mx(c[:, 4]):9.2f} {mx(c[:, 5]):9.2f} "
          f"{mx(c[:, 6]):9.2f} {mx(c[:, 3]):9.2f}")
agg = {}
for i in range(1, ph.value):
    c = t[:, i, :]
    a = agg.setdefault(names[i], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += mx(c[:, 6]) - mn(c[:, 1]) if names[i] != "attn" else mx(c[:, 2]) - mn(c[:, 1])
    a[2] += mx(c[:, 6]) - mx(c[:, 2]) if names[i] != "attn" else 0.0
    a[3] += np.nanmean(c[:, 1] - c[:, 0])
for n, (k, span, lag, wait) in agg.items():
    print(f"{n:5s} x{k:3d}  start->done {span / k:7.2f} us  last-consumer->done {lag / k:6.2f} us  "
          f"mean dependency wait {wait / k:7.2f} us")
m.close()
