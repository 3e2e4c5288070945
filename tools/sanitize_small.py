"""Small end-to-end workload for compute-sanitizer: decode (graph off), prefill, int8 and TP-local."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200 import engine as E  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402

rng = np.random.default_rng(0)
for dt, B, tp in [(2, 1, 1), (1, 3, 1), (2, 5, 1), (1, 8, 1), (2, 2, 2)]:
    m = DecoderModel(256, 2, 4, 1000, dtype_bytes=dt, batch=B, max_ctx=24, use_cuda_graph=False,
                     tp_size=tp, tp_mode=capi.TP_LOCAL if tp > 1 else capi.TP_NONE)
    m.set_prompt(rng.integers(0, 1000, (B, 9)).astype(np.int32))
    m.prefill()
    m.step(3)
    m.set_prompt(rng.integers(0, 1000, (B, 5)).astype(np.int32))
    m.step(7)
    torch.cuda.synchronize()
    m.close()
# round-2 paths: full 32-position attention stages (one context chunk per (row, head)), the QKV
# attention tail, the tensor-core attention stage, INT8 K-group W8A16 and INT8 AUTO at B = 16
for env, kw in [({"DSINF_ATTN_CTAS": "1"}, dict(dtype_bytes=2, batch=2)),
                ({"DSINF_ATTN_FUSE": "1"}, dict(dtype_bytes=2, batch=1)),
                ({"DSINF_ATTN_FUSE": "1"}, dict(dtype_bytes=1, batch=2, int8_act=capi.INT8_W8A16)),
                ({"DSINF_ATTN_MMA": "1", "DSINF_ATTN_CTAS": "1"}, dict(dtype_bytes=2, batch=2)),
                ({}, dict(dtype_bytes=1, batch=1, int8_act=capi.INT8_W8A16, int8_group=128)),
                ({}, dict(dtype_bytes=1, batch=16, int8_act=capi.INT8_AUTO))]:
    os.environ.update(env)
    m = DecoderModel(512, 2, 4, 1000, max_ctx=80, use_cuda_graph=False, **kw)
    m.set_prompt(rng.integers(0, 1000, (kw["batch"], 40)).astype(np.int32))
    m.step(44)
    torch.cuda.synchronize()
    m.close()
    for k in env:
        del os.environ[k]
dev = torch.device("cuda")
w = (torch.randn(640, 320, device=dev) * 0.05).half()
x = torch.randn(3, 320, device=dev).half()
wp = E.pack_weights_device(w, 2)
E.gemm(wp, x, 640, 320)
wq, ws = E.quantize_weights_int8(w)
E.gemm(wq, x, 640, 320, w_scales=ws)
E.gemm(wq, x, 640, 320, w_scales=ws, a16=True)
E.gemm_large_batch(w, torch.randn(130, 320, device=dev).half())
E.gemm_large_batch(torch.randn(512, 2048, device=dev).half(), torch.randn(64, 2048, device=dev).half())
torch.cuda.synchronize()
print("sanitize workload ok")
