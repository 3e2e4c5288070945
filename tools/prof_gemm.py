"""Run one SBI-GeMM shape a few times (for ncu captures):  python tools/prof_gemm.py N K B [fp16|int8] [ksplit]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2207_00032_b200 import engine as E  # noqa: E402

N, K, B = (int(v) for v in sys.argv[1:4])
dt = sys.argv[4] if len(sys.argv) > 4 else "fp16"
ks = int(sys.argv[5]) if len(sys.argv) > 5 else 0
iters = int(os.environ.get("ITERS", "6"))
w = (torch.randn(N, K, device="cuda") * 0.02).half()
if dt == "int8":
    wq, ws = E.quantize_weights_int8(w)
else:
    wq, ws = E.pack_weights_device(w, 2), None
x = torch.randn(B, K, device="cuda").half()
out = torch.empty(B, N, device="cuda")
for _ in range(iters):
    E.gemm(wq, x, N, K, w_scales=ws, out=out, ksplit=ks)
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(20):
    E.gemm(wq, x, N, K, w_scales=ws, out=out, ksplit=ks)
en.record()
en.synchronize()
ms = st.elapsed_time(en) / 20
print(f"N={N} K={K} B={B} {dt}: {ms*1e3:.1f} us  {N*K*(1 if dt=='int8' else 2)/ms/1e6:.1f} GB/s  plan={E.launch_plan(N,K,B,dt=='int8').__dict__ if hasattr(E.launch_plan(N,K,B),'__dict__') else ''}")
p = E.launch_plan(N, K, B, dt == "int8")
print("plan", p.col_tile, p.ksplit, p.rows_per_split, p.ctas, p.stages)
