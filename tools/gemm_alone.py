#!/usr/bin/env python3
"""Drop-in dsinf_gemm timed alone (CUDA events; 4 rotating weight copies > L2) for one shape:
  python tools/gemm_alone.py N K B {fp16|w8a8|w8a16|w8a16g} [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_00032_b200 import engine as E  # noqa: E402

N, K, B = (int(v) for v in sys.argv[1:4])
mode = sys.argv[4]
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 20
dev = torch.device("cuda")
copies = []
for c in range(4):
    w = (torch.randn(N, K, device=dev) * 0.02).half()
    if mode == "fp16":
        copies.append((E.pack_weights_device(w, 2), None, None))
    elif mode == "w8a16g":
        q, g = E.quantize_weights_int8_groups(w)
        copies.append((q, None, g))
    else:
        q, s = E.quantize_weights_int8(w)
        copies.append((q, s, None))
x = torch.randn(B, K, device=dev).half()
out = torch.empty(B, N, device=dev, dtype=torch.float32)
s = torch.cuda.current_stream()


def call(i):
    wq, ws, g = copies[i % 4]
    E.gemm(wq, x, N, K, w_scales=ws, out=out, a16=mode == "w8a16", w_group_scales=g, stream=s)


for i in range(3):
    call(i)
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
st.record(s)
for i in range(iters):
    call(i)
en.record(s)
en.synchronize()
us_host = st.elapsed_time(en) / iters * 1e3
g = torch.cuda.CUDAGraph()
gs = torch.cuda.Stream()
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=gs):
    s = gs
    for i in range(iters):
        call(i)
with torch.cuda.stream(gs):  # replay() launches on the current stream
    g.replay()
    torch.cuda.synchronize()
    st.record(gs)
    g.replay()
    en.record(gs)
en.synchronize()
us = st.elapsed_time(en) / iters * 1e3
byts = N * K * (2 if mode == "fp16" else 1) + B * K * 2 + B * N * 4
print(f"{mode} N={N} K={K} B={B}: graph {us:.2f} us/call, {byts / us / 1e3:.0f} GB/s (host-launched {us_host:.2f} us)")
