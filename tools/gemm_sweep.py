"""SBI-GeMM launch-plan sweep at the decode shapes, timed like the decode step runs them:
CUDA-graph replays of back-to-back launches, weights rotated over > 2x L2 so each launch
streams from HBM.  python tools/gemm_sweep.py [fp16|int8] [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2207_00032_b200 import engine as E  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "fp16"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
i8 = dt == "int8"
SHAPES = {"qkv": (12288, 4096), "o": (4096, 4096), "up": (16384, 4096), "down": (4096, 16384)}
stage_list = [int(s) for s in os.environ.get("SW_STAGES", "2,4,6").split(",")]
split_list = [int(s) for s in os.environ.get("SW_SPLITS", "0,1,2,4,8,16").split(",")]
only = os.environ.get("SW_ONLY")


def time_graph(fn, n=20, reps=3):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / n)
    return best


for name, (N, K) in SHAPES.items():
    if only and name not in only.split(","):
        continue
    wbytes = N * K * (1 if i8 else 2)
    copies = max(2, (400 << 20) // wbytes + 1)
    if i8:
        ws = [torch.randint(-127, 128, (N * ((K + 3) // 4) * 4,), dtype=torch.int8, device="cuda") for _ in range(copies)]
        sc = torch.rand(N, device="cuda") * 1e-3
    else:
        ws = [(torch.randn(N * ((K + 1) // 2) * 2, device="cuda") * 0.02).half() for _ in range(copies)]
        sc = None
    x = torch.randn(B, K, device="cuda").half()
    out = torch.empty(B, N, device="cuda")
    for st in stage_list:
        os.environ["DSINF_STAGES"] = str(st)
        for ks in split_list:
            try:
                p = E.launch_plan(N, K, B, i8) if ks == 0 else None
                us = time_graph(lambda i: E.gemm(ws[i % copies], x, N, K, w_scales=sc, out=out, ksplit=ks))
            except Exception as e:  # invalid split for this shape
                continue
            plan = E.launch_plan(N, K, B, i8)
            tag = f"auto({plan.ksplit})" if ks == 0 else str(ks)
            print(f"{name:5s} {dt} B={B} stages<={st} split={tag:8s} {us:7.2f} us {wbytes / us / 1e3:7.1f} GB/s", flush=True)
