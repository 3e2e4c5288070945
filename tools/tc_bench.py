"""Throughput of the tcgen05 large-batch GEMM at the prefill shapes (M = batch x prompt tokens).
python tools/tc_bench.py [fp16|int8] [M]   -- CUDA-graph replays, CUDA events, TFLOP/s (TOP/s)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2207_00032_b200 import engine as E  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "fp16"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
i8 = dt == "int8"
SHAPES = {"qkv": (12288, 4096), "attn_out": (4096, 4096), "mlp_up": (16384, 4096), "mlp_down": (4096, 16384),
          "175b_qkv_t8": (4608, 12288), "square8k": (8192, 8192)}
dev = torch.device("cuda")
for name, (N, K) in SHAPES.items():
    if i8:
        w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
        x = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
        ws = torch.rand(N, device=dev) * 1e-3
        xs = torch.rand(M, device=dev) * 1e-2
    else:
        w = (torch.randn(N, K, device=dev) * 0.02).half()
        x = torch.randn(M, K, device=dev).half()
        ws = xs = None
    out = torch.empty(M, N, dtype=torch.float16, device=dev)
    fn = lambda: E.gemm_large_batch(w, x, w_scales=ws, x_scales=xs, out=out)  # noqa: E731
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    reps = 10
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    tf = 2.0 * M * N * K / (best * 1e-3) / 1e12
    print(f"{name:12s} {dt} M={M} N={N} K={K}: {best * 1e3:8.1f} us  {tf:7.1f} T{'OP' if i8 else 'FLOP'}/s")
