"""Split-K tcgen05 GEMM at M = 128: time vs K (fixed cost vs per-stage cost).
python tools/tc_kscan.py [fp16|int8] [N ...]   -- CUDA-graph replays, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2207_00032_b200 import engine as E  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "fp16"
Ns = [int(v) for v in sys.argv[2:]] or [4096, 16384]
i8 = dt == "int8"
M = 128
dev = torch.device("cuda")
for N in Ns:
    for K in (1024, 2048, 4096, 8192, 16384):
        if i8:
            w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
            x = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
            ws, xs = torch.rand(N, device=dev) * 1e-3, torch.rand(M, device=dev) * 1e-2
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
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                a.record()
                g.replay()
                b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) / reps)
        gbs = w.numel() * w.element_size() / (best * 1e-3) / 1e9
        print(f"N={N:6d} K={K:6d}: {best * 1e3:7.2f} us  W {gbs:6.0f} GB/s")
