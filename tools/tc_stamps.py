"""Per-CTA phase stamps of one split-K tcgen05 launch at M = 128 (needs `make DIAG=1 lib`).
Phases (globaltimer, µs from the earliest CTA entry): entry, setup done, producer past the PDL wait,
first full stage at the MMA thread, last MMA issued, accumulator ready, partials exchanged (cluster
barrier), partial sums reduced (before the epilogue stores).
python tools/tc_stamps.py [fp16|int8] N K"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200 import engine as E  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "fp16"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
K = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
M = 128
dev = torch.device("cuda")
i8 = dt == "int8"
if i8:
    w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
    x = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
    ws, xs = torch.rand(N, device=dev) * 1e-3, torch.rand(M, device=dev) * 1e-2
else:
    w = (torch.randn(N, K, device=dev) * 0.02).half()
    x = torch.randn(M, K, device=dev).half()
    ws = xs = None
out = torch.empty(M, N, dtype=torch.float16, device=dev)
lib = capi.lib
fn = lib.dsinf_debug_tc_stamps
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["setup", "wait", "first", "lastmma", "acc", "xchg", "reduced"]
for rep in range(4):
    torch.cuda.synchronize()
    E.gemm_large_batch(w, x, w_scales=ws, x_scales=xs, out=out)
    torch.cuda.synchronize()
buf = np.zeros(4096 * 8, dtype=np.uint64)
assert fn(buf.ctypes.data, buf.size) == 0
st = buf.reshape(4096, 8)
n = int((st[:, 0] > 0).sum())
st = st[:n].astype(np.float64)
t0 = st[:, 0].min()
rel = (st - t0) / 1e3
print(f"{dt} N={N} K={K}: {n} CTAs, entry spread {rel[:, 0].max():.2f} us")
for i, nm in enumerate(names, start=1):
    c = rel[:, i]
    c = c[c > -1e6]
    print(f"  {nm:8s} median {np.median(c):7.2f}  max {c.max():7.2f} us")
print(f"  per-CTA main loop (first -> lastmma) median {np.median(rel[:, 4] - rel[:, 3]):.2f} us")
