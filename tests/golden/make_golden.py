"""Generate tests/golden/reference_golden.json by running the UNMODIFIED reference headers
(compiled into oracle/_ref/libinfersim_ref.so by `make ref`) on fixed inputs.

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
The JSON is committed; the CPU tests compare the C ABI and the oracle against it, so parity is
pinned even on machines without the reference tree (the GPU box).
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

ref = O.ref_lib()
assert ref is not None, "build oracle/_ref first (make ref)"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")

BASELINE = [  # (name, hidden, layers, heads, tp) — BASELINE.json configs
    ("gpt2-1.5b", 1600, 48, 25, 1), ("gptj-6b", 4096, 32, 32, 1), ("gpt-neox-20b", 6144, 44, 64, 2),
    ("gpt-50b", 8192, 62, 64, 4), ("gpt3-175b", 12288, 96, 96, 8)]


def sched(N, K, B, dt, sm):
    rc, s = O.ref_derive_schedule(N, K, B, dt, sm)
    return {"N": N, "K": K, "B": B, "dtype": dt, "sm": sm, "rc": rc, "schedule": s}


g = {"generator": "tests/golden/make_golden.py over oracle/_ref (reference headers proj/include/infersim)"}

# derive_schedule (gemm.hpp:65-96): every per-rank GEMM of every BASELINE config on B200 (148 SMs)
# and A100 (108 SMs, the reference's test device), plus the SPEC example and edge shapes.
shapes = []
for name, h, L, H, t in BASELINE:
    vpad = (50257 + 128 * t - 1) // (128 * t) * (128 * t)
    for (N, K) in [(3 * h // t, h), (h, h // t), (4 * h // t, h), (h, 4 * h // t), (vpad // t, h)]:
        for dt in (1, 2, 4):
            for sm in (148, 108):
                shapes.append(sched(N, K, 1, dt, sm))
for (N, K, B, dt, sm) in [(256, 4096, 1, 2, 108), (1, 1, 1, 2, 148), (32, 7, 3, 1, 148), (5000, 3, 2, 4, 148),
                          (100, 100, 1, 3, 148), (0, 5, 1, 2, 148), (4736, 64, 1, 2, 148), (4735, 64, 1, 2, 148)]:
    shapes.append(sched(N, K, B, dt, sm))
g["derive_schedule"] = shapes

# pack_weights (gemm.hpp:113-130): the (n+1)*10+k vectors of SURVEY §8a-a4 plus random shapes
packs = []
rng = np.random.default_rng(20220701)
for (N, K, M) in [(2, 4, 2), (2, 8, 4), (2, 3, 2), (2, 4, 1), (3, 5, 4), (4, 7, 2), (1, 1, 4)]:
    W = np.array([[(n + 1) * 10 + k for k in range(K)] for n in range(N)], dtype=np.float64)
    kp = (K + M - 1) // M * M
    out = np.zeros(N * kp)
    rc = ref.ref_pack_weights(W.ctypes.data_as(O.f64p), N, K, 2, M, out.ctypes.data_as(O.f64p), out.size)
    packs.append({"N": N, "K": K, "M": M, "rc": rc, "matrix": W.ravel().tolist(), "packed": out.tolist()})
g["pack_weights"] = packs

# exec_reference (gemm.hpp:147-202): integer data (exact) and random doubles (bit patterns)
execs = []
for (N, K, B, dt, integer) in [(37, 101, 3, 2, True), (64, 64, 1, 1, True), (5, 403, 2, 2, False),
                               (7, 211, 3, 4, False), (40, 48, 5, 2, False), (1, 17, 1, 1, False)]:
    if integer:
        W = rng.integers(-8, 9, (N, K)).astype(np.float64)
        x = rng.integers(-8, 9, (B, K)).astype(np.float64)
    else:
        W = rng.standard_normal((N, K))
        x = rng.standard_normal((B, K))
    rc, s6 = O.ref_derive_schedule(N, K, B, dt, 148)
    out = O.ref_exec_reference(W, dt, s6, x, B)
    execs.append({"N": N, "K": K, "B": B, "dtype": dt, "schedule": s6, "W": [float.hex(v) for v in W.ravel()],
                  "x": [float.hex(v) for v in x.ravel()], "out": [float.hex(v) for v in out.ravel()]})
g["exec_reference"] = execs

# canonical_layer_graph -> partition_layer -> fusion_savings (fusion.hpp:140-357)
canon = []
for hidden in (512, 1600, 4096, 12288):
    for batch in (1, 8, 16, 32):
        for regime in (0, 1):
            for dt in (1, 2):
                ro = (C.c_int32 * 8)()
                nr, la, by = C.c_int32(), C.c_int64(), C.c_int64()
                rc = ref.ref_canonical_partition(hidden, batch, dt, regime, ro, C.byref(nr), C.byref(la), C.byref(by))
                canon.append({"hidden": hidden, "batch": batch, "regime": regime, "dtype": dt, "rc": rc,
                              "region_of": list(ro), "regions": nr.value, "launches_saved": la.value,
                              "bytes_saved": by.value})
g["canonical_partition"] = canon

# model.hpp accounting
acc = []
for name, h, L, H, t in BASELINE:
    for dt in (1, 2, 4):
        pc = C.c_int64()
        ref.ref_param_count(h, L, H, 50257, 2048, dt, C.byref(pc))
        entry = {"name": name, "hidden": h, "layers": L, "heads": H, "dtype": dt, "param_count": pc.value}
        for (B, P, G, ph) in [(1, 128, 8, 1), (16, 128, 8, 1), (8, 128, 0, 0), (1, 2048, 0, 1)]:
            fl = C.c_double()
            ref.ref_layer_flops(h, L, H, 50257, 2048, dt, B, P, G, ph, C.byref(fl))
            kv = C.c_int64()
            ref.ref_kv_cache_bytes(h, L, H, 50257, 2048, dt, B, P, G, C.byref(kv))
            entry.setdefault("flops", []).append([B, P, G, ph, fl.value])
            entry.setdefault("kv", []).append([B, P, G, kv.value])
        acc.append(entry)
g["model"] = acc

# costmodel.hpp
kt = []
for (flops, by, bw, dt, la, cg) in [(1e9, 1e6, 8e12, 2, 1, 0), (7e12, 1e9, 1.55e12, 2, 4, 1), (0.0, 5e8, 6.45e12, 1, 3, 0),
                                    (1e15, 1e3, 8e12, 4, 1, 0)]:
    o = (C.c_double * 4)()
    rc = ref.ref_kernel_time(flops, by, bw, 148, dt, la, cg, o)
    kt.append({"args": [flops, by, bw, dt, la, cg], "rc": rc, "out": list(o)})
g["kernel_time"] = kt
ct = []
for kind in range(5):
    for grp, nodes, gpus in [([0, 1], 1, 8), ([0, 1, 2, 3, 4, 5, 6, 7], 1, 8), ([0, 9], 2, 8), ([3], 1, 8)]:
        for by in (24576.0, 393216.0, 1.0e9):
            o = C.c_double()
            arr = (C.c_int * len(grp))(*grp)
            rc = ref.ref_collective_time(kind, by, arr, len(grp), nodes, gpus, 900e9, 2e-6, 50e9, 5e-6, C.byref(o))
            ct.append({"kind": kind, "group": grp, "nodes": nodes, "gpus": gpus, "bytes": by, "rc": rc, "out": o.value})
g["collective_time"] = ct
ml = []
for name, h, L, H, t in BASELINE:
    for dt in (1, 2):
        for tp in (1, 2, 4, 8):
            o = C.c_double()
            rc = ref.ref_min_latency_bound(h, L, H, 50257, dt, tp, 1, 8e12, 192_000_000_000, C.byref(o))
            ml.append({"name": name, "dtype": dt, "tp": tp, "rc": rc, "out": o.value})
g["min_latency_bound"] = ml

with open(OUT, "w") as f:
    json.dump(g, f, indent=0)
print("wrote", OUT, os.path.getsize(OUT), "bytes")
