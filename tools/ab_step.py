#!/usr/bin/env python3
"""In-process A/B of environment variants of the decode step (same weights, prompt 128, ms/step by
CUDA events over 32 graph-replayed steps, variants interleaved over 2 repetitions):
  python tools/ab_step.py CFG DTYPE B "VAR=v,VAR2=w" "VAR=u" ...   (an empty string = defaults)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg, dt, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
variants = sys.argv[4:] or [""]
p = PRESETS[cfg]
prompt = np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32)
s = torch.cuda.Stream()
base_env = dict(os.environ)
res = {v: [] for v in variants}
for rep in range(2):
    for v in variants:
        os.environ.clear()
        os.environ.update(base_env)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=", 1)
            os.environ[k] = val
        m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B,
                         max_ctx=200, int8_act=capi.INT8_AUTO)
        m.set_prompt(prompt, stream=s)
        m.prefill(stream=s)
        m.step(8, stream=s)
        s.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(s)
        m.step(32, stream=s)
        en.record(s)
        en.synchronize()
        res[v].append(st.elapsed_time(en) / 32)
        m.close()
        del m
        torch.cuda.empty_cache()
for v, t in res.items():
    print(f"{cfg} {dt} B={B} [{v or 'default'}]: {min(t):.4f} ms/step ({', '.join(f'{x:.4f}' for x in t)})", flush=True)
