#!/usr/bin/env python3
"""Per-rank decode step of a TP config on one GPU (DSINF_TP_SLICE, rank 0's shard alone) under
environment variants, in process (ms/step by CUDA events over 32 graph-replayed steps):
  python tools/slice_ab.py CFG DTYPE B "VAR=v,..." ...   e.g. gpt3-175b fp16 1 "" "DSINF_FUSED_AR=1"
With DSINF_FUSED_AR=1 the rank's row-parallel epilogues push into its own t slots and it waits on its
own counters: the fused all-reduce's per-rank cost without the NVLink hop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

cfg, dt, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
p = PRESETS[cfg]
base = dict(os.environ)
s = torch.cuda.Stream()
for rep in range(2):
    for v in sys.argv[4:] or [""]:
        os.environ.clear()
        os.environ.update(base)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=", 1)
            os.environ[k] = val
        m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, dtype_bytes=1 if dt == "int8" else 2, batch=B,
                         max_ctx=200, tp_size=p.tp, tp_rank=0, tp_mode=capi.TP_SLICE, int8_act=capi.INT8_AUTO)
        m.set_prompt(np.random.default_rng(0).integers(0, p.vocab, (B, 128)).astype(np.int32), stream=s)
        m.step(136, stream=s)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        m.step(32, stream=s)
        e1.record(s)
        e1.synchronize()
        info = m.get_info()
        print(f"rep {rep} {cfg} t={p.tp} {dt} B={B} [{v or 'default'}]: {e0.elapsed_time(e1) / 32:.3f} ms/step, "
              f"fused_allreduce={info.fused_allreduce}", flush=True)
        m.close()
        del m
        torch.cuda.empty_cache()
