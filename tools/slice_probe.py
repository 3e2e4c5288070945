"""Per-rank (DSINF_TP_SLICE) decode step time of one TP config (TP=1 configs: the whole model):
tools/slice_probe.py <config> <fp16|int8> <batch> [w8a8|w8a16]."""
import sys, os, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2207_00032_b200 import engine as E, _capi as capi
name, dtype, batch = sys.argv[1], sys.argv[2], int(sys.argv[3])
pr = E.PRESETS[name]
stream = torch.cuda.Stream()
m = E.DecoderModel(pr.hidden, pr.layers, pr.heads, pr.vocab, dtype_bytes=1 if dtype == "int8" else 2, batch=batch,
                   max_ctx=200, tp_size=pr.tp, tp_rank=0, tp_mode=capi.TP_SLICE, seed=1,
                   int8_act={"w8a8": capi.INT8_W8A8, "w8a16": capi.INT8_W8A16}.get(sys.argv[4] if len(sys.argv) > 4 else "", capi.INT8_AUTO))
prompt = np.random.default_rng(1).integers(0, pr.vocab, (batch, 128)).astype(np.int32)
m.set_prompt(prompt, stream=stream); m.prefill(stream=stream); m.step(4, stream=stream); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream); m.step(32, stream=stream); b.record(stream); b.synchronize()
ms = a.elapsed_time(b) / 32
print(name, dtype, batch, os.environ.get("DSINF_XS", "-"), f"{ms:.3f} ms", m.get_info().kernels_per_step)
m.close()
