"""In-process A/B of decode-step variants (same weights seed, same prompt): python tools/ab_inproc.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_00032_b200.engine import DecoderModel
from paper_2207_00032_b200.presets import PRESETS  # noqa: E402

p = PRESETS[os.environ.get("CFG", "gptj-6b")]
variants = {"pdl": (dict(use_pdl=True), None), "nopdl": (dict(use_pdl=False), None), "pdl_mask0": (dict(use_pdl=True), "0"), "pdl_mask4": (dict(use_pdl=True), "4")}
prompt = np.random.default_rng(0).integers(0, p.vocab, (1, 128)).astype(np.int32)
s = torch.cuda.Stream()
for rep in range(2):
    for name, (kw, mask) in variants.items():
        if mask is None:
            os.environ.pop('DSINF_PDL_MASK', None)
        else:
            os.environ['DSINF_PDL_MASK'] = mask
        m = DecoderModel(p.hidden, p.layers, p.heads, p.vocab, batch=1, max_ctx=200, **kw)
        m.set_prompt(prompt, stream=s)
        m.step(136, stream=s)
        s.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(s)
        m.step(32, stream=s)
        en.record(s)
        en.synchronize()
        print(rep, name, round(st.elapsed_time(en) / 32, 4), "ms/step", flush=True)
        m.close()
        del m
        torch.cuda.empty_cache()
