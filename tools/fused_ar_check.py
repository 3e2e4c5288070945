import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2207_00032_b200 import _capi as capi
from paper_2207_00032_b200.engine import DecoderModel
for fused in ("1", "0"):
    os.environ["DSINF_FUSED_AR"] = fused
    os.environ["DSINF_XS"] = "0" if fused == "1" else "-1"  # fused slots are summed by the LN prologues
    m = DecoderModel(4096, 4, 32, 50257, batch=1, max_ctx=200, tp_size=4, tp_mode=capi.TP_LOCAL)
    m.set_prompt(np.random.default_rng(0).integers(0, 50257, (1, 128)).astype(np.int32))
    m.step(130)
    import torch
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); m.step(32); b.record(); b.synchronize()
    print("fused", fused, "kernels/step", m.get_info().kernels_per_step, "ms/step", a.elapsed_time(b) / 32)
    m.close()
