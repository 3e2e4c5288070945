"""Cross-process tensor parallelism without NCCL (DSINF_TP_IPC): two processes, one rank each, on
the same B200 (CUDA IPC works within one device), exchange CUDA-IPC handles over gloo; every per-layer
all-reduce runs fused in the attn-out / MLP-down epilogues over peer memory (system-scope flags,
costmodel.hpp:84-85), and the vocab-parallel argmax keys are all-gathered by the select kernel.
Both ranks' logit slices and greedy tokens against the TP-aware CPU oracle (tp = 2), with the
tolerances of test_gpu_model.py."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 20220701


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_ranks(tmp_path, world, **kw):
    args = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
            "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
            os.path.join(ROOT, "tools", "tp_ipc_check.py"), "--out", str(tmp_path)]
    for k, v in kw.items():
        args += ["--" + k.replace("_", "-"), str(v)]
    r = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{q}.npz"))) for q in range(world)]


@pytest.mark.parametrize("dtype_bytes", [2, 1])
def test_tp_ipc_two_processes_match_oracle(tmp_path, dtype_bytes):
    hidden, layers, heads, vocab, batch, prompt, gen = 512, 2, 8, 1000, 2, 5, 4
    res = _run_ranks(tmp_path, 2, hidden=hidden, layers=layers, heads=heads, vocab=vocab, batch=batch,
                     dtype_bytes=dtype_bytes, prompt=prompt, gen=gen, max_ctx=32)
    assert all(int(r["fused_allreduce"]) == 1 for r in res)
    # both ranks select the same tokens (the key all-gather) and agree on the history
    assert np.array_equal(res[0]["hist"], res[1]["hist"])
    vl = int(res[0]["vocab_local"])
    tol_rel, tol_abs = (0.03, 0.01) if dtype_bytes == 2 else (0.06, 0.02)
    ora = O.OracleModel(hidden, layers, heads, vocab, dtype_bytes=dtype_bytes, tp=2, batch=batch, max_ctx=32,
                        seed=SEED)
    hist = res[0]["hist"]
    for pos in range(prompt + gen - 1):
        ol, onext = ora.step(hist[:, pos], pos)
        lg = np.concatenate([res[0]["logits"][pos], res[1]["logits"][pos]], axis=1)[:, :vocab]
        assert lg.shape == (batch, vocab) and vl * 2 >= vocab
        tol = tol_rel * float(ol.std()) + tol_abs
        err = float(np.abs(lg - ol).max())
        assert err <= tol, f"pos {pos}: max|dlogit| {err:.4g} > tol {tol:.4g}"
        srt = np.sort(ol, axis=1)
        for b in range(batch):
            if srt[b, -1] - srt[b, -2] > tol:
                assert res[0]["tokens"][pos][b] == onext[b], f"pos {pos} b {b}"
    ora.close()
