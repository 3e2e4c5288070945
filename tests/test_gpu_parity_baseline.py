"""Parity of the benched decode path at BASELINE.json's configs (tools/parity_baseline.py):

- GPT-J-6B at full depth (32 layers), batch 1 / 8 / 16, fp16 and int8 (AUTO activation modes),
  128-token prompt prefilled on the tcgen05 tensor cores, 8 greedy tokens through the CUDA-graph /
  PDL / x-streaming decode step -- the exact path bench.py times;
- GPT-NeoX-20B t=2 (head dim 96), GPT-50B t=4 and GPT3-175B t=8 at full width and 2 layers, all
  shards on this GPU (DSINF_TP_LOCAL), batch 1 / 16, fp16 and int8.

Against the teacher-forced fp64 oracle (oracle/seq_oracle.py, pinned to or_model_step).  Stated
tolerance per position: max |dlogit| <= 0.03 std + 0.01 (fp16), 0.06 std + 0.02 (int8), for INT8 at
least 3x the oracle's own fp32-vs-fp64 accumulation spread at that position (the W8A8 activation
quantisation noise floor, tools/parity_baseline.py).  Greedy
tokens identical, or a near tie within 2 max|dlogit| (each one logged).  Logs: profiles/.
"""
import json
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu]

# The whole suite (~15 min: GPT-J B=8/16 and the three TP configs) runs with DSINF_PARITY_SUITE=1 or
# `python tools/parity_baseline.py --suite all` (its last log: profiles/r2_parity_baseline.*); the
# GPT-J B=1 cases (the headline bench line, ~2 min) always run.
FULL = os.environ.get("DSINF_PARITY_SUITE", "0") not in ("", "0")
full_suite = pytest.mark.skipif(not FULL, reason="set DSINF_PARITY_SUITE=1 (log: profiles/r2_parity_baseline.*)")

from tools import parity_baseline as PB  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check(results, tag):
    out = os.path.join(ROOT, "gpurun_out") if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else None
    if out:
        with open(os.path.join(out, f"parity_{tag}.json"), "w") as f:
            json.dump(results, f, indent=1)
    for r in results:
        print(f"{r['case']}: worst err/tol {r['worst_err_over_tol']}, tokens identical {r['tokens_identical']}/"
              f"{r['positions']}, near ties {r['near_ties_below_tol']}, mismatches {r['token_mismatches']}")
    bad = [f for r in results for f in r["failures"]]
    assert not bad, bad


@pytest.mark.parametrize("dtype", ["fp16", "int8"])
def test_gptj_full_depth_bench_path_b1(dtype):
    label, h, L, H, V, tp, bs = PB.SUITES["gptj"][0]
    _check(PB.run_config(label, h, L, H, V, tp=tp, dtypes=[dtype], batches=(1,)), f"gptj_{dtype}_b1")


@full_suite
@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["fp16", "int8"])
def test_gptj_full_depth_bench_path(dtype):
    label, h, L, H, V, tp, bs = PB.SUITES["gptj"][0]
    _check(PB.run_config(label, h, L, H, V, tp=tp, dtypes=[dtype], batches=bs), f"gptj_{dtype}")


@full_suite
@pytest.mark.slow
@pytest.mark.parametrize("cfg", range(len(PB.SUITES["tp"])), ids=["neox_t2", "gpt50b_t4", "gpt175b_t8"])
def test_tp_configs_full_width(cfg):
    label, h, L, H, V, tp, bs = PB.SUITES["tp"][cfg]
    _check(PB.run_config(label, h, L, H, V, tp=tp, dtypes=["fp16", "int8"], batches=bs), f"tp{tp}")
