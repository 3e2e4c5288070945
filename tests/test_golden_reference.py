"""The host operator API (C ABI) and the CPU oracle against golden vectors produced by the reference
headers themselves (tests/golden/make_golden.py over oracle/_ref).  Runs without a GPU and without
the reference tree.  Mirrors the reference's own tests: test_fusion.cpp:103-243, test_model.cpp:54-179,
test_costmodel.cpp:75-153, and the SPEC gemm examples."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_00032_b200 import infersim as I

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _dev(sm):
    return I.DeviceSpec(192_000_000_000, 8e12, sm, 5e-6, {4: 80e12, 2: 2.25e15, 1: 4.5e15})


@pytest.mark.parametrize("case", G["derive_schedule"], ids=lambda c: f"{c['N']}x{c['K']}d{c['dtype']}s{c['sm']}")
def test_derive_schedule_matches_reference(case):
    shape = I.GemmShape(case["N"], case["K"], case["B"], case["dtype"])
    if case["rc"] != 0:
        with pytest.raises(I.ConfigError):
            I.derive_schedule(shape, _dev(case["sm"]))
        return
    s = I.derive_schedule(shape, _dev(case["sm"]))
    assert [int(s.mode), s.output_tiles, s.input_tiles, s.warps_per_block, s.kernel_count, s.pack_M] == case["schedule"]
    o = O.derive_schedule(case["N"], case["K"], case["B"], case["dtype"], case["sm"])
    assert [o.two_d, o.output_tiles, o.input_tiles, o.warps_per_block, o.kernel_count, o.pack_M] == case["schedule"]


def test_cache_line_pack_values():  # gemm.hpp:57-60; "2 for half precision and 4 for the INT8"
    assert [I.cache_line_pack(d) for d in (1, 2, 4)] == [4, 2, 1]


@pytest.mark.parametrize("case", G["pack_weights"], ids=lambda c: f"{c['N']}x{c['K']}M{c['M']}")
def test_pack_weights_golden(case):
    N, K, M = case["N"], case["K"], case["M"]
    W = np.array(case["matrix"]).reshape(N, K)
    p = I.pack_weights(W, I.GemmShape(N, K, 1, 2), M)
    assert p.data.tolist() == case["packed"]
    assert p.padded_in_dim == (K + M - 1) // M * M
    assert np.array_equal(I.unpack_weights(p), W.ravel())  # round trip
    assert O.pack(W, M).tolist() == case["packed"]
    for n in range(N):
        for k in range(K):
            assert p.data[I.packed_index(n, k, N, M)] == W[n, k]


def test_pack_rejects_bad_pack_m():
    with pytest.raises(I.ConfigError, match="pack_M must be one of"):
        I.pack_weights(np.zeros(8), I.GemmShape(2, 4, 1, 2), 3)
    with pytest.raises(I.ConfigError, match="does not match"):
        I.pack_weights(np.zeros(7), I.GemmShape(2, 4, 1, 2), 2)


@pytest.mark.parametrize("case", G["exec_reference"], ids=lambda c: f"{c['N']}x{c['K']}B{c['B']}d{c['dtype']}")
def test_oracle_exec_is_bit_identical_to_exec_reference(case):
    N, K, B = case["N"], case["K"], case["B"]
    W = np.array([float.fromhex(v) for v in case["W"]]).reshape(N, K)
    x = np.array([float.fromhex(v) for v in case["x"]]).reshape(B, K)
    ref = np.array([float.fromhex(v) for v in case["out"]]).reshape(B, N)
    s = O.derive_schedule(N, K, B, case["dtype"])
    got = O.exec_sameorder(O.pack(W, s.pack_M), N, K, s.pack_M, s, x, B)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("case", G["canonical_partition"],
                         ids=lambda c: f"h{c['hidden']}b{c['batch']}r{c['regime']}d{c['dtype']}")
def test_canonical_partition_matches_reference(case):
    regions, sav = I.canonical_layer_partition(case["hidden"], case["batch"], I.BatchRegime(case["regime"]),
                                               case["dtype"])
    region_of = [0] * 8
    for r, names in enumerate(regions):
        for nm in names:
            region_of[I.CANONICAL_NODE_NAMES.index(nm)] = r
    assert region_of == case["region_of"]
    assert (sav.launches_saved, sav.bytes_saved) == (case["launches_saved"], case["bytes_saved"])


def test_small_batch_four_regions_in_order():  # test_fusion.cpp:103-121
    regions, sav = I.canonical_layer_partition(1600, 1, I.BatchRegime.small_batch)
    assert regions == [["input_layernorm", "qkv_gemm"], ["attn_transpose", "attention"],
                       ["post_attn_layernorm", "intermediate_gemm"], ["bias_add", "residual_add"]]
    assert sav.launches_saved == 4


@pytest.mark.parametrize("case", G["model"], ids=lambda c: f"{c['name']}d{c['dtype']}")
def test_model_accounting_matches_reference(case):
    cfg = I.ModelConfig(case["name"], case["hidden"], case["layers"], case["heads"], 50257, 2048, case["dtype"])
    assert I.param_count(cfg) == case["param_count"]
    assert I.param_bytes(cfg) == case["param_count"] * case["dtype"]
    for B, P, Gn, ph, fl in case["flops"]:
        assert I.layer_flops(cfg, I.SeqWorkload(B, P, Gn), I.Phase(ph)) == fl
    for B, P, Gn, kv in case["kv"]:
        assert I.kv_cache_bytes(cfg, I.SeqWorkload(B, P, Gn)) == kv


def test_gpt2_param_count_anchor():  # test_model.cpp:54-58
    assert I.param_count(I.ModelConfig("gpt2", 1600, 48, 25)) == 1_554_971_200


def test_kv_cache_anchor():  # test_model.cpp:167-179
    cfg = I.ModelConfig("x", 4096, 32, 32, 50257, 2048, 2)
    assert I.kv_cache_bytes(cfg, I.SeqWorkload(8, 2048, 0)) == 8_589_934_592


@pytest.mark.parametrize("case", G["kernel_time"], ids=lambda c: str(c["args"]))
def test_kernel_time_matches_reference(case):
    flops, by, bw, dt, la, cg = case["args"]
    dev = _dev(148)
    dev.mem_bw = bw
    c = I.kernel_time(flops, by, dev, dt, la, bool(cg))
    assert [c.compute_time, c.memory_time, c.launch_overhead, c.total] == case["out"]


@pytest.mark.parametrize("case", G["collective_time"], ids=lambda c: f"k{c['kind']}n{len(c['group'])}b{c['bytes']}")
def test_collective_time_matches_reference(case):
    topo = I.Topology(case["nodes"], case["gpus"], _dev(148), I.LinkSpec(900e9, 2e-6), I.LinkSpec(50e9, 5e-6))
    assert I.collective_time(I.CollectiveKind(case["kind"]), case["bytes"], case["group"], topo) == case["out"]


@pytest.mark.parametrize("case", G["min_latency_bound"], ids=lambda c: f"{c['name']}d{c['dtype']}tp{c['tp']}")
def test_min_latency_bound_matches_reference(case):
    name = case["name"]
    h, L, H = {"gpt2-1.5b": (1600, 48, 25), "gptj-6b": (4096, 32, 32), "gpt-neox-20b": (6144, 44, 64),
               "gpt-50b": (8192, 62, 64), "gpt3-175b": (12288, 96, 96)}[name]
    cfg = I.ModelConfig(name, h, L, H, 50257, 2048, case["dtype"])
    topo = I.Topology(1, 8, _dev(148), I.LinkSpec(900e9, 2e-6), I.LinkSpec(50e9, 5e-6))
    if case["rc"] == 3:
        with pytest.raises(I.InfeasibleError):
            I.min_latency_bound(cfg, I.ParallelismPlan(case["tp"], 1), topo)
    else:
        assert I.min_latency_bound(cfg, I.ParallelismPlan(case["tp"], 1), topo) == case["out"]
