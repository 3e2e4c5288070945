"""SBI-GeMM parity on the GPU, through the C ABI, against the CPU oracle.

fp16 path: tolerance |gpu - oracle| <= 2e-3 * (sum_k |w_k x_k|) + 1e-3 (fp32 accumulation of
fp16 products vs the oracle's fp64 exec_reference order; outputs written fp32).
INT8 path: bit-exact (int32 accumulation and the fixed fp32 dequant order).
"""
import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2207_00032_b200 import engine as E  # noqa: E402
from paper_2207_00032_b200 import infersim as I  # noqa: E402


def _rand_f16(rng, shape, scale=1.0):
    return (rng.standard_normal(shape) * scale).astype(np.float16)


SHAPES = [
    (128, 64, 1), (256, 128, 1), (4096, 4096, 1), (12288, 4096, 1), (4096, 16384, 1),
    (1600, 1600, 3), (4800, 1600, 8), (6400, 1600, 16), (1000, 96, 5), (132, 40, 2),
    (4096, 1024, 16), (50304, 256, 1), (512, 2000, 9),
]


@pytest.mark.parametrize("N,K,B", SHAPES)
def test_fp16_gemm_matches_oracle(N, K, B):
    rng = np.random.default_rng(N * 7 + K * 3 + B)
    W = _rand_f16(rng, (N, K), 0.05)
    x = _rand_f16(rng, (B, K))
    dev = torch.device("cuda")
    wp = E.pack_weights_device(torch.from_numpy(W).to(dev), pack_M=2)
    out = E.gemm(wp, torch.from_numpy(x).to(dev), N, K).cpu().numpy()
    s = O.derive_schedule(N, K, B, 2)
    ref = O.gemm_f64(W.astype(np.float32), x.astype(np.float64), s)
    bound = np.abs(x.astype(np.float64)) @ np.abs(W.astype(np.float64)).T
    err = np.abs(out - ref)
    assert np.all(err <= 2e-3 * bound + 1e-3), float((err / (bound + 1e-9)).max())


@pytest.mark.parametrize("ksplit", [1, 2, 4, 8, 16])
def test_fp16_gemm_every_split_agrees(ksplit):
    rng = np.random.default_rng(11)
    N, K, B = 384, 2048, 4
    W = _rand_f16(rng, (N, K), 0.05)
    x = _rand_f16(rng, (B, K))
    dev = torch.device("cuda")
    wp = E.pack_weights_device(torch.from_numpy(W).to(dev), pack_M=2)
    out = E.gemm(wp, torch.from_numpy(x).to(dev), N, K, ksplit=ksplit).cpu().numpy()
    ref = x.astype(np.float64) @ W.astype(np.float64).T
    assert np.allclose(out, ref, rtol=2e-3, atol=2e-2)


def test_fp16_gemm_bias_gelu_f16_out():
    rng = np.random.default_rng(5)
    N, K, B = 640, 320, 3
    W = _rand_f16(rng, (N, K), 0.05)
    x = _rand_f16(rng, (B, K))
    b = _rand_f16(rng, (N,), 0.1)
    dev = torch.device("cuda")
    wp = E.pack_weights_device(torch.from_numpy(W).to(dev), pack_M=2)
    out = E.gemm(wp, torch.from_numpy(x).to(dev), N, K, bias=torch.from_numpy(b).to(dev), gelu=True)
    y = x.astype(np.float64) @ W.astype(np.float64).T + b.astype(np.float64)
    g = 0.5 * y * (1 + np.tanh(0.7978845608028654 * (y + 0.044715 * y ** 3)))
    assert out.dtype == torch.float16
    assert np.allclose(out.float().cpu().numpy(), g, rtol=4e-3, atol=4e-3)


def test_pack_device_matches_reference_layout():
    rng = np.random.default_rng(3)
    for (N, K, M) in [(5, 7, 2), (33, 64, 2), (8, 9, 4), (16, 3, 1)]:
        W = _rand_f16(rng, (N, K))
        packed = E.pack_weights_device(torch.from_numpy(W).cuda(), pack_M=M).cpu().numpy().astype(np.float64)
        host = I.pack_weights(W.astype(np.float64), I.GemmShape(N, K, 1, 2), M).data
        assert np.array_equal(packed, host)


@pytest.mark.parametrize("N,K,B", [(256, 256, 1), (4096, 4096, 1), (1600, 6400, 16), (1000, 100, 3),
                                   (12288, 4096, 8), (4096, 16384, 2)])
def test_int8_gemm_bit_exact(N, K, B):
    rng = np.random.default_rng(N + K + B)
    W = _rand_f16(rng, (N, K), 0.05)
    x = _rand_f16(rng, (B, K))
    dev = torch.device("cuda")
    wq, ws = E.quantize_weights_int8(torch.from_numpy(W).to(dev))
    xq, xs = E.quantize_activations_int8(torch.from_numpy(x).to(dev))
    # quantisation itself is bit-exact against the oracle
    owq, ows = O.quant_rows(W.astype(np.float32))
    oxq, oxs = O.quant_rows(x.astype(np.float32))
    assert np.array_equal(xq.cpu().numpy(), oxq) and np.array_equal(xs.cpu().numpy(), oxs)
    assert np.array_equal(ws.cpu().numpy(), ows)
    packed_host = I.pack_weights(owq.astype(np.float64), I.GemmShape(N, K, 1, 1), 4).data
    assert np.array_equal(wq.cpu().numpy().astype(np.float64), packed_host)
    _, y_oracle = O.gemm_i8(owq, ows, oxq, oxs)
    # pre-quantised activations (PRO_I8) and on-the-fly quantisation (PRO_QUANT)
    y1 = E.gemm(wq, xq, N, K, w_scales=ws, x_scales=xs).cpu().numpy()
    y2 = E.gemm(wq, torch.from_numpy(x).to(dev), N, K, w_scales=ws).cpu().numpy()
    assert np.array_equal(y1, y_oracle)
    assert np.array_equal(y2, y_oracle)


def test_exec_device_matches_exec_reference():
    rng = np.random.default_rng(17)
    N, K, B = 300, 200, 4
    W = rng.integers(-8, 9, (N, K)).astype(np.float64)
    x = rng.integers(-8, 9, (B, K)).astype(np.float64)
    shape = I.GemmShape(N, K, B, 2)
    sch = I.derive_schedule(shape, I.b200_device())
    packed = I.pack_weights(W, shape, sch.pack_M)
    out = I.exec_device(packed, x, B, sch).reshape(B, N)
    # small integers: fp16 exact, fp32 accumulation exact -> identical to the fp64 reference
    assert np.array_equal(out, x @ W.T)


@pytest.mark.parametrize("pack_m", [1, 2, 4])
@pytest.mark.parametrize("sched_m", [1, 2, 4])
def test_exec_device_any_packed_layout(pack_m, sched_m):
    """exec_reference reads the data with packed.pack_M (gemm.hpp:186): weights packed with any M in
    {1, 2, 4} give the same result under any schedule (whose pack_M only groups the iteration)."""
    rng = np.random.default_rng(pack_m * 10 + sched_m)
    N, K, B = 130, 67, 3  # K a multiple of none of 2, 4: the padded sizes differ per M
    W = rng.integers(-8, 9, (N, K)).astype(np.float64)
    x = rng.integers(-8, 9, (B, K)).astype(np.float64)
    shape = I.GemmShape(N, K, B, 2)
    sch = I.derive_schedule(shape, I.b200_device())
    sch.pack_M = sched_m
    packed = I.pack_weights(W, shape, pack_m)
    out = I.exec_device(packed, x, B, sch).reshape(B, N)
    assert np.array_equal(out, x @ W.T)


@pytest.mark.parametrize("N,K,B", [(4096, 4096, 1), (12288, 4096, 1), (4096, 16384, 1), (1024, 2048, 3),
                                   (4096, 4096, 8), (16384, 4096, 16), (640, 320, 5)])
def test_int8_weight_only_w8a16(N, K, B):
    """W8A16: int8 weights (per-row scale) x fp16 activations, fp32 accumulation -- within
    2e-3 * sum|q x| * s + 1e-3 of the exact product (both the smem-slice and the streamed-x plans)."""
    rng = np.random.default_rng(N + K + B)
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float16)
    x = rng.standard_normal((B, K)).astype(np.float16)
    dev = torch.device("cuda")
    wq, ws = E.quantize_weights_int8(torch.from_numpy(W).to(dev))
    out = E.gemm(wq, torch.from_numpy(x).to(dev), N, K, w_scales=ws, a16=True).cpu().numpy()
    q_rm, s_rm = O.quant_rows(W.astype(np.float32))
    ref = (x.astype(np.float64) @ q_rm.astype(np.float64).T) * s_rm.astype(np.float64)
    bound = (np.abs(x.astype(np.float64)) @ np.abs(q_rm.astype(np.float64)).T) * s_rm.astype(np.float64)
    err = np.abs(out - ref)
    assert np.all(err <= 2e-3 * bound + 1e-3), float((err / (bound + 1e-9)).max())


@pytest.mark.parametrize("ksplit", [1, 2, 4, 8, 16])
def test_int8_w8a16_every_split_agrees(ksplit):
    rng = np.random.default_rng(21)
    N, K, B = 512, 4096, 2
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float16)
    x = rng.standard_normal((B, K)).astype(np.float16)
    dev = torch.device("cuda")
    wq, ws = E.quantize_weights_int8(torch.from_numpy(W).to(dev))
    out = E.gemm(wq, torch.from_numpy(x).to(dev), N, K, w_scales=ws, a16=True, ksplit=ksplit).cpu().numpy()
    q_rm, s_rm = O.quant_rows(W.astype(np.float32))
    ref = (x.astype(np.float64) @ q_rm.astype(np.float64).T) * s_rm.astype(np.float64)
    assert np.allclose(out, ref, rtol=2e-3, atol=2e-2)


@pytest.mark.parametrize("N,K", [(4096, 4096), (1000, 300), (12288, 4096), (640, 16384)])
def test_int8_group_quantisation_bit_exact(N, K):
    """K-group quantisation (128 k per fp16 scale): q and the scales are bit-identical to the oracle,
    in the pack_M = 4 layout of the row mode (a heavy-tailed matrix, so the groups differ)."""
    rng = np.random.default_rng(N + K)
    W = (rng.standard_normal((N, K)) * 0.05 * np.exp(rng.standard_normal((N, K)))).astype(np.float16)
    dev = torch.device("cuda")
    wq, gs = E.quantize_weights_int8_groups(torch.from_numpy(W).to(dev))
    oq, os_ = O.quant_groups(W.astype(np.float32))
    assert np.array_equal(gs.cpu().numpy().view(np.uint16), os_.view(np.uint16))
    packed_host = I.pack_weights(oq.astype(np.float64), I.GemmShape(N, K, 1, 1), 4).data
    assert np.array_equal(wq.cpu().numpy().astype(np.float64), packed_host)


@pytest.mark.parametrize("N,K,B,ksplit", [(4096, 4096, 1, 0), (12288, 4096, 1, 0), (4096, 16384, 1, 0),
                                          (1000, 300, 3, 0), (4096, 4096, 8, 0), (16384, 4096, 16, 0),
                                          (512, 4096, 2, 1), (512, 4096, 2, 4), (512, 4096, 2, 16)])
def test_int8_group_w8a16_gemm(N, K, B, ksplit):
    """W8A16 with K-group scales: y = sum_g s_g sum_{k in g} q_k x_k (each group's exact int8 x fp16
    products in fp32, scaled per group) -- within 2e-3 * sum|q s x| + 1e-3 of the oracle's fp64 sum, for
    every split (a split boundary is a group boundary) and both x plans."""
    rng = np.random.default_rng(N * 7 + K + B)
    W = (rng.standard_normal((N, K)) * 0.05 * np.exp(rng.standard_normal((N, K)))).astype(np.float16)
    x = rng.standard_normal((B, K)).astype(np.float16)
    dev = torch.device("cuda")
    wq, gs = E.quantize_weights_int8_groups(torch.from_numpy(W).to(dev))
    out = E.gemm(wq, torch.from_numpy(x).to(dev), N, K, w_group_scales=gs, ksplit=ksplit).cpu().numpy()
    oq, os_ = O.quant_groups(W.astype(np.float32))
    ref = O.gemm_a16_groups(oq, os_, x).astype(np.float64)
    weff = O.dequant_groups(oq, os_).astype(np.float64)
    bound = np.abs(x.astype(np.float64)) @ np.abs(weff).T
    err = np.abs(out - ref)
    assert np.all(err <= 2e-3 * bound + 1e-3), float((err / (bound + 1e-9)).max())
