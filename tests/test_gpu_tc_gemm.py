"""Large-batch tensor-core GEMM (tcgen05 + TMEM) through the C ABI, against the CPU oracle.

fp16: |gpu - ref| <= 2e-3 * sum_k |w_k x_k| + 1e-3 against an fp64 product of the same fp16
operands (fp32 tensor-core accumulation).  INT8 (W8A8): bit-exact against oracle.gemm_i8 --
exact int32 accumulation, then the fixed fp32 dequant order y = fp32(fp32(acc) * s_x) * s_w.
"""
import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2207_00032_b200 import engine as E  # noqa: E402

SHAPES = [(256, 64, 128), (512, 128, 256), (1024, 4096, 128), (4800, 1600, 300), (12288, 4096, 256),
          (300, 200, 77), (256, 64, 1), (4096, 16384, 128), (4800, 1600, 3), (16384, 4096, 100)]


def _rand_f16(rng, shape, scale=1.0):
    return (rng.standard_normal(shape) * scale).astype(np.float16)


@pytest.mark.parametrize("N,K,M", SHAPES)
def test_tc_fp16_matches_reference(N, K, M):
    rng = np.random.default_rng(N + 3 * K + 7 * M)
    W = _rand_f16(rng, (N, K), 0.05)
    x = _rand_f16(rng, (M, K))
    dev = torch.device("cuda")
    out = E.gemm_large_batch(torch.from_numpy(W).to(dev), torch.from_numpy(x).to(dev)).cpu().numpy()
    ref = x.astype(np.float64) @ W.astype(np.float64).T
    bound = np.abs(x.astype(np.float64)) @ np.abs(W.astype(np.float64)).T
    err = np.abs(out - ref)
    assert np.all(err <= 2e-3 * bound + 1e-3), float((err / (bound + 1e-9)).max())


@pytest.mark.parametrize("N,K,M", [(256, 128, 128), (1024, 4096, 256), (4800, 1600, 300), (300, 208, 77),
                                   (1024, 4096, 64), (4096, 16384, 16), (12288, 4096, 128)])
def test_tc_int8_bit_exact(N, K, M):
    """(M <= 128 with long K runs the split-K cluster mode: int32 partials summed through DSMEM.)"""
    rng = np.random.default_rng(N * 5 + K + M)
    W = rng.standard_normal((N, K)).astype(np.float32) * 0.05
    x = rng.standard_normal((M, K)).astype(np.float32)
    wq, ws = O.quant_rows(W)
    xq, xs = O.quant_rows(x)
    _, ref = O.gemm_i8(wq, ws, xq, xs)
    dev = torch.device("cuda")
    out = E.gemm_large_batch(torch.from_numpy(wq).to(dev), torch.from_numpy(xq).to(dev),
                             w_scales=torch.from_numpy(ws).to(dev), x_scales=torch.from_numpy(xs).to(dev)).cpu().numpy()
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


def test_tc_rejects_unaligned_rows():
    """TMA needs 16-byte row strides: int8 K must be a multiple of 16 (fp16: 8) -> ConfigError."""
    from paper_2207_00032_b200 import _capi as capi
    dev = torch.device("cuda")
    wq = torch.zeros((64, 200), dtype=torch.int8, device=dev)
    s = torch.ones(64, dtype=torch.float32, device=dev)
    with pytest.raises(capi.ConfigError):
        E.gemm_large_batch(wq, wq, w_scales=s, x_scales=s)


def test_tc_epilogues_bias_gelu_resid():
    rng = np.random.default_rng(3)
    N, K, M = 512, 256, 200
    W = _rand_f16(rng, (N, K), 0.05)
    x = _rand_f16(rng, (M, K))
    b = _rand_f16(rng, (N,), 0.1)
    dev = torch.device("cuda")
    Wd, xd, bd = (torch.from_numpy(a).to(dev) for a in (W, x, b))
    y = x.astype(np.float64) @ W.astype(np.float64).T + b.astype(np.float64)
    g = E.gemm_large_batch(Wd, xd, bias=bd, gelu=True).cpu().numpy().astype(np.float64)
    gref = 0.5 * y * (1 + np.tanh(0.7978845608028654 * (y + 0.044715 * y ** 3)))
    assert np.allclose(g, gref, rtol=5e-3, atol=5e-3)
    r0 = rng.standard_normal((M, N)).astype(np.float32)
    r = torch.from_numpy(r0.copy()).to(dev)
    E.gemm_large_batch(Wd, xd, bias=bd, out=r, resid=True)
    assert np.allclose(r.cpu().numpy(), r0 + y, rtol=2e-3, atol=2e-3)


def test_tc_int8_matches_decode_sbi_gemm():
    """The same W8A8 problem through the decode SBI-GeMM (packed layout) and the tensor-core
    path: identical bits (both exact int32 + the same dequant order)."""
    rng = np.random.default_rng(9)
    N, K, M = 1024, 2048, 16
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float16)
    x = rng.standard_normal((M, K)).astype(np.float16)
    dev = torch.device("cuda")
    Wd, xd = torch.from_numpy(W).to(dev), torch.from_numpy(x).to(dev)
    wp, ws = E.quantize_weights_int8(Wd)
    xq, xs = E.quantize_activations_int8(xd)
    wq_rm, ws_rm = E.quantize_activations_int8(Wd)  # per-row quantisation of W, row-major
    assert torch.equal(ws, ws_rm)
    a = E.gemm(wp, xq, N, K, w_scales=ws, x_scales=xs).cpu().numpy()
    b = E.gemm_large_batch(wq_rm, xq, w_scales=ws_rm, x_scales=xs).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("N,K,M", [(1024, 4096, 256), (4800, 1600, 128), (12288, 4096, 64)])
def test_tc_bf16(N, K, M):
    """BF16 operands on the same tcgen05 path (kind::f16 with BF16 A/B formats), fp32 out:
    within 2e-3 * sum|w x| + 1e-3 of the fp64 product of the same bf16 values."""
    g = torch.Generator().manual_seed(N + K + M)
    W = (torch.randn(N, K, generator=g) * 0.05).bfloat16()
    x = torch.randn(M, K, generator=g).bfloat16()
    dev = torch.device("cuda")
    out = E.gemm_large_batch(W.to(dev), x.to(dev)).cpu().double().numpy()
    Wd, xd = W.double().numpy(), x.double().numpy()
    ref = xd @ Wd.T
    bound = np.abs(xd) @ np.abs(Wd).T
    assert np.all(np.abs(out - ref) <= 2e-3 * bound + 1e-3)
