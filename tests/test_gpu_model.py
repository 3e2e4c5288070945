"""End-to-end decode parity: the B200 model (through the C ABI) against the CPU oracle on identical
synthetic weights and prompts.

Stated tolerances (fp16 weights, fp32 accumulation, fp16 activations at the storage points):
  max |logit_gpu - logit_oracle| <= 0.03 * std(logits) + 0.01   (fp16 path)
  max |logit_gpu - logit_oracle| <= 0.06 * std(logits) + 0.02   (int8 W8A8 path)
Greedy token ids are checked at EVERY position: they must be identical, or the GPU's token must be a
near tie whose oracle logit is within 2 x the measured max|dlogit| of the oracle's top token (the
number of such flips is printed); the oracle is always fed the same tokens as the GPU.
"""
import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2207_00032_b200 import _capi as capi  # noqa: E402
from paper_2207_00032_b200.engine import DecoderModel  # noqa: E402

SEED = 20220701


def run_parity(hidden, layers, heads, vocab, *, batch=1, dtype_bytes=2, tp=1, prompt_len=6, gen=4,
               use_graph=True, use_pdl=True, max_ctx=32, step_kernel=False, int8_act=0, oracle_int8_act=None,
               int8_group=0):
    tol_rel, tol_abs = (0.03, 0.01) if dtype_bytes == 2 else (0.06, 0.02)
    if step_kernel and dtype_bytes == 1 and int8_act == capi.INT8_W8A8:
        int8_act = capi.INT8_W8A16  # the persistent step kernel runs INT8 weight-only
    rng = np.random.default_rng(hidden + layers + batch)
    prompt = rng.integers(0, vocab, (batch, prompt_len)).astype(np.int32)
    mode = capi.TP_LOCAL if tp > 1 else capi.TP_NONE
    gpu = DecoderModel(hidden, layers, heads, vocab, dtype_bytes=dtype_bytes, batch=batch, max_ctx=max_ctx,
                       tp_size=tp, tp_mode=mode, use_cuda_graph=use_graph, use_pdl=use_pdl, seed=SEED,
                       use_step_kernel=step_kernel, int8_act=int8_act, int8_group=int8_group)
    ora = O.OracleModel(hidden, layers, heads, vocab, dtype_bytes=dtype_bytes, tp=tp, batch=batch, max_ctx=max_ctx,
                        seed=SEED, int8_act=int8_act if oracle_int8_act is None else oracle_int8_act,
                        int8_group=int8_group)
    gpu.set_prompt(prompt)
    worst = 0.0
    margins = []
    checks = flips = 0
    for pos in range(prompt_len + gen - 1):
        gpu.step(1)
        torch.cuda.synchronize()
        lg = gpu.full_logits()
        nxt, hist = gpu.read_tokens()
        tokens = hist[:, pos]
        ol, onext = ora.step(tokens, pos)
        tol = tol_rel * float(ol.std()) + tol_abs
        err = float(np.abs(lg - ol).max())
        worst = max(worst, err / tol)
        assert err <= tol, f"pos {pos}: max|dlogit| {err:.4g} > tol {tol:.4g}"
        srt = np.sort(ol, axis=1)
        margin = srt[:, -1] - srt[:, -2]
        margins.extend(margin.tolist())
        for b in range(batch):
            checks += 1
            if nxt[b] != onext[b]:
                # only a near tie may flip: the oracle's logit of the GPU's token within 2 max|dlogit|
                gap = float(ol[b, onext[b]] - ol[b, nxt[b]])
                assert gap <= 2 * err, f"pos {pos} b {b}: token {nxt[b]} != oracle {onext[b]} (gap {gap:.4g})"
                flips += 1
    gpu.close()
    ora.close()
    print(f"worst err/tol {worst:.3f}; min top1-top2 margin {min(margins):.4f}; greedy tokens checked {checks}, "
          f"near-tie flips {flips}")
    return worst


PATHS = pytest.mark.parametrize("step_kernel", [True, False], ids=["step_kernel", "per_kernel"])


@PATHS
def test_small_fp16_b1(step_kernel):
    run_parity(256, 2, 4, 1000, step_kernel=step_kernel)


@PATHS
def test_small_fp16_batch3_eager(step_kernel):
    run_parity(256, 2, 4, 1000, batch=3, use_graph=False, use_pdl=False, step_kernel=step_kernel)


@PATHS
def test_small_fp16_batch16(step_kernel):
    run_parity(512, 2, 8, 2000, batch=16, step_kernel=step_kernel)


@PATHS
def test_small_int8_b1(step_kernel):
    run_parity(256, 2, 4, 1000, dtype_bytes=1, step_kernel=step_kernel)


@PATHS
def test_small_int8_batch8(step_kernel):
    run_parity(512, 2, 8, 2000, batch=8, dtype_bytes=1, step_kernel=step_kernel)


@PATHS
def test_gpt2_shape_two_layers(step_kernel):
    """GPT-2 1.5B widths (h=1600, 25 heads, d=64): N and K not multiples of 128, TPP=8 attention."""
    run_parity(1600, 2, 25, 50257, prompt_len=4, gen=3, max_ctx=16, step_kernel=step_kernel)


@PATHS
def test_gpt2_shape_int8_partial_stage(step_kernel):
    """INT8 at GPT-2 widths: K = 1600 ends in a partial 128-k weight stage (zero-filled by TMA), whose
    x words must be zero too (the persistent kernel's whole-row LayerNorm slice)."""
    run_parity(1600, 2, 25, 50257, dtype_bytes=1, prompt_len=4, gen=3, max_ctx=16, step_kernel=step_kernel,
               int8_act=capi.INT8_W8A16)


def test_step_kernel_matches_per_kernel_path():
    """Both TP=1 paths give the same greedy tokens and logits within fp32 split-K reordering."""
    prompt = np.random.default_rng(3).integers(0, 2000, (4, 9)).astype(np.int32)
    res = []
    for sk in (True, False):
        m = DecoderModel(512, 3, 8, 2000, batch=4, max_ctx=32, seed=SEED, use_step_kernel=sk)
        m.set_prompt(prompt)
        m.step(20)
        _, hist = m.read_tokens()
        res.append((hist.copy(), m.full_logits().copy(), m.get_info().kernels_per_step))
        m.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert np.abs(res[0][1] - res[1][1]).max() <= 1e-3 * np.abs(res[1][1]).max()
    assert res[0][2] == 1 and res[1][2] > 1


@pytest.mark.parametrize("tp", [2, 4])
def test_tp_local_fp16(tp):
    run_parity(512, 2, 8, 1000, tp=tp, batch=2)


def test_tp_local_int8():
    run_parity(512, 2, 8, 1000, tp=2, dtype_bytes=1)


def test_gptj_width_one_layer():
    run_parity(4096, 1, 32, 50257, prompt_len=3, gen=2, max_ctx=8)


def test_graph_replay_is_deterministic():
    m = DecoderModel(256, 2, 4, 1000, batch=2, max_ctx=32, seed=SEED)
    prompt = np.arange(10, dtype=np.int32).reshape(2, 5)
    outs = []
    for _ in range(2):
        m.set_prompt(prompt)
        m.step(12)
        _, hist = m.read_tokens()
        outs.append((hist.copy(), m.full_logits().copy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    m.close()


def test_context_capacity_is_enforced():
    m = DecoderModel(256, 1, 4, 1000, max_ctx=8, seed=SEED)
    m.set_prompt(np.zeros((1, 4), dtype=np.int32))
    m.step(8)
    with pytest.raises(capi.InfeasibleError):
        m.step(1)
    m.close()


# Both GEMM plans on both sides of the default batch threshold (gemm::kXsMinBatch = 2):
#   xs:    x streamed by TMA per stage (row_prep launches for LayerNorm / int8 quantisation)
#   slice: x normalised / quantised into a per-CTA smem slice by the GEMM prologue
PLANS = {"xs": {"DSINF_XS": "1", "DSINF_XS_OD": "1"}, "slice": {"DSINF_XS": "0", "DSINF_XS_OD": "0"}}


@pytest.mark.parametrize("plan", list(PLANS))
@pytest.mark.parametrize("dtype_bytes,batch", [(2, 1), (2, 16), (1, 1), (1, 8)], ids=["f16b1", "f16b16", "i8b1", "i8b8"])
def test_gemm_plans(monkeypatch, plan, dtype_bytes, batch):
    for k, v in PLANS[plan].items():
        monkeypatch.setenv(k, v)
    run_parity(512, 2, 8, 2000, batch=batch, dtype_bytes=dtype_bytes, step_kernel=False)


@pytest.mark.parametrize("dtype_bytes", [2, 1], ids=["f16", "i8"])
def test_tp_local_x_stream(monkeypatch, dtype_bytes):
    """TP without producer statistics: row_prep sums the residual itself and writes it back."""
    monkeypatch.setenv("DSINF_XS", "1")
    run_parity(512, 2, 8, 1000, tp=2, batch=4, dtype_bytes=dtype_bytes, step_kernel=False)


def run_prefill_parity(hidden, layers, heads, vocab, *, batch=1, dtype_bytes=2, prompt_len=40, gen=3, max_ctx=64,
                       tp=1):
    """Prefill (tcgen05 large-batch path) vs the oracle stepping through the prompt token by token;
    then `gen` decode steps from the prefilled KV cache.  Same tolerances as run_parity."""
    tol_rel, tol_abs = (0.03, 0.01) if dtype_bytes == 2 else (0.06, 0.02)
    rng = np.random.default_rng(hidden * 3 + layers + batch + prompt_len)
    prompt = rng.integers(0, vocab, (batch, prompt_len)).astype(np.int32)
    gpu = DecoderModel(hidden, layers, heads, vocab, dtype_bytes=dtype_bytes, batch=batch, max_ctx=max_ctx, seed=SEED,
                       tp_size=tp, tp_mode=capi.TP_LOCAL if tp > 1 else capi.TP_NONE)
    ora = O.OracleModel(hidden, layers, heads, vocab, dtype_bytes=dtype_bytes, batch=batch, max_ctx=max_ctx, seed=SEED,
                        tp=tp)
    gpu.set_prompt(prompt)
    gpu.prefill()
    torch.cuda.synchronize()
    for pos in range(prompt_len):
        ol, onext = ora.step(prompt[:, pos], pos)
    worst = 0.0
    for g in range(gen + 1):
        pos = prompt_len - 1 + g
        if g > 0:
            gpu.step(1)
            torch.cuda.synchronize()
        lg = gpu.full_logits()
        nxt, hist = gpu.read_tokens()
        if g > 0:
            ol, onext = ora.step(hist[:, pos], pos)
        else:
            assert np.array_equal(hist[:, :prompt_len], prompt)
        tol = tol_rel * float(ol.std()) + tol_abs
        err = float(np.abs(lg - ol).max())
        worst = max(worst, err / tol)
        assert err <= tol, f"pos {pos}: max|dlogit| {err:.4g} > tol {tol:.4g}"
        srt = np.sort(ol, axis=1)
        for b in range(batch):
            if srt[b, -1] - srt[b, -2] > tol:
                assert nxt[b] == onext[b], f"pos {pos} b {b}: token {nxt[b]} != oracle {onext[b]}"
    assert int(gpu.read_tokens()[1][0, prompt_len]) == int(hist[0, prompt_len])
    gpu.close()
    ora.close()
    return worst


@pytest.mark.parametrize("dtype_bytes", [2, 1])
@pytest.mark.parametrize("batch,prompt_len", [(1, 40), (3, 50), (2, 130)])
def test_prefill_matches_oracle_small(dtype_bytes, batch, prompt_len):
    run_prefill_parity(256, 2, 4, 1000, batch=batch, dtype_bytes=dtype_bytes, prompt_len=prompt_len,
                       max_ctx=prompt_len + 8)


@pytest.mark.parametrize("dtype_bytes", [2, 1])
def test_prefill_matches_oracle_head_dim_128(dtype_bytes):
    run_prefill_parity(1024, 2, 8, 2000, batch=2, dtype_bytes=dtype_bytes, prompt_len=96, max_ctx=104)


@pytest.mark.parametrize("dtype_bytes", [2, 1])
def test_prefill_equals_token_by_token_decode(dtype_bytes):
    """The large-batch prefill and P decode steps over the prompt leave the same state: same
    history and greedy continuation, logits within the fp16 / int8 tolerance."""
    hidden, layers, heads, vocab, B, P = 512, 3, 8, 3000, 4, 64
    rng = np.random.default_rng(77)
    prompt = rng.integers(0, vocab, (B, P)).astype(np.int32)
    a = DecoderModel(hidden, layers, heads, vocab, dtype_bytes=dtype_bytes, batch=B, max_ctx=80, seed=SEED)
    b = DecoderModel(hidden, layers, heads, vocab, dtype_bytes=dtype_bytes, batch=B, max_ctx=80, seed=SEED)
    a.set_prompt(prompt)
    b.set_prompt(prompt)
    a.prefill()
    b.step(P)
    torch.cuda.synchronize()
    la, lb = a.full_logits(), b.full_logits()
    tol = (0.03 if dtype_bytes == 2 else 0.06) * float(lb.std()) + (0.01 if dtype_bytes == 2 else 0.02)
    assert float(np.abs(la - lb).max()) <= tol
    ha, hb = a.read_tokens()[1], b.read_tokens()[1]
    assert np.array_equal(ha[:, :P], hb[:, :P])
    srt = np.sort(lb, axis=1)
    for i in range(B):  # greedy token identical unless the top-1/top-2 margin is inside the tolerance
        if srt[i, -1] - srt[i, -2] > tol:
            assert ha[i, P] == hb[i, P]
    a.close()
    b.close()


def test_prefill_rejects_bad_state():
    gpu = DecoderModel(256, 1, 4, 1000, batch=1, max_ctx=16, seed=SEED)
    with pytest.raises(capi.ConfigError):
        gpu.prefill()  # no prompt
    gpu.set_prompt(np.array([[1, 2, 3]], dtype=np.int32))
    gpu.step(1)
    with pytest.raises(capi.ConfigError):
        gpu.prefill()  # not at position 0
    gpu.close()


@pytest.mark.parametrize("batch", [1, 3, 8, 16])
def test_int8_weight_only_model_matches_oracle(batch):
    """W8A16 decode (int8 weights, fp16 activations) against the oracle's W8A16 mode."""
    run_parity(256, 2, 4, 1000, batch=batch, dtype_bytes=1, int8_act=1, step_kernel=False)


def test_int8_weight_only_gptj_width_layer():
    run_parity(4096, 1, 32, 2000, batch=1, dtype_bytes=1, int8_act=1, step_kernel=False, prompt_len=4, gen=3)


@pytest.mark.parametrize("dtype_bytes", [2, 1])
@pytest.mark.parametrize("tp", [2, 4])
def test_prefill_tensor_parallel_matches_oracle(dtype_bytes, tp):
    """Prefill with Megatron TP (column-parallel QKV / up, row-parallel attn-out / down with an
    all-reduce of the [M][h] partials, vocab-parallel LM head) on one device, vs the TP-aware oracle."""
    run_prefill_parity(512, 2, 8, 1000, batch=2, dtype_bytes=dtype_bytes, prompt_len=48, max_ctx=56, tp=tp)


@pytest.mark.parametrize("dtype_bytes", [2, 1])
@pytest.mark.parametrize("tp,batch", [(2, 1), (4, 3), (8, 2)])
@pytest.mark.parametrize("xs", ["0", "1"])
def test_fused_allreduce_tp_matches_oracle(dtype_bytes, tp, batch, xs, monkeypatch):
    """Tensor parallelism with the fused all-reduce (row-parallel epilogues push their partials into
    every rank's slots and bump a counter; the next LayerNorm prologue waits and sums the slots in
    rank order) against the TP-aware oracle, graph-replayed over several steps."""
    monkeypatch.setenv("DSINF_FUSED_AR", "1")
    # the fused slots are summed by the per-CTA LayerNorm prologues (slice plan, DSINF_XS=0) or by
    # the row_prep launches of the x-streaming plan (DSINF_XS=1)
    monkeypatch.setenv("DSINF_XS", xs)
    run_parity(512, 3, 8, 1000, batch=batch, dtype_bytes=dtype_bytes, tp=tp, step_kernel=False, prompt_len=5, gen=4)


@pytest.mark.parametrize("xs", ["0", "1"])
def test_fused_allreduce_equals_explicit_allreduce(monkeypatch, xs):
    """Same TP=4 model and plan with the fused all-reduce and with explicit on-device all-reduce
    launches: identical greedy tokens, logits within fp32 summation-order noise, and exactly the
    all-reduce launches (2 per layer) fewer."""
    rng = np.random.default_rng(5)
    prompt = rng.integers(0, 1000, (2, 6)).astype(np.int32)
    outs, launches = [], []
    monkeypatch.setenv("DSINF_XS", xs)
    for fused in ("1", "0"):
        monkeypatch.setenv("DSINF_FUSED_AR", fused)
        m = DecoderModel(512, 2, 8, 1000, batch=2, max_ctx=24, tp_size=4, tp_mode=capi.TP_LOCAL, seed=SEED)
        m.set_prompt(prompt)
        m.step(10)
        torch.cuda.synchronize()
        outs.append((m.full_logits(), m.read_tokens()[1]))
        info = m.get_info()
        launches.append(info.kernels_per_step)
        assert info.fused_allreduce == (1 if fused == "1" else 0)
        m.close()
    assert launches[1] - launches[0] == 2 * 2, launches  # 2 layers x (attn-out, MLP-down) all-reduces
    (la, ha), (lb, hb) = outs
    assert np.array_equal(ha, hb)
    assert float(np.abs(la - lb).max()) <= 1e-3 * float(np.abs(lb).max()) + 1e-4


@pytest.mark.parametrize("batch,oracle_act", [(1, 1), (8, 1), (16, 1)])
def test_int8_auto_mode_matches_oracle(batch, oracle_act):
    """DSINF_INT8_AUTO at TP = 1: weight-only (W8A16) at every batch (B = 16 was W8A8 QKV + W8A16 the
    rest until the round-2 tuning pass) -- against the oracle's same per-GEMM modes."""
    run_parity(256, 2, 4, 1000, batch=batch, dtype_bytes=1, int8_act=capi.INT8_AUTO, step_kernel=False,
               oracle_int8_act=oracle_act)


@pytest.mark.parametrize("dtype_bytes", [2, 1])
def test_tp_slice_mode(dtype_bytes):
    """DSINF_TP_SLICE (per-rank timing of a TP model on one GPU): rank r's shard alone, collectives
    skipped.  Deterministic, greedy tokens come from the rank's own vocab slice, and the per-rank
    step bytes equal 1/t of the TP=1 weight stream plus the replicated parts."""
    rng = np.random.default_rng(9)
    V, t = 1000, 4
    prompt = rng.integers(0, V, (2, 6)).astype(np.int32)
    vl = (V + 128 * t - 1) // (128 * t) * 128
    for rank in (0, 3):
        hists = []
        for _ in range(2):
            m = DecoderModel(512, 2, 8, V, dtype_bytes=dtype_bytes, batch=2, max_ctx=24, tp_size=t, tp_rank=rank,
                             tp_mode=capi.TP_SLICE, seed=SEED)
            m.set_prompt(prompt)
            m.prefill()
            m.step(6)
            torch.cuda.synchronize()
            _, hist = m.read_tokens()
            hists.append(hist[:, 6:12].copy())
            m.close()
        assert np.array_equal(hists[0], hists[1])
        lo, hi = rank * vl, min(V, (rank + 1) * vl)
        assert ((hists[0] >= lo) & (hists[0] < hi)).all(), (rank, hists[0])


@pytest.mark.parametrize("split", [2, 8])
@pytest.mark.parametrize("dtype_bytes,tp", [(2, 1), (1, 1), (2, 2), (1, 2)], ids=["f16", "i8", "f16tp2", "i8tp2"])
def test_row_prep_cluster_split(monkeypatch, split, dtype_bytes, tp):
    """row_prep with each row split over a cluster of CTAs (row sums / maxima exchanged through
    DSMEM; TP = 2 exercises the sums computed in the kernel) gives the same parity as one CTA."""
    monkeypatch.setenv("DSINF_PREP_SPLIT", str(split))
    monkeypatch.setenv("DSINF_XS", "1")
    run_parity(512, 2, 8, 1000, tp=tp, batch=4, dtype_bytes=dtype_bytes, step_kernel=False)


def test_int8_auto_mode_tp_matches_oracle():
    """DSINF_INT8_AUTO at TP > 1 and batch 16: W8A8 everywhere."""
    run_parity(256, 2, 4, 1000, batch=16, dtype_bytes=1, tp=2, int8_act=capi.INT8_AUTO, step_kernel=False,
               oracle_int8_act=0)


@pytest.mark.parametrize("mask", [0x5, 0xa])
def test_int8_mixed_mask_matches_oracle(monkeypatch, mask):
    """Per-GEMM activation modes (DSINF_A16_MASK) against the oracle's per-GEMM mask."""
    monkeypatch.setenv("DSINF_A16_MASK", hex(mask))
    run_parity(256, 2, 4, 1000, batch=4, dtype_bytes=1, int8_act=capi.INT8_W8A8, step_kernel=False,
               oracle_int8_act=0x100 | mask)


def test_generate_fills_max_ctx_and_rejects_beyond():
    """generate() returns exactly gen_tokens columns up to P + gen == max_ctx and raises past it."""
    m = DecoderModel(256, 1, 4, 1000, max_ctx=12, seed=SEED)
    prompt = np.arange(1, 5, dtype=np.int32).reshape(1, 4)
    out = m.generate(prompt, 8)
    assert out.shape == (1, 8)
    with pytest.raises(capi.InfeasibleError):
        m.generate(prompt, 9)
    m.close()


@pytest.mark.parametrize("dtype_bytes", [2, 1])
def test_prefill_single_weight_copy_identical(dtype_bytes, monkeypatch):
    """DSINF_PREFILL_REPACK=1 (chosen automatically when the row-major prefill copies of every layer
    do not fit): the tensor-core prefill re-fills ONE layer's row-major operands from the packed
    decode weights before each layer, so the model holds a single resident weight copy.  Same GEMM
    operands, so the prefill logits and the following decode are bit-identical to the copy mode."""
    rng = np.random.default_rng(17)
    prompt = rng.integers(0, 1000, (2, 40)).astype(np.int32)
    outs = []
    for rp in ("0", "1"):
        monkeypatch.setenv("DSINF_PREFILL_REPACK", rp)
        m = DecoderModel(512, 2, 8, 1000, dtype_bytes=dtype_bytes, batch=2, max_ctx=48, seed=SEED)
        m.set_prompt(prompt)
        m.prefill()
        torch.cuda.synchronize()
        lg = m.full_logits()
        m.step(3)
        torch.cuda.synchronize()
        outs.append((lg, m.full_logits(), m.read_tokens()[1]))
        m.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("tp,batch", [(1, 1), (1, 5), (2, 3), (4, 2)])
def test_int8_k_group_decode_matches_oracle(tp, batch):
    """INT8 decode with K-group weight scales (int8_group = 128, "per-group
    dequant"): every layer GEMM weight-only with the per-group dequant in the SBI-GeMM main loop,
    against the oracle's K-group restatement (same q and fp16 scales, fp64 sums), TP shards on one
    device included (a group never straddles a shard)."""
    run_parity(512, 2, 8, 1000, batch=batch, dtype_bytes=1, tp=tp, int8_act=capi.INT8_W8A16, int8_group=128)


def test_int8_k_group_rejects_w8a8():
    with pytest.raises(capi.ConfigError):
        DecoderModel(256, 1, 4, 1000, dtype_bytes=1, batch=1, max_ctx=16, int8_act=capi.INT8_W8A8, int8_group=128)


@pytest.mark.parametrize("batch,d_heads", [(1, 4), (5, 8), (16, 4)])
def test_attention_bulk_copy_variant(batch, d_heads, monkeypatch):
    """DSINF_ATTN_TMA=1: decode attention streaming each chunk's contiguous K/V rows through a
    2-stage shared-memory ring with 1-D bulk copies (cp.async.bulk + mbarrier) -- against the oracle,
    head dims 128 and 64, contexts longer than one 32-row stage."""
    monkeypatch.setenv("DSINF_ATTN_TMA", "1")
    run_parity(512, 2, d_heads, 1000, batch=batch, prompt_len=40, gen=4, max_ctx=48)


@pytest.mark.parametrize("dtype_bytes,batch,int8_act", [(2, 1, 0), (2, 16, 0), (1, 1, capi.INT8_W8A16),
                                                         (1, 16, capi.INT8_AUTO)])
def test_layernorm_streaming_plan(dtype_bytes, batch, int8_act, monkeypatch):
    """LayerNorm-streaming (TP = 1): the LayerNorm GEMMs stream the fp32 residual with their weights
    and normalise each stage in shared memory with the producer's row sums -- the row_prep launches
    of Deep-Fusion regions 1 and 3 (and the LM head's) disappear.  Same LayerNorm expression as
    row_prep: identical greedy tokens, logits equal to fp32 rounding, 2L + 1 fewer launches; and against
    the oracle."""
    rng = np.random.default_rng(31)
    prompt = rng.integers(0, 1000, (batch, 6)).astype(np.int32)
    outs, launches = [], []
    for ls in ("0", "1"):
        monkeypatch.setenv("DSINF_LN_STREAM", ls)
        m = DecoderModel(512, 3, 8, 1000, dtype_bytes=dtype_bytes, batch=batch, max_ctx=24, seed=SEED,
                         int8_act=int8_act)
        m.set_prompt(prompt)
        m.step(9)
        torch.cuda.synchronize()
        outs.append((m.full_logits(), m.read_tokens()[1]))
        launches.append(m.get_info().kernels_per_step)
        m.close()
    (la, ha), (lb, hb) = outs
    assert np.array_equal(ha, hb)
    assert float(np.abs(la - lb).max()) <= 1e-3 * float(np.abs(la).max()) + 1e-4
    fewer = 2 * 3 + 1
    assert launches[0] - launches[1] == fewer, launches
    monkeypatch.setenv("DSINF_LN_STREAM", "1")
    run_parity(512, 2, 8, 1000, batch=batch, dtype_bytes=dtype_bytes, int8_act=int8_act,
               oracle_int8_act=None if int8_act != capi.INT8_AUTO else 0x10f)


@pytest.mark.parametrize("dtype_bytes,batch,int8_act", [(2, 1, 0), (2, 8, 0), (1, 1, capi.INT8_W8A16)])
def test_down_flag_dependency(dtype_bytes, batch, int8_act, monkeypatch):
    """DSINF_DOWN_FLAGS=1: MLP-down is PDL-launched and its producer waits only for the MLP-up column
    tiles of its k range (monotonic per-tile counters, +1 per MLP-up CTA after its epilogue stores),
    the epilogue for the whole MLP-up grid.  Same arithmetic: bit-identical logits and tokens over
    many graph-replayed steps (the counters carry across steps), and against the oracle."""
    rng = np.random.default_rng(41)
    prompt = rng.integers(0, 1000, (batch, 6)).astype(np.int32)
    outs = []
    for df in ("0", "1"):
        monkeypatch.setenv("DSINF_DOWN_FLAGS", df)
        m = DecoderModel(512, 3, 8, 1000, dtype_bytes=dtype_bytes, batch=batch, max_ctx=40, seed=SEED,
                         int8_act=int8_act)
        m.set_prompt(prompt)
        m.step(12)
        torch.cuda.synchronize()
        m.set_prompt(prompt)  # a second sequence on the same counters (re-captured graph)
        m.step(20)
        torch.cuda.synchronize()
        outs.append((m.full_logits(), m.read_tokens()[1]))
        m.close()
    assert np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][0], outs[1][0])
    monkeypatch.setenv("DSINF_DOWN_FLAGS", "1")
    run_parity(512, 2, 8, 1000, batch=batch, dtype_bytes=dtype_bytes, int8_act=int8_act)


@pytest.mark.parametrize("hidden,heads,dtype_bytes,batch,int8_act", [(512, 4, 2, 1, 0), (512, 8, 2, 3, 0),
                                                                     (768, 8, 2, 1, 0),
                                                                     (512, 4, 1, 1, capi.INT8_W8A16),
                                                                     (512, 8, 1, 2, capi.INT8_W8A16)])
def test_qkv_attention_tail(hidden, heads, dtype_bytes, batch, int8_act, monkeypatch):
    """DSINF_ATTN_FUSE=1: decode attention runs in the tail of the QKV launch (the cluster completing a
    head's q / k / v column tiles attends for it, its K splits merging the context chunks through
    DSMEM); one launch per layer fewer, same tokens as the standalone attention and the oracle.  Head
    dims 128, 64 and 96 (768 / 8: tiles straddle heads)."""
    rng = np.random.default_rng(53)
    prompt = rng.integers(0, 1000, (batch, 5)).astype(np.int32)
    outs, launches = [], []
    for f in ("0", "1"):
        monkeypatch.setenv("DSINF_ATTN_FUSE", f)
        m = DecoderModel(hidden, 3, heads, 1000, dtype_bytes=dtype_bytes, batch=batch, max_ctx=40, seed=SEED,
                         int8_act=int8_act)
        m.set_prompt(prompt)
        m.step(20)  # graph replays: the head counters must return to zero every step
        torch.cuda.synchronize()
        outs.append((m.full_logits(), m.read_tokens()[1]))
        launches.append(m.get_info().kernels_per_step)
        m.close()
    (la, ha), (lb, hb) = outs
    assert launches[0] - launches[1] == 3, launches
    assert np.array_equal(ha, hb)
    assert float(np.abs(la - lb).max()) <= 2e-3 * float(np.abs(la).max()) + 1e-3
    monkeypatch.setenv("DSINF_ATTN_FUSE", "1")
    run_parity(hidden, 2, heads, 1000, batch=batch, dtype_bytes=dtype_bytes, int8_act=int8_act)
