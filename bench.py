#!/usr/bin/env python3
"""Decode benchmark of the B200 DeepSpeed-Inference hot path (BASELINE.json configs[1]: GPT-J-6B shape).

One "step" = one greedy decode step (one token per sequence) through every layer, the LM head and
the argmax, replayed from a CUDA graph.  Default: N=1, GPT-J-6B fp16, batch 1, 128-token prompt.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config gptj-6b] [--dtype fp16|int8] [--batch 1]

N > 1 is launched by torchrun (one process per GPU, NCCL over NVLink): tensor parallel TP=N of the
same model (strong scaling), timed on the device as the max over ranks.
`--impl reference` times the reference's own CPU implementation of the path (exec_reference from
the reference headers, oracle/_ref) on the host cores, for the same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20220701
METRIC = "decode_tokens_per_s"


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def measured_tensor_peak():
    """Dense bf16 TFLOP/s for a kernel timed alone (burst), measured or the recipe's fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["bf16_tflops"]), "measured"
    return 1590.0, "fallback"


def tc_roofline(E, torch, preset, M, dtype, stream):
    """The prefill's dominant kernel: the tcgen05 GEMM at the layer shapes with M = batch x prompt,
    each timed alone (CUDA-graph replays, CUDA events on the launching stream).  Returns the
    flop-weighted TFLOP/s (TOP/s for int8) and the per-shape table."""
    i8 = dtype == "int8"
    dev = torch.device("cuda")
    rows = []
    tot_f = tot_t = 0.0
    for name, N, K in gemm_shapes(preset, 1)[0]:
        if i8:
            w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
            x = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
            ws, xs = torch.rand(N, device=dev) * 1e-3, torch.rand(M, device=dev) * 1e-2
        else:
            w = (torch.randn(N, K, device=dev) * 0.02).half()
            x = torch.randn(M, K, device=dev).half()
            ws = xs = None
        out = torch.empty(M, N, dtype=torch.float16, device=dev)
        reps = 10
        with torch.cuda.stream(stream):
            for _ in range(3):
                E.gemm_large_batch(w, x, w_scales=ws, x_scales=xs, out=out, stream=stream)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(reps):
                    E.gemm_large_batch(w, x, w_scales=ws, x_scales=xs, out=out, stream=stream)
        torch.cuda.synchronize()
        best = 1e9
        with torch.cuda.stream(stream):  # replay on the stream the events are recorded on
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g.replay()
                b.record(stream)
                b.synchronize()
                best = min(best, a.elapsed_time(b) / reps)
        f = 2.0 * M * N * K
        rows.append({"kernel": f"tc_gemm[{name}] M={M} N={N} K={K}", "us": round(best * 1e3, 2),
                     "tflops": round(f / (best * 1e-3) / 1e12, 1)})
        tot_f += f
        tot_t += best * 1e-3
        del g
    return tot_f / tot_t / 1e12, rows


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a while to start: wait for its first sample, then count only the
            # samples taken from here on (inside the caller's timed region)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.005)
            self.first = len(self.lines)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines[getattr(self, "first", 0):]
        outside = not lines
        if outside:  # timed region shorter than one sampling period: the last sample before it
            lines = self.lines[-1:]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": 0 if outside else len(sm)}


# ---------------------------------------------------------------- CPU reference path (exec_reference)

def gemm_shapes(preset, tp):
    h = preset.hidden
    vpad = (preset.vocab + 128 * tp - 1) // (128 * tp) * (128 * tp)
    layer = [("qkv", 3 * h // tp, h), ("attn_out", h, h // tp), ("mlp_up", 4 * h // tp, h), ("mlp_down", h, 4 * h // tp)]
    return layer, ("lm_head", vpad // tp, h)


def reference_ms_per_token(preset, tp, batch, dtype_bytes, budget_s, threads, rows_cache=None):
    """exec_reference (gemm.hpp:147-202, compiled from the reference headers) on a row sample of every
    per-rank GEMM of one decode step; per-token time = L * sum(layer GEMMs) + LM head, each scaled
    from its row sample (every output row costs the same).  Returns (ms_per_token, kind, sample).
    `rows_cache` (dict) keeps the calibrated sample sizes across calls."""
    from oracle import oracle as O

    layer, lm = gemm_shapes(preset, tp)
    shapes = layer + [lm]
    ref = O.ref_lib()
    kind = "reference" if ref is not None else "port"
    per_shape = budget_s / len(shapes)
    total_ms = 0.0
    rows_used = {}
    for name, N, K in shapes:
        if rows_cache is not None and name in rows_cache:
            rows = rows_cache[name]
        else:
            # calibrate: time a small sample, then size the real sample to the per-shape budget
            rows = max(threads, 64)
            t = _time_rows(O, ref, N, K, batch, dtype_bytes, rows, threads)
            rate = t / rows
            rows = int(min(N, max(threads, per_shape / max(rate, 1e-9))))
            if rows_cache is not None:
                rows_cache[name] = rows
        t = _time_rows(O, ref, N, K, batch, dtype_bytes, rows, threads)
        ms_full = t * (N / rows) * 1e3
        rows_used[name] = rows
        total_ms += ms_full * (preset.layers if name != "lm_head" else 1)
    sample = "exec_reference on row samples " + ", ".join(f"{k}:{v}" for k, v in rows_used.items()) + \
             f" of each per-rank GEMM (B={batch}), x{threads} threads, extrapolated to L={preset.layers} layers + LM head"
    return total_ms, kind, sample


def _time_rows(O, ref, N, K, B, dtype_bytes, rows, threads):
    import ctypes as C

    if ref is not None:
        cs = C.c_double()
        return float(ref.ref_time_exec(N, K, B, dtype_bytes, 148, rows, threads, SEED, C.byref(cs)))
    # port: the oracle's same-order restatement (multi-threaded)
    W = np.random.default_rng(0).standard_normal((rows, K)).astype(np.float32)
    x = np.random.default_rng(1).standard_normal((B, K))
    s = O.derive_schedule(N, K, B, dtype_bytes)
    t0 = time.perf_counter()
    O.gemm_f64(W, x, s)
    return time.perf_counter() - t0


def cpu_model_name():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ReferenceStep:
    """One whole decode step of the reference's CPU path (oracle/_ref, compiled from the reference
    headers): every per-rank GEMM of all L layers plus the LM head, each a full exec_reference over all
    its output rows, rows split across `threads` host threads.  Weights of each distinct shape are
    generated and packed once, outside the timed calls."""

    def __init__(self, preset, tp, batch, dtype_bytes, threads):
        import ctypes as C

        from oracle import oracle as O

        self.ref = O.ref_lib()
        if self.ref is None:
            raise RuntimeError("oracle/_ref is not built")
        layer, lm = gemm_shapes(preset, tp)
        shapes = layer + [lm]
        nk = (C.c_int64 * (2 * len(shapes)))(*[v for _, N, K in shapes for v in (N, K)])
        reps = (C.c_int64 * len(shapes))(*[preset.layers] * len(layer) + [1])
        self.threads = threads
        self.h = self.ref.ref_step_create(nk, reps, len(shapes), batch, dtype_bytes, 148, threads, SEED)
        self.desc = (f"whole decode steps: exec_reference over every output row of the {len(layer)} per-rank layer "
                     f"GEMMs x {preset.layers} layers + the LM head (B={batch}), rows split over {threads} threads")

    def run(self):
        return float(self.ref.ref_step_run(self.h, self.threads))

    def close(self):
        if self.h:
            self.ref.ref_step_destroy(self.h)
            self.h = None


def run_reference(args, preset, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    dtype_bytes = 1 if args.dtype == "int8" else 2
    # estimate one whole step from a short row sample; time whole steps when the full --warmup +
    # --steps run fits in ~3 minutes of host time, else time bounded row samples and extrapolate
    est_ms, kind, _ = reference_ms_per_token(preset, world, args.batch, dtype_bytes, 2.0, threads)
    runs = args.warmup + args.steps
    vals = []
    if est_ms * 1e-3 * runs <= args.ref_full_budget:
        st = ReferenceStep(preset, world, args.batch, dtype_bytes, threads)
        for i in range(runs):
            t = st.run()
            if i >= args.warmup:
                vals.append(t * 1e3)
        sample = st.desc
        st.close()
    else:
        budget = max(1.0, min(args.ref_step_budget, 50.0 / max(1, runs)))
        rows_cache = {}
        for i in range(runs):
            ms, kind, sample = reference_ms_per_token(preset, world, args.batch, dtype_bytes, budget, threads, rows_cache)
            if i >= args.warmup:
                vals.append(ms)
        sample = "extrapolated (a whole step exceeds the time budget): " + sample
    ms = statistics.median(vals)
    value = args.batch * 1e3 / ms
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, preset, world),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": kind, "sample": sample,
                         "cpu_model": cpu_model_name()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def auto_act(batch, tp):
    """The per-GEMM INT8 activation modes DSINF_INT8_AUTO picks (model.cu, dsinf_model_create)."""
    if batch <= 8 or tp == 1:
        return "w8a16"
    return "w8a8"


def workload_config(args, preset, world):
    cfg = {"workload": f"{preset.name} {args.dtype} greedy decode, batch {args.batch}, {args.prompt}-token prompt, "
                       f"TP={world}", "model": args.config, "global_batch": args.batch, "seq_len": args.prompt,
           "parallelism": f"tp{world}", "l2": "weights per step (GB) >> 126 MB L2; no flush needed"}
    if world > 1:
        cfg["collectives"] = ("all-reduces fused into the row-parallel GEMM epilogues over CUDA-IPC peer memory "
                              "(DSINF_TP_IPC)" if args.tp_mode == "ipc" else "NCCL all-reduce / all-gather launches")
    if args.dtype == "int8":
        cfg["int8_act"] = auto_act(args.batch, world) if args.int8_act == "auto" else args.int8_act
        cfg["int8_scales"] = "K-group 128 (fp16)" if args.int8_group else "per output row (fp32)"
    return cfg


# ---------------------------------------------------------------- our path

def decode_sweep(E, capi, torch, preset, args, stream, peak_gbs, skip):
    """BASELINE.json's full decode metric on one GPU: ms/token, tokens/s and step GB/s (fraction of
    the measured HBM peak) for fp16 / int8 at batch 1 / 8 / 16, each a fresh model (prompt prefilled
    on the tensor cores), device-timed over args.steps decode steps with CUDA events."""
    rows = []
    for dtype in ("fp16", "int8"):
        for batch in (1, 8, 16):
            if (dtype, batch) == skip:
                continue
            m = E.DecoderModel(preset.hidden, preset.layers, preset.heads, preset.vocab,
                               dtype_bytes=1 if dtype == "int8" else 2, batch=batch,
                               max_ctx=args.prompt + args.warmup + args.steps + 8, seed=SEED,
                               int8_act={"w8a8": capi.INT8_W8A8, "w8a16": capi.INT8_W8A16,
                                         "auto": capi.INT8_AUTO}[args.int8_act])
            prompt = np.random.default_rng(SEED + batch).integers(0, preset.vocab, (batch, args.prompt)).astype(np.int32)
            m.set_prompt(prompt, stream=stream)
            m.prefill(stream=stream)
            m.step(args.warmup, stream=stream)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m.step(args.steps, stream=stream)
            b.record(stream)
            b.synchronize()
            ms = a.elapsed_time(b)
            pos0 = args.prompt + args.warmup
            gb = sum(m.bytes_per_step(q) for q in range(pos0, pos0 + args.steps)) / (ms * 1e-3) / 1e9
            mode = (auto_act(batch, 1) if args.int8_act == "auto" else args.int8_act) \
                if dtype == "int8" else None
            rows.append({"dtype": dtype, "batch": batch, "int8_act": mode, "ms_per_token": round(ms / args.steps, 4),
                         "tokens_per_s": round(batch * args.steps * 1e3 / ms, 1), "step_gbs": round(gb, 1),
                         "frac": round(gb / peak_gbs, 4)})
            m.close()
    return rows


def tp_slice_sweep(E, capi, torch, args, stream, peak_gbs):
    """The TP configs of BASELINE.json (NeoX-20B t=2, GPT-50B t=4, GPT3-175B t=8) measured per rank
    on this one GPU: rank 0's shard alone (DSINF_TP_SLICE -- the same kernels and per-rank bytes,
    the two per-layer all-reduces and the argmax all-gather skipped), device-timed like the main
    line.  It is the compute floor of each rank's step; the TP=t step adds the collectives."""
    rows = []
    for name in ("gpt-neox-20b", "gpt-50b", "gpt3-175b"):
        pr = E.PRESETS[name]
        for dtype in ("fp16", "int8"):
            for batch in (1, 16):
                m = E.DecoderModel(pr.hidden, pr.layers, pr.heads, pr.vocab, dtype_bytes=1 if dtype == "int8" else 2,
                                   batch=batch, max_ctx=args.prompt + args.warmup + args.steps + 8, tp_size=pr.tp,
                                   tp_rank=0, tp_mode=capi.TP_SLICE, seed=SEED,
                                   int8_act={"w8a8": capi.INT8_W8A8, "w8a16": capi.INT8_W8A16,
                                             "auto": capi.INT8_AUTO}[args.int8_act])
                prompt = np.random.default_rng(SEED + batch).integers(0, pr.vocab, (batch, args.prompt)).astype(np.int32)
                m.set_prompt(prompt, stream=stream)
                m.prefill(stream=stream)
                m.step(args.warmup, stream=stream)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                m.step(args.steps, stream=stream)
                b.record(stream)
                b.synchronize()
                ms = a.elapsed_time(b)
                pos0 = args.prompt + args.warmup
                gb = sum(m.bytes_per_step(q) for q in range(pos0, pos0 + args.steps)) / (ms * 1e-3) / 1e9
                rows.append({"config": name, "tp": pr.tp, "dtype": dtype, "batch": batch,
                             "rank_ms_per_token": round(ms / args.steps, 4), "rank_step_gbs": round(gb, 1),
                             "frac": round(gb / peak_gbs, 4)})
                m.close()
    return rows


def kernel_roofline(E, torch, preset, tp, batch, dtype, peak_gbs, stream):
    """Times each SBI-GeMM shape of one layer (+ LM head) alone with CUDA events on the launching
    stream (20 drop-in dsinf_gemm calls captured in a CUDA graph and replayed); 4 rotating weight
    copies (> L2) per shape.  Returns the per-kernel list and the byte-weighted
    aggregate for the dominant kernel family (sbi_gemm_kernel)."""
    layer, lm = gemm_shapes(preset, tp)
    dev = torch.device("cuda")
    res = []
    tot_b, tot_t = 0.0, 0.0
    for name, N, K in layer + [lm]:
        int8 = dtype == "int8" and name != "lm_head"
        copies = []
        for c in range(4):
            w = (torch.randn(N, K, device=dev) * 0.02).half()
            if int8:
                copies.append(E.quantize_weights_int8(w))
            else:
                copies.append((E.pack_weights_device(w, 2), None))
            del w
        x = torch.randn(batch, K, device=dev).half()
        out = torch.empty(batch, N, device=dev, dtype=torch.float32)
        for i in range(3):
            wq, ws = copies[i % 4]
            E.gemm(wq, x, N, K, w_scales=ws, out=out, stream=stream)
        # the n calls captured once into a CUDA graph and replayed: device time of the launches,
        # not the host's ctypes / launch overhead between back-to-back small calls
        n = 20
        graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(n):
                wq, ws = copies[i % 4]
                E.gemm(wq, x, N, K, w_scales=ws, out=out, stream=stream)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):  # replay() launches on the current stream
            graph.replay()
            torch.cuda.synchronize()
            st.record(stream)
            graph.replay()
            en.record(stream)
        en.synchronize()
        ms = st.elapsed_time(en) / n
        algo = gemm_algo_bytes(N, K, batch, int8)
        gbs = algo / (ms * 1e-3) / 1e9
        res.append({"kernel": f"sbi_gemm[{name}] N={N} K={K}", "us": round(ms * 1e3, 2), "bytes": algo,
                    "gbs": round(gbs, 1), "frac": round(gbs / peak_gbs, 3)})
        mult = preset.layers if name != "lm_head" else 1
        tot_b += algo * mult
        tot_t += ms * 1e-3 * mult
        del copies
        torch.cuda.empty_cache()
    agg = tot_b / tot_t / 1e9
    return res, agg


def gemm_algo_bytes(N, K, batch, int8):
    """Algorithmic bytes of one SBI-GeMM launch: packed weights (+ int8 row scales), x in, y out."""
    return N * K * (1 if int8 else 2) + (N * 4 if int8 else 0) + batch * K * 2 + batch * N * 4


def insitu_roofline(model, preset, tp, batch, dtype, peak_gbs, stream, steps=8):
    """Per-launch device timeline of `steps` decode steps replayed right after the timed region from
    the same CUDA graph (re-captured with timestamp atomics per CTA; globaltimer).

    Launches overlap (programmatic dependent launch starts a GEMM's CTAs, and their weight prefetch,
    while the previous kernel still runs), so each launch is charged the INTERVAL from the previous
    launch's last-CTA end to its own last-CTA end: the intervals tile the step exactly, with no
    double counting.  `achieved` = SBI-GeMM algorithmic bytes / (SBI-GeMM intervals + the row_prep
    intervals: those launches exist only to feed the x-streamed GEMMs, and the GEMMs prefetch their
    first ring stages under them, so charging the GEMMs alone would overstate them).  The GEMM-only
    figure and the first-CTA-start -> last-CTA-end spans are reported beside it.
    Returns (GB/s, table) or None."""
    from paper_2207_00032_b200 import _capi as capi

    tr = model.launch_trace(steps, stream=stream).astype(np.float64)
    kinds = [capi.LK_NAMES[int(k)] for k in tr[0, :, 2]]
    dur = (tr[:, :, 1] - tr[:, :, 0]) / 1e3
    ends = tr[:, :, 1]
    first = np.minimum.accumulate(tr[:, :, 0], axis=1)[:, :1]
    prev_end = np.concatenate([first, np.maximum.accumulate(ends, axis=1)[:, :-1]], axis=1)
    interval = np.maximum(ends - prev_end, 0.0) / 1e3
    span = float(np.median((tr[:, -1, 1] - tr[:, 0, 0]) / 1e3))
    layer, lm = gemm_shapes(preset, tp)
    shapes = {n: (N, K) for n, N, K in layer + [lm]}
    tot_b = tot_us = prep_us = 0.0
    table = {}
    for k in dict.fromkeys(kinds):
        idx = [i for i, kk in enumerate(kinds) if kk == k]
        d, iv = dur[:, idx], interval[:, idx]
        row = {"launches_per_step": len(idx), "interval_us_mean": round(float(iv.mean()), 2),
               "span_us_mean": round(float(d.mean()), 2), "share_of_step": round(float(iv.sum() / steps / span), 4)}
        if k in shapes:
            N, K = shapes[k]
            b = gemm_algo_bytes(N, K, batch, dtype == "int8" and k != "lm_head")
            row["bytes"] = b
            row["gbs"] = round(b / (iv.mean() * 1e-6) / 1e9, 1)
            row["frac"] = round(row["gbs"] / peak_gbs, 4)
            tot_b += b * iv.size
            tot_us += float(iv.sum())
        elif k == "prep":
            prep_us += float(iv.sum())
        table[k] = row
    if tot_us == 0:
        return None
    gemm_only = tot_b / (tot_us * 1e-6) / 1e9
    return tot_b / ((tot_us + prep_us) * 1e-6) / 1e9, {"step_span_us": round(span, 1),
                                                        "gemm_only_gbs": round(gemm_only, 1), "kinds": table}


def run_ours(args, preset, rank, world, local_rank):
    import torch

    from paper_2207_00032_b200 import _capi as capi
    from paper_2207_00032_b200 import engine as E

    local_rank = local_rank % max(1, torch.cuda.device_count())  # ranks may share a GPU (functional runs)
    torch.cuda.set_device(local_rank)
    stream = torch.cuda.Stream()
    peak_gbs, peak_kind = measured_peaks()
    dtype_bytes = 1 if args.dtype == "int8" else 2
    comm = None
    ipc_exchange = None
    tp_mode = capi.TP_NONE
    if world > 1 and args.tp_mode == "ipc":
        # the fused all-reduce over CUDA-IPC peer memory (DSINF_TP_IPC): handles all-gathered over gloo
        import torch.distributed as dist

        def ipc_exchange(blob):
            lst = [None] * world
            dist.all_gather_object(lst, blob)
            return lst

        tp_mode = capi.TP_IPC
    elif world > 1:
        import ctypes as C

        import torch.distributed as dist

        tp_mode = capi.TP_NCCL
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            capi.check(capi.lib.dsinf_nccl_get_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * 128)(*obj[0])
        h = C.c_void_p()
        capi.check(capi.lib.dsinf_nccl_comm_create(uid, world, rank, local_rank, C.byref(h)))
        comm = h.value
    max_ctx = args.prompt + 2 * (args.warmup + args.steps) + 8
    model = E.DecoderModel(preset.hidden, preset.layers, preset.heads, preset.vocab, dtype_bytes=dtype_bytes,
                           batch=args.batch, max_ctx=max_ctx, tp_size=world, tp_rank=rank,
                           tp_mode=tp_mode, nccl_comm=comm, ipc_exchange=ipc_exchange,
                           use_cuda_graph=not args.no_graph, use_pdl=not args.no_pdl, seed=SEED, device=local_rank,
                           int8_act={"w8a8": capi.INT8_W8A8, "w8a16": capi.INT8_W8A16, "auto": capi.INT8_AUTO}[args.int8_act],
                           int8_group=args.int8_group if args.dtype == "int8" else 0)
    rng = np.random.default_rng(SEED)
    prompt = rng.integers(0, preset.vocab, (args.batch, args.prompt)).astype(np.int32)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    # ---- prompt prefill: the large-batch (tcgen05) path at TP = 1, else the prompt tokens through
    # the decode step graph
    use_tc_prefill = world == 1 and not args.token_prefill and not (args.dtype == "int8" and args.int8_group)

    def do_prefill():
        model.set_prompt(prompt, stream=stream)
        if use_tc_prefill:
            model.prefill(stream=stream)
        else:
            model.step(args.prompt, stream=stream)

    do_prefill()  # first call builds the row-major weight copies and buffers
    stream.synchronize()
    pst, pen = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pst.record(stream)
    do_prefill()
    pen.record(stream)
    pen.synchronize()
    prefill_ms = pst.elapsed_time(pen)

    # ---- device-timed decode (inputs resident in HBM)
    model.step(args.warmup, stream=stream)
    pos0 = args.prompt + args.warmup
    barrier()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        st.record(stream)
        model.step(args.steps, stream=stream)
        en.record(stream)
        en.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = args.batch * args.steps * 1e3 / ms  # whole-job tokens/s (every rank serves the same tokens)
    info = model.get_info()
    step_bytes = sum(model.bytes_per_step(p) for p in range(pos0, pos0 + args.steps))
    step_gbs = step_bytes / (ms * 1e-3) / 1e9
    _, hist = model.read_tokens(stream=stream)
    gen_sample = hist[0, args.prompt: args.prompt + 8].tolist()

    # ---- end to end through the C ABI with host buffers (H2D tokens in, D2H tokens out each step)
    import ctypes as C

    do_prefill()
    stream.synchronize()
    tin = torch.empty(args.batch, dtype=torch.int32, pin_memory=True)
    tout = torch.empty(args.batch, dtype=torch.int32, pin_memory=True)
    nxt, _ = model.read_tokens(stream=stream)
    tin.numpy()[:] = nxt
    pin = C.cast(tin.data_ptr(), C.POINTER(C.c_int32))
    pout = C.cast(tout.data_ptr(), C.POINTER(C.c_int32))
    sp = stream.cuda_stream
    for _ in range(args.warmup):
        capi.check(capi.lib.dsinf_decode_step_host(model._h, pin, pout, sp))
        tin.copy_(tout)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        capi.check(capi.lib.dsinf_decode_step_host(model._h, pin, pout, sp))
        tin.copy_(tout)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch

        import torch.distributed as dist

        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = args.batch * args.steps / e2e_s

    # ---- dominant-kernel roofline: SBI-GeMM launches inside the decode step (device timeline),
    # plus each shape timed alone; and the CPU baseline: rank 0
    insitu = insitu_roofline(model, preset, world, args.batch, args.dtype, peak_gbs, stream)
    roof = None
    cpu = None
    prefill = {"ms": round(prefill_ms, 3), "tokens_per_s": round(args.batch * args.prompt * 1e3 / prefill_ms, 1),
               "path": "decode step graph, token by token"}
    if rank == 0:
        per_kernel, agg_alone = kernel_roofline(E, torch, preset, world, args.batch, args.dtype, peak_gbs, stream)
        # roofline.frac: the dominant kernel's algorithmic bytes over its CUDA-event launch time (each
        # layer shape timed alone, byte-weighted) -- the figure the ncu launch list reproduces; the
        # in-step interval accounting is reported beside it (in_step_interval), never as frac
        agg = agg_alone
        traffic = traffic_note = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                traffic = json.load(f).get(f"{args.config}-{args.dtype}-b{args.batch}")
            if isinstance(traffic, dict):  # bytes of the one captured launch, with its algorithmic bytes
                traffic_note = traffic
                traffic = traffic.get("bytes")
            else:
                traffic_note = None
        roof = {"bound": "hbm", "achieved": round(agg, 1), "peak": peak_gbs, "unit": "GB/s",
                "frac": round(agg / peak_gbs, 4), "traffic": traffic, "traffic_launch": traffic_note,
                "peak_kind": peak_kind,
                "kernel": ("sbi_gemm_kernel: algorithmic bytes of one step's SBI-GeMM launches over their "
                           "CUDA-event launch times (each shape timed alone on the launching stream, byte-weighted)"),
                "in_step_interval": ({"achieved": round(insitu[0], 1), "frac": round(insitu[0] / peak_gbs, 4),
                                      "how": "SBI-GeMM bytes of 8 graph-replayed decode steps over the device-"
                                             "timeline intervals the GEMMs and their row_preps own (previous "
                                             "launch's last-CTA end -> own last-CTA end, globaltimer)",
                                      **insitu[1]} if insitu else None),
                "alone": {"achieved": round(agg_alone, 1), "per_kernel": per_kernel},
                "step": {"achieved": round(step_gbs, 1), "frac": round(step_gbs / peak_gbs, 4),
                         "bytes_per_step": int(step_bytes / args.steps)}}
        if use_tc_prefill:
            M = args.batch * args.prompt
            tpk, tkind = measured_tensor_peak()
            if args.dtype == "int8":
                tpk, tkind = 2 * tpk, f"2x {tkind} bf16 (int8 tensor rate)"
            agg_tc, rows_tc = tc_roofline(E, torch, preset, M, args.dtype, stream)
            h, L = preset.hidden, preset.layers
            pf_flops = 2.0 * M * 12 * h * h * L + 2.0 * M * args.prompt * h * L
            # arithmetic intensity of the layer GEMMs is ~M flop per weight element: below the ridge
            # (peak flop/s over peak bytes/s) they are bound by streaming the weights, not the tensor pipe
            wbytes = 1 if args.dtype == "int8" else 2
            ridge = tpk * 1e12 / (peak_gbs * 1e9)
            if 2.0 * M / wbytes < ridge:
                tot_b = sum(N * K * wbytes for _, N, K in gemm_shapes(preset, 1)[0])
                tot_us = sum(r["us"] for r in rows_tc)
                gbs = tot_b / (tot_us * 1e-6) / 1e9
                roof_pf = {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak_gbs, "unit": "GB/s",
                           "frac": round(gbs / peak_gbs, 4), "peak_kind": peak_kind,
                           "tensor_achieved": round(agg_tc, 1), "tensor_peak": tpk, "tensor_peak_kind": tkind}
            else:
                roof_pf = {"bound": "tensor", "achieved": round(agg_tc, 1), "peak": tpk,
                           "unit": "TOP/s" if args.dtype == "int8" else "TFLOP/s", "frac": round(agg_tc / tpk, 4),
                           "peak_kind": tkind}
            roof_pf["kernel"] = ("tc_gemm_kernel (tcgen05.mma + TMEM) over the layer GEMMs at M = batch x prompt, "
                                 "each timed alone; bound by arithmetic intensity 2M/w vs the ridge "
                                 f"{ridge:.0f} flop/B")
            roof_pf["per_kernel"] = rows_tc
            prefill = {"ms": round(prefill_ms, 3), "tokens_per_s": round(M * 1e3 / prefill_ms, 1),
                       "tflops": round(pf_flops / (prefill_ms * 1e-3) / 1e12, 1), "path": "tcgen05 large-batch",
                       "roofline": roof_pf}
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            est_ms, kind, sample = reference_ms_per_token(preset, 1, args.batch, dtype_bytes, 2.0, threads)
            if est_ms * 1e-3 * 3 <= args.cpu_budget:  # median of 3 whole reference steps
                st = ReferenceStep(preset, 1, args.batch, dtype_bytes, threads)
                cms = statistics.median([st.run() * 1e3 for _ in range(3)])
                sample = "median of 3 " + st.desc
                st.close()
            else:
                cms, kind, sample = reference_ms_per_token(preset, 1, args.batch, dtype_bytes, args.cpu_budget, threads)
            cpu = {"value": args.batch * 1e3 / cms, "unit": "tokens/s", "cores": threads, "kind": kind,
                   "sample": sample, "ms_per_token": cms, "cpu_model": cpu_model_name()}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f16" if args.dtype == "fp16" else "int8", "data": "synthetic",
        "config": workload_config(args, preset, world),
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": 4 * args.batch,
                "d2h_bytes_per_step": 4 * args.batch, "ms_per_step": e2e_s * 1e3 / args.steps},
        "gpu_launches": int(info.kernels_per_step) * args.steps,
        "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
        "prefill": prefill, "generated_sample": gen_sample,
    }
    model.close()
    if world == 1 and rank == 0 and not args.no_sweep:
        sweep = decode_sweep(E, capi, torch, preset, args, stream, peak_gbs, (args.dtype, args.batch))
        sweep.insert(0, {"dtype": args.dtype, "batch": args.batch, "ms_per_token": round(ms_step, 4),
                         "tokens_per_s": round(value, 1), "step_gbs": round(step_gbs, 1),
                         "frac": round(step_gbs / peak_gbs, 4)})
        line["decode_sweep"] = {"note": "BASELINE metric matrix on this GPU, same timing rules; frac = step GB/s "
                                        "(algorithmic bytes) / measured HBM peak", "rows": sweep}
    if world == 1 and rank == 0 and not args.no_tp_slices:
        line["tp_rank_slices"] = {
            "note": "per-rank step of the TP configs on this one GPU: rank 0's shard alone (same kernels and "
                    "per-rank bytes; the per-layer all-reduces and the argmax all-gather are skipped, so this "
                    "is each rank's compute floor, not a TP=t number)",
            "rows": tp_slice_sweep(E, capi, torch, args, stream, peak_gbs)}
    if comm is not None:
        capi.lib.dsinf_nccl_comm_destroy(comm)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="gptj-6b")
    ap.add_argument("--dtype", choices=["fp16", "int8"], default="fp16")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the fp16/int8 x batch 1/8/16 decode matrix")
    ap.add_argument("--int8-act", choices=["w8a8", "w8a16", "auto"], default="auto",
                    help="int8 decode GEMMs: per-token int8 activations (int32 accumulate), weight-only, or the "
                         "measured per-batch choice (W8A16 for batch <= 8, W8A8 above)")
    ap.add_argument("--int8-group", type=int, choices=[0, 128], default=0,
                    help="int8: 128 = K-group weight scales (weight-only GEMMs, per-group dequant; the prompt goes "
                         "through the decode step)")
    ap.add_argument("--tp-mode", choices=["ipc", "nccl"], default="ipc",
                    help="N > 1: all-reduces fused into the GEMM epilogues over CUDA-IPC peer memory (default), "
                         "or NCCL all-reduce launches between the GEMMs")
    ap.add_argument("--no-tp-slices", action="store_true", help="skip the per-rank TP slice measurements")
    ap.add_argument("--token-prefill", action="store_true", help="prefill the prompt through the decode step graph")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU work for cpu_baseline")
    ap.add_argument("--ref-full-budget", type=float, default=180.0,
                    help="--impl reference times whole steps when warmup + steps of them fit in this many seconds")
    ap.add_argument("--ref-step-budget", type=float, default=2.0, help="seconds per --impl reference step")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    # the presets module loads no native code: the reference arm must not map libdsinf.so
    import importlib.util

    spec = importlib.util.spec_from_file_location("dsinf_presets", os.path.join(ROOT, "paper_2207_00032_b200",
                                                                                 "presets.py"))
    presets = importlib.util.module_from_spec(spec)
    sys.modules["dsinf_presets"] = presets  # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(presets)
    preset = presets.PRESETS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1:
        world = 1
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    if args.impl == "reference":
        run_reference(args, preset, rank, world)
    else:
        run_ours(args, preset, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
