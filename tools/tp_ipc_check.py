#!/usr/bin/env python3
"""One rank of a DSINF_TP_IPC decode (launch with torch.distributed.run, one process per rank; the
ranks may share a GPU): gloo exchanges the CUDA-IPC handles, then every cross-rank exchange of the
decode step (the per-layer all-reduces fused into the attn-out / MLP-down epilogues, the argmax keys
of the vocab-parallel LM head) goes over peer memory.  Each rank saves its vocab slice of the logits
and the greedy tokens per position to <out>/rank<r>.npz (tests/test_gpu_tp_ipc.py compares them
with the TP-aware oracle).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P \\
      tools/tp_ipc_check.py --hidden 512 --layers 2 --heads 8 --vocab 1000 --batch 2 --out DIR
With --bench N: also time N decode steps (CUDA events, max over ranks) and print ms/step.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    for k, v in (("hidden", 512), ("layers", 2), ("heads", 8), ("vocab", 1000), ("batch", 2), ("dtype_bytes", 2),
                 ("prompt", 5), ("gen", 4), ("max_ctx", 32), ("bench", 0), ("seed", 20220701), ("int8_act", 0)):
        ap.add_argument("--" + k.replace("_", "-"), type=int, default=v)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2207_00032_b200 import _capi as capi
    from paper_2207_00032_b200.engine import DecoderModel

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)

    def exchange(blob):
        lst = [None] * world
        dist.all_gather_object(lst, blob)
        return lst

    m = DecoderModel(a.hidden, a.layers, a.heads, a.vocab, dtype_bytes=a.dtype_bytes, batch=a.batch,
                     max_ctx=a.max_ctx, tp_size=world, tp_rank=rank, tp_mode=capi.TP_IPC, seed=a.seed, device=dev,
                     int8_act=a.int8_act, ipc_exchange=exchange)
    info = m.get_info()
    prompt = np.random.default_rng(a.hidden + a.layers + a.batch).integers(0, a.vocab, (a.batch, a.prompt))
    m.set_prompt(prompt.astype(np.int32))
    logits, tokens = [], []
    for _ in range(a.prompt + a.gen - 1):
        m.step(1)
        torch.cuda.synchronize()
        logits.append(m.read_logits()[0].copy())
        tokens.append(m.read_tokens()[0].copy())
    _, hist = m.read_tokens()
    res = {"logits": np.stack(logits), "tokens": np.stack(tokens), "hist": hist, "prompt": prompt,
           "vocab_local": info.vocab_local, "fused_allreduce": int(info.fused_allreduce)}
    if a.bench > 0:
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(s)
        m.step(a.bench, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.bench])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["ms_per_step"] = float(t)
        if rank == 0:
            print(f"TP_IPC t={world} h={a.hidden} L={a.layers} B={a.batch}: {float(t):.3f} ms/step (max over ranks)")
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        np.savez(os.path.join(a.out, f"rank{rank}.npz"), **res)
    m.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
