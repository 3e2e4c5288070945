"""Tensor-parallel sharding on CPU with world_size 2 (gloo, 127.0.0.1): each rank takes its shards
from the C ABI (dsinf_shard_tensor — the same Megatron map the device generator uses), runs its part
of the layer GEMMs, and the collectives the B200 path issues (all-reduce after the row-parallel
attn-out / MLP-down, all-gather of the vocab-parallel argmax) rebuild the unsharded results."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_00032_b200 import _capi as capi
from paper_2207_00032_b200 import engine as E

H_, NH, V, SEED = 256, 8, 500, 99


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sh = lambda tensor, tp, r, layer=0: E.shard_tensor(H_, NH, V, tp, r, layer, tensor, SEED).astype(np.float64)  # noqa
        rng = np.random.default_rng(0)
        x = rng.standard_normal((3, H_))
        d, Hl, Fl = H_ // NH, NH // world, 4 * H_ // world
        # column-parallel QKV: local rows [q_r | k_r | v_r]
        full = sh(capi.T_QKV, 1, 0)
        y = torch.from_numpy(x @ sh(capi.T_QKV, world, rank).T)
        parts = [torch.zeros_like(y) for _ in range(world)]
        dist.all_gather(parts, y)
        ref = x @ full.T
        for r, p in enumerate(parts):
            for sec in range(3):
                cols = slice(sec * H_ + r * Hl * d, sec * H_ + (r + 1) * Hl * d)
                np.testing.assert_allclose(p.numpy()[:, sec * Hl * d:(sec + 1) * Hl * d], ref[:, cols], rtol=1e-12)
        # row-parallel attn-out and MLP-down: partial sums + all-reduce
        for tensor, kdim, klocal in ((capi.T_O, H_, Hl * d), (capi.T_DOWN, 4 * H_, Fl)):
            a = rng.standard_normal((3, kdim))
            part = torch.from_numpy(a[:, rank * klocal:(rank + 1) * klocal] @ sh(tensor, world, rank).T)
            dist.all_reduce(part)
            np.testing.assert_allclose(part.numpy(), a @ sh(tensor, 1, 0).T, rtol=1e-10, atol=1e-12)
        # column-parallel MLP-up
        up = torch.from_numpy(x @ sh(capi.T_UP, world, rank).T)
        parts = [torch.zeros_like(up) for _ in range(world)]
        dist.all_gather(parts, up)
        np.testing.assert_allclose(torch.cat(parts, 1).numpy(), x @ sh(capi.T_UP, 1, 0).T, rtol=1e-12)
        # vocab-parallel LM head + argmax combine (ties -> lowest id), as select_kernel does
        wl = sh(capi.T_WTE, world, rank, -1)
        vl = wl.shape[0]
        logits = x @ wl.T
        valid = max(0, min(vl, V - rank * vl))
        loc = logits[:, :valid]
        pair = torch.tensor(np.stack([loc.max(1), loc.argmax(1) + rank * vl], 1))
        pairs = [torch.zeros_like(pair) for _ in range(world)]
        dist.all_gather(pairs, pair)
        best = []
        for b in range(3):
            bv, bi = -np.inf, 1 << 30
            for p in pairs:
                v, i = float(p[b, 0]), int(p[b, 1])
                if v > bv or (v == bv and i < bi):
                    bv, bi = v, i
            best.append(bi)
        full_logits = x @ sh(capi.T_WTE, 1, 0, -1)[:V].T
        assert best == list(full_logits.argmax(1))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        errq.put(f"rank {rank}: {e!r}")
        raise


@pytest.mark.parametrize("world", [2])
def test_tp_shards_and_collectives_rebuild_unsharded_layer(world):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    assert not errors, errors
    assert all(p.exitcode == 0 for p in procs)
