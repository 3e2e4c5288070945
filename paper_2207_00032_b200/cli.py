"""Command line over the C ABI (SPEC `run(subcommand, RunConfig)`):

  python -m paper_2207_00032_b200.cli params        MODEL.toml
  python -m paper_2207_00032_b200.cli gemm-schedule --out-dim N --in-dim K [--batch B] [--dtype-bytes 2]
  python -m paper_2207_00032_b200.cli fuse          (--graph GRAPH.json | --hidden H --batch B) [--regime small|large]
  python -m paper_2207_00032_b200.cli decode        MODEL.toml [--batch B] [--prompt P] [--gen G] [--int8]  (GPU)

Reports are deterministic JSON on stdout with a `schema_version`.  Exit codes follow the SPEC:
0 success, 1 unknown subcommand (usage on stderr), 2 ConfigError, 3 InfeasibleError, with no partial
report on failure.  The subcommands of the reference's other modules (estimate, schedule, moe-sim,
pcc, offload-plan) are off the decode hot path and answer with exit 1.
"""
from __future__ import annotations

import argparse
import json
import sys

from . import _capi as capi
from . import config_io as cio
from . import infersim as I

SUBCOMMANDS = ("params", "gemm-schedule", "fuse", "decode")


def _dump(obj) -> str:
    return json.dumps(dict(obj, schema_version=cio.SCHEMA_VERSION), indent=2, sort_keys=False)


def cmd_params(a) -> str:
    f = cio.load_model_file(a.model)
    c = f.config
    out = {"name": c.name, "hidden_dim": c.hidden_dim, "num_layers": c.num_layers, "num_heads": c.num_heads,
           "vocab_size": c.vocab_size, "max_seq": c.max_seq, "dtype_bytes": c.dtype_bytes,
           "param_count": I.param_count(c), "param_bytes": I.param_bytes(c)}
    if f.params_reported is not None:
        out["params_reported"] = f.params_reported
        out["relative_error"] = abs(out["param_count"] - f.params_reported) / f.params_reported
    if f.grid is not None:
        out["grid"] = {"mp_degree": f.grid.mp_degree, "ep_degree": f.grid.ep_degree,
                       "expert_slicing": f.grid.expert_slicing, "gpus": f.grid.gpus}
    return _dump(out)


def cmd_gemm_schedule(a) -> str:
    sch = I.derive_schedule(I.GemmShape(a.out_dim, a.in_dim, a.batch, a.dtype_bytes), I.b200_device())
    return _dump({"shape": {"out_dim": a.out_dim, "in_dim": a.in_dim, "batch": a.batch, "dtype_bytes": a.dtype_bytes},
                  "schedule": {"mode": "twoD" if sch.mode == I.TilingMode.twoD else "oneD",
                               "output_tiles": sch.output_tiles, "input_tiles": sch.input_tiles,
                               "warps_per_block": sch.warps_per_block, "kernel_count": sch.kernel_count,
                               "pack_M": sch.pack_M},
                  "device": "B200 (148 SMs)"})


def cmd_fuse(a) -> str:
    if a.graph:
        try:
            with open(a.graph) as fh:
                j = json.load(fh)
        except FileNotFoundError:
            raise capi.ConfigError(f"cannot open '{a.graph}'") from None
        except json.JSONDecodeError as ex:
            raise capi.ConfigError(f"bad graph JSON: {ex}") from None
        g = cio.graph_from_json(j)
    else:
        if a.hidden is None:
            raise capi.ConfigError("fuse needs --graph or --hidden/--batch")
        g = I.canonical_layer_graph(a.hidden, a.batch, a.dtype_bytes)
    regime = I.BatchRegime.small_batch if a.regime == "small" else I.BatchRegime.large_batch
    regions = I.partition_layer(g, regime)
    sav = I.fusion_savings(regions, g)
    return _dump({"regime": a.regime, "graph": cio.graph_to_json(g),
                  "regions": [[g.nodes[i].name for i in r.node_ids] for r in regions],
                  "savings": {"launches_saved": sav.launches_saved, "bytes_saved": sav.bytes_saved}})


def cmd_decode(a) -> str:
    import numpy as np

    from .engine import DecoderModel

    c = cio.load_model_file(a.model).config
    m = DecoderModel(c.hidden_dim, c.num_layers, c.num_heads, c.vocab_size, c.max_seq,
                     dtype_bytes=1 if a.int8 else c.dtype_bytes, batch=a.batch,
                     max_ctx=a.prompt + a.gen + 1, int8_act=capi.INT8_AUTO)
    prompt = np.random.default_rng(a.seed).integers(0, c.vocab_size, (a.batch, a.prompt)).astype(np.int32)
    m.set_prompt(prompt)
    m.prefill()
    m.step(a.gen - 1)
    _, hist = m.read_tokens()
    m.close()
    return _dump({"model": c.name, "batch": a.batch, "prompt_len": a.prompt, "seed": a.seed,
                  "tokens": hist[:, a.prompt:a.prompt + a.gen].tolist()})


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if not argv or argv[0] not in SUBCOMMANDS:
        sys.stderr.write(__doc__)
        return 1
    ap = argparse.ArgumentParser(prog=f"paper_2207_00032_b200.cli {argv[0]}")
    sub = argv[0]
    if sub in ("params", "decode"):
        ap.add_argument("model")
    if sub == "gemm-schedule":
        ap.add_argument("--out-dim", type=int, required=True)
        ap.add_argument("--in-dim", type=int, required=True)
        ap.add_argument("--batch", type=int, default=1)
        ap.add_argument("--dtype-bytes", type=int, default=2)
    if sub == "fuse":
        ap.add_argument("--graph")
        ap.add_argument("--hidden", type=int)
        ap.add_argument("--batch", type=int, default=1)
        ap.add_argument("--dtype-bytes", type=int, default=2)
        ap.add_argument("--regime", choices=["small", "large"], default="small")
    if sub == "decode":
        ap.add_argument("--batch", type=int, default=1)
        ap.add_argument("--prompt", type=int, default=128)
        ap.add_argument("--gen", type=int, default=8)
        ap.add_argument("--seed", type=int, default=20220701)
        ap.add_argument("--int8", action="store_true")
    try:
        a = ap.parse_args(argv[1:])
    except SystemExit:
        return 2
    fn = {"params": cmd_params, "gemm-schedule": cmd_gemm_schedule, "fuse": cmd_fuse, "decode": cmd_decode}[sub]
    try:
        report = fn(a)
    except capi.InfeasibleError as ex:
        sys.stderr.write(f"infeasible: {ex}\n")
        return 3
    except capi.ConfigError as ex:
        sys.stderr.write(f"config error: {ex}\n")
        return 2
    sys.stdout.write(report + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
