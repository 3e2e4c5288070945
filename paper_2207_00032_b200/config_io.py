"""Model presets from TOML and machine-readable JSON reports.

Restates the reference's user-facing input/output formats over this repo's C ABI:
- `load_model_file` reads the TOML model file of `config.hpp:58-100` (`parse_model_file`): the same
  keys, defaults (vocab_size 50257, max_seq 2048, dtype_bytes 2) and optional `params_reported`,
  `[parallelism]` grid hints and `[moe]` table; the dense fields are validated by the library
  (`dsinf_param_count`, the reference's `ModelConfig::validate` error messages).
- `graph_to_json` / `graph_from_json` follow the OpGraph schema of `json_io.hpp:51-83` (nodes with
  kind / out_elems / tile_count, edges with sparse `[consumer, [producers]]` tile-dependency pairs).
- Reports carry a `schema_version` (SPEC "External Interfaces").

Bundled presets of BASELINE.json's shapes live in `configs/*.toml` (`preset_path`).
"""
from __future__ import annotations

import os
import tomllib
from dataclasses import dataclass, field
from typing import Any, Dict, Optional

from . import infersim as I
from ._capi import ConfigError

SCHEMA_VERSION = 1
CONFIG_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs")


@dataclass
class GridHints:  # config.hpp: GridHints
    mp_degree: int = 1
    ep_degree: int = 1
    expert_slicing: int = 1
    gpus: int = 1


@dataclass
class ModelFile:  # config.hpp: ModelFile
    config: I.ModelConfig
    params_reported: Optional[float] = None
    grid: Optional[GridHints] = None
    moe: Dict[str, Any] = field(default_factory=dict)  # parsed, not used by the dense decode path


def _get(t: Dict[str, Any], dotted: str, default=None, required=False):
    cur: Any = t
    for part in dotted.split("."):
        if not isinstance(cur, dict) or part not in cur:
            if required:
                raise ConfigError(f"missing key '{dotted}'")
            return default
        cur = cur[part]
    return cur


def _int(t, key, default=None, required=False) -> Optional[int]:
    v = _get(t, key, default, required)
    if v is None:
        return None
    if isinstance(v, bool) or not isinstance(v, (int, float)) or int(v) != v:
        raise ConfigError(f"key '{key}' must be an integer")
    return int(v)


def parse_model_file(t: Dict[str, Any]) -> ModelFile:
    """config.hpp:58-100 over a parsed TOML table."""
    cfg = I.ModelConfig()
    cfg.name = str(_get(t, "name", ""))
    cfg.hidden_dim = _int(t, "hidden_dim", required=True)
    cfg.num_layers = _int(t, "num_layers", required=True)
    cfg.num_heads = _int(t, "num_heads", required=True)
    cfg.vocab_size = _int(t, "vocab_size", 50257)
    cfg.max_seq = _int(t, "max_seq", 2048)
    cfg.dtype_bytes = _int(t, "dtype_bytes", 2)
    I.param_count(cfg)  # ModelConfig::validate through the library (raises ConfigError)
    f = ModelFile(cfg)
    if _get(t, "moe.num_experts") is not None:
        f.moe = {"num_experts": _int(t, "moe.num_experts"), "expert_interval": _int(t, "moe.expert_interval", 2),
                 "capacity_factor": float(_get(t, "moe.capacity_factor", 1.0)), "top_k": _int(t, "moe.top_k", 1)}
    if _get(t, "params_reported") is not None:
        f.params_reported = float(_get(t, "params_reported"))
    if _get(t, "parallelism.mp_degree") is not None:
        f.grid = GridHints(_int(t, "parallelism.mp_degree"), _int(t, "parallelism.ep_degree", 1),
                           _int(t, "parallelism.expert_slicing", 1), _int(t, "parallelism.gpus", 1))
    return f


def load_model_file(path: str) -> ModelFile:
    """config.hpp: load_model_file (a missing or malformed file is a ConfigError)."""
    try:
        with open(path, "rb") as fh:
            t = tomllib.load(fh)
    except FileNotFoundError:
        raise ConfigError(f"cannot open '{path}'") from None
    except tomllib.TOMLDecodeError as ex:
        raise ConfigError(f"bad TOML in '{path}': {ex}") from None
    return parse_model_file(t)


def preset_path(name: str) -> str:
    """Bundled preset TOML (INFERSIM_FIXTURES overrides the directory, SPEC External Interfaces)."""
    d = os.environ.get("INFERSIM_FIXTURES", CONFIG_DIR)
    return os.path.join(d, name if name.endswith(".toml") else name + ".toml")


def graph_to_json(g: I.OpGraph) -> Dict[str, Any]:
    """json_io.hpp:51-83 schema."""
    return {
        "dtype_bytes": g.dtype_bytes,
        "nodes": [{"name": n.name, "kind": n.kind.name, "iter_dims": [], "tileable_dims": [], "reduce_dims": [],
                   "out_elems": n.out_elems, "tile_count": n.tile_count} for n in g.nodes],
        "edges": [{"from": e.from_, "to": e.to,
                   "tile_dep": [[c, sorted(p)] for c, p in sorted(e.tile_dep.items())]} for e in g.edges],
    }


def graph_from_json(j: Dict[str, Any]) -> I.OpGraph:
    """json_io.hpp graph_from_json: unknown kinds and malformed entries are ConfigErrors."""
    try:
        g = I.OpGraph(dtype_bytes=int(j.get("dtype_bytes", 2)))
        for n in j["nodes"]:
            kind = n["kind"]
            if kind not in I.OpKind.__members__:
                raise ConfigError(f"unknown op kind '{kind}'")
            g.nodes.append(I.OpNode(str(n["name"]), I.OpKind[kind], int(n.get("out_elems", 0)),
                                    int(n.get("tile_count", 1))))
        for e in j["edges"]:
            dep = {}
            for pair in e.get("tile_dep", []):
                dep.setdefault(int(pair[0]), set()).update(int(p) for p in pair[1])
            g.edges.append(I.GraphEdge(int(e["from"]), int(e["to"]), dep))
    except (KeyError, TypeError, ValueError, IndexError) as ex:
        raise ConfigError(f"bad graph JSON: {ex}") from None
    for e in g.edges:
        if not (0 <= e.from_ < len(g.nodes) and 0 <= e.to < len(g.nodes)):
            raise ConfigError("graph edge endpoint out of range")
    return g
