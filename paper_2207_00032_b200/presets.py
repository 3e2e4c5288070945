"""Model presets of BASELINE.json's configs (shapes only; pure Python, loads no native code, so the
reference arm of bench.py can read them without mapping libdsinf.so)."""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Preset:
    name: str
    hidden: int
    layers: int
    heads: int
    tp: int
    vocab: int = 50257
    max_seq: int = 2048


PRESETS = {
    "gpt2-1.5b": Preset("GPT-2 1.5B", 1600, 48, 25, 1),
    "gptj-6b": Preset("GPT-J 6B", 4096, 32, 32, 1),
    "gpt-neox-20b": Preset("GPT-NeoX 20B", 6144, 44, 64, 2),
    "gpt-50b": Preset("GPT-50B", 8192, 62, 64, 4),
    "gpt3-175b": Preset("GPT3-175B", 12288, 96, 96, 8),
}
