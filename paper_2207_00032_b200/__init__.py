"""B200-native (sm_100a) decoder-layer decode hot path of DeepSpeed-Inference (arXiv 2207.00032).

The product is the C ABI library `libdsinf.so` (include/dsinf.h): SBI-GeMM kernels over the
reference's packed weight layout, Deep-Fusion layer kernels, INT8 W8A8 GEMMs, decode attention,
tensor-parallel NCCL sharding and a CUDA-graph decode loop.  `infersim` mirrors the reference's
operator API; `engine` drives a model.
"""
from . import _capi  # noqa: F401  (loads libdsinf.so; fails loudly if it was not built)
from . import infersim  # noqa: F401
from .engine import PRESETS, DecoderModel  # noqa: F401

__all__ = ["infersim", "DecoderModel", "PRESETS"]
