"""cuDNN fp32 precision for the dense comparators.

torch 2.11 governs cuDNN convolutions with ``torch.backends.cudnn.conv.fp32_precision``
("ieee" | "tf32" | "none").  The legacy switch ``cudnn.allow_tf32 = False`` only sets it
to "none" (inherit), and measured on B200 that still ran TF32 (max relative error ~1e-3
against the fp64-accurate oracle on a 1152-tap layer), so round-1 "IEEE fp32" cuDNN
baselines were TF32.  Every dense fp32 comparator now pins the mode explicitly.
"""
from __future__ import annotations

from contextlib import contextmanager


@contextmanager
def cudnn_fp32(mode: str):
    """Run cuDNN fp32 convolutions in `mode` ("ieee" or "tf32") inside the block."""
    import torch
    if mode not in ("ieee", "tf32"):
        raise ValueError(mode)
    conv = torch.backends.cudnn.conv
    old = conv.fp32_precision
    conv.fp32_precision = mode
    try:
        yield
    finally:
        conv.fp32_precision = old
