"""Measured launch tuner (replaces the reference's tune_sub_batch,
engine.py:143-166, and the paper's hand-picked subBatchSize).

For one layer and batch size it times every launch configuration the C
library reports as valid (tiled variant x warp groups x images per CTA x
output block x channels per stage, scb_launch_candidates) with CUDA events
on the launching stream, keeps the median of `repetitions` after `warmups`,
and records the argmin in ``engine.TUNED`` so later ``conv_sparse`` calls on
the same (layer signature, batch, flags) use it.  Ties go to the earlier
candidate.  Results are bit-identical across candidates (exact mode), which
tests/test_gpu_parity.py checks.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from . import _abi, engine
from .device import device_layer
from .geometry import check_nchw, dtype_of


def time_call(fn, repetitions: int = 5, warmups: int = 2) -> float:
    """Median seconds of fn() measured with CUDA events on the current stream."""
    import torch
    for _ in range(warmups):
        fn()
    torch.cuda.synchronize()
    samples = []
    for _ in range(repetitions):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        samples.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(samples))


def tune_launch(x, kernel, bias=None, plan: engine.EnginePlan = engine.EnginePlan(), *,
                relu: bool = False, pool: bool = False, repetitions: int = 5, warmups: int = 2,
                max_candidates: int | None = None, include_generic: bool = False,
                layout: str = "nchw"):
    """Time every valid launch for (x, kernel) and cache the fastest.

    x must be a CUDA tensor (NCHW).  Returns (best_launch, {launch: median_seconds});
    best_launch None means the generic kernel won.  layout = "minor" times the kernels
    that read and write image-minor activations (FLAG_IMAGE_MINOR, kind 7) on an
    image-minor copy of x instead; (None, {}) when the layer has none.
    """
    import torch
    x = check_nchw(x)
    sh = kernel.shape
    x_dt = dtype_of(x)
    io = engine._io_dtype(x_dt, kernel)
    dev = x.device.index
    layer = device_layer(kernel, dev, io, plan.weight_format)
    flags = engine._flags(plan, relu, pool, False)
    minor = layout == "minor"
    if minor:
        flags |= _abi.FLAG_IMAGE_MINOR
        include_generic = False
    n = int(x.shape[0])
    cands = layer.candidates(n, flags)
    if max_candidates is not None:
        cands = cands[:max_candidates]
    xin = x.to(engine._torch_dtype(io)).contiguous()
    e, f = (sh.e // 2, sh.f // 2) if pool else (sh.e, sh.f)
    y = torch.empty((n, sh.k, e, f), dtype=engine._torch_dtype(io), device=x.device)
    ld = n
    if minor:
        ld = engine.minor_ld(n)
        xm = torch.empty((sh.c * sh.h * sh.w, ld), dtype=xin.dtype, device=x.device)
        xm[:, :n] = xin.reshape(n, -1).t()
        xin = xm
        y = torch.empty((sh.k * e * f, ld), dtype=xin.dtype, device=x.device)
    if bias is not None:
        bnp = np.ascontiguousarray(bias.detach().cpu().numpy() if hasattr(bias, "detach") else bias,
                                   dtype=np.float64 if io == np.float64 else np.float32)
        bdev = torch.from_numpy(bnp).to(x.device)
        bptr = bdev.data_ptr()
    else:
        bptr = 0
    stream = torch.cuda.current_stream(dev).cuda_stream
    timings = {}
    for c in cands:
        timings[c] = time_call(lambda: layer.launch(xin.data_ptr(), bptr, y.data_ptr(), n, flags,
                                                    c, stream, ldx=ld, ldy=ld), repetitions, warmups)
    if include_generic:
        # the generic kernel has no fused pool: conv + ReLU, then scb_maxpool2
        yfull = torch.empty((n, sh.k, sh.e, sh.f), dtype=engine._torch_dtype(io), device=x.device) \
            if pool else y
        gflags = (flags & ~_abi.FLAG_POOL2) | _abi.FLAG_GENERIC

        def run_generic():
            layer.launch(xin.data_ptr(), bptr, yfull.data_ptr(), n, gflags, None, stream)
            if pool:
                _abi.maxpool2(io, yfull.data_ptr(), y.data_ptr(), n * sh.k, sh.e, sh.f, stream)
        timings[None] = time_call(run_generic, repetitions, warmups)
    if not timings:
        return None, {}
    # refine: the closest few re-timed with more repetitions (single-digit-percent gaps
    # between neighbouring launches are within one short median's noise)
    top = sorted(timings, key=lambda c: timings[c])[:4]
    if len(top) > 1:
        for c in top:
            if c is None:
                continue
            timings[c] = min(timings[c], time_call(
                lambda: layer.launch(xin.data_ptr(), bptr, y.data_ptr(), n, flags, c, stream, ldx=ld, ldy=ld),
                3 * repetitions, warmups))
    best = min(timings, key=lambda c: timings[c])
    engine.TUNED[(layer.signature(), n, flags)] = best
    return best, timings


def save_tuned(path) -> None:
    rows = [{"sig": list(k[0]), "n": k[1], "flags": k[2], "launch": None if v is None else list(v)}
            for k, v in engine.TUNED.items()]
    Path(path).write_text(json.dumps(rows, indent=1))


def load_tuned(path) -> int:
    rows = json.loads(Path(path).read_text())
    for r in rows:
        engine.TUNED[(tuple(r["sig"]), r["n"], r["flags"])] = None if r["launch"] is None else tuple(r["launch"])
    return len(rows)
