"""Operator API: direct sparse convolution on B200 (drop-in for the
reference's engine.py).

``conv_sparse(x, kernel, bias, plan)`` keeps the reference's contract
(engine.py:68-87): batch taken from ``x`` (``kernel.shape.n`` ignored), bias
optional (zeros), output dtype = input dtype, f16 storage computed in f32,
outputs independent of ``sub_batch_size`` / ``worker_count``.  What changes is
where it runs: one asynchronous launch of an sm_100a kernel from
libsparseconv_b200 (no CPU fallback).

Inputs may be
  * numpy arrays  -> copied to the GPU, result copied back (numpy out);
  * torch CUDA tensors -> zero-copy on their device and current stream
    (torch tensor out, nothing synchronised).
"""
from __future__ import annotations

import logging
import time
from dataclasses import dataclass

import numpy as np

from . import _abi
from .device import device_layer
from .errors import ShapeError
from .geometry import check_nchw, compute_dtype, dtype_of
from .weights import CsrKernel

log = logging.getLogger(__name__)

SUB_BATCH_CANDIDATES = (1, 2, 4, 8, 16)
WEIGHT_FORMATS = ("native", "cb4", "lin16", "aff16")


@dataclass(frozen=True)
class EnginePlan:
    """Execution plan.  ``sub_batch_size`` and ``worker_count`` keep the
    reference's validation (engine.py:28-39).  On the GPU, ``sub_batch_size``
    > 1 asks for that many images per CTA (the paper's subBatchSize,
    PAPER.md:151) and ``worker_count`` is accepted and ignored.

    GPU-only fields: ``launch`` (explicit scb_launch tuple, see
    tuner.tune_launch), ``fast_math`` (f32 single-rounding FMA instead of the
    reference's separately rounded multiply and add), ``weight_format``
    ("native" | "cb4" 4-bit codebook | "lin16" int16 fixed point, decoded in
    registers) and ``device`` (CUDA device for numpy inputs)."""

    sub_batch_size: int = 1
    worker_count: int = 1
    launch: tuple | None = None
    fast_math: bool = False
    weight_format: str = "native"
    device: int | None = None

    def __post_init__(self):
        if self.sub_batch_size not in SUB_BATCH_CANDIDATES:
            raise ShapeError(f"sub_batch_size must be in {SUB_BATCH_CANDIDATES}")
        if self.worker_count < 1:
            raise ShapeError("worker_count must be >= 1")
        if self.weight_format not in WEIGHT_FORMATS:
            raise ShapeError(f"weight_format must be in {WEIGHT_FORMATS}")


# launches chosen by tuner.tune_launch: (layer signature, n, flags) -> launch
TUNED: dict = {}


def _torch():
    import torch
    return torch


_TORCH_DT = None


def _torch_dtype(dt: np.dtype):
    global _TORCH_DT
    torch = _torch()
    if _TORCH_DT is None:
        _TORCH_DT = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
                     np.dtype(np.float16): torch.float16}
    return _TORCH_DT[np.dtype(dt)]


def _io_dtype(x_dtype: np.dtype, kernel: CsrKernel) -> np.dtype:
    """Activation dtype the device kernel runs in.  f16 activations with f16
    values use the f16 kernels (f16*f16 products are exact in f32, so FFMA is
    bit-equal to the reference); any other f16 combination computes on f32
    copies exactly like the reference's astype(f32) (engine.py:62-64)."""
    x_dtype = np.dtype(x_dtype)
    if x_dtype == np.float16:
        return np.dtype(np.float16) if kernel.values.dtype == np.float16 else np.dtype(np.float32)
    return x_dtype


def _flags(plan: EnginePlan, relu: bool, pool: bool, generic: bool) -> int:
    f = 0
    if relu:
        f |= _abi.FLAG_RELU
    if pool:
        f |= _abi.FLAG_POOL2
    if plan.fast_math:
        f |= _abi.FLAG_FAST
    if generic:
        f |= _abi.FLAG_GENERIC
    return f


def _check_geometry(x, kernel: CsrKernel):
    sh = kernel.shape
    if tuple(x.shape[1:]) != (sh.c, sh.h, sh.w):
        raise ShapeError(f"input {tuple(x.shape)} does not match kernel geometry "
                         f"(C,H,W)=({sh.c},{sh.h},{sh.w})")


def _check_out(out, shape, dt, tdev) -> None:
    """A caller-provided output buffer is written by the kernels through a raw pointer:
    it must be a contiguous CUDA tensor of exactly the output shape and dtype on the
    input's device, 16-byte aligned (the vectorised epilogue stores)."""
    torch = _torch()
    if not isinstance(out, torch.Tensor) or not out.is_cuda:
        raise ShapeError("out must be a CUDA torch tensor")
    if tuple(out.shape) != tuple(shape):
        raise ShapeError(f"out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.dtype != _torch_dtype(dt):
        raise ShapeError(f"out has dtype {out.dtype}, expected {_torch_dtype(dt)}")
    if out.device != tdev:
        raise ShapeError(f"out is on {out.device}, the input on {tdev}")
    if not out.is_contiguous() or out.data_ptr() % 16:
        raise ShapeError("out must be contiguous and 16-byte aligned")


def _run(x, kernel: CsrKernel, bias, plan: EnginePlan, *, relu=False, pool=False,
         generic=False, out=None):
    torch = _torch()
    x = check_nchw(x)
    _check_geometry(x, kernel)
    sh = kernel.shape
    x_dt = dtype_of(x)
    ct = compute_dtype(x_dt)
    io = _io_dtype(x_dt, kernel)
    n = int(x.shape[0])
    is_torch = not isinstance(x, np.ndarray)
    if is_torch and x.is_cuda:
        dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
    else:
        if not torch.cuda.is_available():
            from .errors import SparseConvError
            raise SparseConvError("no CUDA device: the B200 engine has no CPU fallback")
        dev = plan.device if plan.device is not None else torch.cuda.current_device()
    tdev = torch.device("cuda", dev)
    # bias in the compute dtype (engine.py:55-60)
    if bias is None:
        b_dev = None
    else:
        b_np = bias.detach().cpu().numpy() if hasattr(bias, "detach") else np.asarray(bias)
        b_np = np.ascontiguousarray(b_np, dtype=ct if io != np.float64 else np.float64)
        if b_np.shape != (sh.k,):
            raise ShapeError(f"bias must have shape ({sh.k},)")
        if io == np.float16:
            b_np = b_np.astype(np.float32)
        b_dev = torch.from_numpy(b_np).to(tdev)
    layer = device_layer(kernel, dev, io, plan.weight_format)
    flags = _flags(plan, relu, pool, generic)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        if is_torch:
            x_dev = x.to(tdev)
        else:
            x_dev = torch.from_numpy(np.ascontiguousarray(x)).to(tdev, non_blocking=False)
        if dtype_of(x_dev) != io:
            x_dev = x_dev.to(_torch_dtype(io))
        x_dev = x_dev.contiguous()
        if x_dev.data_ptr() % 16:
            x_dev = x_dev.clone()  # a sliced view: the tiled kernels stage 16-byte chunks
        e, f = (sh.e // 2, sh.f // 2) if pool else (sh.e, sh.f)
        if out is not None:
            _check_out(out, (n, sh.k, e, f), x_dt, tdev)
        if out is None or io != x_dt:
            y = torch.empty((n, sh.k, e, f), dtype=_torch_dtype(io), device=tdev)
        else:
            y = out
        launch = _choose_launch(layer, n, flags, plan)
        run_layer(layer, x_dev.data_ptr(), b_dev.data_ptr() if b_dev is not None else 0,
                  y, n, flags, launch, stream.cuda_stream)
        if io != x_dt:
            y = y.to(_torch_dtype(x_dt))
            if out is not None:
                out.copy_(y)
                y = out
    if is_torch:
        return y
    return y.cpu().numpy()


_KINDS = None


def launch_kind(launch) -> int:
    """Kernel kind of a launch tuple (-1 = generic)."""
    global _KINDS
    if launch is None:
        return -1
    if _KINDS is None:
        _KINDS = [v["kind"] for v in _abi.variants()]
    return _KINDS[launch[0]]


def minor_ld(n: int) -> int:
    """Row stride of an image-minor buffer for n images: a multiple of 8 (16-byte TMA rows
    in f32 and f16)."""
    return (int(n) + 7) // 8 * 8


def run_layer(layer, x_ptr: int, b_ptr: int, y, n: int, flags: int, launch, stream: int,
              scratch=None) -> None:
    """One layer on `stream` with NCHW activations: a tiled launch (tuple), or the
    generic kernel (launch None) followed by scb_maxpool2 when the pool is requested
    (the generic kernel has no fused pool epilogue).  A kind-7 launch (image-minor
    activations) runs between two layout conversions (scb_to_image_minor /
    scb_from_image_minor) through temporary image-minor buffers."""
    if launch is None and flags & _abi.FLAG_POOL2:
        sh = layer.shape
        tmp = scratch if scratch is not None else \
            _torch().empty((n, sh.k, sh.e, sh.f), dtype=y.dtype, device=y.device)
        layer.launch(x_ptr, b_ptr, tmp.data_ptr(), n, (flags & ~_abi.FLAG_POOL2) | _abi.FLAG_GENERIC,
                     None, stream)
        _abi.maxpool2(layer.io_dtype, tmp.data_ptr(), y.data_ptr(), n * sh.k, sh.e, sh.f, stream)
        return
    if launch_kind(launch) == _abi.KIND_LANE and not flags & _abi.FLAG_IMAGE_MINOR:
        sh = layer.shape
        ld = minor_ld(n)
        chw_in = sh.c * sh.h * sh.w
        chw_out = int(np.prod(y.shape[1:]))
        xm = _torch().empty((chw_in, ld), dtype=y.dtype, device=y.device)
        ym = _torch().empty((chw_out, ld), dtype=y.dtype, device=y.device)
        _abi.to_image_minor(layer.io_dtype, x_ptr, xm.data_ptr(), n, chw_in, ld, stream)
        layer.launch(xm.data_ptr(), b_ptr, ym.data_ptr(), n, flags | _abi.FLAG_IMAGE_MINOR, launch, stream,
                     ldx=ld, ldy=ld)
        _abi.from_image_minor(layer.io_dtype, ym.data_ptr(), ld, y.data_ptr(), n, chw_out, stream)
        return
    layer.launch(x_ptr, b_ptr, y.data_ptr(), n, flags | (_abi.FLAG_GENERIC if launch is None else 0),
                 launch, stream)


def _choose_launch(layer, n, flags, plan: EnginePlan):
    """tuple = tiled launch, None = generic kernel."""
    if flags & _abi.FLAG_GENERIC:
        return None
    if plan.launch is not None:
        return tuple(plan.launch)
    key = (layer.signature(), n, flags)
    if key in TUNED:
        return TUNED[key]
    hit = _builtin().get(_builtin_key(layer.signature(), flags))
    # the shipped table is keyed on geometry, not sparsity: a launch tuned at 90-95 % may not
    # fit (shared memory) a denser layer of the same shape -- then the heuristic decides
    if hit is not None and layer.launch_ok(n, flags, hit):
        return hit
    d = layer.default_launch(n, flags, plan.sub_batch_size if plan.sub_batch_size > 1 else 0)
    return None if d[0] < 0 else d


_BUILTIN = None


def _builtin_key(sig, flags):
    s = list(sig)
    return (tuple(s[:8] + s[9:]), int(flags))  # geometry + dtype + format, not the sparse level


def _builtin() -> dict:
    """Launch table measured on B200 for the VGG-16/CIFAR geometries
    (tools/tune_table.py -> tuned/b200_vgg_cifar.json); the fallback when the
    tuner has not run in this process.  The C library re-validates every
    launch, so a stale entry fails loudly rather than computing wrongly."""
    global _BUILTIN
    if _BUILTIN is None:
        import json
        from pathlib import Path
        _BUILTIN = {}
        p = Path(__file__).resolve().parent / "tuned" / "b200_vgg_cifar.json"
        if p.exists():
            # launches name their kernel by its description, not the compiled-table index
            index = {tuple(sorted(v.items())): i for i, v in reversed(list(enumerate(_abi.variants())))}
            for r in json.loads(p.read_text())["rows"]:
                launch = r["launch"]
                if launch is not None:
                    vi = index.get(tuple(sorted(r["variant"].items())))
                    if vi is None:
                        continue  # kernel no longer compiled: fall back to the heuristic
                    launch = (vi, *launch[1:])
                _BUILTIN[(tuple(r["sig"]), int(r["flags"]))] = None if launch is None else tuple(launch)
    return _BUILTIN


def conv_sparse(x, kernel: CsrKernel, bias=None, plan: EnginePlan = EnginePlan(), *,
                relu: bool = False, pool: bool = False, out=None):
    """Direct sparse convolution of an NCHW batch against a CsrKernel
    (engine.py:68-87).  ``relu`` / ``pool`` fuse Model.forward's ReLU
    (store.py:284) and a 2x2 max-pool into the epilogue."""
    return _run(x, kernel, bias, plan, relu=relu, pool=pool, out=out)


def conv_sparse_1d(x, kernel: CsrKernel, bias=None, plan: EnginePlan = EnginePlan(), *,
                   relu: bool = False, out=None):
    """1D specialisation: H=1, R=1 (engine.py:90-106); bit-identical to
    conv_sparse on the same inputs."""
    sh = kernel.shape
    if sh.h != 1 or sh.r != 1:
        raise ShapeError("conv_sparse_1d requires H=1 and R=1")
    return _run(x, kernel, bias, plan, relu=relu, out=out)


def conv_sparse_reference(x, kernel: CsrKernel, bias=None):
    """Instrumented path (engine.py:109-128): runs the generic one-thread-
    per-output kernel -- independent of the tiled kernels -- and returns
    (output, exact multiply-accumulate count)."""
    out = _run(x, kernel, bias, EnginePlan(), generic=True)
    sh = kernel.shape
    per_ch = np.diff(np.asarray(kernel.rowptr, np.int64))
    macs = int(x.shape[0]) * int(per_ch.sum()) * sh.e * sh.f
    return out, macs


def sparse_mac_count(kernel: CsrKernel, batch: int) -> int:
    """Executed MACs: N*K*E*F*L for unified kernels (engine.py:131-136)."""
    sh = kernel.shape
    if kernel.unified:
        return batch * sh.k * sh.e * sh.f * kernel.sparse_level
    return batch * sh.e * sh.f * int(kernel.nnz)


def dense_mac_count(shape, batch: int) -> int:
    return batch * shape.k * shape.e * shape.f * shape.kernel_volume


def tune_sub_batch(x, kernel: CsrKernel, bias=None, candidates=SUB_BATCH_CANDIDATES,
                   worker_count: int = 1, repetitions: int = 5,
                   warmups: int = 2) -> tuple[int, dict[int, float]]:
    """Timed argmin over images-per-CTA candidates (engine.py:143-166
    contract: median of `repetitions` after `warmups`, ties to the smaller).
    Timing uses CUDA events around each launch.  For the full launch search
    see tuner.tune_launch."""
    if not candidates:
        raise ShapeError("candidate set must be non-empty")
    from .tuner import time_call
    timings: dict[int, float] = {}
    for sb in sorted(candidates):
        plan = EnginePlan(sub_batch_size=sb, worker_count=worker_count)
        timings[sb] = time_call(lambda: conv_sparse(x, kernel, bias, plan),
                                repetitions=max(repetitions, 1), warmups=warmups)
    best = min(timings, key=lambda sb: (timings[sb], sb))
    return best, timings
