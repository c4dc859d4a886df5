"""Device-side residency of CsrKernel weights.

A ``DeviceLayer`` owns one ``scb_layer`` handle: the CSR uploaded to one GPU
as the tap programs of the tiled kernels plus the arrays of the generic
kernel.  It is built once per (CsrKernel, device, activation dtype, weight
format) and cached on the CsrKernel -- the reference rebuilds CSR per forward
for dense-stored layers (store.py:178-182); here the upload happens once and
every call after that is a single asynchronous launch.
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _abi
from .errors import ShapeError

_WFMT = {"native": _abi.SCB_W_NATIVE, "cb4": _abi.SCB_W_CB4, "lin16": _abi.SCB_W_LIN16,
         "aff16": _abi.SCB_W_AFF16}
_IO = {np.dtype(np.float32): _abi.SCB_F32, np.dtype(np.float64): _abi.SCB_F64,
       np.dtype(np.float16): _abi.SCB_F16}


def _destroy(handle: int) -> None:
    try:
        _abi.lib().scb_layer_destroy(ctypes.c_void_p(handle))
    except Exception:
        pass


class DeviceLayer:
    """Handle of one uploaded layer (see include/sparseconv_b200.h)."""

    def __init__(self, kernel, device: int, io_dtype, weight_format: str = "native"):
        io_dtype = np.dtype(io_dtype)
        if weight_format not in _WFMT:
            raise ShapeError(f"unknown weight format {weight_format!r}")
        self.shape = kernel.shape
        self.device = int(device)
        self.io_dtype = io_dtype
        self.weight_format = weight_format
        self.sparse_level = int(kernel.sparse_level)
        self.unified = bool(kernel.unified)
        vals = np.ascontiguousarray(kernel.values, dtype=io_dtype)
        colidx = np.ascontiguousarray(kernel.colidx, dtype=np.int32)
        rowptr = np.ascontiguousarray(kernel.rowptr, dtype=np.int32)
        self.nnz = int(len(vals))
        self.rowptr = rowptr.copy()
        st = _abi.shape_struct(kernel.shape)
        h = ctypes.c_void_p()
        # affine int16 codes need the quantizer's step (quantize.py:137-138)
        self.qstep = float((kernel.quant or {}).get("step", 0.0)) if weight_format == "aff16" else 0.0
        if weight_format == "aff16" and not self.qstep > 0:
            raise ShapeError("weight_format 'aff16' needs kernel.quant['step'] (the affine quantizer's step)")
        _abi.check(_abi.lib().scb_layer_create_q(
            ctypes.byref(st), _IO[io_dtype], _WFMT[weight_format],
            ctypes.c_void_p(vals.ctypes.data), ctypes.c_void_p(colidx.ctypes.data),
            ctypes.c_void_p(rowptr.ctypes.data), self.nnz, int(kernel.unified),
            self.device, ctypes.c_double(self.qstep), ctypes.byref(h)), "scb_layer_create")
        self.handle = h.value
        self._fin = weakref.finalize(self, _destroy, self.handle)
        self._prepared = set()

    # ---- launches -------------------------------------------------------
    def prepare(self, n: int, flags: int, launch=None) -> None:
        """Build the device tables of `launch` once (scb_layer_prepare); the launch
        itself then never allocates or synchronises (CUDA-graph capturable)."""
        key = (int(n), int(flags), None if launch is None else tuple(launch))
        if key in self._prepared:
            return
        cfg = None if launch is None else ctypes.byref(_abi.Launch.from_tuple(launch))
        _abi.check(_abi.lib().scb_layer_prepare(ctypes.c_void_p(self.handle), int(n), int(flags), cfg),
                   "scb_layer_prepare")
        self._prepared.add(key)

    def launch_ok(self, n: int, flags: int, launch) -> bool:
        """Whether `launch` is valid for this layer at batch n (scb_launch_check)."""
        if launch is None:
            return True
        st = _abi.lib().scb_launch_check(ctypes.c_void_p(self.handle), int(n), int(flags),
                                         ctypes.byref(_abi.Launch.from_tuple(launch)))
        return st == 0

    def launch(self, x_ptr: int, bias_ptr: int | None, y_ptr: int, n: int, flags: int,
               launch=None, stream: int = 0, ldx: int | None = None, ldy: int | None = None) -> None:
        """scb_conv_sparse_ld; ldx / ldy are the image-minor row strides (FLAG_IMAGE_MINOR,
        default n), ignored for NCHW activations."""
        if launch is not None or not (flags & _abi.FLAG_GENERIC):
            self.prepare(n, flags, launch)
        cfg = None if launch is None else ctypes.byref(_abi.Launch.from_tuple(launch))
        _abi.check(_abi.lib().scb_conv_sparse_ld(
            ctypes.c_void_p(self.handle), ctypes.c_void_p(x_ptr), int(n if ldx is None else ldx),
            ctypes.c_void_p(bias_ptr) if bias_ptr else None, ctypes.c_void_p(y_ptr),
            int(n if ldy is None else ldy), int(n), int(flags), cfg, ctypes.c_void_p(stream)), "scb_conv_sparse")

    def candidates(self, n: int, flags: int = 0, cap: int = 4096):
        buf = (_abi.Launch * cap)()
        cnt = ctypes.c_int32(0)
        _abi.check(_abi.lib().scb_launch_candidates(ctypes.c_void_p(self.handle), int(n),
                                                    int(flags), buf, cap, ctypes.byref(cnt)))
        return [buf[i].as_tuple() for i in range(min(cnt.value, cap))]

    def default_launch(self, n: int, flags: int = 0, prefer_imgs: int = 0):
        out = _abi.Launch()
        _abi.check(_abi.lib().scb_default_launch(ctypes.c_void_p(self.handle), int(n), int(flags),
                                                 int(prefer_imgs), ctypes.byref(out)))
        return out.as_tuple()

    def weight_bytes(self, variant: int) -> int:
        b = ctypes.c_int64(0)
        _abi.check(_abi.lib().scb_layer_weight_bytes(ctypes.c_void_p(self.handle), int(variant),
                                                     ctypes.byref(b)))
        return int(b.value)

    def set_act_quant(self, aq: dict | None) -> None:
        """Attach (dict as in the reference's layer.act_quant, quantize.py:324-326)
        or clear (None) the activation fake-quant applied under FLAG_ACT_QUANT."""
        q = None if aq is None else ctypes.byref(_abi.ActQuant.from_dict(aq))
        _abi.check(_abi.lib().scb_layer_set_act_quant(ctypes.c_void_p(self.handle), q),
                   "scb_layer_set_act_quant")

    def signature(self):
        """Key of the tuner cache: everything the best launch depends on."""
        sh = self.shape
        return (sh.c, sh.h, sh.w, sh.k, sh.r, sh.s, sh.stride, sh.padding, self.sparse_level,
                self.unified, str(self.io_dtype), self.weight_format)


def device_layer(kernel, device: int, io_dtype, weight_format: str = "native") -> DeviceLayer:
    """Cached DeviceLayer of `kernel` (keyed on the identity of its arrays)."""
    io_dtype = np.dtype(io_dtype)
    key = (int(device), str(io_dtype), weight_format, float((kernel.quant or {}).get("step", 0.0)))
    ident = (id(kernel.values), id(kernel.colidx), id(kernel.rowptr), int(kernel.sparse_level),
             bool(kernel.unified), kernel.shape)
    cache = kernel._device_cache
    hit = cache.get(key)
    if hit is not None and hit[0] == ident:
        return hit[1]
    kernel.validate()
    layer = DeviceLayer(kernel, device, io_dtype, weight_format)
    # keep the arrays alive with the entry so their ids cannot be recycled
    cache[key] = (ident, layer, (kernel.values, kernel.colidx, kernel.rowptr))
    return layer
