"""Unified-sparsity CSR weight format (drop-in for the reference's csr.py).

The arrays and their invariants are the reference's (csr.py:33-77):
``values`` (the weight dtype), ``colidx`` int32 offsets ``c*Hp*Wp + r*Wp + s``
into the padded input plane, ``rowptr`` int32 (K+1), ``sparse_level`` = the
unified per-channel count.  Building, validation and decompression run in the
C++ builder of libsparseconv_b200 (csrc/builder.cpp), bit-exact with the
reference including the zero-promotion order (csr.py:94-117) and the sign bit
of promoted -0.0 entries.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import ShapeError
from .geometry import ConvShape

_DT = {np.dtype(np.float32): _abi.SCB_F32, np.dtype(np.float64): _abi.SCB_F64,
       np.dtype(np.float16): _abi.SCB_F16}


def _code(dtype) -> int:
    try:
        return _DT[np.dtype(dtype)]
    except KeyError:
        raise ShapeError(f"weight dtype {dtype} not in f32/f64/f16") from None


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class SparsityReport:
    """Zero statistics of one KCRS weight tensor."""

    per_channel_nnz: np.ndarray
    unified_nnz: int
    padded_zero_count: int
    layer_sparsity: float


@dataclass
class CsrKernel:
    """Compressed weights of one layer; treat as immutable once built (the
    device copy is cached per CsrKernel and keyed on the array objects)."""

    values: np.ndarray
    colidx: np.ndarray
    rowptr: np.ndarray
    sparse_level: int
    shape: ConvShape
    unified: bool = True
    _device_cache: dict = field(default_factory=dict, repr=False, compare=False)
    # quantizer metadata of the values (the reference's quantize_weights_array meta, e.g.
    # {"scheme": "affine", "bits": 16, "step": s}, quantize.py:265-288); None = plain floats
    quant: dict | None = field(default=None, repr=False, compare=False)

    def validate(self) -> None:
        """Structural invariants (csr.py:50-73); raises FormatError."""
        from .errors import FormatError
        sh = self.shape
        if self.values.ndim != 1 or self.values.shape != self.colidx.shape:
            raise FormatError("values/colidx must be parallel 1D arrays")
        if self.rowptr.shape != (sh.k + 1,):
            raise FormatError(f"rowptr must have length K+1={sh.k + 1}")
        colidx = np.ascontiguousarray(self.colidx, dtype=np.int32)
        rowptr = np.ascontiguousarray(self.rowptr, dtype=np.int32)
        st = _abi.shape_struct(sh)
        _abi.check(_abi.lib().scb_validate_csr(ctypes.byref(st), _ptr(colidx), _ptr(rowptr),
                                               len(colidx), int(bool(self.unified)),
                                               int(self.sparse_level)))

    @property
    def nnz(self) -> int:
        return len(self.values)


def analyze_sparsity(weights: np.ndarray) -> SparsityReport:
    """Per-channel nonzero counts and the unified count (csr.py:80-91)."""
    weights = np.asarray(weights)
    if weights.ndim != 4 or weights.size == 0:
        raise ShapeError("weights must be a non-empty KCRS tensor")
    w = np.ascontiguousarray(weights)
    k = w.shape[0]
    vol = w.size // k
    nnz = np.empty(k, np.int64)
    _abi.check(_abi.lib().scb_channel_nnz(_ptr(w), _code(w.dtype), k, vol, _ptr(nnz)))
    unified = int(nnz.max())
    return SparsityReport(per_channel_nnz=nnz, unified_nnz=unified,
                          padded_zero_count=int(np.sum(unified - nnz)),
                          layer_sparsity=1.0 - int(nnz.sum()) / w.size)


def select_padding_zeros(channel_weights: np.ndarray, deficit: int) -> np.ndarray:
    """Zero positions promoted to stored entries (csr.py:94-117), ascending."""
    flat = np.ascontiguousarray(np.asarray(channel_weights).ravel())
    if flat.dtype not in _DT:
        flat = flat.astype(np.float64)
    out = np.empty(max(int(deficit), 1), np.int64)
    _abi.check(_abi.lib().scb_select_padding_zeros(_ptr(flat), _code(flat.dtype), flat.size,
                                                   int(deficit), _ptr(out)))
    return out[:int(deficit)]


def build_csr(weights: np.ndarray, shape: ConvShape, unify: bool = True) -> CsrKernel:
    """Compress a KCRS tensor for `shape` (csr.py:120-165)."""
    weights = np.asarray(weights)
    if weights.ndim != 4:
        raise ShapeError("weights must be KCRS 4D")
    k, c, r, s = weights.shape
    if (k, c, r, s) != (shape.k, shape.c, shape.r, shape.s):
        raise ShapeError(f"weights {weights.shape} inconsistent with shape KCRS="
                         f"({shape.k},{shape.c},{shape.r},{shape.s})")
    w = np.ascontiguousarray(weights)
    code = _code(w.dtype)
    st = _abi.shape_struct(shape)
    L = _abi.lib()
    nnz, level = ctypes.c_int64(0), ctypes.c_int32(0)
    _abi.check(L.scb_csr_count(_ptr(w), code, ctypes.byref(st), int(unify),
                               ctypes.byref(nnz), ctypes.byref(level)))
    values = np.empty(nnz.value, w.dtype)
    colidx = np.empty(nnz.value, np.int32)
    rowptr = np.empty(k + 1, np.int32)
    _abi.check(L.scb_build_csr(_ptr(w), code, ctypes.byref(st), int(unify), nnz.value,
                               _ptr(values), _ptr(colidx), _ptr(rowptr)))
    kern = CsrKernel(values=values, colidx=colidx, rowptr=rowptr,
                     sparse_level=int(level.value), shape=shape, unified=bool(unify))
    kern.validate()
    return kern


def decompress(kernel: CsrKernel) -> np.ndarray:
    """Exact inverse of build_csr (csr.py:168-178)."""
    kernel.validate()
    sh = kernel.shape
    out = np.empty((sh.k, sh.c, sh.r, sh.s), kernel.values.dtype)
    vals = np.ascontiguousarray(kernel.values)
    colidx = np.ascontiguousarray(kernel.colidx, dtype=np.int32)
    rowptr = np.ascontiguousarray(kernel.rowptr, dtype=np.int32)
    st = _abi.shape_struct(sh)
    _abi.check(_abi.lib().scb_decompress(ctypes.byref(st), _code(vals.dtype), _ptr(vals),
                                         _ptr(colidx), _ptr(rowptr), len(vals), _ptr(out)))
    return out
