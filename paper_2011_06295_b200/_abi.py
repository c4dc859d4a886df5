"""ctypes binding of the C ABI in include/sparseconv_b200.h.

The shared library is built in-tree (paper_2011_06295_b200/_lib/) by
``paper_2011_06295_b200/csrc/Makefile`` (``__graft_entry__.build()``).  There
is no CPU fallback: if the library is missing every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

from .errors import FormatError, IntegrityError, ShapeError, SparseConvError

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SCB_LIB"]) if os.environ.get("SCB_LIB") else PKG / "_lib" / "libsparseconv_b200.so"
CSRC = PKG / "csrc"

SCB_OK, SCB_ERR_SHAPE, SCB_ERR_FORMAT, SCB_ERR_INTEGRITY = 0, 1, 2, 3
SCB_ERR_CUDA, SCB_ERR_ARG, SCB_ERR_UNSUPPORTED = 4, 5, 6

SCB_F32, SCB_F64, SCB_F16 = 0, 1, 2
SCB_W_NATIVE, SCB_W_CB4, SCB_W_LIN16, SCB_W_AFF16 = 0, 1, 2, 3

FLAG_RELU, FLAG_FAST, FLAG_POOL2, FLAG_GENERIC, FLAG_NO_PDL = 0x1, 0x2, 0x4, 0x8, 0x10
FLAG_ACT_QUANT = 0x20
FLAG_IMAGE_MINOR = 0x40  # x / y image-minor: ((c*H + h)*W + w)*ld + n (kind-7 launches)
FLAG_Y_IMAGE_MINOR = 0x80  # NCHW x, image-minor y (narrow direct kernels)
FLAG_Y_NCHW = 0x100  # with FLAG_IMAGE_MINOR: NCHW y (kind-7 kernels)
KIND_LANE = 7

# every symbol include/sparseconv_b200.h declares
EXPORTS = (
    "scb_channel_nnz", "scb_select_padding_zeros", "scb_csr_count", "scb_build_csr",
    "scb_validate_csr", "scb_decompress", "scb_layer_create", "scb_layer_create_q", "scb_layer_destroy",
    "scb_layer_weight_bytes", "scb_conv_sparse", "scb_launch_candidates",
    "scb_default_launch", "scb_layer_prepare", "scb_launch_check", "scb_variant_count", "scb_variant_get", "scb_maxpool2",
    "scb_fma_peaks", "scb_fnv1a64", "scb_last_error", "scb_version", "scb_fake_quant",
    "scb_layer_set_act_quant", "scb_conv_sparse_ld", "scb_to_image_minor", "scb_from_image_minor",
)


class Shape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("n", "c", "h", "w", "k", "r", "s", "stride", "padding")]


class Launch(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("variant", "warps_k", "imgs", "bh", "bw", "cc", "stages")]

    def as_tuple(self):
        return (self.variant, self.warps_k, self.imgs, self.bh, self.bw, self.cc, self.stages)

    @classmethod
    def from_tuple(cls, t):
        return cls(*[int(v) for v in t])


class ActQuant(ctypes.Structure):
    """scb_act_quant: the reference's layer.act_quant dict (quantize.py:324-326)."""
    _fields_ = [("bits", ctypes.c_int32), ("symmetric", ctypes.c_int32), ("clip_lo", ctypes.c_double),
                ("clip_hi", ctypes.c_double), ("mu", ctypes.c_double), ("step", ctypes.c_double)]

    @classmethod
    def from_dict(cls, aq: dict):
        mode = aq.get("mode", "asymmetric")
        if mode not in ("asymmetric", "symmetric"):
            raise ValueError(f"unknown activation quantization mode {mode!r}")
        return cls(int(aq["bits"]), 1 if mode == "symmetric" else 0, float(aq["clip_lo"]),
                   float(aq["clip_hi"]), float(aq["mu"]), float(aq["step"]))


class VariantInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("r", "s", "kt", "nbt", "th", "tw", "io", "wf", "mode", "dispatch", "pad", "kind")]


_lock = threading.Lock()
_lib = None


def build(quiet: bool = True) -> Path:
    """Compile the CUDA library for sm_100a in place (nvcc cross-compiles; no GPU needed)."""
    cmd = ["make", "-C", str(CSRC), f"-j{min(8, os.cpu_count() or 1)}"]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL if quiet else None)
    return LIB_PATH


def lib():
    """Load libsparseconv_b200.so; raise loudly if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise SparseConvError(
                f"CUDA library {LIB_PATH} is missing: run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        P = ctypes.POINTER
        sig = {
            "scb_channel_nnz": [vp, i32, i32, i64, vp],
            "scb_select_padding_zeros": [vp, i32, i64, i64, vp],
            "scb_csr_count": [vp, i32, P(Shape), i32, P(i64), P(i32)],
            "scb_build_csr": [vp, i32, P(Shape), i32, i64, vp, vp, vp],
            "scb_validate_csr": [P(Shape), vp, vp, i64, i32, i32],
            "scb_decompress": [P(Shape), i32, vp, vp, vp, i64, vp],
            "scb_layer_create": [P(Shape), i32, i32, vp, vp, vp, i64, i32, i32, P(vp)],
            "scb_layer_create_q": [P(Shape), i32, i32, vp, vp, vp, i64, i32, i32, ctypes.c_double, P(vp)],
            "scb_layer_destroy": [vp],
            "scb_layer_weight_bytes": [vp, i32, P(i64)],
            "scb_conv_sparse": [vp, vp, vp, vp, i32, u32, P(Launch), vp],
            "scb_conv_sparse_ld": [vp, vp, i64, vp, vp, i64, i32, u32, P(Launch), vp],
            "scb_to_image_minor": [i32, vp, vp, i32, i64, i64, vp],
            "scb_from_image_minor": [i32, vp, i64, vp, i32, i64, vp],
            "scb_launch_candidates": [vp, i32, u32, P(Launch), i32, P(i32)],
            "scb_default_launch": [vp, i32, u32, i32, P(Launch)],
            "scb_layer_prepare": [vp, i32, u32, P(Launch)],
            "scb_launch_check": [vp, i32, u32, P(Launch)],
            "scb_variant_get": [i32, P(VariantInfo)],
            "scb_maxpool2": [i32, vp, vp, i64, i32, i32, vp],
            "scb_fma_peaks": [i32, vp, vp, i32, P(i32)],
            "scb_fnv1a64": [vp, i64, P(ctypes.c_uint64)],
            "scb_fake_quant": [i32, vp, i64, P(ActQuant), vp],
            "scb_layer_set_act_quant": [vp, P(ActQuant)],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.scb_variant_count.restype = i32
        L.scb_variant_count.argtypes = []
        L.scb_last_error.restype = ctypes.c_char_p
        L.scb_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def last_error() -> str:
    return lib().scb_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map a C status onto the reference exception hierarchy (errors.py)."""
    if status == SCB_OK:
        return
    msg = last_error() or what
    if status == SCB_ERR_SHAPE:
        raise ShapeError(msg)
    if status == SCB_ERR_FORMAT:
        raise FormatError(msg)
    if status == SCB_ERR_INTEGRITY:
        raise IntegrityError(msg)
    raise SparseConvError(f"{what}: {msg}" if what else msg)


def shape_struct(sh) -> Shape:
    return Shape(int(sh.n), int(sh.c), int(sh.h), int(sh.w), int(sh.k), int(sh.r), int(sh.s),
                 int(sh.stride), int(sh.padding))


def variants():
    L = lib()
    out = []
    for i in range(L.scb_variant_count()):
        v = VariantInfo()
        check(L.scb_variant_get(i, ctypes.byref(v)))
        out.append({f: getattr(v, f) for f, _ in VariantInfo._fields_})
    return out


_DT_CODE = {"float32": SCB_F32, "float64": SCB_F64, "float16": SCB_F16}


def fake_quant(dtype, y_ptr: int, count: int, aq: dict, stream: int = 0) -> None:
    """In-place activation fake-quant of `count` device values (scb_fake_quant,
    the reference's fake_quant_activation, quantize.py:332-338)."""
    import numpy as np
    q = ActQuant.from_dict(aq)
    check(lib().scb_fake_quant(_DT_CODE[str(np.dtype(dtype))], ctypes.c_void_p(y_ptr), int(count),
                               ctypes.byref(q), ctypes.c_void_p(stream)), "scb_fake_quant")


def maxpool2(dtype, x_ptr: int, y_ptr: int, planes: int, h: int, w: int, stream: int = 0) -> None:
    """2x2 stride-2 max pool over `planes` h x w planes (scb_maxpool2)."""
    import numpy as np
    check(lib().scb_maxpool2(_DT_CODE[str(np.dtype(dtype))], ctypes.c_void_p(x_ptr),
                             ctypes.c_void_p(y_ptr), int(planes), int(h), int(w),
                             ctypes.c_void_p(stream)), "scb_maxpool2")


def to_image_minor(dtype, x_ptr: int, y_ptr: int, n: int, chw: int, ldy: int, stream: int = 0) -> None:
    """NCHW (n, chw) -> image-minor y[j*ldy + i] (scb_to_image_minor)."""
    import numpy as np
    check(lib().scb_to_image_minor(_DT_CODE[str(np.dtype(dtype))], ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                   int(n), int(chw), int(ldy), ctypes.c_void_p(stream)), "scb_to_image_minor")


def from_image_minor(dtype, x_ptr: int, ldx: int, y_ptr: int, n: int, chw: int, stream: int = 0) -> None:
    """image-minor x[j*ldx + i] -> NCHW (n, chw) (scb_from_image_minor)."""
    import numpy as np
    check(lib().scb_from_image_minor(_DT_CODE[str(np.dtype(dtype))], ctypes.c_void_p(x_ptr), int(ldx),
                                     ctypes.c_void_p(y_ptr), int(n), int(chw), ctypes.c_void_p(stream)),
          "scb_from_image_minor")
