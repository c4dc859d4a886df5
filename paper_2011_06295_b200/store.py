"""Model-store loader: the reference's on-disk model directory
(manifest.json + 64-byte-header blobs, pkg/docs/format.md; writer
sc/store.py:323-372) read straight into device-ready layers.

Only what the hot path needs is read: the conv layers (CSR triplet or dense
KCRS weights, bias, activation) in order.  Every blob is FNV-1a-64 verified
with the native ``scb_fnv1a64`` before use and every CSR kernel is
re-validated (``CsrKernel.validate``, csr.py:50-73), exactly the reference's
loading guarantees (format.md "Loading guarantees", store.py:375-434).
Dense-stored conv layers are converted with the C++ ``build_csr`` once here,
for the input geometry propagated from the recorded architecture -- the
reference rebuilds them on every forward (store.py:178-182).  Codebook
layers need nothing extra: the reference stores their dequantized values
(quantize.py:275-288), which the device layer can also re-encode as 4-bit
codes (weight_format="cb4").  Layers with an activation quantizer (the
manifest's act_quant, fitted by apply_quantization) get the fused fake-quant
epilogue (quantize.py:332-338; store.py:285-286).  The fully connected head is
out of scope.
"""
from __future__ import annotations

import ctypes
import json
from pathlib import Path

import numpy as np

from . import _abi
from .errors import FormatError, ShapeError
from .geometry import ConvShape
from .weights import CsrKernel, build_csr

FORMAT_VERSION = 1
_MAGIC = b"SCBLOB01"
_HEADER = 64
_DTYPES = {"f32": np.dtype("<f4"), "f16": np.dtype("<f2"), "f64": np.dtype("<f8"),
           "i32": np.dtype("<i4"), "i64": np.dtype("<i8"), "u8": np.dtype("u1")}


def fnv1a64(data: bytes) -> int:
    """64-bit FNV-1a (store.py:46-51) computed by the native library."""
    buf = np.frombuffer(data, dtype=np.uint8)
    out = ctypes.c_uint64(0)
    _abi.check(_abi.lib().scb_fnv1a64(ctypes.c_void_p(buf.ctypes.data) if buf.size else None,
                                      int(buf.size), ctypes.byref(out)), "scb_fnv1a64")
    return int(out.value)


def read_blob(path: Path, entry: dict) -> np.ndarray:
    """One blob: checksum, magic, tag and size checks (format.md), then the
    payload (nibble-unpacked for u8-packed-codes)."""
    blob = Path(path).read_bytes()
    if f"{fnv1a64(blob):016x}" != entry["checksum"]:
        raise FormatError(f"checksum mismatch for {Path(path).name}")
    if blob[:8] != _MAGIC:
        raise FormatError(f"{Path(path).name}: bad blob magic")
    tag = entry["dtype"]
    if blob[8:16].rstrip(b"\0").decode() != tag[:8]:
        raise FormatError(f"{Path(path).name}: dtype tag disagrees with manifest")
    shape = tuple(entry["shape"])
    count = int(np.prod(shape)) if shape else 1
    payload = blob[_HEADER:]
    if tag == "u8-packed-codes":
        packed = np.frombuffer(payload, dtype=np.uint8)
        flat = np.empty(packed.size * 2, dtype=np.uint8)
        flat[0::2] = packed & 0x0F
        flat[1::2] = packed >> 4
        if flat.size < count:
            raise FormatError(f"{Path(path).name}: payload size disagrees with shape")
        return flat[:count].reshape(shape).astype(np.int64)
    dt = _DTYPES.get(tag)
    if dt is None:
        raise FormatError(f"{Path(path).name}: unknown dtype tag {tag!r}")
    arr = np.frombuffer(payload, dtype=dt)
    if arr.size != count:
        raise FormatError(f"{Path(path).name}: payload size disagrees with shape")
    return arr.reshape(shape).astype(dt.newbyteorder("="))


def load_conv_layers(path, input_chw: tuple | None = None):
    """[NetLayer] of the model's conv stack (no pooling: Model.forward has none).
    `input_chw` overrides the manifest's meta.architecture input geometry."""
    from .network import NetLayer
    path = Path(path)
    mpath = path / "manifest.json"
    if not mpath.exists():
        raise FormatError(f"{path} has no manifest.json")
    manifest = json.loads(mpath.read_text())
    if manifest.get("format_version") != FORMAT_VERSION:
        raise FormatError(f"unsupported format version {manifest.get('format_version')!r}")
    blobs = manifest["blobs"]

    def get(key):
        if key not in blobs:
            raise FormatError(f"manifest references missing blob entry {key!r}")
        entry = blobs[key]
        bp = path / entry["file"]
        if not bp.exists():
            raise FormatError(f"missing blob file {entry['file']}")
        return read_blob(bp, entry)

    if input_chw is None:
        arch = manifest.get("meta", {}).get("architecture")
        if arch is not None:
            input_chw = (arch["in_channels"], arch["image_size"], arch["image_size"])
    layers = []
    chw = input_chw
    for rec in manifest["layers"]:
        if rec["type"] != "conv":
            continue
        bias = get(rec["bias"])
        if rec["storage"] == "csr":
            sh = ConvShape(**rec["conv_shape"])
            kern = CsrKernel(values=get(rec["values"]), colidx=get(rec["colidx"]).astype(np.int32),
                             rowptr=get(rec["rowptr"]).astype(np.int32), sparse_level=rec["sparse_level"],
                             shape=sh, unified=rec["unified"])
            kern.validate()
        elif rec["storage"] == "dense":
            w = get(rec["weights"])
            if chw is None:
                raise ShapeError("dense-stored conv layer needs the input geometry (meta.architecture)")
            k, c, r, s = w.shape
            sh = ConvShape(n=1, c=c, h=chw[1], w=chw[2], k=k, r=r, s=s, stride=rec["stride"],
                           padding=rec["padding"])
            kern = build_csr(w, sh)
        else:
            raise FormatError(f"unknown storage {rec['storage']!r}")
        layers.append(NetLayer(rec["name"], kern, bias, relu=rec.get("activation", "relu") == "relu", pool=False,
                               act_quant=rec.get("act_quant")))
        chw = (kern.shape.k, kern.shape.e, kern.shape.f)
    if not layers:
        raise FormatError("model has no conv layers")
    return layers


def load_net(path, device: int = 0, weight_format: str = "native", input_chw=None, dtype=None):
    """SparseConvNet of a stored model's conv stack, resident on `device`.

    The reference's Model.forward computes in the dtype of the input it is given
    (store.py:263-286); a device network fixes its activation dtype up front, so pass the
    dtype of the inputs you will feed (`dtype`).  Default: f16 when the stored weights are
    f16, else f32; SparseConvNet.forward refuses an input of another dtype rather than
    casting it.  Dense-stored conv layers are converted with build_csr on load and run on
    the sparse kernels (the reference runs them dense-gemm); the result is the same
    convolution, summed in the reference's colidx order."""
    from .network import SparseConvNet
    layers = load_conv_layers(path, input_chw)
    if dtype is None:
        dtype = np.float16 if layers[0].kernel.values.dtype == np.float16 else np.float32
    return SparseConvNet(layers, device=device, dtype=dtype, weight_format=weight_format)
