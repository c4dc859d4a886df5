"""Synthetic workloads of BASELINE.json (weights and inputs are synthetic:
there is no network for datasets or checkpoints).

* ``make_layer_weights`` restates the reference generator bench.py:105-116:
  every output channel gets exactly ``vol - round(sparsity*vol)`` N(0,1)
  nonzeros at ``rng.choice`` positions, same rng call order, so the weights
  are bit-identical to the reference's for the same seed
  (tests/test_gpu_parity.py checks the digest recorded from the reference).
* ``bench_inputs`` restates bench.py:175-177 (x, bias ~ N(0,1) from
  ``default_rng(seed+1)``).
* The CIFAR-10 stacks are builder-defined: the reference only
  ships ImageNet shapes (bench.py:74-102).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ShapeError
from .geometry import ConvShape


@dataclass(frozen=True)
class LayerSpec:
    """One benchmark subject: geometry (batch replaced at run time) + sparsity."""

    name: str
    shape: ConvShape
    sparsity: float
    source: str = "builder-defined"

    def __post_init__(self):
        if not 0.0 <= self.sparsity <= 1.0:
            raise ShapeError(f"sparsity must be in [0,1], got {self.sparsity}")


def make_layer_weights(spec: LayerSpec, seed: int = 0) -> np.ndarray:
    sh = spec.shape
    rng = np.random.default_rng(seed)
    vol = sh.c * sh.r * sh.s
    keep = vol - int(round(spec.sparsity * vol))
    w = np.zeros((sh.k, vol), np.float32)
    for k in range(sh.k):
        pos = rng.choice(vol, size=keep, replace=False)
        w[k, pos] = rng.standard_normal(keep)
    return w.reshape(sh.k, sh.c, sh.r, sh.s)


def bench_inputs(shape: ConvShape, batch: int, seed: int = 0):
    rng = np.random.default_rng(seed + 1)
    x = rng.standard_normal((batch, shape.c, shape.h, shape.w)).astype(np.float32)
    bias = rng.standard_normal(shape.k).astype(np.float32)
    return x, bias


def _vgg(c, hw, k):
    return ConvShape(n=1, c=c, h=hw, w=hw, k=k, r=3, s=3, stride=1, padding=1)


# (name, C, H, K, pool after)
VGG16_CIFAR_LAYERS = [
    ("conv1_1", 3, 32, 64, False), ("conv1_2", 64, 32, 64, True),
    ("conv2_1", 64, 16, 128, False), ("conv2_2", 128, 16, 128, True),
    ("conv3_1", 128, 8, 256, False), ("conv3_2", 256, 8, 256, False), ("conv3_3", 256, 8, 256, True),
    ("conv4_1", 256, 4, 512, False), ("conv4_2", 512, 4, 512, False), ("conv4_3", 512, 4, 512, True),
    ("conv5_1", 512, 2, 512, False), ("conv5_2", 512, 2, 512, False), ("conv5_3", 512, 2, 512, True),
]

# AlexNet-style CIFAR-10 stack: 5x5 then 3x3, "same" padding
ALEXNET_CIFAR_LAYERS = [
    ("conv1", 3, 32, 64, 5, True), ("conv2", 64, 16, 192, 5, True),
    ("conv3", 192, 8, 384, 3, False), ("conv4", 384, 8, 256, 3, False),
    ("conv5", 256, 8, 256, 3, False),
]


def vgg16_cifar(sparsity: float = 0.9):
    """[(LayerSpec, pool_after)] of the 13 VGG-16 convs on 32x32 inputs."""
    return [(LayerSpec(n, _vgg(c, h, k), sparsity), pool) for n, c, h, k, pool in VGG16_CIFAR_LAYERS]


def alexnet_cifar(sparsity: float = 0.9):
    out = []
    for n, c, h, k, ks, pool in ALEXNET_CIFAR_LAYERS:
        sh = ConvShape(n=1, c=c, h=h, w=h, k=k, r=ks, s=ks, stride=1, padding=ks // 2)
        out.append((LayerSpec(n, sh, sparsity), pool))
    return out


SWEEP_SPARSITIES = (0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.97, 0.98, 0.99)


def sweep_layer(sparsity: float) -> LayerSpec:
    """BASELINE config 5: 256->256, 3x3, 32x32."""
    return LayerSpec(f"sweep256_s{sparsity:g}", _vgg(256, 32, 256), sparsity)


def _shape(c, h, w, k, r, s, padding=0):
    return ConvShape(n=1, c=c, h=h, w=w, k=k, r=r, s=s, stride=1, padding=padding)


# The reference's named layer presets (pkg/src/sparseconv/bench.py:74-102),
# timed at its DEFAULT_BATCH = 128 (bench.py:29) by tools/bench_presets.py.
PRESET_BATCH = 128
PRESETS = {
    "vgg16": [LayerSpec(f"{c}x{hw}x{hw}x{k}", _vgg(c, hw, k), 0.90)
              for c, hw, k in [(3, 224, 64), (64, 224, 64), (64, 112, 128), (128, 112, 128), (128, 56, 256),
                               (256, 56, 256), (256, 28, 512), (512, 28, 512), (512, 14, 512)]],
    "vgg16-mini": [LayerSpec("64x28x28x64", _vgg(64, 28, 64), 0.90)],
    "resnet-1x1": [LayerSpec("256-filters-1x1x64", _shape(64, 56, 56, 256, 1, 1), 0.90),
                   LayerSpec("64-filters-1x1x256", _shape(256, 56, 56, 64, 1, 1), 0.90)],
    "densenet-1x1": [LayerSpec("densenet121-block3-layer24", _shape(992, 14, 14, 128, 1, 1), 0.875),
                     LayerSpec("densenet121-block3-layer24-r91", _shape(992, 14, 14, 128, 1, 1), 0.91),
                     LayerSpec("densenet161-block4-layer16", _shape(1776, 7, 7, 192, 1, 1), 0.91),
                     LayerSpec("densenet161-block3-layer16", _shape(1104, 14, 14, 192, 1, 1), 0.93)],
    "cnn-non-static": [LayerSpec(f"300x64-kernel{s}-s{sp * 100:g}", _shape(64, 1, 300, 100, 1, s), sp)
                       for s in (2, 3) for sp in (0.77, 0.83, 0.875)],
}


def codebook16(w: np.ndarray) -> np.ndarray:
    """Synthetic 4-bit-codebook weights (config 4, the paper's "4b/16b"): every nonzero
    mapped to the nearest of 14 f16 centroids spread over [-max|w|, max|w|] (zero excluded),
    so a layer holds <= 16 distinct values with the +-0.0 of promoted zeros -- what
    quantize_weights_array("codebook", 16) produces in form (quantize.py:284-288)."""
    w = np.asarray(w)
    m = float(np.abs(w).max()) or 1.0
    cent = np.concatenate([-np.geomspace(m, m / 16, 7), np.geomspace(m / 16, m, 7)]).astype(np.float16)
    out = w.astype(np.float32).copy()
    nz = out != 0
    idx = np.abs(out[nz][:, None] - cent.astype(np.float32)[None, :]).argmin(axis=1)
    out[nz] = cent[idx].astype(np.float32)
    return out.astype(w.dtype)


def linear16(w: np.ndarray, frac: int = 8) -> np.ndarray:
    """Synthetic linear 16-bit weights (config 4, quantize_fixed's sigma * code with
    sigma = 2^-frac, quantize.py:48-71): multiples of 2^-frac, |w| < 2^(15-frac)."""
    w = np.asarray(w)
    s = 2.0 ** frac
    q = np.clip(np.round(w.astype(np.float64) * s), -(2 ** 15 - 1), 2 ** 15 - 1) / s
    q[(w != 0) & (q == 0)] = 1.0 / s  # keep the sparsity pattern
    return q.astype(w.dtype)


def f16_scaled(w: np.ndarray) -> np.ndarray:
    """Config-4 weights in f16 storage: make_layer_weights' N(0,1) nonzeros scaled by
    sqrt(2 / L) (L = nonzeros per output channel, He-style) in float32, then rounded to
    f16.  Unscaled N(0,1) weights overflow f16 by conv3_3 of the VGG stack (inf, then
    NaN), which no fp16 deployment would run; the f32 stack keeps the unscaled weights.
    Restated identically by tests/golden/make_quant_vgg.py."""
    w = np.asarray(w, dtype=np.float32)
    L = int(np.count_nonzero(w.reshape(w.shape[0], -1)[0]))
    return (w * np.float32(math.sqrt(2.0 / max(L, 1)))).astype(np.float16)


def reference_quantize(values: np.ndarray, kind: str, centers=None, pin_zero: bool = False,
                       bits: int = 16) -> np.ndarray:
    """Restates quantize_weights_array(values, kind, bits) (quantize.py:265-288) on a CSR
    values array, bit for bit (pinned by tests/golden/quant_vgg.json digests):

    * "fixed": fit_fixed_point (int_bits = ceil(log2 max|x|), clamped at 0) and
      quantize_fixed (mu + sigma * round((x - mu) / sigma), saturated), quantize.py:48-71,
      computed in float64, then cast to the storage dtype;
    * "codebook": the decode of build_codebook (quantize.py:217-246): every value takes
      the float64 k-means center nearest to it (squared distance, first on ties -- the
      final assignment of _cluster.py:45-47), the table is stored as float16; with
      pin_zero the zeros keep centroid 0 = 0.0.  `centers` are the reference's k-means
      centers (they come from its seeded k-means++ run, recorded by
      tests/golden/make_quant_vgg.py)."""
    dtype = values.dtype
    x = np.asarray(values, dtype=np.float64).ravel()
    if kind == "affine":  # symmetric int (fit_affine_int / quantize_affine_int / dequantize, quantize.py:99-138)
        return affine_quantize(values, bits)[0]
    if kind == "fixed":
        m = float(np.max(np.abs(x))) if x.size else 0.0
        int_bits = 0 if m == 0 else max(0, math.ceil(math.log2(m)))
        sigma = 2.0 ** (-(bits - int_bits - 1))
        mu = 0.0
        q = mu + sigma * np.round((x - mu) / sigma)
        return np.clip(q, -(2.0 ** int_bits), 2.0 ** int_bits - sigma).astype(dtype).reshape(values.shape)
    if kind != "codebook":
        raise ShapeError(f"unknown quantizer {kind!r}")
    c = np.asarray(centers, dtype=np.float64).ravel()
    labels = np.zeros(x.size, dtype=np.int64)
    sel = x != 0 if pin_zero else np.ones(x.size, bool)
    pts = x[sel]
    best = np.full(pts.size, np.inf)
    lab = np.zeros(pts.size, dtype=np.int64)
    for j, cj in enumerate(c):  # argmin over centers, first on ties
        d = (pts - cj) ** 2
        upd = d < best
        best[upd] = d[upd]
        lab[upd] = j
    table = np.concatenate([[0.0], c]) if pin_zero else c
    labels[sel] = lab + (1 if pin_zero else 0)
    return table.astype(np.float16)[labels].astype(dtype).reshape(values.shape)


def affine_quantize(values: np.ndarray, bits: int = 16):
    """quantize_weights_array(values, "affine", bits) restated (quantize.py:99-138, 279-283):
    symmetric fit (mu = 0, step = max|x| / (2^(bits-1) - 1), 1 if that is 0), codes
    round-to-nearest clipped to +-(2^(bits-1) - 1), value = mu + float64(code) * step cast
    to the storage dtype.  Returns (values, step)."""
    x = np.asarray(values, dtype=np.float64).ravel()
    vmin, vmax = float(x.min()), float(x.max())
    mu = 0.0
    step = max(abs(vmin), abs(vmax)) / (2 ** (bits - 1) - 1)
    if step == 0:
        step = 1.0
    lim = 2 ** (bits - 1) - 1
    codes = np.clip(np.round((x - mu) / step), -lim, lim).astype(np.int64)
    out = (mu + codes.astype(np.float64) * step).astype(values.dtype).reshape(values.shape)
    return out, step


def reference_quantized_values_fn(kind: str, fixture) -> "callable":
    """values_fn for network.build_net: replaces each layer's CSR values by the
    reference quantizer's output (config 4 with the reference's own "fixed:16" /
    "codebook:16" weights), using the recorded k-means centers of `fixture`
    (tests/golden/quant_vgg.json)."""
    import json
    from pathlib import Path
    recs = {r["name"]: r for r in json.loads(Path(fixture).read_text())["layers"]}

    def fn(name, values):
        r = recs[name]
        if kind == "fixed":
            return reference_quantize(values, "fixed")
        if kind == "affine":
            out, step = affine_quantize(values, 16)
            return out, {"scheme": "affine", "bits": 16, "mode": "symmetric", "step": step}
        return reference_quantize(values, "codebook", r["codebook"]["centers"], r["codebook"]["pin_zero"])
    return fn
