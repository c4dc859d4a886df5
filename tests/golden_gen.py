"""Seeded input generators restated from the reference test-suite (test
infrastructure; shared by tests/ and tests/golden/make_golden.py).

Each generator consumes numpy's ``default_rng`` stream in exactly the order
the reference does, so the golden digests recorded from the reference can be
re-derived on the GPU box without the reference present:

* ``random_sparse_weights``  -- pkg/tests/conftest.py:36-40
* ``make_case``              -- pkg/tests/test_engine.py:10-18
* ``c1_configs``             -- pkg/tests/test_acceptance.py:42-92
  (``random_config`` retry loop; ConvShape validity rules of shapes.py:35-51)
* ``lenet_conv2_case``       -- BASELINE config 0 (LeNet-5 conv2, 6->16, 5x5,
  12x12, 90% Bernoulli sparsity, default_rng(0)), SURVEY.md 8(d)
"""
from __future__ import annotations

import hashlib

import numpy as np


class Shape(dict):
    """Plain geometry record with attribute access (n,c,h,w,k,r,s,stride,padding)."""

    __getattr__ = dict.__getitem__

    @property
    def e(self):
        return (self["h"] + 2 * self["padding"] - self["r"]) // self["stride"] + 1

    @property
    def f(self):
        return (self["w"] + 2 * self["padding"] - self["s"]) // self["stride"] + 1


def shape_valid(n, c, h, w, k, r, s, stride, padding) -> bool:
    if min(n, c, h, w, k, r, s, stride) < 1 or padding < 0:
        return False
    if r > h + 2 * padding or s > w + 2 * padding:
        return False
    return (h + 2 * padding - r) % stride == 0 and (w + 2 * padding - s) % stride == 0


def sha256(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def random_sparse_weights(rng, k, c, r, s, sparsity, dtype=np.float32):
    w = rng.standard_normal((k, c, r, s)).astype(dtype)
    mask = rng.random((k, c, r, s)) < sparsity
    w[mask] = 0
    return w


def _conv_shape(**kw):
    """Reference ConvShape when importable (golden generation), else Shape."""
    try:
        from sparseconv.shapes import ConvShape  # only present when generating
        return ConvShape(**kw)
    except ImportError:
        return Shape(**kw)


def make_case(seed, n=2, c=3, h=8, w=8, k=4, r=3, s=3, stride=1, padding=1,
              sparsity=0.7, dtype=np.float32, shape_factory=None):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, c, h, w)).astype(dtype)
    wt = random_sparse_weights(rng, k, c, r, s, sparsity, dtype)
    bias = rng.standard_normal(k).astype(dtype)
    mk = shape_factory or _conv_shape
    sh = mk(n=n, c=c, h=h, w=w, k=k, r=r, s=s, stride=stride, padding=padding)
    return x, wt, bias, sh


def _random_config(rng):
    while True:
        n = int(rng.integers(1, 5))
        c = int(rng.integers(1, 33))
        k = int(rng.integers(1, 33))
        r = int(rng.choice([1, 2, 3, 5]))
        s = int(rng.choice([1, 2, 3, 5]))
        h = int(rng.integers(1, 33))
        w = int(rng.integers(1, 33))
        stride = int(rng.integers(1, 3))
        padding = int(rng.integers(0, 3))
        sparsity = float(rng.choice([0.0, 0.5, 0.77, 0.9, 0.95, 1.0]))
        if shape_valid(n, c, h, w, k, r, s, stride, padding):
            return dict(n=n, c=c, h=h, w=w, k=k, r=r, s=s, stride=stride,
                        padding=padding), sparsity


def c1_configs(n_configs=200, seed=0):
    """Yield the acceptance-C1 configs with their inputs (same rng order)."""
    rng = np.random.default_rng(seed)
    for i in range(n_configs):
        shape, sparsity = _random_config(rng)
        x = rng.standard_normal((shape["n"], shape["c"], shape["h"], shape["w"])).astype(np.float32)
        w = random_sparse_weights(rng, shape["k"], shape["c"], shape["r"], shape["s"], sparsity)
        bias = rng.standard_normal(shape["k"]).astype(np.float32)
        yield {"shape": shape, "sparsity": sparsity, "x": x, "w": w, "bias": bias,
               "f16": i % 5 == 0}


def lenet_conv2_case():
    rng = np.random.default_rng(0)
    w = random_sparse_weights(rng, 16, 6, 5, 5, 0.9)
    x = rng.standard_normal((1, 6, 12, 12)).astype(np.float32)
    bias = rng.standard_normal(16).astype(np.float32)
    sh = _conv_shape(n=1, c=6, h=12, w=12, k=16, r=5, s=5, stride=1, padding=0)
    return x, w, bias, sh
