"""Golden data for BASELINE config 4 with the REFERENCE's own weight quantizers.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_quant_vgg.py

For every VGG-16/CIFAR layer at 90 % unified sparsity (make_layer_weights,
bench.py:105-116, seed 0, scaled by sqrt(2/L) as synth.f16_scaled does) in f16
storage, the CSR values (build_csr) are passed
through quantize_weights_array(values, "fixed", 16), ("codebook", 16, seed=0) and
("affine", 16)
(quantize.py:265-288).  Stored per layer: the sha256 of both reference outputs
(bit patterns), the fixed-point split, and the codebook's float64 k-means centers
(the labels are the final argmin against them, _cluster.py:45-47), which is what
synth.reference_quantize restates.  quant_vgg.json is ~10 KB.
"""
from __future__ import annotations

import hashlib
import json
import math
from pathlib import Path

import numpy as np

from sparseconv._cluster import kmeans
from sparseconv.bench import LayerSpec, make_layer_weights
from sparseconv.csr import build_csr
from sparseconv.quantize import quantize_weights_array
from sparseconv.shapes import ConvShape

OUT = Path(__file__).resolve().parent
LAYERS = [("conv1_1", 3, 32, 64), ("conv1_2", 64, 32, 64), ("conv2_1", 64, 16, 128), ("conv2_2", 128, 16, 128),
          ("conv3_1", 128, 8, 256), ("conv3_2", 256, 8, 256), ("conv3_3", 256, 8, 256), ("conv4_1", 256, 4, 512),
          ("conv4_2", 512, 4, 512), ("conv4_3", 512, 4, 512), ("conv5_1", 512, 2, 512), ("conv5_2", 512, 2, 512),
          ("conv5_3", 512, 2, 512)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    recs = []
    for name, c, h, k in LAYERS:
        sh = ConvShape(n=1, c=c, h=h, w=h, k=k, r=3, s=3, stride=1, padding=1)
        w = make_layer_weights(LayerSpec(name, sh, 0.9), seed=0)
        # = synth.f16_scaled: N(0,1) nonzeros x sqrt(2/L) in f32, rounded to f16
        L = int(np.count_nonzero(w.reshape(w.shape[0], -1)[0]))
        w16 = (w.astype(np.float32) * np.float32(math.sqrt(2.0 / max(L, 1)))).astype(np.float16)
        vals = build_csr(w16, sh).values
        fixed, fmeta, _ = quantize_weights_array(vals, "fixed", 16)
        cbv, cmeta, cb = quantize_weights_array(vals, "codebook", 16, seed=0)
        aff, ameta, _ = quantize_weights_array(vals, "affine", 16)
        # the float64 centers build_codebook's kmeans call returns (quantize.py:229-243)
        flat = np.asarray(vals, dtype=np.float64).ravel()
        k_eff = min(16, len(np.unique(flat)))
        rng = np.random.default_rng(0)
        pin = bool(np.any(flat == 0))
        if pin:
            centers, labels, _ = kmeans(flat[flat != 0], k_eff - 1, rng)
        else:
            centers, labels, _ = kmeans(flat, k_eff, rng)
        assert np.array_equal(cb.centroids[1:] if pin else cb.centroids, centers.ravel().astype(np.float16))
        recs.append({"name": name, "nnz": int(vals.size), "values_sha": sha(vals),
                     "fixed": {"int_bits": fmeta["int_bits"], "frac_bits": fmeta["frac_bits"], "sha": sha(fixed)},
                     "codebook": {"pin_zero": pin, "centers": [float(v) for v in centers.ravel()],
                                  "sha": sha(cbv)},
                     "affine": {"step": ameta["step"], "sha": sha(aff)}})
        print(name, vals.size, fmeta, cmeta, pin)
    (OUT / "quant_vgg.json").write_text(json.dumps({"sparsity": 0.9, "seed": 0, "dtype": "float16",
                                                    "layers": recs}, indent=1))


if __name__ == "__main__":
    main()
