"""Golden vectors for the activation fake-quant epilogue, made WITH THE
REFERENCE PACKAGE (run here, not on the GPU box):
PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_fake_quant.py

* fake_quant_cases.npz: fake_quant_activation (quantize.py:332-338) on seeded
  f32 / f16 / f64 arrays (incl. exact code ties and out-of-clip values) for
  asymmetric and symmetric parameter sets;
* store_aq/ + store_aq_expected.npz: a model with 8-bit activation quantizers
  fitted by apply_quantization(..., targets=("activations",)) (quantize.py:314-328),
  saved with save_model, and its conv-stack output per Model.forward
  (conv_sparse -> ReLU -> fake_quant_activation, store.py:276-286)."""
import json
import shutil
import sys
from pathlib import Path

import numpy as np

import sparseconv as sc
from sparseconv.quantize import apply_quantization, fake_quant_activation
from sparseconv.store import ConvLayerRecord, DenseLayerRecord, Model, load_model, save_model

HERE = Path(__file__).resolve().parent
rng = np.random.default_rng(11)

PARAMS = [
    {"bits": 8, "clip_lo": -0.75, "clip_hi": 2.5, "mu": -0.75, "step": 3.25 / 255, "mode": "asymmetric"},
    {"bits": 4, "clip_lo": 0.0, "clip_hi": 1.3, "mu": 0.0, "step": 1.3 / 15, "mode": "asymmetric"},
    {"bits": 8, "clip_lo": -2.0, "clip_hi": 2.0, "mu": 0.0, "step": 2.0 / 127, "mode": "symmetric"},
    {"bits": 6, "clip_lo": 0.1, "clip_hi": 0.7, "mu": 0.1, "step": 0.0095, "mode": "asymmetric"},
]
cases = {}
meta = []
i = 0
for dt in (np.float32, np.float16, np.float64):
    for p in PARAMS:
        x = (rng.standard_normal(4099) * 1.5).astype(dt)
        # exact ties of the code grid and values outside the clip range
        ties = (p["mu"] + (np.arange(40) + 0.5) * p["step"]).astype(dt)
        x = np.concatenate([x, ties, np.array([-1e4, 1e4, 0.0, -0.0], dt)])
        cases[f"x{i}"] = x
        cases[f"y{i}"] = fake_quant_activation(x, p)
        meta.append({"dtype": np.dtype(dt).name, "params": p})
        i += 1
cases["meta"] = np.array(json.dumps(meta))
np.savez(HERE / "fake_quant_cases.npz", **cases)

# a small model with fitted activation quantizers
rng = np.random.default_rng(13)


def pruned(k, c, r, s, sp):
    w = rng.standard_normal((k, c, r, s)).astype(np.float32)
    w[rng.random(w.shape) < sp] = 0
    return w


convs = []
for name, c, k in (("conv0", 3, 16), ("conv1", 16, 24), ("conv2", 24, 32)):
    sh = sc.ConvShape(n=1, c=c, h=16, w=16, k=k, r=3, s=3, padding=1)
    convs.append(ConvLayerRecord(name=name, bias=rng.standard_normal(k).astype(np.float32), padding=1,
                                 kernel=sc.build_csr(pruned(k, c, 3, 3, 0.8), sh)))
dense = [DenseLayerRecord(name="fc", weights=rng.standard_normal((10, 32)).astype(np.float32),
                          bias=np.zeros(10, np.float32))]
model = Model(convs, dense, {"architecture": {"in_channels": 3, "image_size": 16}})
calib = rng.standard_normal((8, 3, 16, 16)).astype(np.float32)
apply_quantization(model, "affine:8", targets=("activations",), calib_data=calib)
out = HERE / "store_aq"
if out.exists():
    shutil.rmtree(out)
save_model(model, out)
back = load_model(out)
x = rng.standard_normal((3, 3, 16, 16)).astype(np.float32)
a = x
for L in back.conv_layers:
    a = np.maximum(sc.conv_sparse(a, L.csr_kernel(a), L.bias), 0)
    a = fake_quant_activation(a, L.act_quant)
np.savez(HERE / "store_aq_expected.npz", x=x, conv_out=a)
print("wrote fake_quant_cases.npz, store_aq/, store_aq_expected.npz", file=sys.stderr)
