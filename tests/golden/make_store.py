"""Generate a small model-store fixture WITH THE REFERENCE PACKAGE (run here,
not on the GPU box): PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
    python tests/golden/make_store.py

Writes tests/golden/store_small/ (manifest.json + blobs, reference
save_model, sc/store.py:323-372) and tests/golden/store_small_expected.npz:
the reference's own load_model arrays per conv layer and the conv-stack
output (conv_sparse -> ReLU per layer, store.py:276-284) on a seeded input."""
import shutil
import sys
from pathlib import Path

import numpy as np

import sparseconv as sc
from sparseconv.quantize import apply_quantization
from sparseconv.store import ConvLayerRecord, DenseLayerRecord, Model, load_model, save_model

HERE = Path(__file__).resolve().parent
OUT = HERE / "store_small"

rng = np.random.default_rng(7)


def pruned(k, c, r, s, sp):
    w = rng.standard_normal((k, c, r, s)).astype(np.float32)
    w[rng.random(w.shape) < sp] = 0
    return w


convs = []
# conv0: 3->16, 3x3, stored as CSR (unified)
w0 = pruned(16, 3, 3, 3, 0.5)
sh0 = sc.ConvShape(n=1, c=3, h=16, w=16, k=16, r=3, s=3, padding=1)
convs.append(ConvLayerRecord(name="conv0", bias=rng.standard_normal(16).astype(np.float32), padding=1,
                             kernel=sc.build_csr(w0, sh0)))
# conv1: 16->24, 3x3, stored dense (CSR built per forward)
convs.append(ConvLayerRecord(name="conv1", bias=rng.standard_normal(24).astype(np.float32), padding=1,
                             weights=pruned(24, 16, 3, 3, 0.85)))
# conv2: 24->32, 3x3, CSR, non-unified
w2 = pruned(32, 24, 3, 3, 0.9)
sh2 = sc.ConvShape(n=1, c=24, h=16, w=16, k=32, r=3, s=3, padding=1)
convs.append(ConvLayerRecord(name="conv2", bias=rng.standard_normal(32).astype(np.float32), padding=1,
                             kernel=sc.build_csr(w2, sh2, unify=False)))
dense = [DenseLayerRecord(name="fc", weights=rng.standard_normal((10, 32)).astype(np.float32),
                          bias=np.zeros(10, np.float32))]
model = Model(convs, dense, {"architecture": {"in_channels": 3, "image_size": 16}})
apply_quantization(model, "codebook:16", targets=("weights",), seed=0)  # 16-centroid codebooks
if OUT.exists():
    shutil.rmtree(OUT)
save_model(model, OUT)

back = load_model(OUT)
x = rng.standard_normal((2, 3, 16, 16)).astype(np.float32)
a = x
arrays = {"x": x}
for L in back.conv_layers:
    kern = L.csr_kernel(a)
    arrays[f"{L.name}.values"] = kern.values
    arrays[f"{L.name}.colidx"] = kern.colidx
    arrays[f"{L.name}.rowptr"] = kern.rowptr
    arrays[f"{L.name}.bias"] = L.bias
    a = np.maximum(sc.conv_sparse(a, kern, L.bias), 0)
arrays["conv_out"] = a
np.savez(HERE / "store_small_expected.npz", **arrays)
print("wrote", OUT, "and expected output", a.shape, file=sys.stderr)
