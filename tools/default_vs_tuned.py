"""Default launch (C heuristic, scb_default_launch) vs the tuned best for the
reference presets and the VGG-CIFAR layers (debug helper for pick_default):
python tools/default_vs_tuned.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06295_b200 as sc  # noqa: E402
from paper_2011_06295_b200 import _abi  # noqa: E402
from paper_2011_06295_b200.device import device_layer  # noqa: E402
from paper_2011_06295_b200.synth import PRESETS, make_layer_weights, vgg16_cifar  # noqa: E402
from paper_2011_06295_b200.tuner import time_call  # noqa: E402

vs = _abi.variants()
st = torch.cuda.current_stream().cuda_stream
specs = [(s, 256) for s, _ in vgg16_cifar(0.9)] + [(s, 128) for p in PRESETS.values() for s in p]
for spec, n in specs:
    sh = spec.shape.with_batch(n)
    kern = sc.build_csr(make_layer_weights(spec, 0), sh)
    layer = device_layer(kern, 0, np.float32)
    xd = torch.randn((n, sh.c, sh.h, sh.w), device="cuda")
    bd = torch.randn(sh.k, device="cuda")
    y = torch.empty((n, sh.k, sh.e, sh.f), device="cuda")
    d = layer.default_launch(n, 0)
    run = lambda c: layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), n, 0, c, st)  # noqa: E731
    td = time_call(lambda: run(d), 5, 2)
    cands = layer.candidates(n)
    best, tb = d, td
    for c in cands[:: max(1, len(cands) // 60)]:
        t = time_call(lambda: run(c), 3, 1)
        if t < tb:
            best, tb = c, t
    v, w = vs[d[0]], vs[best[0]]
    print(f"{spec.name:32s} default {td * 1e6:9.1f}us k{v['kind']}d{v['dispatch']} {d}  best {tb * 1e6:9.1f}us "
          f"k{w['kind']}d{w['dispatch']} {best}  ratio {td / tb:.2f}", flush=True)
    del xd, y
    torch.cuda.empty_cache()
