"""Launch every direct-kind candidate (narrow, WIDE, ONED) once on small
shapes, for `compute-sanitizer --tool memcheck python tools/sanitize_direct.py`
(debug helper; correctness is checked by tests/test_gpu_parity.py)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06295_b200 as sc  # noqa: E402
from paper_2011_06295_b200 import _abi  # noqa: E402
from paper_2011_06295_b200.device import device_layer  # noqa: E402
from paper_2011_06295_b200.synth import LayerSpec, make_layer_weights  # noqa: E402

SHAPES = [(64, 2, 2, 64, 3, 1, 17), (64, 4, 4, 64, 3, 1, 9), (32, 8, 8, 32, 3, 1, 5), (16, 28, 28, 16, 3, 1, 2),
          (16, 40, 36, 16, 3, 1, 2), (16, 7, 7, 16, 1, 0, 3), (8, 1, 37, 8, 1, 3, 0, 3)]
vs = _abi.variants()
st = torch.cuda.current_stream().cuda_stream
total = 0
for spec in SHAPES:
    if len(spec) == 8:
        c, h, w, k, r, s, pad, n = spec
    else:
        c, h, w, k, r, pad, n = spec
        s = r
    sh = sc.ConvShape(n=n, c=c, h=h, w=w, k=k, r=r, s=s, padding=pad)
    kern = sc.build_csr(make_layer_weights(LayerSpec("l", sh, 0.8), 0), sh)
    layer = device_layer(kern, 0, np.float32)
    # exact-size allocations: no slack around the activations
    x = torch.randn(n * c * h * w, device="cuda")
    b = torch.randn(k, device="cuda")
    for flags in (0, 5):
        cands = [cf for cf in layer.candidates(n, flags) if vs[cf[0]]["kind"] == 2]
        e, f = (sh.e // 2, sh.f // 2) if flags & 4 else (sh.e, sh.f)
        y = torch.empty(n * k * e * f, device="cuda")
        for cf in cands:
            layer.launch(x.data_ptr(), b.data_ptr(), y.data_ptr(), n, flags, cf, st)
            torch.cuda.synchronize()
            total += 1
    print(spec, "ok", flush=True)
print("launched", total)
