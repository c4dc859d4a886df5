"""Time every launch candidate of one kernel kind on chosen VGG-CIFAR layers
(debug helper): python tools/probe_kind.py <kind> [layer ...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06295_b200 as sc  # noqa: E402
from paper_2011_06295_b200 import _abi  # noqa: E402
from paper_2011_06295_b200.device import device_layer  # noqa: E402
from paper_2011_06295_b200.synth import bench_inputs, make_layer_weights, vgg16_cifar  # noqa: E402
from paper_2011_06295_b200.tuner import time_call  # noqa: E402

kind = int(sys.argv[1])
names = sys.argv[2:] or ["conv1_2", "conv3_2"]
vs = _abi.variants()
N = 256
for spec, _ in vgg16_cifar(0.9):
    if spec.name not in names:
        continue
    sh = spec.shape.with_batch(N)
    kern = sc.build_csr(make_layer_weights(spec, 0), sh)
    x, b = bench_inputs(sh, N)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    layer = device_layer(kern, 0, np.float32)
    y = torch.empty((N, sh.k, sh.e, sh.f), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    macs = sc.sparse_mac_count(kern, N)
    res = []
    for c in layer.candidates(N):
        if vs[c[0]]["kind"] != kind:
            continue
        t = time_call(lambda: layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), N, 0, c, st), 3, 1)
        v = vs[c[0]]
        res.append((t, c, (v["th"], v["tw"], v["kt"], v["nbt"], v["dispatch"])))
    for t, c, v in sorted(res)[:8]:
        print(f"{spec.name} {t * 1e6:8.1f}us {macs / t / 1e12:5.2f}TMAC/s {c} th,tw,kt,nbt,disp={v}", flush=True)
