"""Time and parity-check the TMEM image-lane kernel (kind 6) on VGG-CIFAR
layers at batch 256 (debug helper): python tools/probe_tmi.py [layer ...]

Every candidate's output is compared bit for bit with the oracle
(oracle/oracle.c conv_sparse) -- plain, and with the fused ReLU + 2x2 pool."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06295_b200 as sc  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2011_06295_b200 import _abi  # noqa: E402
from paper_2011_06295_b200.device import device_layer  # noqa: E402
from paper_2011_06295_b200.synth import bench_inputs, make_layer_weights, vgg16_cifar  # noqa: E402
from paper_2011_06295_b200.tuner import time_call  # noqa: E402

names = sys.argv[1:] or ["conv3_2", "conv4_1", "conv4_2", "conv5_1"]
N = int(__import__("os").environ.get("PROBE_N", "256"))
vs = _abi.variants()
for spec, _ in vgg16_cifar(0.9):
    if spec.name not in names:
        continue
    sh = spec.shape.with_batch(N)
    kern = sc.build_csr(make_layer_weights(spec, 0), sh)
    x, b = bench_inputs(sh, N)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, sh.k, 3, 3, 1, 1, b)
    refp = np.maximum(ref, 0).reshape(N, sh.k, sh.e // 2, 2, sh.f // 2, 2).max(axis=(3, 5))
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    layer = device_layer(kern, 0, np.float32)
    y = torch.empty((N, sh.k, sh.e, sh.f), device="cuda")
    yp = torch.empty((N, sh.k, sh.e // 2, sh.f // 2), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    macs = sc.sparse_mac_count(kern, N)
    best_other = None
    res = []
    for c in layer.candidates(N):
        v = vs[c[0]]
        if v["kind"] != 6:
            continue
        y.fill_(float("nan"))
        layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), N, 0, c, st)
        torch.cuda.synchronize()
        ok = np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        yp.fill_(float("nan"))
        layer.launch(xd.data_ptr(), bd.data_ptr(), yp.data_ptr(), N, _abi.FLAG_RELU | _abi.FLAG_POOL2, c, st)
        torch.cuda.synchronize()
        okp = np.array_equal(yp.cpu().numpy().view(np.uint32), refp.view(np.uint32))
        if not ok:
            got = y.cpu().numpy()
            bad = np.argwhere(got.view(np.uint32) != ref.view(np.uint32))
            print(f"  MISMATCH {c}: {len(bad)} of {got.size}, first {bad[:3].tolist()} "
                  f"got {got[tuple(bad[0])]} want {ref[tuple(bad[0])]}", flush=True)
        t = time_call(lambda: layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), N, 0, c, st), 5, 2)
        res.append((t, c, ok, okp, (v["tw"], v["th"], v["nbt"], v["kt"], v["dispatch"])))
    for t, c, ok, okp, v in sorted(res):
        print(f"{spec.name} {t * 1e6:8.1f}us {macs / t / 1e12:5.2f}TMAC/s ({macs / t / 1e12 / 18.02:.2f} of FMUL+FADD) "
              f"bitwise={ok} pooled={okp} {c} W,TE,J,KW,WQ={v}", flush=True)
