"""Per-layer times of the tuned f16-storage VGG-CIFAR stack (config 4) next to
the f32 exact stack (debug helper): python tools/probe_f16.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_06295_b200 import _abi  # noqa: E402
from paper_2011_06295_b200.network import build_net  # noqa: E402
from paper_2011_06295_b200.synth import vgg16_cifar  # noqa: E402

vs = _abi.variants()
N = 256
for dt in (np.float16, np.float32):
    net = build_net(vgg16_cifar(0.9), seed=0, dtype=dt)
    net.plan(N, tune=True)
    x = torch.randn((N, 3, 32, 32), device="cuda").to(net.tdtype)
    for _ in range(3):
        net.forward_device(x)
    nl = len(net.layers)
    reps = 10
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)] for _ in range(reps)]
    for k in range(reps):
        net.forward_device(x, events=ev[k])
    torch.cuda.synchronize()
    tot = 0
    for i, L in enumerate(net.layers):
        us = 1e3 * float(np.median([ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(reps)]))
        tot += us
        l = net.launches[i]
        v = vs[l[0]] if l is not None else None
        desc = "generic" if v is None else f"kind{v['kind']} th{v['th']} tw{v['tw']} kt{v['kt']} nbt{v['nbt']} d{v['dispatch']}"
        print(f"{np.dtype(dt).name} {L.name:8s} {us:8.1f}us  {l}  {desc}", flush=True)
    print(f"{np.dtype(dt).name} total {tot:.1f}us", flush=True)
