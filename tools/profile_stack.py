"""One forward of the VGG-CIFAR sparse stack with fixed launches (for ncu:
every layer's kernel launches exactly once after one untimed warm pass)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_06295_b200.network import build_net  # noqa: E402
from paper_2011_06295_b200.synth import vgg16_cifar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--launches", required=True)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--sparsity", type=float, default=0.9)
ap.add_argument("--passes", type=int, default=1)
ap.add_argument("--f16", action="store_true", help="f16 storage stack (config 4); --launches may be 'tune'")
a = ap.parse_args()
dt = np.float16 if a.f16 else np.float32
net = build_net(vgg16_cifar(a.sparsity), dtype=dt)
if a.launches == "tune":
    net.plan(a.batch, tune=True)
else:
    net.plan(a.batch, tune=False)
    net.set_launches([None if l is None else tuple(l) for l in json.loads(Path(a.launches).read_text())])
x = torch.randn((a.batch, 3, 32, 32), device="cuda").to(net.tdtype)
for _ in range(a.passes):
    net.forward_device(x)
torch.cuda.synchronize()
print("ok", net.launches)
