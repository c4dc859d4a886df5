"""Debug helper: the launch the network planner picks for conv1_2 vs a direct tune_launch."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2011_06295_b200.network import build_net  # noqa: E402
from paper_2011_06295_b200.synth import vgg16_cifar  # noqa: E402
from paper_2011_06295_b200 import tuner  # noqa: E402

orig = tuner.tune_launch
log = {}


def spy(x, kernel, *a, **k):
    best, t = orig(x, kernel, *a, **k)
    log[kernel.shape.c, kernel.shape.h] = sorted((v, c) for c, v in t.items() if c is not None)[:5]
    return best, t


tuner.tune_launch = spy
net = build_net(vgg16_cifar(0.9), seed=0)
net.plan(256, tune=True)
print("planned conv1_2:", net.launches[1])
for v, c in log[(64, 32)]:
    print("   %.1f us" % (v * 1e6), c)
