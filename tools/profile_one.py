"""Launch one VGG-CIFAR layer with an explicit launch a few times (for ncu):
python tools/profile_one.py <layer> <v,wk,imgs,bh,bw,cc,stages> [f16]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06295_b200 as sc  # noqa: E402
from paper_2011_06295_b200.device import device_layer  # noqa: E402
from paper_2011_06295_b200.synth import bench_inputs, make_layer_weights, vgg16_cifar  # noqa: E402

name, launch = sys.argv[1], tuple(int(v) for v in sys.argv[2].split(","))
spec = [s for s, _ in vgg16_cifar(0.9) if s.name == name][0]
N = 256
sh = spec.shape.with_batch(N)
dt = np.float16 if sys.argv[3:] == ["f16"] else np.float32
kern = sc.build_csr(make_layer_weights(spec, 0).astype(dt), sh)
x, b = bench_inputs(sh, N)
xd, bd = torch.from_numpy(x.astype(dt)).cuda(), torch.from_numpy(b).cuda()
layer = device_layer(kern, 0, dt)
y = torch.empty((N, sh.k, sh.e, sh.f), device="cuda", dtype=xd.dtype)
for _ in range(3):
    layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), N, 0, launch, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
