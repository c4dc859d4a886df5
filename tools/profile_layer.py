"""Run one VGG-CIFAR layer's sparse conv a few times (for ncu captures)."""
import sys, argparse
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2011_06295_b200 as sc
from paper_2011_06295_b200.synth import vgg16_cifar, make_layer_weights, bench_inputs
from paper_2011_06295_b200.device import device_layer
ap = argparse.ArgumentParser()
ap.add_argument('--layer', default='conv3_2'); ap.add_argument('--n', type=int, default=256)
ap.add_argument('--launch', default=''); ap.add_argument('--reps', type=int, default=3)
ap.add_argument('--flags', type=int, default=0); ap.add_argument('--f16', action='store_true')
a = ap.parse_args()
spec = [s for s, _ in vgg16_cifar(0.9) if s.name == a.layer][0]
sh = spec.shape.with_batch(a.n)
w = make_layer_weights(spec, 0); x, b = bench_inputs(sh, a.n)
dt = np.float16 if a.f16 else np.float32
kern = sc.build_csr(w.astype(dt), sh)
xd = torch.from_numpy(x.astype(dt)).cuda(); bd = torch.from_numpy(b).cuda()
layer = device_layer(kern, 0, dt)
launch = tuple(int(v) for v in a.launch.split(',')) if a.launch else layer.default_launch(a.n, a.flags)
print("launch", launch)
y = torch.empty((a.n, sh.k, sh.e, sh.f), device='cuda', dtype=xd.dtype)
st = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), a.n, a.flags, launch if launch[0] >= 0 else None, st)
torch.cuda.synchronize()
print("ok")
