import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '.')
import numpy as np, torch
from oracle import oracle as orc
from paper_2011_06295_b200.network import build_net
from paper_2011_06295_b200.synth import vgg16_cifar
for n in (8, 256):
    net = build_net(vgg16_cifar(0.9), seed=0, dtype=np.float16)
    net.plan(n, tune=False)
    x = np.random.default_rng(12).standard_normal((n, 3, 32, 32)).astype(np.float16)
    cur = torch.from_numpy(x).cuda()
    a = x
    st = torch.cuda.current_stream().cuda_stream
    for i, L in enumerate(net.layers):
        sh = L.kernel.shape
        got = torch.empty(net.out_shape(i, n), dtype=net.tdtype, device='cuda')
        net.launch_layer(i, cur, got, st)
        torch.cuda.synchronize()
        z = orc.conv_sparse(a, L.kernel.values, L.kernel.colidx, L.kernel.rowptr, sh.k, 3, 3, 1, 1, L.bias)
        z = np.maximum(z, z.dtype.type(0))
        if L.pool:
            nn, k, e, f = z.shape
            z = z.reshape(nn, k, e // 2, 2, f // 2, 2).max(axis=(3, 5))
        g = got.cpu().numpy()
        bad = np.count_nonzero(g.view(np.uint16) != z.view(np.uint16))
        print(n, L.name, net.launches[i], 'bad', bad, 'of', z.size, g.dtype, z.dtype, flush=True)
        if bad:
            idx = np.argwhere(g.view(np.uint16) != z.view(np.uint16))[:3]
            for t in idx: print('   ', t, g[tuple(t)], z[tuple(t)])
        cur = got
        a = z
