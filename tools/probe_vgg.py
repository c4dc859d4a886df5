import sys, time, json
sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__file__), '..'))
import numpy as np, torch, ctypes
import paper_2011_06295_b200 as sc
from paper_2011_06295_b200 import _abi
from paper_2011_06295_b200.synth import vgg16_cifar, make_layer_weights, bench_inputs
from paper_2011_06295_b200.device import device_layer
from paper_2011_06295_b200.tuner import time_call
p = torch.cuda.get_device_properties(0)
print("DEVICE", p.name, p.multi_processor_count, p.L2_cache_size if hasattr(p,'L2_cache_size') else '', flush=True)
# peaks
names = ctypes.create_string_buffer(16*8); vals=(ctypes.c_double*8)(); cnt=ctypes.c_int32()
_abi.check(_abi.lib().scb_fma_peaks(0, names, vals, 8, ctypes.byref(cnt)))
pk = {names.raw[16*i:16*i+16].split(b'\0')[0].decode(): vals[i] for i in range(cnt.value)}
print("PEAKS_GMACS", json.dumps({k: round(v/1e9,1) for k,v in pk.items()}), flush=True)
N = 256
DT = np.float16 if '--f16' in sys.argv else np.float32
FL = 2 if '--fast' in sys.argv else 0
tot = 0
for spec, pool in vgg16_cifar(0.9):
    sh = spec.shape.with_batch(N)
    w = make_layer_weights(spec, 0); x, b = bench_inputs(sh, N)
    kern = sc.build_csr(w.astype(DT), sh)
    xd = torch.from_numpy(x.astype(DT)).cuda(); bd = torch.from_numpy(b).cuda()
    layer = device_layer(kern, 0, DT)
    cands = layer.candidates(N, FL)
    y = torch.empty((N, sh.k, sh.e, sh.f), device='cuda', dtype=xd.dtype)
    st = torch.cuda.current_stream().cuda_stream
    best = None
    res = []
    for c in cands:
        t = time_call(lambda: layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), N, FL, c, st), 3, 1)
        res.append((t, c))
    res.sort()
    tg = time_call(lambda: layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), N, 8, None, st), 3, 1)
    td = time_call(lambda: layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), N, 0, None, st), 3, 1)
    macs = sc.sparse_mac_count(kern, N)
    t = res[0][0] if res else tg
    tot += t
    print(f"{spec.name:8s} L={kern.sparse_level:4d} ncand={len(cands):3d} best={t*1e6:8.1f}us {macs/t/1e12:6.2f}TMAC/s default={td*1e6:8.1f}us generic={tg*1e6:9.1f}us best_cfg={res[0][1] if res else None} v={_abi.variants()[res[0][1][0]] if res else None} top3={[ (round(a*1e6,1), c) for a,c in res[1:3]]}", flush=True)
print("TOTAL_us", tot*1e6, "img/s", N/tot)
