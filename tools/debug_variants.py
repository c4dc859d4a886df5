"""Run one launch candidate per (variant, first config) in a subprocess and
report pass / bitwise-mismatch / crash (debug helper for new kernels)."""
import os, subprocess, sys, json
sys.path.insert(0, '/root/repo')
if len(sys.argv) > 1 and sys.argv[1] == 'one':
    import numpy as np, torch
    import paper_2011_06295_b200 as sc
    from paper_2011_06295_b200.device import device_layer
    from oracle import oracle as orc
    from paper_2011_06295_b200.synth import LayerSpec, make_layer_weights, bench_inputs
    c, hw, k, n, f16, idx = [int(v) for v in sys.argv[2:8]]
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec('l', sh, 0.9), 0); x, b = bench_inputs(sh, n)
    dt = np.float16 if f16 else np.float32
    w, x = w.astype(dt), x.astype(dt)
    kern = sc.build_csr(w, sh)
    layer = device_layer(kern, 0, dt)
    cands = layer.candidates(n)
    cfg = cands[idx]
    out = sc.conv_sparse(torch.from_numpy(x).cuda(), kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b.astype(dt) if f16 else b)
    ok = np.array_equal(out.view(np.uint16 if f16 else np.uint32), ref.view(np.uint16 if f16 else np.uint32))
    print(json.dumps({"cfg": cfg, "ok": bool(ok), "maxdiff": float(np.max(np.abs(out.astype(np.float64) - ref)))}))
    sys.exit(0)
import numpy as np
import paper_2011_06295_b200 as sc
from paper_2011_06295_b200 import _abi
from paper_2011_06295_b200.device import device_layer
vs = _abi.variants()
for (c, hw, k, n, f16) in [(8, 8, 16, 4, 0), (16, 2, 16, 64, 0), (16, 4, 16, 64, 0), (16, 32, 16, 2, 0), (16, 8, 16, 8, 1)]:
    # enumerate candidates on the CPU side is impossible (needs device layer) -> spawn a lister
    lister = subprocess.run([sys.executable, '-c', f'''
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, paper_2011_06295_b200 as sc, json
from paper_2011_06295_b200.device import device_layer
sh = sc.ConvShape(n={n}, c={c}, h={hw}, w={hw}, k={k}, r=3, s=3, padding=1)
w = np.zeros(({k},{c},3,3), np.float32); w[:, :, 1, 1] = 1
dt = np.float16 if {f16} else np.float32
kern = sc.build_csr(w.astype(dt), sh)
print(json.dumps(device_layer(kern, 0, dt).candidates({n})))
'''], capture_output=True, text=True)
    cands = json.loads(lister.stdout.strip().splitlines()[-1])
    seen = set()
    for i, cf in enumerate(cands):
        v = vs[cf[0]]
        key = (cf[0],)
        if key in seen:
            continue
        seen.add(key)
        r = subprocess.run([sys.executable, __file__, 'one', str(c), str(hw), str(k), str(n), str(f16), str(i)],
                           capture_output=True, text=True, env=dict(os.environ, CUDA_LAUNCH_BLOCKING='1'), timeout=120)
        tail = (r.stdout.strip().splitlines() or [''])[-1] if r.returncode == 0 else ('CRASH ' + (r.stderr.strip().splitlines() or [''])[-1][:150])
        print(f"layer c{c} hw{hw} f16={f16} v{cf[0]} disp={v['dispatch']} tile=({v['kt']},{v['nbt']},{v['th']},{v['tw']}) mode={v['mode']} cfg={cf}: {tail}", flush=True)
