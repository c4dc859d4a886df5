"""Build the shipped launch table (paper_2011_06295_b200/tuned/b200_vgg_cifar.json):
tune every VGG-16/CIFAR layer geometry at batch 256 for the flag sets the
network and the plain operator use (0, ReLU, ReLU+pool), f32 exact and f16.
conv_sparse falls back to this table when the tuner has not run in-process
(engine._choose_launch), so the operator is fast by default on these shapes."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06295_b200 as sc  # noqa: E402
from paper_2011_06295_b200 import _abi, engine  # noqa: E402
from paper_2011_06295_b200.synth import bench_inputs, make_layer_weights, vgg16_cifar  # noqa: E402
from paper_2011_06295_b200.tuner import tune_launch  # noqa: E402

rows = []
for dt in (np.float32, np.float16):
    for spec, pool in vgg16_cifar(0.9):
        sh = spec.shape.with_batch(256)
        w = make_layer_weights(spec, 0).astype(dt)
        x, b = bench_inputs(sh, 256)
        kern = sc.build_csr(w, sh)
        xd = torch.from_numpy(x.astype(dt)).cuda()
        for relu, pl in ((False, False), (True, False)) + (((True, True),) if pool else ()):
            best, _ = tune_launch(xd, kern, b, relu=relu, pool=pl, repetitions=3, warmups=1, include_generic=True)
            flags = engine._flags(sc.EnginePlan(), relu, pl, False)
            sig = list(engine.device_layer(kern, 0, engine._io_dtype(xd.numpy().dtype if False else np.dtype(dt), kern)).signature())
            sig = [s if not isinstance(s, (np.integer,)) else int(s) for s in sig]
            # the table is keyed without the sparse level: the best launch depends on geometry and dtype
            row = {"sig": sig[:8] + sig[9:], "flags": flags, "launch": None if best is None else list(best)}
            if best is not None:
                row["variant"] = _abi.variants()[best[0]]
            rows.append(row)
            print(spec.name, str(np.dtype(dt)), flags, best, flush=True)
out = ROOT / "paper_2011_06295_b200" / "tuned" / "b200_vgg_cifar.json"
out.parent.mkdir(exist_ok=True)
out.write_text(json.dumps({"gpu": torch.cuda.get_device_name(0), "batch": 256, "rows": rows}, indent=1))
print("wrote", out)
