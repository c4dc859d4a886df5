#!/usr/bin/env python3
"""BASELINE config 5: sparsity sweep of one 256->256 3x3 conv at 32x32, batch
512, sparse (this engine) vs dense cuDNN, with the crossover the paper studies
(sc/bench.py:235-274 sparsity_sweep semantics: dense timed once, crossover =
linear interpolation where sparse time == dense time).

Per sparsity: L = 2304 - round(sp*2304) (make_layer_weights), sparse time with
a launch tuned at the full batch, dense fp32 (cuDNN, TF32 off), dense TF32 and dense fp16
(channels_last, tensor cores) for reference.  Every sparse result is checked
bit-for-bit against the engine's independent generic kernel before timing.

Usage: python tools/sweep.py [--batch 512] [--out profiles/r01_sweep.json]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2011_06295_b200 as sc  # noqa: E402
from paper_2011_06295_b200 import _abi, engine  # noqa: E402
from paper_2011_06295_b200.device import device_layer  # noqa: E402
from paper_2011_06295_b200.synth import SWEEP_SPARSITIES, make_layer_weights, sweep_layer  # noqa: E402
from paper_2011_06295_b200.tuner import time_call  # noqa: E402


def ev_time(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts)


def tune(layer, x64, y64, bptr, kinds, per_kind=40):
    """Sampled pass over every (kind, dispatch) group, then every launch of the 3 best variants,
    timed at the batch of x64 (the full sweep batch: a 64-image slice misranks launches)."""
    vs = _abi.variants()
    st = torch.cuda.current_stream().cuda_stream
    nb = x64.shape[0]
    cands = [c for c in layer.candidates(nb) if vs[c[0]]["kind"] in kinds]
    timed = {}

    def run(cs):
        for c in cs:
            if c in timed:
                continue
            try:
                timed[c] = time_call(lambda: layer.launch(x64.data_ptr(), bptr, y64.data_ptr(), nb, 0, c, st), 2, 1)
            except Exception as e:  # a candidate the device cannot launch is skipped, not fatal
                print("skip", c, e, file=sys.stderr)
    groups = {}
    for c in cands:
        groups.setdefault((vs[c[0]]["kind"], vs[c[0]]["dispatch"]), []).append(c)
    run([c for lst in groups.values() for c in lst[:: max(1, len(lst) // per_kind)]])
    top = {c[0] for c in sorted(timed, key=timed.get)[:3]}
    run([c for c in cands if c[0] in top])
    return min(timed, key=timed.get)


def crossover(sps, sparse, dense):
    """Interpolated sparsity where sparse time == dense (None = never)."""
    pts = list(zip(sps, sparse))
    for (s0, t0), (s1, t1) in zip(pts, pts[1:]):
        if (t0 - dense) * (t1 - dense) <= 0 and t0 != t1:
            return s0 + (dense - t0) * (s1 - s0) / (t1 - t0)
    return None if sparse[-1] > dense else sps[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r01_sweep.json"))
    ap.add_argument("--sparsities", default=",".join(str(s) for s in SWEEP_SPARSITIES))
    a = ap.parse_args()
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda", 0)
    n = a.batch
    sps = [float(s) for s in a.sparsities.split(",")]
    g = torch.Generator(device="cpu").manual_seed(1)
    x32 = torch.randn((n, 256, 32, 32), generator=g).to(dev)
    x16 = x32.half()
    bias = torch.randn(256, generator=g).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    for sp in sps:
        spec = sweep_layer(sp)
        sh = spec.shape
        w = make_layer_weights(spec, 0)
        row = {"sparsity": sp}
        for name, dt, x in (("f32", np.float32, x32), ("f16", np.float16, x16)):
            kern = sc.build_csr(w.astype(dt), sh)
            layer = device_layer(kern, 0, dt)
            y = torch.empty((n, 256, 32, 32), device=dev, dtype=x.dtype)
            y64 = torch.empty((64, 256, 32, 32), device=dev, dtype=x.dtype)
            best = tune(layer, x, y, bias.data_ptr(), kinds=(0, 1, 2, 3))
            # integrity gate: tuned launch == generic kernel, bitwise (64 images)
            ref = torch.empty_like(y64)
            layer.launch(x[:64].data_ptr(), bias.data_ptr(), y64.data_ptr(), 64, 0, best, st)
            layer.launch(x[:64].data_ptr(), bias.data_ptr(), ref.data_ptr(), 64, _abi.FLAG_GENERIC, None, st)
            torch.cuda.synchronize()
            assert torch.equal(y64.view(torch.int16 if name == "f16" else torch.int32),
                               ref.view(torch.int16 if name == "f16" else torch.int32)), (sp, name, best)
            t = ev_time(lambda: layer.launch(x.data_ptr(), bias.data_ptr(), y.data_ptr(), n, 0, best, st))
            macs = sc.sparse_mac_count(kern, n)
            row[f"sparse_{name}_us"] = round(t * 1e6, 1)
            row[f"sparse_{name}_tmacs"] = round(macs / t / 1e12, 3)
            es = np.dtype(dt).itemsize  # algorithmic bytes: x + y once, taps {value, index}
            nbytes = 2 * n * 256 * 32 * 32 * es + kern.nnz * (es + 4) + 4 * 257 + 4 * 256
            row[f"sparse_{name}_hbm_gbs"] = round(nbytes / t / 1e9, 1)
            row[f"launch_{name}"] = list(best)
            row["L"] = int(kern.sparse_level)
            del layer
        rows.append(row)
        print(json.dumps(row), flush=True)
    # dense comparators (timed once: they do not depend on sparsity)
    wd = torch.randn((256, 256, 3, 3), generator=g).to(dev)
    from paper_2011_06295_b200.cudnn_mode import cudnn_fp32
    with cudnn_fp32("ieee"):
        d32 = ev_time(lambda: torch.nn.functional.conv2d(x32, wd, bias, padding=1))
    with cudnn_fp32("tf32"):
        dtf = ev_time(lambda: torch.nn.functional.conv2d(x32, wd, bias, padding=1))
    xcl = x16.to(memory_format=torch.channels_last)
    wcl = wd.half().to(memory_format=torch.channels_last)
    d16 = ev_time(lambda: torch.nn.functional.conv2d(xcl, wcl, bias.half(), padding=1))
    out = {
        "config": "BASELINE config 5: 256->256 3x3 conv @32x32, batch %d, unified sparsity sweep" % n,
        "dense_us": {"cudnn_fp32_ieee": round(d32 * 1e6, 1), "cudnn_tf32": round(dtf * 1e6, 1),
                     "cudnn_fp16_tensorcore": round(d16 * 1e6, 1)},
        "rows": rows,
        "crossover": {
            "f32_vs_cudnn_fp32": crossover(sps, [r["sparse_f32_us"] for r in rows], d32 * 1e6),
            "f16_vs_cudnn_fp16": crossover(sps, [r["sparse_f16_us"] for r in rows], d16 * 1e6),
            "f32_vs_cudnn_tf32": crossover(sps, [r["sparse_f32_us"] for r in rows], dtf * 1e6),
        },
        "gpu": torch.cuda.get_device_name(0),
        "note": "sparse f32 = exact mode (bit-identical to the reference); f16 = f16 storage, FHFMA f32 "
                "accumulation (bit-identical to the reference f16 profile)",
    }
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(out, indent=1))
    print(json.dumps(out["dense_us"]), json.dumps(out["crossover"]))


if __name__ == "__main__":
    main()
